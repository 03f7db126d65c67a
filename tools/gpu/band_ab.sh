python -m pytest tests/test_gpu_config_scale.py tests/test_gpu_setup.py tests/test_gpu_golden.py -q -x -k "masked_band or ledger or golden or full_size" > gpurun_out/tb.log 2>&1
tail -2 gpurun_out/tb.log
for c in "5 1024" "2 1024" "4 2048"; do set -- $c
python tools/family_times.py --config $1 --size $2 --tag c$1 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "emin_|total" | tr '\n' ' '; echo
done
for c in "5 1024" "4 2048"; do set -- $c
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4_c$1.csv -k regex:k_masked python tools/profile_step.py --config $1 --size $2 --reps 1 > gpurun_out/ncu4_c$1.log 2>&1
done
