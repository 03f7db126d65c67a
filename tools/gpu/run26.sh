python -m pytest tests/test_gpu_config_scale.py tests/test_gpu_setup.py tests/test_gpu_golden.py -q -x -k "masked_band or ledger or golden or full_size or default_mode" > gpurun_out/t26.log 2>&1
tail -2 gpurun_out/t26.log
for c in "4 2048" "3 1024" "5 1024"; do set -- $c
AMGCU_BAND_TRACE=1 python tools/family_times.py --config $1 --size $2 --tag c$1 > gpurun_out/fam26_c$1.txt 2>&1
grep "^\[c" gpurun_out/fam26_c$1.txt | tr ' ' '\n' | grep -E "emin_|total" | tr '\n' ' '; echo
grep "direct 1" gpurun_out/fam26_c$1.txt | sort | uniq -c | head -5
done
