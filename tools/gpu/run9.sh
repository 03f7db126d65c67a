for c in "5 1024" "4 2048"; do set -- $c
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2_c$1.csv -k regex:k_masked python tools/profile_step.py --config $1 --size $2 --reps 1 > gpurun_out/ncu2_c$1.log 2>&1
done
