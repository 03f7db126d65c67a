for c in "5 1024" "4 2048"; do set -- $c
  AMGCU_BAND_TRACE=1 python tools/profile_step.py --config $1 --size $2 --reps 1 > gpurun_out/trace_c$1.txt 2>&1
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$1.csv python tools/profile_step.py --config $1 --size $2 --reps 1 > gpurun_out/ncu_c$1.log 2>&1
  python tools/launch_summary.py gpurun_out/launches_c$1.csv gpurun_out/launch_summary_c$1.txt > /dev/null
done
grep -h "band" gpurun_out/trace_c5.txt gpurun_out/trace_c4.txt
