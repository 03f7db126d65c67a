timeout 300 python tools/profile_step.py --config 5 --size 1024 --reps 1 > /dev/null 2>&1 || echo "plain run failed" > gpurun_out/g25_fail.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03_c5_launches.csv python tools/profile_step.py --config 5 --size 1024 --reps 1 > gpurun_out/g25_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/g25_ncu.log
