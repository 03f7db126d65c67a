rm -f gpurun_out/r04_*.ncu-rep
bash tools/ncu_capture_c5.sh r04
cap2() {  # cfg size name regex skip count
    timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
        -k "regex:$4" -s "$5" -c "$6" -o "gpurun_out/r04_c$1_$3" python tools/profile_step.py --config $1 --size $2 --reps 1 > "gpurun_out/r04_c$1_$3.log" 2>&1
    echo "$3 c$1 rc=$?"
}
cap2 2 1024 band 'k_masked_band' 1 1
cap2 4 2048 band 'k_masked_band' 1 1
cap2 4 2048 band_l1 'k_masked_band' 12 1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r04_launches_c5.csv python tools/profile_step.py --config 5 --size 1024 --reps 1 > gpurun_out/r04_ncu_c5.log 2>&1
python tools/launch_summary.py gpurun_out/r04_launches_c5.csv gpurun_out/r04_c5_launch_summary.txt > /dev/null
