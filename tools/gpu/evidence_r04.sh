# Round-end evidence set (r04): GPU tests, bench lines of every config and the reference arm,
# ncu --set full captures summarised on the box (the .ncu-rep files exceed the 64 MiB that
# come back), launch lists.  Run as: gpurun --timeout 5400 -- "bash tools/gpu/evidence_r04.sh"
python -m pytest tests -m gpu -x -q > gpurun_out/t27.log 2>&1
tail -2 gpurun_out/t27.log
python bench.py > gpurun_out/r04_bench_c5.json 2> gpurun_out/r04_bench_c5.err
for c in 1 2 4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/r04_bench_c$c.json 2> gpurun_out/r04_bench_c$c.err; done
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r04_reference_arm.json 2> gpurun_out/r04_reference_arm.err
bash tools/ncu_capture_c5.sh r04 > gpurun_out/r04_capture.log 2>&1
cap2() {  # cfg size name regex skip count
    timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
        -k "regex:$4" -s "$5" -c "$6" -o "gpurun_out/r04_c$1_$3" python tools/profile_step.py --config $1 --size $2 --reps 1 > "gpurun_out/r04_c$1_$3.log" 2>&1
    echo "$3 c$1 rc=$?" >> gpurun_out/r04_capture.log
}
cap2 2 1024 band 'k_masked_band' 1 1
cap2 4 2048 band 'k_masked_band' 1 1
cap2 4 2048 band_l1 'k_masked_band' 12 1
cap2 4 2048 band_direct 'k_masked_band' 23 1
python tools/ncu_summary.py r04 > gpurun_out/r04_ncu_summary_table.md 2> gpurun_out/r04_ncu_summary.err
cp profiles/r04_traffic.json gpurun_out/r04_traffic.json
rm -f gpurun_out/r04_*.ncu-rep
for c in "5 1024" "4 2048"; do set -- $c
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r04_launches_c$1.csv python tools/profile_step.py --config $1 --size $2 --reps 1 > gpurun_out/r04_ncu_c$1.log 2>&1
python tools/launch_summary.py gpurun_out/r04_launches_c$1.csv gpurun_out/r04_c$1_launch_summary.txt > /dev/null
done
rm -f gpurun_out/r04_launches_c4.csv
du -sh gpurun_out
