python -m pytest tests -m gpu -x -q > gpurun_out/t32.log 2>&1
tail -2 gpurun_out/t32.log
python bench.py > gpurun_out/r04_bench_c5.json 2> gpurun_out/r04_bench_c5.err
for c in 2 4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/r04_bench_c$c.json 2> gpurun_out/r04_bench_c$c.err; done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k "regex:k_gs_seg_warp" -s 0 -c 2 -o gpurun_out/r04_gs_segwarp python tools/profile_step.py --config 5 --size 1024 --reps 1 > gpurun_out/r04_gs_segwarp.log 2>&1
python tools/ncu_summary.py r04 > gpurun_out/r04_gs_table.md 2>/dev/null
rm -f gpurun_out/r04_*.ncu-rep
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r04_launches_c5.csv python tools/profile_step.py --config 5 --size 1024 --reps 1 > gpurun_out/r04_ncu_c5.log 2>&1
python tools/launch_summary.py gpurun_out/r04_launches_c5.csv gpurun_out/r04_c5_launch_summary.txt > /dev/null
