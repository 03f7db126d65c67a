python -m pytest tests -m gpu -x -q > gpurun_out/t_final.log 2>&1
tail -2 gpurun_out/t_final.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/r04_bench_c5.json 2> gpurun_out/r04_bench_c5.err
for c in 2 4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/r04_bench_c$c.json 2> gpurun_out/r04_bench_c$c.err; done
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r04_reference_arm.json 2> gpurun_out/r04_reference_arm.err
