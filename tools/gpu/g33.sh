for cfg in 1 2 3 4 5; do python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --max-restarts 3 > gpurun_out/g33_bench_c$cfg.json 2> gpurun_out/g33_bench_c$cfg.err; done
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/g33_ref.json 2> gpurun_out/g33_ref.err
