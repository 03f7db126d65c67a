for cfg in 5 2; do python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g40_bench_c$cfg.json 2> gpurun_out/g40_bench_c$cfg.err; done
AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 4 > gpurun_out/g40_phases.log 2>&1
