python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g3_bench_a.json 2> gpurun_out/g3_bench_a.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --family-timing 0 > gpurun_out/g3_bench_b.json 2> gpurun_out/g3_bench_b.err
timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 5 > gpurun_out/g3_steps_c5.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_config_scale.py tests/test_gpu_setup.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "C2-1024 or C5-1024 or overlap or setup or gauss or relax or candidates" > gpurun_out/g3_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g3_pytest.log
