timeout 1200 python -m pytest tests/test_gpu_setup.py tests/test_gpu_kernels.py tests/test_gpu_golden.py tests/test_gpu_seqsum.py -q -x -p no:cacheprovider > gpurun_out/g20_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g20_pytest.log
timeout 900 python -m pytest tests/test_gpu_config_scale.py -q -x -p no:cacheprovider -k "C5-1024 or C2-1024 or C1-96 or C3-512 or C4-512 or overlap" >> gpurun_out/g20_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g20_pytest.log
AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 6 > gpurun_out/g20_phases.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g20_bench.json 2> gpurun_out/g20_bench.err
