timeout 1500 python -m pytest tests/test_gpu_config_scale.py tests/test_gpu_setup.py tests/test_cpp_dropin.py -q -x -p no:cacheprovider > gpurun_out/g27_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g27_pytest.log
AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 5 > gpurun_out/g27_phases.log 2>&1
AMGCU_PCG_SPEC=0 AMGCU_WARP_ROW_MAX=100000000 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 5 > gpurun_out/g27_phases_old.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g27_bench.json 2> gpurun_out/g27_bench.err
