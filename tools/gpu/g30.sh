timeout 300 python tools/gs_levels.py 5 1024 > gpurun_out/g30_gs_c5.log 2>&1
timeout 300 python tools/gs_levels.py 2 1024 > gpurun_out/g30_gs_c2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_setup.py tests/test_gpu_golden.py -q -x -p no:cacheprovider > gpurun_out/g30_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g30_pytest.log
timeout 1500 python -m pytest tests/test_gpu_config_scale.py -q -x -p no:cacheprovider -k "dump or overlap" >> gpurun_out/g30_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g30_pytest.log
AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 4 > gpurun_out/g30_phases.log 2>&1
