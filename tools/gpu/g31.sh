timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_setup.py tests/test_gpu_golden.py -q -x -p no:cacheprovider > gpurun_out/g31_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g31_pytest.log
timeout 1500 python -m pytest tests/test_gpu_config_scale.py -q -x -p no:cacheprovider -k "dump or bitwise" >> gpurun_out/g31_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g31_pytest.log
AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 4 > gpurun_out/g31_phases.log 2>&1
AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 2 --size 1024 --reps 4 > gpurun_out/g31_phases_c2.log 2>&1
