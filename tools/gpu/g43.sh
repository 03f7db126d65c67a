timeout 900 python -m pytest tests/test_gpu_setup.py -q -x -p no:cacheprovider -k "gauss_jordan" > gpurun_out/g43_pytest.log 2>&1; echo "exit $?" >> gpurun_out/g43_pytest.log
timeout 900 python -m pytest tests/test_gpu_config_scale.py -q -x -p no:cacheprovider -k "C5 or C1" >> gpurun_out/g43_pytest.log 2>&1; echo "exit $?" >> gpurun_out/g43_pytest.log
AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 3 > gpurun_out/g43_phases.log 2>&1
