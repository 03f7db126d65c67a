AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 4 > gpurun_out/g42_phases.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "matmul or galerkin or spgemm" > gpurun_out/g42_pytest.log 2>&1; echo "exit $?" >> gpurun_out/g42_pytest.log
