timeout 1200 python -m pytest tests/test_gpu_setup.py tests/test_gpu_kernels.py tests/test_gpu_golden.py -v -x -p no:cacheprovider --timeout 120 > gpurun_out/g7_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g7_pytest.log
timeout 300 python tools/gs_levels.py 5 1024 > gpurun_out/g7_gs_levels_c5.log 2>&1
