timeout 300 python tools/gs_levels.py 5 1024 > gpurun_out/g44_gs_c5.log 2>&1
timeout 300 python tools/gs_levels.py 2 1024 >> gpurun_out/g44_gs_c5.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "gauss or candidates or segment or cta" > gpurun_out/g44_pytest.log 2>&1; echo "exit $?" >> gpurun_out/g44_pytest.log
timeout 900 python -m pytest tests/test_gpu_config_scale.py -q -x -p no:cacheprovider -k "C5 or C2" >> gpurun_out/g44_pytest.log 2>&1; echo "exit $?" >> gpurun_out/g44_pytest.log
