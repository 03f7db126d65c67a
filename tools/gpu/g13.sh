timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "segment_warps or gauss_seidel_cta or improve_candidates" > gpurun_out/g13_pytest.log 2>&1; echo "exit $?" >> gpurun_out/g13_pytest.log
timeout 300 python tools/gs_levels.py 5 1024 > gpurun_out/g13_gs_levels_c5.log 2>&1
