for env in "AMGCU_GS_LANES=0 AMGCU_GS_SEGWARP=2"; do echo "== $env" >> gpurun_out/g17.log; env $env timeout 300 python tools/gs_l0_repeat.py 5 1024 3 >> gpurun_out/g17.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "segment_warps or gauss_seidel or improve_candidates" >> gpurun_out/g17.log 2>&1; echo "exit $?" >> gpurun_out/g17.log
