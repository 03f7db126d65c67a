SS_MODES=seq SS_SIZES=1000,16385,30000,100000,234000,1046529,2099200,4194304 timeout 300 python tools/seqsum_bench.py > gpurun_out/g35_ss.log 2>&1
timeout 600 python -m pytest tests/test_gpu_seqsum.py -q -x -p no:cacheprovider >> gpurun_out/g35_ss.log 2>&1
