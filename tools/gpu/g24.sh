AMGCU_SS_TRACE=1 SS_MODES=seq SS_SIZES=30000,234000,2099200 timeout 300 python tools/seqsum_bench.py > gpurun_out/g24_sstrace.log 2>&1
