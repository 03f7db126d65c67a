AMGCU_SS_TRACE=1 timeout 600 python tools/ss_solve_trace.py 1024 > gpurun_out/g34_sstrace.log 2>&1
