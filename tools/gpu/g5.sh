for ns in 32 256 1024 4096; do echo "WR_NS $ns"; AMGCU_GS_WR_NS=$ns timeout 300 python tools/gs_levels.py 5 1024; done > gpurun_out/g5_wr_ns.log 2>&1
for rm in 0 1; do echo "ROWMAJOR $rm"; AMGCU_GS_ROWMAJOR=$rm timeout 300 python tools/gs_levels.py 5 1024; done > gpurun_out/g5_rowmajor.log 2>&1
