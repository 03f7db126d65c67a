for ns in 32 0 8 128; do echo "CTA_NS $ns SW_NS $ns" >> gpurun_out/g28.log; AMGCU_GS_CTA_NS=$ns AMGCU_GS_SW_NS=$ns timeout 300 python tools/gs_levels.py 5 1024 >> gpurun_out/g28.log 2>&1; done
