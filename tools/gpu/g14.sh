AMGCU_GS_LANES=0 AMGCU_GS_SEGWARP=2 timeout 300 python tools/gs_levels.py 5 1024 > gpurun_out/g14_segwarp_all_c5.log 2>&1
AMGCU_GS_LANES=0 AMGCU_GS_SEGWARP=2 timeout 300 python tools/gs_levels.py 2 1024 > gpurun_out/g14_segwarp_all_c2.log 2>&1
AMGCU_GS_CTA=0 timeout 300 python tools/gs_levels.py 5 1024 > gpurun_out/g14_nocta_c5.log 2>&1
