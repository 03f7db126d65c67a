echo "CTA=0 MINLEN=1" >> gpurun_out/g29.log; AMGCU_GS_CTA=0 AMGCU_GS_SW_MINLEN=1 timeout 300 python tools/gs_levels.py 5 1024 >> gpurun_out/g29.log 2>&1
echo "CTA=0 MINLEN=1 C2" >> gpurun_out/g29.log; AMGCU_GS_CTA=0 AMGCU_GS_SW_MINLEN=1 timeout 300 python tools/gs_levels.py 2 1024 >> gpurun_out/g29.log 2>&1
