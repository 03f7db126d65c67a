for env in "X=1" "AMGCU_GS_LANES=0 AMGCU_GS_SEGWARP=2"; do echo "== $env" >> gpurun_out/g16.log; env $env timeout 300 python tools/gs_l0_repeat.py 5 1024 5 >> gpurun_out/g16.log 2>&1; done
for env in "X=1" "AMGCU_GS_LANES=0 AMGCU_GS_SEGWARP=2"; do echo "== C2 $env" >> gpurun_out/g16.log; env $env timeout 300 python tools/gs_l0_repeat.py 2 1024 3 >> gpurun_out/g16.log 2>&1; done
