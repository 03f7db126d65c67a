timeout 60 python tools/gs_small_check.py > gpurun_out/g8_small.log 2>&1; echo "exit $?" >> gpurun_out/g8_small.log
AMGCU_GS_CTA=0 timeout 60 python tools/gs_small_check.py > gpurun_out/g8_small_nocta.log 2>&1; echo "exit $?" >> gpurun_out/g8_small_nocta.log
