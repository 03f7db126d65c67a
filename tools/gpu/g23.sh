AMGCU_HOST_TRACE=1 AMGCU_SYNC_TRACE=1 AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 12 > gpurun_out/g23.log 2>&1
