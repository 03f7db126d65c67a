AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 6 > gpurun_out/g12_phases.log 2>&1
