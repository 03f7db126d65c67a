AMGCU_PHASE_TRACE=1 AMGCU_SYNC_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 8 > gpurun_out/g19_phases_lazy.log 2>&1
CUDA_MODULE_LOADING=EAGER AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 8 > gpurun_out/g19_phases_eager.log 2>&1
