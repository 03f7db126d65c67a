AMGCU_PROF_OTHER=1 python tools/family_times.py --config 5 --size 1024 --tag other > gpurun_out/other_c5.txt 2>&1
AMGCU_SYNC_TRACE=1 python tools/profile_step.py --config 5 --size 1024 --reps 2 > gpurun_out/sync_c5.txt 2>&1
AMGCU_PHASE_TRACE=1 python tools/profile_step.py --config 5 --size 1024 --reps 2 > gpurun_out/phase_c5.txt 2>&1
