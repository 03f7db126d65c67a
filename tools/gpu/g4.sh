timeout 600 python tools/prof_overhead.py 5 1024 > gpurun_out/g4_prof_overhead.log 2>&1
timeout 600 python tools/gs_levels.py 5 1024 > gpurun_out/g4_gs_levels_c5.log 2>&1
timeout 600 python tools/level_stats.py 5 1024 > gpurun_out/g4_level_stats_c5.log 2>&1
SS_SIZES=100,1000,4000,16384,16385,30000,100000,300000,1046529,2099200 timeout 600 python tools/seqsum_bench.py > gpurun_out/g4_seqsum.log 2>&1
