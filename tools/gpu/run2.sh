python -m pytest tests/test_gpu_config_scale.py -q -x -k "masked_band" > gpurun_out/t2.log 2>&1
tail -5 gpurun_out/t2.log
for c in "5 1024" "2 1024" "4 2048"; do set -- $c
  AMGCU_PROF_OTHER=1 python tools/family_times.py --config $1 --size $2 --tag band > gpurun_out/fam_c$1_band.txt 2>&1
  AMGCU_MASKED_BAND=0 python tools/family_times.py --config $1 --size $2 --tag noband > gpurun_out/fam_c$1_noband.txt 2>&1
  grep -h "^\[" gpurun_out/fam_c$1_band.txt gpurun_out/fam_c$1_noband.txt
done
