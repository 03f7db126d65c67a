python -m pytest tests -m gpu -x -q > gpurun_out/t4.log 2>&1
tail -4 gpurun_out/t4.log
for c in "5 1024" "2 1024" "4 2048" "1 256"; do set -- $c
  AMGCU_BAND_TRACE=1 python tools/family_times.py --config $1 --size $2 --tag band > gpurun_out/fam_c$1_band.txt 2>&1
  grep -h "^\[band\] C" gpurun_out/fam_c$1_band.txt
done
grep -h "band\] n" gpurun_out/fam_c5_band.txt gpurun_out/fam_c4_band.txt | sort | uniq -c
