timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k "regex:k_masked_band" -s 1 -c 1 -o gpurun_out/x_band python tools/profile_step.py --config 5 --size 1024 --reps 1 > gpurun_out/x_band.log 2>&1
ncu -i gpurun_out/x_band.ncu-rep --page source --csv > gpurun_out/x_band_source.csv 2>/dev/null
ncu -i gpurun_out/x_band.ncu-rep --page raw --csv > gpurun_out/x_band_raw.csv 2>/dev/null
rm -f gpurun_out/x_band.ncu-rep
