# ncu --set full of the band masked product / cg columns on C5, C2, C4 level 0, then the sanitizer runs
cap() {  # tag cfg size name regex skip count
    timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
        -k "regex:$5" -s "$6" -c "$7" -o "gpurun_out/r04_c$2_$4" python tools/profile_step.py --config $2 --size $3 --reps 1 > "gpurun_out/r04_c$2_$4.log" 2>&1
    echo "$4 c$2 rc=$?"
}
cap r04 5 1024 band 'k_masked_band' 1 1
cap r04 5 1024 band_l1 'k_masked_band' 6 1
cap r04 5 1024 cgcol 'k_cg_columns' 0 1
cap r04 2 1024 band 'k_masked_band' 1 1
cap r04 4 2048 band 'k_masked_band' 1 1
for f in gpurun_out/r04_*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}.raw.csv 2>/dev/null
done
bash tools/sanitize.sh memcheck racecheck synccheck
cat gpurun_out/sanitize_*.log
