for b in 2 3 4 6 8; do
AMGCU_CGCOL_BLOCKS_PER_SM=$b timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/cg_$b.csv -k regex:k_cg_columns -c 4 python tools/profile_step.py --config 5 --size 1024 --reps 1 > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.DictReader([l for l in open('gpurun_out/cg_$b.csv') if l.startswith('"')])]
t=[float(r['Metric Value'].replace(',',''))/1000 for r in rows if r['Metric Name']=='gpu__time_duration.sum']
d=[float(r['Metric Value'].replace(',','')) for r in rows if r['Metric Name']=='dram__bytes_read.sum']
print('blocks/SM $b', [round(x,1) for x in t], [round(x,1) for x in d], rows[0]['Metric Unit'] if rows else '')
PY
done
