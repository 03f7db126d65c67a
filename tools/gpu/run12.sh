python -m pytest tests -m gpu -x -q > gpurun_out/t12.log 2>&1
tail -3 gpurun_out/t12.log
python bench.py > gpurun_out/b5.json 2> gpurun_out/b5.err
for c in 1 2 4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/b$c.json 2> gpurun_out/b$c.err; done
python - <<'PY'
import json
for c in (5,1,2,4):
    try:
        d=json.loads(open(f'gpurun_out/b{c}.json').read().strip().splitlines()[-1])
        print(c, d['ms_per_step'], d['e2e']['value'], d['result'], d['roofline']['kernel'], d['roofline']['frac'])
    except Exception as e: print(c,'ERR',e)
PY
