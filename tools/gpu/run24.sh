python -m pytest tests -m gpu -x -q > gpurun_out/t24.log 2>&1
tail -2 gpurun_out/t24.log
python bench.py --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', d['ms_per_step'], d['e2e']['value'], d['result'])"
python bench.py --config 2 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2', d['ms_per_step'], d['e2e']['value'], d['result'])"
