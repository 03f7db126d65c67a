python tools/family_times.py --config 2 --size 1024 --tag a 2>&1 | grep "^\["
python tools/family_times.py --config 2 --size 1024 --tag b 2>&1 | grep "^\["
for i in 1 2; do python bench.py --config 2 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2', d['ms_per_step'], d['e2e']['value'], d['clocks'])"; done
