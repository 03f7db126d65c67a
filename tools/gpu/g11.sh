for ft in 1 0 1 0; do python bench.py --steps 3 --warmup 3 --no-cpu-baseline --family-timing $ft > gpurun_out/g11_bench_$ft.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/g11_bench_$ft.json').read().strip().splitlines()[-1]); print('ft $ft', d['value'], d['e2e']['value'])" >> gpurun_out/g11.log; done
