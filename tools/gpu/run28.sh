timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_setup.py -q -x -k "gauss_seidel or relax or improve or remaining" > gpurun_out/t28.log 2>&1
tail -2 gpurun_out/t28.log
timeout 1500 python -m pytest tests/test_gpu_config_scale.py -q -x >> gpurun_out/t28.log 2>&1
tail -2 gpurun_out/t28.log
python tools/gs_levels.py 5 1024 2>&1 | tail -9
AMGCU_GS_SW_WIDE=0 python tools/gs_levels.py 5 1024 2>&1 | tail -9
for c in "5 1024" "3 1024"; do set -- $c
timeout 600 python tools/family_times.py --config $1 --size $2 --tag c$1 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "gauss|total" | tr '\n' ' '; echo
done
python bench.py --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5', d['ms_per_step'], d['e2e']['value'], d['result'])"
