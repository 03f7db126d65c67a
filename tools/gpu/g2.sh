# round 2, call 2: C5 bench in the default (reference-exact) mode, host/sync traces, full-size parity for C2/C5 + overlap
python bench.py --steps 3 --warmup 3 > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err
AMGCU_HOST_TRACE=1 AMGCU_SYNC_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 2 > gpurun_out/g2_trace_c5.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_config_scale.py -q -x -p no:cacheprovider -k "C2-1024 or C5-1024 or overlap or tree" > gpurun_out/g2_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g2_pytest.log
