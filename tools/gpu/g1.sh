nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/g1_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g1_pytest.log
timeout 600 python tools/mode_timing.py --config 2 --reps 2 > gpurun_out/g1_mode_c2.log 2>&1
timeout 900 python tools/mode_timing.py --config 5 --reps 2 > gpurun_out/g1_mode_c5.log 2>&1
