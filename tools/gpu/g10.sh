timeout 60 python tools/gs_small_check.py > gpurun_out/g10_small.log 2>&1; echo "exit $?" >> gpurun_out/g10_small.log
timeout 1500 python -m pytest tests/test_gpu_setup.py tests/test_gpu_kernels.py tests/test_gpu_golden.py tests/test_gpu_seqsum.py -q -x -p no:cacheprovider > gpurun_out/g10_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g10_pytest.log
timeout 900 python -m pytest tests/test_gpu_config_scale.py -q -x -p no:cacheprovider -k "C5-1024 or C2-1024 or C1-96 or C3-512 or C4-512 or overlap" >> gpurun_out/g10_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g10_pytest.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g10_bench.json 2> gpurun_out/g10_bench.err
