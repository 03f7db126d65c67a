timeout 1500 python -m pytest tests/test_gpu_config_scale.py -v -p no:cacheprovider > gpurun_out/g26_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g26_pytest.log
