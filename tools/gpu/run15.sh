timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gauss_seidel or relax or improve" > gpurun_out/t15.log 2>&1
tail -2 gpurun_out/t15.log
timeout 1200 python -m pytest tests/test_gpu_config_scale.py -q -x -k "full_size or default_mode" >> gpurun_out/t15.log 2>&1
tail -2 gpurun_out/t15.log
for c in "5 1024" "2 1024" "3 1024"; do set -- $c
timeout 600 python tools/family_times.py --config $1 --size $2 --tag c$1 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "gauss|total" | tr '\n' ' '; echo
done
