timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_setup.py -q -x -k "gauss_seidel or relax or improve or remaining" > gpurun_out/t20.log 2>&1
tail -2 gpurun_out/t20.log
timeout 1200 python -m pytest tests/test_gpu_config_scale.py -q -x -k "full_size or default_mode" >> gpurun_out/t20.log 2>&1
tail -2 gpurun_out/t20.log
python tools/gs_chain_rate.py 2>&1 | tail -6
for c in "5 1024" "2 1024" "3 1024"; do set -- $c
timeout 600 python tools/family_times.py --config $1 --size $2 --tag c$1 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "gauss|total" | tr '\n' ' '; echo
done
