timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "matmul or transpose or spmv" > gpurun_out/t17.log 2>&1
tail -2 gpurun_out/t17.log
timeout 1200 python -m pytest tests/test_gpu_config_scale.py tests/test_gpu_golden.py -q -x -k "full_size or default_mode or golden" >> gpurun_out/t17.log 2>&1
tail -2 gpurun_out/t17.log
for c in "5 1024" "2 1024" "4 2048"; do set -- $c
timeout 600 python tools/family_times.py --config $1 --size $2 --tag c$1 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "spgemm|total|gauss" | tr '\n' ' '; echo
done
for g in 148 74; do AMGCU_FUSED_GRID=$g timeout 600 python tools/family_times.py --config 5 --size 1024 --tag fg$g 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "fused|fg" | tr '\n' ' '; echo; done
