timeout 900 python -m pytest tests/test_gpu_seqsum.py tests/test_gpu_kernels.py -q -x -k "seqsum or dot or spectral" > gpurun_out/t_ss.log 2>&1
tail -2 gpurun_out/t_ss.log
python tools/ss_trace_cfg.py 3 2048 30 3 2>/dev/null
for c in "5 1024" "2 1024"; do set -- $c
python tools/family_times.py --config $1 --size $2 --tag c$1 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "blas1|total" | tr '\n' ' '; echo
done
timeout 1200 python -m pytest tests/test_gpu_config_scale.py -q -x -k "full_size" >> gpurun_out/t_ss.log 2>&1
tail -2 gpurun_out/t_ss.log
