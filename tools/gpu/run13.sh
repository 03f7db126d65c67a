python -m pytest tests/test_gpu_setup.py tests/test_gpu_golden.py -q -x -k "fused or golden" > gpurun_out/t13.log 2>&1
tail -2 gpurun_out/t13.log
for nz in 100000000 1500000 300000; do
for c in "5 1024" "2 1024" "4 2048"; do set -- $c
AMGCU_FUSED_MAX_NNZ=$nz python tools/family_times.py --config $1 --size $2 --tag nnz$nz-c$1 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "nnz|vcycle|total" | tr '\n' ' '; echo
done; done
