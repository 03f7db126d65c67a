python -m pytest tests/test_gpu_config_scale.py tests/test_gpu_setup.py tests/test_gpu_golden.py -q -x -k "masked_band or ledger or golden or full_size" > gpurun_out/t6.log 2>&1
tail -3 gpurun_out/t6.log
for b in 2 4 8; do
  AMGCU_CGCOL_BLOCKS_PER_SM=$b python tools/family_times.py --config 5 --size 1024 --tag cgcol$b 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "cgcol|emin_" | tr '\n' ' '; echo
done
AMGCU_CGCOL_BLOCKS_PER_SM=4 python tools/family_times.py --config 2 --size 1024 --tag c2cg4 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "emin_" | tr '\n' ' '; echo
python tools/family_times.py --config 2 --size 1024 --tag c2cg2 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "emin_" | tr '\n' ' '; echo
python tools/family_times.py --config 4 --size 2048 --tag c4 2>&1 | grep "^\[" | tr ' ' '\n' | grep -E "emin_" | tr '\n' ' '; echo
AMGCU_FUSED_TRACE=1 python tools/profile_step.py --config 5 --size 1024 --reps 1 2>&1 | grep "fused" | tail -3
