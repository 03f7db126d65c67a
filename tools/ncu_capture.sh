#!/bin/bash
# Full ncu captures of the hot kernels of one C2 setup+solve (tools/profile_step.py),
# after a plain run of the same command has exited 0.  Output: gpurun_out/<tag>_<kernel>.ncu-rep
set -u
tag=${1:-r02}
cmd="python tools/profile_step.py --reps 1"
timeout 300 $cmd > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
cap() {  # name regex skip count
    timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
        -k "regex:$2" -s "$3" -c "$4" -o "gpurun_out/${tag}_$1" $cmd > "gpurun_out/${tag}_$1.log" 2>&1
    echo "$1 rc=$?"
}
cap gs 'k_gs_lanes' 0 2
cap gs_seg 'k_gs_segments|k_gs_warp_rows' 0 2
cap lfmis 'k_lfmis_lists' 0 1
cap evolution 'k_evolution2' 0 1
cap spgemm_hash 'k_spgemm_hash' 3 1
cap spgemm_sort 'k_spgemm_small' 2 1
cap arnoldi 'k_arnoldi_coop' 0 1
cap masked 'k_masked_rows' 0 1
cap relax0 'k_relax0_residual' 0 1
cap jacobi 'k_jacobi_sweep' 0 6
cap prolong 'k_prolong' 0 6
cap sell_spmv 'k_sell_spmv' 0 8
cap vcycle_fused 'k_vcycle_fused' 0 1
cap count 'k_evolution_count' 0 1
