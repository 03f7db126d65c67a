#!/bin/bash
# Full ncu captures of the hot kernels of one C5 setup+solve (tools/profile_step.py,
# config 5 at 1024^2 -- the bench workload), after a plain run of the same command has
# exited 0.  Output: gpurun_out/<tag>_<name>.ncu-rep; summarised by tools/ncu_summary.py.
set -u
tag=${1:-r04}
cmd="python tools/profile_step.py --config 5 --size 1024 --reps 1"
timeout 300 $cmd > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
cap() {  # name regex skip count
    timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
        -k "regex:$2" -s "$3" -c "$4" -o "gpurun_out/${tag}_$1" $cmd > "gpurun_out/${tag}_$1.log" 2>&1
    echo "$1 rc=$?"
}
cap seqsum 'k_seqsum$' 0 3
cap gs_segwarp 'k_gs_seg_warp' 0 1
cap spgemm_bitmap 'k_spgemm_bitmap' 0 4
cap masked_band 'k_masked_band' 1 2
cap relax0 'k_relax0_residual' 0 1
cap jacobi 'k_jacobi_sweep' 0 1
cap prolong 'k_prolong' 0 2
cap sell_spmv 'k_sell_spmv' 0 3
cap vcycle_fused 'k_vcycle_fused' 0 1
cap lfmis 'k_lfmis_lists' 0 1
cap gauss_jordan 'k_gauss_jordan' 0 1
cap cg_columns 'k_cg_columns' 0 1
