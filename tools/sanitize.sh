#!/bin/bash
# compute-sanitizer over the sync-free kernels (spin-on-flag wavefronts: aggregation
# pass 1, Gauss-Seidel lanes / segments / single CTA, gsne and block GS) and the TMA
# band kernel, on small cases, on a B200 box.  Writes gpurun_out/sanitize_<tool>.log;
# summaries are copied to profiles/ by hand.
#   usage: tools/sanitize.sh [memcheck|racecheck|synccheck ...]
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TOOLS=${@:-memcheck racecheck synccheck}
SEL='aggregation_known or aggregation_random or gauss_seidel_cta or gauss_seidel_segment or gauss_seidel_lane or relax'
for t in $TOOLS; do
  timeout 1500 compute-sanitizer --tool $t --target-processes all --error-exitcode 7 \
    --log-file gpurun_out/sanitize_$t.raw \
    python -m pytest tests/test_gpu_kernels.py -q -x -k "$SEL" -p no:cacheprovider > gpurun_out/sanitize_$t.pytest 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$t.pytest
  timeout 1500 compute-sanitizer --tool $t --target-processes all --error-exitcode 7 \
    --log-file gpurun_out/sanitize_${t}_setup.raw \
    python -m pytest tests/test_gpu_config_scale.py -q -x -k "masked_band and (C1-96 or C5-96)" -p no:cacheprovider > gpurun_out/sanitize_${t}_setup.pytest 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${t}_setup.pytest
  for f in gpurun_out/sanitize_$t.raw gpurun_out/sanitize_${t}_setup.raw; do
    { echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Invalid|error" $f | sort | uniq -c | head -40; } >> gpurun_out/sanitize_$t.log
  done
  tail -3 gpurun_out/sanitize_$t.pytest gpurun_out/sanitize_${t}_setup.pytest >> gpurun_out/sanitize_$t.log
done
