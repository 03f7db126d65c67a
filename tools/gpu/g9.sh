for args in "p1d3 2 1" "p1d30 2 1" "p1d30 1 8" "spd40 2 1" "aniso8 2 1"; do
  timeout 30 python tools/gs_small_check.py $args >> gpurun_out/g9_small.log 2>&1; echo "[$args] exit $?" >> gpurun_out/g9_small.log
done
timeout 120 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python tools/gs_small_check.py p1d3 2 1 > gpurun_out/g9_racecheck.log 2>&1; echo "exit $?" >> gpurun_out/g9_racecheck.log
