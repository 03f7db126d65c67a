for v in "A" "B" "C"; do
  case $v in
    A) ENV="X=1"; EXTRA="";;
    B) ENV="AMGCU_RHO_OVERLAP=0"; EXTRA="";;
    C) ENV="AMGCU_RHO_OVERLAP=0"; EXTRA="--no-cand-overlap";;
  esac
  env $ENV AMGCU_PHASE_TRACE=1 timeout 600 python tools/profile_step.py --config 5 --size 1024 --reps 10 $EXTRA > gpurun_out/g21_$v.log 2>&1
done
