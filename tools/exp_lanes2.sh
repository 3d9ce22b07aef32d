#!/bin/bash
# Part-A overlap on the small lanes: colour-group size and the prefetch cells-per-thread rule.
out=${1:-gpurun_out/exp_lanes2}; mkdir -p "$out"
run() { echo "== NB=$NB LAM=$LAM $*"; env "$@" python tools/profile_fit.py --fits 2 --lam $LAM --n-blocks $NB 2>&1 | tail -1; }
{
for NB in 41 30 22; do
  for LAM in 0.3 0.15; do
    export NB LAM
    run X=1
    run CONCORD_QB_PF_CELLS=8
    run CONCORD_QB_PF_CELLS=12
    run CONCORD_QB_PF_CELLS=20 CONCORD_QB_CW=-2
    run CONCORD_QB_PF_CELLS=20 CONCORD_QB_CW=-1
    run CONCORD_QB_PF_CELLS=20 CONCORD_QB_CW=-3
  done
done
for NB in 41; do LAM=0.3; export NB LAM
  CONCORD_PHASE_PROFILE=1 CONCORD_QB_PF_CELLS=20 CONCORD_QB_CW=-2 python tools/profile_fit.py --lam 0.3 --n-blocks 41 2>&1 | tail -20
done
} > "$out/knobs.log" 2>&1
