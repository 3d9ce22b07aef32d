#!/bin/bash
# Kernel knobs at the lanes' CTA counts (41: the sparse lanes, 66: the dense lane).
# Usage (GPU box): tools/exp_lanes.sh OUTDIR
out=${1:-gpurun_out/exp_lanes}; mkdir -p "$out"
run() { echo "== $*"; env "$@" python tools/profile_fit.py --fits 2 --lam $LAM --n-blocks $NB 2>&1 | tail -1; }
{
for NB in 41 66; do
  for LAM in 0.3 0.1; do
    export NB LAM
    run X=1
    run CONCORD_QB_D=3
    run CONCORD_QB_CW=1
    run CONCORD_QB_CW=2
    run CONCORD_QB_CW=3
    run CONCORD_QB_NBUF=1
    run CONCORD_QB_RING=8
  done
done
} > "$out/knobs.log" 2>&1
