#!/bin/bash
# In-kernel phase profiles (CONCORD_PHASE_PROFILE=1, CTA 0 cycle counters) of single fits at the
# CTA counts the bench's lanes use.  Usage (GPU box): tools/phase_sweep.sh OUTDIR [lam...]
out=${1:-gpurun_out/phase}; shift
lams=${@:-0.3 0.2 0.1}
mkdir -p "$out"
for nb in 148 66 41; do
  for lam in $lams; do
    CONCORD_PHASE_PROFILE=1 timeout 120 python tools/profile_fit.py --lam "$lam" --n-blocks "$nb" \
      > "$out/phase_nb${nb}_l${lam}.log" 2>&1
    python tools/profile_fit.py --lam "$lam" --n-blocks "$nb" --fits 2 > "$out/time_nb${nb}_l${lam}.log" 2>&1
  done
done
