#!/bin/bash
# Row-major vs slab storage (CONCORD_LAYOUT=slab) for single fits at the lanes' CTA counts and full device.
out=${1:-gpurun_out/exp_layout}; mkdir -p "$out"
{
for rep in 1 2; do
for lay in rowmajor slab; do
  for cfg in "0 0.1" "0 0.3" "66 0.1" "41 0.3" "41 0.15"; do
    set -- $cfg
    echo "== $lay nb=$1 lam=$2"
    CONCORD_LAYOUT=$lay python tools/profile_fit.py --fits 2 --lam $2 --n-blocks $1 2>&1 | tail -1
  done
done
done
} > "$out/layout.log" 2>&1
