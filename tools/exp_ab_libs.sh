#!/bin/bash
# A/B of library builds (build/lib_*.so) on single fits at the lanes' CTA counts.
out=${1:-gpurun_out/exp_ab}; shift; mkdir -p "$out"
libs=${@:-build/lib_preshard.so build/lib_now.so}
{
for rep in 1 2; do
for lib in $libs; do
  for cfg in "41 0.55" "41 0.3" "41 0.15" "66 0.1" "0 0.3"; do
    set -- $cfg
    echo "== $lib nb=$1 lam=$2"
    CONCORD_LIB_PATH=$lib python tools/profile_fit.py --fits 2 --lam $2 --n-blocks $1 2>&1 | tail -1
  done
done
done
} > "$out/ab.log" 2>&1
