#!/bin/bash
# A/B: chain warps of the blocked kernel (build/lib_cwN.so from tools/build_variant.sh) per lane size.
out=${1:-gpurun_out/exp_cw}; mkdir -p "$out"
{
for lib in paper_2106_09382_b200/libconcord_b200.so build/lib_cw5.so build/lib_cw4.so; do
  for cfg in "66 0.1" "148 0.1" "41 0.3" "41 0.15" "148 0.3"; do
    set -- $cfg
    echo "== $lib nb=$1 lam=$2"
    CONCORD_LIB_PATH=$lib python tools/profile_fit.py --fits 2 --lam $2 --n-blocks $1 2>&1 | tail -1
  done
done
} > "$out/cw.log" 2>&1
