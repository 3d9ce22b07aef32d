#!/bin/bash
# Sector alignment of the slab rows: w=34 (148 CTAs, 272-byte rows) vs w=36 (139 CTAs, 288 bytes = 9 sectors).
out=${1:-gpurun_out/exp_align}; mkdir -p "$out"
{
for cfg in "148 0.1" "139 0.1" "148 0.3" "139 0.3" "41 0.3" "42 0.3" "41 0.15" "42 0.15"; do
  set -- $cfg
  echo "== nb=$1 lam=$2"
  python tools/profile_fit.py --fits 2 --lam $2 --n-blocks $1 2>&1 | tail -1
done
} > "$out/align.log" 2>&1
