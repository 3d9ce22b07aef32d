#!/bin/bash
# Quick gpurun: GPU tests + profile fits at p=1000/5000 (+ optional extra command in $EXTRA).
mkdir -p gpurun_out
timeout 300 python tools/profile_fit.py --p 1000 --n 500 --fits 2 > gpurun_out/profile_small.log 2>&1
echo "profile_small rc=$?" > gpurun_out/status.txt
timeout 300 python tools/profile_fit.py --p 5000 --n 2000 --fits 2 > gpurun_out/profile_5000.log 2>&1
echo "profile_5000 rc=$?" >> gpurun_out/status.txt
timeout 300 python tools/profile_fit.py --p 5000 --n 2000 --lam 0.1 --fits 1 > gpurun_out/profile_5000_l01.log 2>&1
echo "profile_5000_l0.1 rc=$?" >> gpurun_out/status.txt
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/status.txt
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; echo "extra rc=$?" >> gpurun_out/status.txt; fi
