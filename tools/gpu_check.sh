#!/bin/bash
# One gpurun call: GPU tests, smoke, quick profile fits, bench, ncu launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
timeout 300 python tools/profile_fit.py --p 1000 --n 500 --fits 2 > gpurun_out/profile_small.log 2>&1
echo "profile_small rc=$?" >> gpurun_out/status.txt
timeout 300 python tools/profile_fit.py --p 5000 --n 2000 --fits 2 > gpurun_out/profile_5000.log 2>&1
echo "profile_5000 rc=$?" >> gpurun_out/status.txt
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_fit.py --p 5000 --n 2000 --fits 1 > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcd_ -c 1 -o gpurun_out/prof_wform python tools/profile_fit.py --p 5000 --n 2000 --fits 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/status.txt
