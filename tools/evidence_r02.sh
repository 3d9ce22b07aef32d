#!/bin/bash
# Round-2 evidence in one gpurun call (final kernel): smoke, bench, reference arm, ncu launch list,
# lambda-path DRAM traffic, one --set full capture of the dense fit on the full device.
o=${EV_OUT:-gpurun_out/ev_r02}; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $o/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/status.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $o/bench.json 2> $o/bench.err; echo "bench rc=$?" >> $o/status.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_ref.json 2>&1; echo "ref rc=$?" >> $o/status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $o/ncu_launch.log 2>&1; echo "launches rc=$?" >> $o/status.txt
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:pcd_ --csv \
    --log-file $o/traffic.csv python tools/ncu_fits.py --out $o/ncu_fits.json > $o/ncu_traffic.log 2>&1; echo "traffic rc=$?" >> $o/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcd_qblock -c 1 -o $o/ncu_full_l0.1 \
    python tools/profile_fit.py --lam 0.1 > $o/ncu_full.log 2>&1; echo "full rc=$?" >> $o/status.txt
