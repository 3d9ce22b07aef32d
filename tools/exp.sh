mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/gpu.txt 2>&1; nproc >> gpurun_out/gpu.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" > gpurun_out/status.txt
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/status.txt
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?" >> gpurun_out/status.txt
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:pcd_wform --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/ncu_fits.py > gpurun_out/ncu_traffic.log 2>&1; echo "traffic rc=$?" >> gpurun_out/status.txt
timeout 900 ncu --set full --import-source on -k regex:pcd_wform --clock-control none -c 1 -o gpurun_out/prof_wform_r01_final python tools/ncu_fits.py --lams 0.3 --out gpurun_out/ncu_fit03.json > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?" >> gpurun_out/status.txt
