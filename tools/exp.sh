mkdir -p gpurun_out
timeout 600 python bench.py --mode sharded --steps 2 --warmup 1 --no-e2e > gpurun_out/bench_sharded1.log 2>&1; echo "sharded rc=$?" > gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/status.txt
