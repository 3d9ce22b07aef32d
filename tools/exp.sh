mkdir -p gpurun_out
CONCORD_SHARE_MIN=64 timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu64.log 2>&1; echo "pytest64 rc=$?" > gpurun_out/status.txt
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
