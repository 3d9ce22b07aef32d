mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/status.txt
