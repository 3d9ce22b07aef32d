mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/status.txt
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests -x -q -m gpu -k "device_check_optimality" > gpurun_out/memcheck_diag.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/status.txt
