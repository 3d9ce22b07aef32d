mkdir -p gpurun_out
export CONCORD_PHASE_PROFILE=1
timeout 60 python tools/profile_fit.py --p 5000 --n 2000 --lam 0.3 --fits 1 > gpurun_out/phase_03.log 2>&1
unset CONCORD_PHASE_PROFILE
for cfg in "--p 5000 --n 2000 --lam 0.1" "--p 1000 --n 500 --lam 0.3"; do
  timeout 60 python tools/profile_fit.py $cfg --fits 1 2>&1 | grep -E "fit lam|Error" | sed 's/per-sweep.*//' >> gpurun_out/ab.log
done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/status.txt
