mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab.log
CONCORD_DENSE_MIN=1 timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_dense1.log 2>&1; echo "pytest dense_min=1 rc=$?" >> gpurun_out/ab.log
for v in base t384; do
  if [ $v = base ]; then lib=paper_2106_09382_b200/libconcord_b200.so; else lib=build/lib_$v.so; fi
  for cfg in "--p 5000 --n 2000 --lam 0.3" "--p 5000 --n 2000 --lam 0.15" "--p 5000 --n 2000 --lam 0.1" "--p 5000 --n 2000 --lam 0.0 --max-iter 2"; do
    echo "== $v $cfg" >> gpurun_out/ab.log
    CONCORD_LIB_PATH=$lib timeout 60 python tools/profile_fit.py $cfg --fits 1 2>&1 | grep "fit lam" | sed 's/per-sweep.*//' >> gpurun_out/ab.log
  done
done
CONCORD_PHASE_PROFILE=1 timeout 60 python tools/profile_fit.py --p 5000 --n 2000 --lam 0.1 --fits 1 > gpurun_out/phase5000_l01.log 2>&1
