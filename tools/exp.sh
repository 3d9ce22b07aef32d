mkdir -p gpurun_out
for v in base t384 t384c2 lag4 t512c2; do
  if [ $v = base ]; then lib=paper_2106_09382_b200/libconcord_b200.so; else lib=build/lib_$v.so; fi
  for cfg in "--p 5000 --n 2000 --lam 0.3" "--p 5000 --n 2000 --lam 0.1" "--p 5000 --n 2000 --lam 0.0 --max-iter 2" "--p 1000 --n 500 --lam 0.3"; do
    echo "== $v $cfg" >> gpurun_out/ab.log
    CONCORD_LIB_PATH=$lib timeout 60 python tools/profile_fit.py $cfg --fits 1 2>&1 | grep "fit lam" | sed 's/per-sweep.*//' >> gpurun_out/ab.log
  done
done
