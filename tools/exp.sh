mkdir -p gpurun_out
for v in base u2 u8; do
  if [ $v = base ]; then lib=paper_2106_09382_b200/libconcord_b200.so; else lib=build/lib_$v.so; fi
  for cfg in "--p 5000 --n 2000 --lam 0.3" "--p 5000 --n 2000 --lam 0.15" "--p 5000 --n 2000 --lam 0.1" "--p 5000 --n 2000 --lam 0.0 --max-iter 2"; do
    echo "== $v $cfg" >> gpurun_out/ab.log
    CONCORD_LIB_PATH=$lib timeout 60 python tools/profile_fit.py $cfg --fits 1 2>&1 | grep -E "fit lam|Error" | sed 's/per-sweep.*//' >> gpurun_out/ab.log
  done
done
