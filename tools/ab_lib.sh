for lib in base new; do
  if [ $lib = base ]; then export CONCORD_LIB_PATH=$PWD/paper_2106_09382_b200/libconcord_base.so; else unset CONCORD_LIB_PATH; fi
  echo "== $lib"
  python tools/profile_fit.py --lam 0.3 --n-blocks 27 --fits 2 2>&1 | grep "fit lam" | cut -c1-75
  python tools/profile_fit.py --lam 0.2 --n-blocks 27 --fits 1 2>&1 | grep "fit lam" | cut -c1-75
  python tools/profile_fit.py --lam 0.3 --fits 2 2>&1 | grep "fit lam" | cut -c1-75
  python tools/profile_fit.py --lam 0.1 --n-blocks 66 --fits 1 2>&1 | grep "fit lam" | cut -c1-75
  LANES=66,28,27,27 PASSES=4 QUIET=1 timeout 200 python tools/lane_probe.py 2>&1 | grep "=="
done

echo skip-tests
