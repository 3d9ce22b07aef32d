#!/bin/bash
# A/B of two builds of the library in one gpurun call: copy the baseline build to
# paper_2106_09382_b200/libconcord_base.so (git-ignored, travels with the snapshot), rebuild the
# candidate in place, run this.  Single fits on a 27-SM lane and the full device, the dense fit on
# a 66-SM lane, and the bench path on 4 lanes (profiles/r02/ab_speculative_T_loads.log).
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
