for L in 66,28,27,27 64,28,28,28 62,29,29,28 68,27,27,26 66,21,21,20,20 58,23,23,22,22; do
  LANES=$L HANDOVER=1 PASSES=4 QUIET=1 timeout 200 python tools/lane_probe.py 2>&1 | grep "=="
done
