for L in 66,28,27,27 74,37,37 74,25,25,24 63,29,28,28 66,30,26,26; do
  LANES=$L HANDOVER=1 PASSES=4 QUIET=1 timeout 200 python tools/lane_probe.py 2>&1 | grep "=="
done
