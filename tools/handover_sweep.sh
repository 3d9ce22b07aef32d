for L in 66,28,27,27 60,30,29,29 56,31,31,30 70,26,26,26 66,41,41 56,46,46 74,74; do
  for H in 1 0; do
    LANES=$L HANDOVER=$H PASSES=4 QUIET=1 timeout 200 python tools/lane_probe.py 2>&1 | grep "=="
  done
done
