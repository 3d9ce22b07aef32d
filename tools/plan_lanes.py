"""Offline lane planner: from tools/fit_matrix.py's solo fit times, the lane split and assignment
that minimise the path's makespan (list scheduling, densest lambda first, each fit to the lane
where it would finish first).  Interference between concurrent lanes (shared HBM) is ignored, so
the ranking is a shortlist for tools/lane_probe.py, not a prediction.

    python tools/plan_lanes.py fit_matrix.json [max_lanes]
"""
import itertools
import json
import sys

m = json.load(open(sys.argv[1]))
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctas = sorted({int(k.split(":")[0]) for k in m})
lams = sorted({float(k.split(":")[1]) for k in m})


def makespan(lanes):
    fin = [0.0] * len(lanes)
    plan = [[] for _ in lanes]
    for lam in lams:  # densest first
        j = min(range(len(lanes)), key=lambda i: fin[i] + m[f"{lanes[i]}:{lam:.2f}"])
        fin[j] += m[f"{lanes[j]}:{lam:.2f}"]
        plan[j].append(lam)
    return max(fin), plan


best = []
for k in range(1, kmax + 1):
    for lanes in itertools.combinations_with_replacement(sorted(ctas, reverse=True), k):
        if sum(lanes) > 148:
            continue
        t, plan = makespan(list(lanes))
        best.append((t, lanes, plan))
best.sort()
for t, lanes, plan in best[:15]:
    print(f"{t:.3f} s  lanes={lanes}  " + "  ".join(f"{c}:{p}" for c, p in zip(lanes, plan)))
