"""Solo fit time for every (lambda of the bench path, CTA count): the input of the lane planner.

    python tools/fit_matrix.py OUT.json [ctas ...]
Probe, not a bench number: each fit runs alone on a solver of n_blocks CTAs (one per SM).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_09382_b200 as cb  # noqa: E402
from paper_2106_09382_b200 import synth  # noqa: E402

out = sys.argv[1]
ctas = [int(v) for v in sys.argv[2:]] or [148, 111, 90, 82, 74, 66, 55, 48, 41, 37, 30, 25, 22, 18]
lams = [0.55, 0.50, 0.45, 0.40, 0.35, 0.30, 0.25, 0.20, 0.15, 0.10]
x, t = synth.portable_problem("ar2", 5000, 2000, seed=0)
g = cb.GramMatrix(t, 2000)
res = {}
for nb in ctas:
    s = cb.Solver(5000, n_blocks=nb)
    s.set_gram(g)
    for lam in lams:
        s.fit_raw(lam, 1e-5, 5000)  # warm
        rc, r, d, o, secs = s.fit_raw(lam, 1e-5, 5000)
        res[f"{nb}:{lam:.2f}"] = r.kernel_ms / 1e3
        print(nb, lam, round(r.kernel_ms / 1e3, 4), r.iterations, flush=True)
    s.close()
json.dump(res, open(out, "w"), indent=1)
