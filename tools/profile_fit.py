"""One CONCORD-PCD fit for ncu / quick timing (not a bench number).

    python tools/profile_fit.py [--p 5000] [--n 2000] [--lam 0.3] [--fits 1]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_09382_b200 as cb  # noqa: E402
from paper_2106_09382_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=5000)
ap.add_argument("--n", type=int, default=2000)
ap.add_argument("--lam", type=float, default=0.3)
ap.add_argument("--fits", type=int, default=1)
ap.add_argument("--n-blocks", type=int, default=0)
ap.add_argument("--max-iter", type=int, default=5000)
a = ap.parse_args()
x = (synth.portable_problem("ar2", a.p, a.n, seed=0)[0] if a.p <= 8000
     else synth.center(synth.sample_mvn_ar2_banded(a.p, a.n, seed=0)))
s = cb.Solver(a.p, n_blocks=a.n_blocks)
t0 = time.perf_counter()
s.gram_from_data(cb.DataMatrix(x))
print(f"gram {time.perf_counter() - t0:.3f}s", flush=True)
for i in range(a.fits):
    rc, res, deltas, objs, secs = s.fit_raw(a.lam, 1e-5, a.max_iter)
    print(f"fit lam={a.lam} iters={res.iterations} conv={res.converged} edges={res.edge_count} "
          f"kernel={res.kernel_ms:.3f}ms setup={res.setup_ms:.3f}ms blocks={res.n_blocks} w={res.slab_width} "
          f"per-sweep(ms)={np.round(secs * 1e3, 3).tolist()[:6]}...", flush=True)
