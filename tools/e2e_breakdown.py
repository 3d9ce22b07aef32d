"""Where the end-to-end pcd_fit time goes at the bench workload (not a bench number)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2106_09382_b200 as cb
from paper_2106_09382_b200 import _lib, synth
from paper_2106_09382_b200.solver import Solver

p, n = 5000, 2000
x = synth.center(synth.sample_mvn(synth.ar2_precision(p), n, seed=0))
s0 = cb.Solver(p)
s0.gram_from_data(cb.DataMatrix(x, centered=True))
tp = _lib.pinned_empty((p, p))
tp[...] = s0.gram().t
s0.close()
g = cb.GramMatrix(tp, n)
cfg = cb.SolverConfig(lam=0.3, max_outer_iterations=5000)
for rep in range(3):
    t0 = time.perf_counter()
    s = Solver(p, device=0)
    t1 = time.perf_counter()
    s.set_gram(g)
    t2 = time.perf_counter()
    rc, res, d, o, secs = s.fit_raw(0.3, 1e-5, 5000)
    t3 = time.perf_counter()
    om = s.omega()
    t4 = time.perf_counter()
    rep_ = cb.pcd_fit(g, cfg)
    t5 = time.perf_counter()
    print(f"pool {1e3*(t1-t0):.1f} set_gram {1e3*(t2-t1):.1f} fit_raw {1e3*(t3-t2):.1f} (kernel {res.kernel_ms:.1f} setup {res.setup_ms:.1f}) "
          f"omega {1e3*(t4-t3):.1f} | pcd_fit total {1e3*(t5-t4):.1f} ms", flush=True)
