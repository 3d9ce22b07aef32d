"""Fit one AR(2) problem generated on the device (large-p timing helper; not a bench number)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2106_09382_b200 as cb
p, n, lam = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
s = cb.Solver(p)
s.gram_from_ar2(n, seed=0)
rc, res, d, o, secs = s.fit_raw(lam, 1e-5, 500)
print(f"p={p} kernel_D={s.layout()['kernel']} lam={lam} iters={res.iterations} edges={res.edge_count} kernel={res.kernel_ms/1e3:.3f}s "
      f"ms/sweep={np.median(secs)*1e3:.1f}", flush=True)
