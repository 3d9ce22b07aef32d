"""More headline-size reference fixtures (run like make_golden_p5000.py; ~5 min per fit on 16 cores).

* odd p at the paper size: AR(2), p=5001, n=2000, lambda=0.3, cold -- the p-colour circle schedule
  with a phantom partner per round (schedule.py:53-88) at scale;
* a warm start at the paper size: AR(2), p=5000, n=2000, lambda=0.25 started from the reference's
  own lambda=0.30 estimate (SolverConfig.init, model.py:143,158-166) -- the warm lambda-path mode of
  pcd_path.
Both through the REAL reference package's stock pcd_fit (solver.py:254-294, compiled backend), on
the portable exact Gram (synth.portable_problem).  Output: tests/golden/p5000/extra_*.npz.
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
OUT = os.environ.get("P5K_OUT", os.path.join(HERE, "p5000"))


def record(path, pc, gram, rep, lam, tol, init_sha=None):
    from make_golden import sha
    from make_golden_p5000 import ambiguity

    om = rep.estimate.omega
    p = om.shape[0]
    iu = np.triu_indices(p, 1)
    upper = om[iu]
    mask = upper != 0.0
    np.savez_compressed(
        path, meta=np.array([p, gram.n, lam, tol]), tsha=np.frombuffer(sha(gram.t).encode(), np.uint8),
        omsha=np.frombuffer(sha(om).encode(), np.uint8), iters=np.array(rep.iterations),
        final_delta=np.array(rep.final_delta), edges=np.array(rep.edge_count), obj=np.array(rep.objective_trace),
        sweep_s=np.array(rep.wall_time_per_iteration), diag=np.diag(om).copy(), support=np.packbits(mask),
        values=upper[mask], ambiguous=ambiguity(om, gram.t, float(gram.n), lam),
        init_sha=np.frombuffer((init_sha or "").encode(), np.uint8))


def main():
    sys.path.insert(0, HERE)
    from make_golden import _import_reference, sha

    pc = _import_reference()
    sys.path.insert(0, REPO)
    from paper_2106_09382_b200 import synth

    os.makedirs(OUT, exist_ok=True)
    workers = int(os.environ.get("P5K_WORKERS", os.cpu_count()))
    # odd p at scale
    path = os.path.join(OUT, "extra_ar2_p5001_n2000_l0.30.npz")
    if not os.path.exists(path):
        x, t = synth.portable_problem("ar2", 5001, 2000, seed=0)
        gram = pc.GramMatrix(t, 2000)
        tic = time.time()
        rep = pc.pcd_fit(gram, pc.SolverConfig(lam=0.3, delta_tol=1e-5, max_outer_iterations=5000, workers=workers),
                         backend="compiled")
        record(path, pc, gram, rep, 0.3, 1e-5)
        print(f"p=5001 lam=0.30: iters={rep.iterations} edges={rep.edge_count} wall={time.time() - tic:.0f}s", flush=True)
    # warm start lambda 0.25 from the reference's own lambda 0.30 estimate
    path = os.path.join(OUT, "extra_ar2_p5000_n2000_l0.25_warm_from_0.30.npz")
    if not os.path.exists(path):
        x, t = synth.portable_problem("ar2", 5000, 2000, seed=0)
        gram = pc.GramMatrix(t, 2000)
        tic = time.time()
        cfg = pc.SolverConfig(lam=0.3, delta_tol=1e-5, max_outer_iterations=5000, workers=workers)
        first = pc.pcd_fit(gram, cfg, backend="compiled")
        cfg = pc.SolverConfig(lam=0.25, delta_tol=1e-5, max_outer_iterations=5000, workers=workers,
                              init=first.estimate)
        rep = pc.pcd_fit(gram, cfg, backend="compiled")
        record(path, pc, gram, rep, 0.25, 1e-5, init_sha=sha(first.estimate.omega))
        print(f"p=5000 lam=0.25 warm: iters={rep.iterations} edges={rep.edge_count} wall={time.time() - tic:.0f}s",
              flush=True)


if __name__ == "__main__":
    main()
