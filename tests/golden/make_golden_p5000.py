"""Reference fixtures for the headline workload (BASELINE configs[2]): AR(2), p=5000, n=2000, seed 0.

Run in the build container (needs /root/reference; about 1 min per sweep on 8 cores) or on
the GPU box's 16 host cores with the reference staged under baseline/_ref/pkg by
tools/stage_reference_suite.py (about 12 s per sweep):

    python tests/golden/make_golden_p5000.py [lam ...]

For every lambda of the bench path it runs the REAL reference package's stock
`pcd_fit` loop (`/root/reference/pkg/src/parconcord/solver.py:254-294`) with the
compiled `_ckernels.pcd_sweep` (`_ckernels.pyx:68-102`), cold from the identity,
delta_tol 1e-5, on the reference's own generators
(`datagen.ar2_precision` -> `sample_mvn` -> `center_columns`), with X rounded
onto the exact-Gram grid of `synth.quantize_exact_gram` so that T = X^T X is
the same bits on every machine (BLAS kernel and thread count change the last
bits of an unrounded Gram); the reference's own `compute_gram` is asserted to
give exactly that T.
It writes one compact fixture per lambda to tests/golden/p5000/:

* meta (p, n, lam, delta_tol), sha256 of T (the GPU test regenerates T from the
  seed with `synth`, which is bitwise the reference generator, and checks it);
* iterations, final_delta, edge_count, the objective trace, the reference's own
  `wall_time_per_iteration` (sweep + delta, `solver.py:284-288`) and workers;
* the diagonal of Omega, the strict-upper support as a packed bitmask
  (row-major over i<j), and the non-zero values in that order;
* an ambiguity census of the final iterate: the pairs whose soft-threshold
  argument |num| sits within 1e-10 / 1e-8 / 1e-6 (relative) of n*lam, where
  `num` is the `_offdiag_value` numerator (`_ckernels.pyx:25-38`) evaluated at
  the final Omega (support flips can only come from those pairs).

Resumable: lambdas whose fixture exists are skipped.
"""

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
OUT = os.environ.get("P5K_OUT", os.path.join(HERE, "p5000"))
P, N, TOL = 5000, 2000, 1e-5
LAMS = [0.30, 0.10, 0.20, 0.15, 0.55, 0.50, 0.45, 0.40, 0.35, 0.25]


def fixture_name(lam):
    return os.path.join(OUT, f"ar2_p{P}_n{N}_l{lam:.2f}.npz")


def ambiguity(omega, t, n, lam):
    w = omega @ t
    num = -(w + w.T - omega * (np.diag(t)[:, None] + np.diag(t)[None, :]))
    iu = np.triu_indices(omega.shape[0], 1)
    shrink = n * lam
    rel = np.abs(np.abs(num[iu]) - shrink) / shrink
    return np.array([int((rel < e).sum()) for e in (1e-10, 1e-8, 1e-6)], dtype=np.int64)


def main():
    sys.path.insert(0, HERE)
    from make_golden import _import_reference, sha

    pc = _import_reference()
    sys.path.insert(0, REPO)
    from paper_2106_09382_b200 import synth

    os.makedirs(OUT, exist_ok=True)
    lams = [float(a) for a in sys.argv[1:]] or LAMS
    x, t = synth.portable_problem("ar2", P, N, seed=0)
    assert np.array_equal(pc.compute_gram(pc.DataMatrix(x)).t, t)  # the reference's own Gram, bitwise
    gram = pc.GramMatrix(t, N)
    tsha = sha(gram.t)
    workers = int(os.environ.get("P5K_WORKERS", os.cpu_count()))
    iu = np.triu_indices(P, 1)
    for lam in lams:
        path = fixture_name(lam)
        if os.path.exists(path):
            print("exists", path)
            continue
        tic = time.time()
        cfg = pc.SolverConfig(lam=lam, delta_tol=TOL, max_outer_iterations=5000, workers=workers)
        rep = pc.pcd_fit(gram, cfg, backend="compiled")  # stock path: builds its own schedule
        om = rep.estimate.omega
        upper = om[iu]
        mask = upper != 0.0
        np.savez_compressed(
            path,
            meta=np.array([P, N, lam, TOL]),
            tsha=np.frombuffer(tsha.encode(), np.uint8),
            omsha=np.frombuffer(sha(om).encode(), np.uint8),
            iters=np.array(rep.iterations),
            final_delta=np.array(rep.final_delta),
            edges=np.array(rep.edge_count),
            obj=np.array(rep.objective_trace),
            sweep_s=np.array(rep.wall_time_per_iteration),
            workers=np.array(workers),
            diag=np.diag(om).copy(),
            support=np.packbits(mask),
            values=upper[mask],
            ambiguous=ambiguity(om, gram.t, float(gram.n), lam),
        )
        print(f"lam={lam:.2f}: iters={rep.iterations} edges={rep.edge_count} delta={rep.final_delta:.3e} "
              f"sum(sweep_s)={sum(rep.wall_time_per_iteration):.1f}s wall={time.time() - tic:.0f}s", flush=True)


if __name__ == "__main__":
    main()
