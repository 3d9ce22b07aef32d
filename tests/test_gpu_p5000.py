"""Parity at the headline workload (BASELINE configs[2]): AR(2), p=5000, n=2000, seed 0.

North-star acceptance criterion: "the p=5000, n=2000 paper workload converges to
the reference's Omega (same support, within tolerance)".  The fixtures in
tests/golden/p5000/ were produced by the REAL reference package's stock
`pcd_fit` loop (`/root/reference/pkg/src/parconcord/solver.py:254-294`, compiled
`_ckernels.pcd_sweep`, `_ckernels.pyx:68-102`) by tests/golden/make_golden_p5000.py,
on the portable exact Gram (synth.portable_problem: the same T bits on every
machine, pinned here by its sha256).

For every fixture lambda, through both the single-fit drop-in
(`pcd_fit`) and the lambda-path lanes (`pcd_path(concurrency=4)`, the bench's):
* identical iteration count and edge count,
* identical support (every exact zero of the reference is an exact zero here),
* max |Omega - Omega_ref| <= 1e-9 * max |Omega_ref| (tolerance stated by
  north_star: 1e-8 relative in FP64; the W-form accumulates the same dot
  products in a different order, so it is not bitwise),
* final delta within 1e-6 relative and the objective trace within 1e-10.
The measured errors are printed (tests/README: profiles/r02/p5000_parity.log).
"""

import glob
import hashlib
import os

import numpy as np
import pytest

import paper_2106_09382_b200 as cb
from paper_2106_09382_b200 import synth

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "p5000", "ar2_p5000_n2000_l*.npz")))
EXTRA = os.path.join(HERE, "golden", "p5000")

pytestmark = pytest.mark.gpu


def _load(path):
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="module")
def gram():
    x, t = synth.portable_problem("ar2", 5000, 2000, seed=0)
    return cb.GramMatrix(t, 2000), hashlib.sha256(t.tobytes()).hexdigest()


def _check(rep, fx, label):
    p = int(fx["meta"][0])
    om = rep.estimate.omega
    iu = np.triu_indices(p, 1)
    mask = np.unpackbits(fx["support"], count=iu[0].size).astype(bool)
    ref_upper = np.zeros(iu[0].size)
    ref_upper[mask] = fx["values"]
    upper = om[iu]
    err_off = float(np.max(np.abs(upper - ref_upper)))
    err_diag = float(np.max(np.abs(np.diag(om) - fx["diag"])))
    scale = float(max(np.max(np.abs(ref_upper)), np.max(np.abs(fx["diag"]))))
    same_support = bool(np.array_equal(upper != 0.0, mask))
    print(f"[p5000 parity] {label} lam={float(fx['meta'][2]):.2f}: iterations {rep.iterations} "
          f"(ref {int(fx['iters'])}), edges {rep.edge_count} (ref {int(fx['edges'])}), support identical "
          f"{same_support}, max|dOmega| off-diagonal {err_off:.3e} diagonal {err_diag:.3e} "
          f"(rel {max(err_off, err_diag) / scale:.3e}), final delta {rep.final_delta:.6e} "
          f"(ref {float(fx['final_delta']):.6e}), ambiguous pairs (1e-10/1e-8/1e-6 rel) "
          f"{fx['ambiguous'].tolist()}")
    assert rep.iterations == int(fx["iters"])
    assert rep.edge_count == int(fx["edges"])
    assert same_support
    assert max(err_off, err_diag) <= 1e-9 * scale
    assert rep.final_delta == pytest.approx(float(fx["final_delta"]), rel=1e-6)
    np.testing.assert_allclose(rep.objective_trace, fx["obj"], rtol=1e-10)


def test_fixtures_present():
    assert FIXTURES, "tests/golden/p5000/ fixtures are missing (tests/golden/make_golden_p5000.py)"


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(f)[:-4] for f in FIXTURES])
def test_p5000_fit_matches_reference(gram, path):
    g, tsha = gram
    fx = _load(path)
    assert tsha == bytes(fx["tsha"]).decode(), "T differs from the reference fixture's T"
    lam = float(fx["meta"][2])
    rep = cb.pcd_fit(g, cb.SolverConfig(lam=lam, delta_tol=float(fx["meta"][3]), max_outer_iterations=5000))
    _check(rep, fx, "pcd_fit")


def test_p5000_path_lanes_match_reference(gram):
    """The bench's scheduler: every fixture lambda in one pcd_path(concurrency=4) call."""
    g, tsha = gram
    fxs = [_load(f) for f in FIXTURES]
    lams = [float(fx["meta"][2]) for fx in fxs]
    reps = cb.pcd_path(g, lams, delta_tol=1e-5, max_outer_iterations=5000, concurrency=4)
    for rep, fx in zip(reps, fxs):
        _check(rep, fx, "pcd_path(concurrency=4)")


def test_p5001_odd_p_matches_reference():
    """Odd p at the paper size (p colours per sweep, a phantom partner in every round)."""
    path = os.path.join(EXTRA, "extra_ar2_p5001_n2000_l0.30.npz")
    if not os.path.exists(path):
        pytest.skip("fixture not generated (tests/golden/make_golden_p5000_extra.py)")
    fx = _load(path)
    x, t = synth.portable_problem("ar2", 5001, 2000, seed=0)
    assert hashlib.sha256(t.tobytes()).hexdigest() == bytes(fx["tsha"]).decode()
    rep = cb.pcd_fit(cb.GramMatrix(t, 2000), cb.SolverConfig(lam=0.3, max_outer_iterations=5000))
    _check(rep, fx, "pcd_fit p=5001")


def test_p5000_warm_start_matches_reference(gram):
    """Warm start at the paper size (SolverConfig.init, model.py:158-166): lambda=0.25 from the
    lambda=0.30 estimate, as pcd_path(warm_start=True) chains them; the reference started from its
    own lambda=0.30 estimate, which equals ours to ~1e-15."""
    path = os.path.join(EXTRA, "extra_ar2_p5000_n2000_l0.25_warm_from_0.30.npz")
    if not os.path.exists(path):
        pytest.skip("fixture not generated (tests/golden/make_golden_p5000_extra.py)")
    fx = _load(path)
    g, tsha = gram
    assert tsha == bytes(fx["tsha"]).decode()
    reps = cb.pcd_path(g, [0.30, 0.25], delta_tol=1e-5, max_outer_iterations=5000, warm_start=True)
    _check(reps[1], fx, "pcd_path(warm_start=True)")
    first = cb.pcd_fit(g, cb.SolverConfig(lam=0.30, max_outer_iterations=5000))
    rep = cb.pcd_fit(g, cb.SolverConfig(lam=0.25, max_outer_iterations=5000, init=first.estimate))
    _check(rep, fx, "pcd_fit(init=lambda 0.30 estimate)")
