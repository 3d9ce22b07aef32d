"""GPU parity: the CUDA path against the reference (golden vectors) and the oracle.

Tolerances (north star: "Omega within a stated relative tolerance, e.g. 1e-8
in FP64", identical sparsity and schedule):
  * exact sweeps (backend "cuda-exact", pcd_exact.cu): BITWISE equal;
  * W-form fit (default backend, pcd_wform.cu): max |dOmega| <= 1e-9 * max |Omega|,
    identical support, edge count and iteration count; objective trace rtol 1e-10.
"""

import os

import numpy as np
import pytest

import paper_2106_09382_b200 as cb
from paper_2106_09382_b200 import cuda_kernels, synth
from conftest import case

pytestmark = pytest.mark.gpu

REL_TOL = 1e-9
FIT_CASES = ["ar2_p100_n50_l0.3", "ar2_p100_n50_l0.1", "ar2_p100_n50_l0.3_tol1e-8", "sf_p101_n50_l0.3",
             "ar2_p9_n70_l0.1", "ar2_p12_n60_l0.1_tol1e-8"]


def assert_close_support(got, want, rel=REL_TOL):
    scale = np.max(np.abs(want))
    err = np.max(np.abs(got - want))
    assert err <= rel * scale, f"max abs diff {err:.3e} > {rel:.0e} * {scale:.3e}"
    assert np.array_equal(got != 0.0, want != 0.0), "support differs"
    assert np.array_equal(got, got.T), "not exactly symmetric"


# ------------------------------------------------------------ exact sweeps


@pytest.mark.parametrize("name", ["ar2_p100_n50_l0.3", "sf_p101_n50_l0.3", "ar2_p9_n70_l0.1"])
def test_exact_sweeps_bitwise_equal_reference(golden, name):
    c = case(golden, name)
    rs, ss, off = cb.flat_circle_schedule(c["p"])
    om = np.eye(c["p"])
    for k in range(3):
        cuda_kernels.pcd_sweep(om, c["t"], c["n"], c["n"] * c["lam"], rs, ss, off, 1)
        assert np.array_equal(om, golden[f"{name}_sweep{k + 1}"]), k


def test_exact_u2_equals_pcd_and_cd_matches_reference(golden):
    c = case(golden, "ar2_p9_n70_l0.1")
    rs, ss, off = cb.flat_circle_schedule(9)
    a, b = np.eye(9), np.eye(9)
    for _ in range(3):
        cuda_kernels.pcd_sweep(a, c["t"], c["n"], c["n"] * 0.1, rs, ss, off, 1)
        cuda_kernels.u2_sweep(b, c["t"], c["n"], c["n"] * 0.1, rs, ss)
        assert np.array_equal(a, b)
    rep = cb.cd_fit(cb.GramMatrix(c["t"], c["n"]), cb.SolverConfig(lam=c["lam"], delta_tol=c["tol"],
                                                                    max_outer_iterations=5000))
    assert rep.iterations == c["cd_iters"]
    assert np.array_equal(rep.estimate.omega, c["cd_omega"])


@pytest.mark.parametrize("name", ["ar2_p100_n50_l0.3", "sf_p101_n50_l0.3", "ar2_p12_n60_l0.1_tol1e-8"])
def test_exact_backend_fit_bitwise_equal_reference(golden, name):
    c = case(golden, name)
    cfg = cb.SolverConfig(lam=c["lam"], delta_tol=c["tol"], max_outer_iterations=5000)
    rep = cb.pcd_fit(cb.GramMatrix(c["t"], c["n"]), cfg, backend="cuda-exact")
    assert rep.iterations == c["iters"]
    assert np.array_equal(rep.estimate.omega, c["omega"])
    assert rep.final_delta == c["delta"]


def test_exact_protocol_rejects_bad_buffers():
    t = np.eye(4)
    rs, ss, off = cb.flat_circle_schedule(4)
    with pytest.raises(ValueError):
        cuda_kernels.pcd_sweep(np.eye(4, dtype=np.float32), t, 10, 1.0, rs, ss, off, 1)
    with pytest.raises(ValueError):
        cuda_kernels.pcd_sweep(np.asfortranarray(np.eye(4) + 0.5), t, 10, 1.0, rs, ss, off, 1)


# ---------------------------------------------------------- W-form fit


@pytest.mark.parametrize("name", FIT_CASES)
def test_wform_fit_matches_reference(golden, name):
    c = case(golden, name)
    cfg = cb.SolverConfig(lam=c["lam"], delta_tol=c["tol"], max_outer_iterations=5000)
    rep = cb.pcd_fit(cb.GramMatrix(c["t"], c["n"]), cfg)
    assert rep.iterations == c["iters"]
    assert rep.edge_count == c["edges"]
    assert rep.converged and rep.final_delta < c["tol"]
    assert_close_support(rep.estimate.omega, c["omega"])
    np.testing.assert_allclose(rep.objective_trace, c["obj"], rtol=1e-10)
    assert len(rep.wall_time_per_iteration) == rep.iterations
    assert all(t > 0 for t in rep.wall_time_per_iteration)


CONFIG2 = [("scale_free", 1000, 500, 0.3), ("scale_free", 1001, 500, 0.3), ("ar2", 1000, 500, 0.3),
           # dense regime: 5-12% of the pairs move per sweep, so the blocked kernel's conflict paths
           # (per-row chains, phase-by-phase passes, multi-entry segments) carry the fit
           ("scale_free", 1000, 500, 0.1), ("scale_free", 1001, 500, 0.1), ("ar2", 1000, 500, 0.1),
           ("ar2", 2001, 1000, 0.1)]


@pytest.mark.parametrize("kind,p,n,lam", CONFIG2)
def test_wform_config2_matches_oracle(oracle, kind, p, n, lam):
    """BASELINE configs[1] (p=1000 / odd 1001, n=500) at lam 0.3 and 0.1, and p=2001 dense: the
    fast fit against the oracle (bitwise the compiled reference) on the same T."""
    _, t = synth.problem(kind, p, n, seed=0)
    ref = oracle.pcd_fit(t, n, lam, 1e-5, 5000, workers=os.cpu_count(), trace=True)
    rep = cb.pcd_fit(cb.GramMatrix(t, n), cb.SolverConfig(lam=lam, max_outer_iterations=5000))
    assert rep.iterations == ref["iterations"]
    assert rep.edge_count == ref["edge_count"]
    assert_close_support(rep.estimate.omega, ref["omega"])
    np.testing.assert_allclose(rep.objective_trace, ref["objective_trace"], rtol=1e-10)


@pytest.mark.parametrize("row", range(6))
def test_config2_reference_summaries(golden, row):
    """`big_summary` recorded from the REAL reference package (make_golden.py): iterations, edges,
    final delta and last objective of the fast fit; the exact backend reproduces the reference's
    Omega bitwise (sha256 `big_*_omsha`)."""
    import hashlib

    kind_id, p, n, lam, iters, edges, delta, obj = golden["big_summary"][row]
    kind = "ar2" if kind_id == 0 else "scale_free"
    p, n = int(p), int(n)
    _, t = synth.portable_problem(kind, p, n, seed=0)  # exact Gram: the same bits on every machine
    assert hashlib.sha256(t.tobytes()).hexdigest() == bytes(golden[f"big_{row}_tsha"]).decode()
    g = cb.GramMatrix(t, n)
    cfg = cb.SolverConfig(lam=lam, max_outer_iterations=5000)
    rep = cb.pcd_fit(g, cfg)
    assert rep.iterations == int(iters) and rep.edge_count == int(edges)
    assert rep.final_delta == pytest.approx(delta, rel=1e-6)
    assert rep.objective_trace[-1] == pytest.approx(obj, rel=1e-10)
    ex = cb.pcd_fit(g, cfg, backend="cuda-exact")
    assert ex.iterations == int(iters) and ex.final_delta == delta
    assert hashlib.sha256(ex.estimate.omega.tobytes()).hexdigest() == bytes(golden[f"big_{row}_omsha"]).decode()


@pytest.mark.parametrize("p,lam", [(2, 0.1), (3, 0.05), (5, 0.0), (64, 0.0), (257, 0.2)])
def test_wform_edge_cases_match_oracle(oracle, p, lam):
    rng = np.random.default_rng(p)
    x = rng.standard_normal((3 * p + 2, p))
    x -= x.mean(axis=0)
    t = synth.host_gram(x)
    n = x.shape[0]
    ref = oracle.pcd_fit(t, n, lam, 1e-7, 20000, trace=True)
    rep = cb.pcd_fit(cb.GramMatrix(t, n), cb.SolverConfig(lam=lam, delta_tol=1e-7, max_outer_iterations=20000))
    assert rep.iterations == ref["iterations"]
    assert_close_support(rep.estimate.omega, ref["omega"], rel=1e-8)
    np.testing.assert_allclose(rep.objective_trace, ref["objective_trace"], rtol=1e-9)


def test_wform_one_sweep_at_p2000_matches_oracle(oracle):
    """Dense-ish first sweep at a size where rows no longer fit one slab."""
    _, t = synth.problem("ar2", 2000, 1000, seed=1)
    om = np.eye(2000)
    rs, ss, off = oracle.circle_flat(2000)
    oracle.pcd_sweep(om, t, 1000, 1000 * 0.1, rs, ss, off, 8)
    with cb.Solver(2000) as s:
        s.set_gram(cb.GramMatrix(t, 1000))
        rc, res, deltas, objs, secs = s.fit_raw(0.1, 1e-5, 1)
        got = s.omega()
    assert res.iterations == 1
    assert_close_support(got, om)


def test_slab_count_never_changes_bits(golden):
    """GPU analogue of worker invariance (test_solver.py:222-230)."""
    c = case(golden, "ar2_p100_n50_l0.1")
    outs = []
    for nb in (0, 1, 3, 7, 50):
        with cb.Solver(100, n_blocks=nb) as s:
            s.set_gram(cb.GramMatrix(c["t"], c["n"]))
            rep = s.fit(c["lam"], c["tol"], 5000)
        outs.append(rep)
    for r in outs[1:]:
        assert np.array_equal(r.estimate.omega, outs[0].estimate.omega)
        assert r.iterations == outs[0].iterations


def test_fit_is_deterministic_and_data_path_equals_gram_path(golden):
    c = case(golden, "sf_p101_n50_l0.3")
    cfg = cb.SolverConfig(lam=0.3)
    dm = cb.DataMatrix(c["x"], centered=True)
    a = cb.pcd_fit(dm, cfg)
    b = cb.pcd_fit(cb.compute_gram(dm), cfg)
    assert np.array_equal(a.estimate.omega, b.estimate.omega)
    assert a.objective_trace == b.objective_trace


def test_device_gram_matches_host(golden):
    rng = np.random.default_rng(3)
    for n, p in ((50, 100), (37, 129), (500, 1000), (7, 65)):
        x = rng.standard_normal((n, p))
        g = cb.compute_gram(cb.DataMatrix(x))
        assert np.array_equal(g.t, g.t.T)
        want = x.T @ x
        np.testing.assert_allclose(g.t, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())
    g2 = cb.compute_gram(cb.DataMatrix(np.array([[1.0, 2.0], [3.0, 4.0]])))
    assert np.array_equal(g2.t, golden["gram_2x2"])


def test_not_converged_carries_partial_report(golden):
    c = case(golden, "ar2_p100_n50_l0.1")
    with pytest.raises(cb.NotConverged) as err:
        cb.pcd_fit(cb.GramMatrix(c["t"], c["n"]), cb.SolverConfig(lam=0.1, max_outer_iterations=2))
    rep = err.value.report
    assert not rep.converged and rep.iterations == 2 and rep.final_delta >= 1e-5
    assert isinstance(rep.estimate, cb.PrecisionEstimate)


def test_huge_lambda_gives_diagonal_fixed_point(golden):
    c = case(golden, "ar2_p100_n50_l0.3")
    rep = cb.pcd_fit(cb.GramMatrix(c["t"], c["n"]), cb.SolverConfig(lam=1e6, delta_tol=1e-8))
    assert rep.edge_count == 0
    np.testing.assert_allclose(np.diag(rep.estimate.omega), np.sqrt(c["n"] / np.diag(c["t"])), rtol=1e-12)


def test_warm_start_matches_oracle(oracle, golden):
    c = case(golden, "ar2_p100_n50_l0.3")
    init = golden["ar2_p100_n50_l0.1_omega"]
    ref = oracle.pcd_fit(c["t"], c["n"], 0.3, 1e-6, 5000, init=init)
    cfg = cb.SolverConfig(lam=0.3, delta_tol=1e-6, max_outer_iterations=5000, init=cb.PrecisionEstimate(init))
    rep = cb.pcd_fit(cb.GramMatrix(c["t"], c["n"]), cfg)
    assert rep.iterations == ref["iterations"]
    assert_close_support(rep.estimate.omega, ref["omega"], rel=1e-8)


def test_lambda_path_cold_equals_independent_fits(golden):
    c = case(golden, "ar2_p100_n50_l0.3")
    g = cb.GramMatrix(c["t"], c["n"])
    lams = [0.5, 0.3, 0.2]
    path = cb.pcd_path(g, lams, delta_tol=1e-6, max_outer_iterations=5000)
    for lam, rep in zip(lams, path):
        one = cb.pcd_fit(g, cb.SolverConfig(lam=lam, delta_tol=1e-6, max_outer_iterations=5000))
        assert np.array_equal(rep.estimate.omega, one.estimate.omega)
    warm = cb.pcd_path(g, lams, delta_tol=1e-6, max_outer_iterations=5000, warm_start=True)
    for a, b in zip(warm, path):
        assert a.converged and np.max(np.abs(a.estimate.omega - b.estimate.omega)) < 1e-3


def test_custom_schedule_runs_bitwise_like_reference(oracle, golden):
    c = case(golden, "ar2_p9_n70_l0.1")
    import dataclasses

    sched = cb.build_circle_schedule(9)
    rev = dataclasses.replace(sched, rounds=sched.rounds[::-1])
    cfg = cb.SolverConfig(lam=0.1, delta_tol=1e-6)
    rep = cb.pcd_fit(cb.GramMatrix(c["t"], c["n"]), cfg, schedule=rev)
    from paper_2106_09382_b200.schedule import flatten_schedule

    rs, ss, off = flatten_schedule(rev)
    om = np.eye(9)
    for _ in range(rep.iterations):
        oracle.pcd_sweep(om, c["t"], c["n"], c["n"] * 0.1, rs, ss, off, 1)
    assert np.array_equal(rep.estimate.omega, om)
    with pytest.raises(cb.ScheduleMismatch):
        cb.pcd_fit(cb.GramMatrix(c["t"], c["n"]), cfg, schedule=cb.build_circle_schedule(5))


def test_objective_monotone_large_p():
    _, t = synth.problem("ar2", 3000, 1500, seed=2)
    rep = cb.pcd_fit(cb.GramMatrix(t, 1500), cb.SolverConfig(lam=0.2, max_outer_iterations=500))
    tr = rep.objective_trace
    assert all(b <= a + 1e-9 * abs(a) for a, b in zip(tr, tr[1:]))
    om = rep.estimate.omega
    assert np.array_equal(om, om.T) and np.all(np.diag(om) > 0)


# ------------------------------------------------- multi-GPU data path (8e)


@pytest.mark.parametrize("name", ["ar2_p100_n50_l0.1", "sf_p101_n50_l0.3", "ar2_p9_n70_l0.1"])
def test_virtual_shards_are_bitwise_invariant(golden, name):
    """Columns split over G shards with replicated exchange buffers (the NVLink
    data flow of dist.py, on one device): bitwise identical for G = 1, 2, 4, 8."""
    c = case(golden, name)
    outs = []
    for g in (1, 2, 4, 8):
        with cb.Solver(c["p"], n_shards=g) as s:
            assert s.layout()["n_shards"] == g
            s.set_gram(cb.GramMatrix(c["t"], c["n"]))
            outs.append(s.fit(c["lam"], c["tol"], 5000))
    for r in outs:
        assert r.iterations == c["iters"]
        assert np.array_equal(r.estimate.omega, outs[0].estimate.omega)
        np.testing.assert_allclose(r.objective_trace, outs[0].objective_trace, rtol=1e-12)
    assert_close_support(outs[0].estimate.omega, c["omega"])


def test_virtual_shards_consecutive_fits_and_large_p(oracle):
    """Barrier/sweep bases carried across fits; a p=2000 sweep split 8 ways."""
    _, t = synth.problem("ar2", 2000, 1000, seed=4)
    g = cb.GramMatrix(t, 1000)
    with cb.Solver(2000) as s1, cb.Solver(2000, n_shards=8) as s8:
        s1.set_gram(g)
        s8.set_gram(g)
        for lam in (0.5, 0.3, 0.25):
            a = s1.fit(lam, 1e-5, 500)
            b = s8.fit(lam, 1e-5, 500)
            assert a.iterations == b.iterations
            assert np.array_equal(a.estimate.omega, b.estimate.omega)
    om = np.eye(2000)
    rs, ss, off = oracle.circle_flat(2000)
    ref = oracle.pcd_fit(t, 1000, 0.25, 1e-5, 500, workers=8, trace=False)
    assert ref["iterations"] == b.iterations
    assert_close_support(b.estimate.omega, ref["omega"])


# ------------------------------------------------ device diagnostics (8f #2, #3)


@pytest.mark.parametrize("name", ["ar2_p100_n50_l0.3", "sf_p101_n50_l0.3", "ar2_p12_n60_l0.1_tol1e-8"])
def test_device_check_optimality_and_entries(golden, name, tmp_path):
    """check_optimality from the maintained W (= Omega T up to rounding) and the
    device-compacted estimate entries, against the reference's own outputs."""
    import os

    from paper_2106_09382_b200 import fileio
    from conftest import REPO

    io = np.load(os.path.join(REPO, "tests", "golden", "reference_io_golden.npz"))
    c = case(golden, name)
    with cb.Solver(c["p"]) as s:
        s.set_gram(cb.GramMatrix(c["t"], c["n"]))
        rep = s.fit(c["lam"], c["tol"], 5000)
        opt = s.check_optimality(c["lam"])
        ents = s.estimate_entries()
    worst, i, j = io[f"{name}_opt"]
    host = cb.check_optimality(rep.estimate, cb.GramMatrix(c["t"], c["n"]), c["lam"])
    assert abs(opt.worst_violation - host.worst_violation) <= 1e-9 * max(1.0, host.worst_violation)
    assert opt.worst_coordinate == host.worst_coordinate
    assert abs(opt.worst_violation - worst) <= 1e-6 * max(1.0, abs(worst))
    h = fileio.estimate_entries(rep.estimate)
    for a, b in zip(ents, h):
        assert np.array_equal(a, b)
    path = tmp_path / "e.txt"
    fileio.write_estimate(str(path), ents, c["lam"], rep.iterations, rep.final_delta, p=c["p"])
    est, _ = fileio.read_estimate(str(path))
    assert np.array_equal(est.omega, rep.estimate.omega)


# ------------------------------------------------- blocked kernel == per-phase kernel


@pytest.mark.parametrize("p,lam", [(1000, 0.03), (1000, 0.3), (777, 0.1), (2001, 0.2)])
def test_blocked_kernel_bitwise_equals_per_phase_kernel(p, lam, monkeypatch):
    """pcd_qblock.cu (temporally blocked, D colours per barrier) against
    pcd_wform.cu (one barrier per colour): the same FMAs in the same order, so
    the same bits, for every D the kernel supports (2..QB_DMAX=4).  lam=0.03 makes most pairs move, so batches
    hit both row-conflict paths (per-row chains and phase-by-phase passes);
    odd p exercises the phantom id."""
    _, t = synth.problem("ar2", p, 400, seed=5)
    g = cb.GramMatrix(t, 400)
    def run():
        with cb.Solver(p) as s:
            kern = s.layout()["kernel"]
            s.set_gram(g)
            rc, res, deltas, objs, _ = s.fit_raw(lam, 1e-5, 30)  # lam=0.03 may not converge: compare anyway
            return kern, res.iterations, s.omega(), np.array(deltas), np.array(objs)

    monkeypatch.setenv("CONCORD_KERNEL", "wform")
    k0, it0, om0, dl0, ob0 = run()
    assert k0 == 0
    monkeypatch.delenv("CONCORD_KERNEL")
    for d in ("2", "3", "4"):
        monkeypatch.setenv("CONCORD_QB_D", d)
        k, it, om, dl, ob = run()
        assert k == int(d)
        assert it == it0, d
        assert np.array_equal(om, om0), d
        assert np.array_equal(dl, dl0), d
        np.testing.assert_allclose(ob, ob0, rtol=1e-12)


def test_result_arrays_are_independent_pinned_pool(golden):
    """Omega results come from a pool of page-locked blocks: a live report's array is never
    reused, and a freed one is recycled without disturbing the others."""
    c = case(golden, "ar2_p100_n50_l0.1")
    with cb.Solver(c["p"]) as s:
        s.set_gram(cb.GramMatrix(c["t"], c["n"]))
        r1 = s.fit(0.3, 1e-5, 5000)
        keep = r1.estimate.omega.copy()
        r2 = s.fit(0.1, 1e-5, 5000)
        assert not np.shares_memory(r1.estimate.omega, r2.estimate.omega)
        assert np.array_equal(r1.estimate.omega, keep)
        del r2
        r3 = s.fit(0.2, 1e-5, 5000)
        assert not np.shares_memory(r1.estimate.omega, r3.estimate.omega)
        assert np.array_equal(r1.estimate.omega, keep)
        r4 = s.fit(0.1, 1e-5, 5000)
        assert_close_support(r4.estimate.omega, c["omega"])


@pytest.mark.parametrize("k,p", [(2, 1000), (3, 1000), (3, 777), (3, 300)])
def test_concurrent_lambda_path_equals_sequential_fits(k, p):
    """pcd_path(concurrency=k) (PathScheduler): k cold fits at a time on SMs/k slabs each, own
    stream and thread, while sparse, then one at a time on all SMs -- the same bits and iteration
    counts as one fit at a time on all SMs."""
    _, t = synth.problem("ar2", p, 400, seed=7)
    g = cb.GramMatrix(t, 400)
    lams = [0.4, 0.3, 0.2, 0.15, 0.1]
    seq = cb.pcd_path(g, lams, max_outer_iterations=300)
    con = cb.pcd_path(g, lams, max_outer_iterations=300, concurrency=k)
    assert len(con) == len(lams)
    for a, b in zip(seq, con):
        assert a.iterations == b.iterations
        assert np.array_equal(a.estimate.omega, b.estimate.omega)
        np.testing.assert_allclose(a.objective_trace, b.objective_trace, rtol=1e-12)
    with pytest.raises(ValueError):
        cb.pcd_path(g, lams, warm_start=True, concurrency=k)


def test_concurrent_lambda_path_from_data_matrix():
    """pcd_path(DataMatrix, concurrency=3) computes the Gram on the device first; same bits as
    sequential fits from the same data."""
    x, _ = synth.problem("ar2", 600, 300, seed=11)
    dm = cb.DataMatrix(x, centered=True)
    lams = [0.3, 0.15]
    seq = cb.pcd_path(dm, lams, max_outer_iterations=300)
    con = cb.pcd_path(dm, lams, max_outer_iterations=300, concurrency=3)
    for a, b in zip(seq, con):
        assert a.iterations == b.iterations
        assert np.array_equal(a.estimate.omega, b.estimate.omega)


@pytest.mark.parametrize("sys_scope", ["0", "1"])
def test_virtual_shards_on_the_blocked_kernel(sys_scope, monkeypatch):
    """The column-sharded fit runs the temporally blocked kernel too (one cross-shard barrier per
    D=4 colours; stage, delta ring and lists written into every shard's copy): bitwise equal to
    the unsharded blocked kernel for G = 2, 4, 8, with GPU-scope and -- forced on one device --
    the multi-GPU system-scope fences and reductions (the reference's worker-invariance contract,
    test_solver.py:222-230)."""
    monkeypatch.setenv("CONCORD_FORCE_SYS_SCOPE", sys_scope)
    _, t = synth.problem("ar2", 1000, 500, seed=6)
    g = cb.GramMatrix(t, 500)
    with cb.Solver(1000) as s1:
        assert s1.layout()["kernel"] == 4
        s1.set_gram(g)
        want = [s1.fit(lam, 1e-5, 500) for lam in (0.3, 0.1)]
    for G in (2, 4, 8):
        with cb.Solver(1000, n_shards=G) as sg:
            lay = sg.layout()
            assert lay["n_shards"] == G and lay["kernel"] == 4
            sg.set_gram(g)
            for lam, w in zip((0.3, 0.1), want):  # consecutive fits: barrier and sweep bases carried
                r = sg.fit(lam, 1e-5, 500)
                assert r.iterations == w.iterations and r.edge_count == w.edge_count
                assert np.array_equal(r.estimate.omega, w.estimate.omega)
                np.testing.assert_allclose(r.objective_trace, w.objective_trace, rtol=1e-12)


@pytest.mark.parametrize("n_blocks", [0, 41])
def test_kernel_variants_are_bitwise_identical(n_blocks):
    """The chain-warp variants of the blocked kernel (6 default; 4 apply-heavy and 8 chain-heavy,
    whose warp groups trade registers with setmaxnreg) evaluate the same FMAs in the same order:
    bitwise the same estimate, iterations and objective trace, also consecutive fits on one solver."""
    _, t = synth.problem("ar2", 1000, 500, seed=7)
    g = cb.GramMatrix(t, 500)
    outs = {}
    for cw in (6, 4, 8):
        with cb.Solver(1000, n_blocks=n_blocks) as s:
            assert s.layout()["kernel"] == 4
            s.set_chain_warps(cw)
            s.set_gram(g)
            outs[cw] = [s.fit(lam, 1e-5, 500) for lam in (0.3, 0.1)]
    for cw in (4, 8):
        for r, w in zip(outs[cw], outs[6]):
            assert r.iterations == w.iterations and r.edge_count == w.edge_count
            assert np.array_equal(r.estimate.omega, w.estimate.omega)
            np.testing.assert_allclose(r.objective_trace, w.objective_trace, rtol=1e-12)
    from paper_2106_09382_b200 import _lib

    with cb.Solver(1000) as s, pytest.raises(_lib.ConcordError):
        s.set_chain_warps(5)
