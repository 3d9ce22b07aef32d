"""Pin the CPU oracle (test infrastructure) to the real reference.

The oracle is the checker of every GPU parity test, so before trusting it we
require it to reproduce, BIT FOR BIT, the vectors the reference package's
compiled backend produced (tests/golden/make_golden.py), and -- when
oracle/_ref was built -- the reference's own compiled kernel on fresh inputs.
"""

import numpy as np
import pytest

from conftest import case

FIT_CASES = ["ar2_p100_n50_l0.3", "ar2_p100_n50_l0.1", "ar2_p100_n50_l0.3_tol1e-8", "sf_p101_n50_l0.3",
             "ar2_p9_n70_l0.1", "ar2_p12_n60_l0.1_tol1e-8"]


@pytest.mark.parametrize("p", list(range(2, 21)) + [101])
def test_oracle_schedule_matches_reference(golden, oracle, p):
    rs, ss, off = oracle.circle_flat(p)
    assert np.array_equal(rs, golden[f"sched_{p}_rs"])
    assert np.array_equal(ss, golden[f"sched_{p}_ss"])
    assert np.array_equal(off, golden[f"sched_{p}_off"])


@pytest.mark.parametrize("name", ["ar2_p100_n50_l0.3", "sf_p101_n50_l0.3", "ar2_p9_n70_l0.1"])
def test_oracle_sweeps_bitwise_equal_reference(golden, oracle, name):
    c = case(golden, name)
    rs, ss, off = oracle.circle_flat(c["p"])
    for workers in (1, 4):
        om = np.eye(c["p"])
        for k in range(3):
            oracle.pcd_sweep(om, c["t"], c["n"], c["n"] * c["lam"], rs, ss, off, workers)
            assert np.array_equal(om, golden[f"{name}_sweep{k + 1}"]), (workers, k)


@pytest.mark.parametrize("name", FIT_CASES)
def test_oracle_fit_bitwise_equal_reference(golden, oracle, name):
    c = case(golden, name)
    rep = oracle.pcd_fit(c["t"], c["n"], c["lam"], c["tol"], 5000)
    assert rep["iterations"] == c["iters"]
    assert np.array_equal(rep["omega"], c["omega"])
    assert rep["edge_count"] == c["edges"]
    assert rep["final_delta"] == c["delta"]
    np.testing.assert_allclose(rep["objective_trace"], c["obj"], rtol=1e-12)


@pytest.mark.parametrize("name", ["ar2_p9_n70_l0.1", "ar2_p12_n60_l0.1_tol1e-8"])
def test_oracle_cd_bitwise_equal_reference(golden, oracle, name):
    c = case(golden, name)
    rep = oracle.cd_fit(c["t"], c["n"], c["lam"], c["tol"], 5000)
    assert rep["iterations"] == c["cd_iters"]
    assert np.array_equal(rep["omega"], c["cd_omega"])


def test_oracle_u2_equals_pcd(golden, oracle):
    c = case(golden, "ar2_p9_n70_l0.1")
    rs, ss, off = oracle.circle_flat(9)
    a, b = np.eye(9), np.eye(9)
    for _ in range(3):
        oracle.pcd_sweep(a, c["t"], c["n"], c["n"] * 0.1, rs, ss, off, 1)
        oracle.u2_sweep(b, c["t"], c["n"], c["n"] * 0.1, rs, ss)
        assert np.array_equal(a, b)


def test_oracle_matches_reference_build_on_random_inputs(oracle):
    ref = oracle.load_ref()
    if ref is None:
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    rng = np.random.default_rng(5)
    for p in (7, 30, 64):
        x = rng.standard_normal((2 * p, p))
        x -= x.mean(axis=0)
        raw = x.T @ x
        t = 0.5 * (raw + raw.T)
        rs, ss, off = oracle.circle_flat(p)
        a = np.eye(p)
        b = np.eye(p)
        for _ in range(4):
            oracle.pcd_sweep(a, t, 2 * p, 2 * p * 0.05, rs, ss, off, 2)
            ref.pcd_sweep(b, t, float(2 * p), 2 * p * 0.05, rs.astype(np.intp), ss.astype(np.intp),
                          off.astype(np.intp), 2)
            assert np.array_equal(a, b)


@pytest.mark.parametrize("row", range(6))
def test_oracle_matches_reference_config2_summaries(golden, oracle, row):
    """BASELINE configs[1] (p=1000 / odd p=1001, n=500, lam=0.3 and 0.1) through the oracle: the same T
    (sha256), iteration count, edges, final delta and Omega bits (sha256) as the real reference
    package recorded in `big_summary` (make_golden.py)."""
    import hashlib
    import os

    from paper_2106_09382_b200 import synth

    kind_id, p, n, lam, iters, edges, delta, obj = golden["big_summary"][row]
    kind = "ar2" if kind_id == 0 else "scale_free"
    p, n = int(p), int(n)
    _, t = synth.portable_problem(kind, p, n, seed=0)
    assert hashlib.sha256(t.tobytes()).hexdigest() == bytes(golden[f"big_{row}_tsha"]).decode()
    rep = oracle.pcd_fit(t, n, lam, 1e-5, 5000, workers=os.cpu_count(), trace=False)
    assert rep["iterations"] == int(iters) and rep["edge_count"] == int(edges)
    assert rep["final_delta"] == delta
    assert hashlib.sha256(rep["omega"].tobytes()).hexdigest() == bytes(golden[f"big_{row}_omsha"]).decode()
