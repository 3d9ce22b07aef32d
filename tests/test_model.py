"""API-type validation (host logic, no GPU), mirroring the reference's test_model."""

import numpy as np
import pytest

import paper_2106_09382_b200 as cb
from paper_2106_09382_b200 import synth


def test_containers_validate():
    with pytest.raises(cb.DimensionError):
        cb.DataMatrix(np.zeros(3))
    with pytest.raises(cb.DimensionError):
        cb.DataMatrix(np.zeros((3, 1)))
    with pytest.raises(ValueError):
        cb.DataMatrix(np.array([[1.0, 2.0], [3.0, 5.0]]), centered=True)
    with pytest.raises(ValueError):
        cb.GramMatrix(np.array([[1.0, 2.0], [3.0, 1.0]]), 3)
    with pytest.raises(cb.ZeroVarianceColumn):
        cb.GramMatrix(np.array([[1.0, 0.0], [0.0, 0.0]]), 3)
    with pytest.raises(ValueError):
        cb.GramMatrix(np.eye(2), 0)
    with pytest.raises(ValueError):
        cb.PrecisionEstimate(np.array([[1.0, 0.0], [0.0, -1.0]]))
    with pytest.raises(ValueError):
        cb.PrecisionEstimate(np.array([[1.0, 0.1], [0.2, 1.0]]))


def test_solver_config_validation_and_init_copy():
    with pytest.raises(ValueError):
        cb.SolverConfig(lam=-1.0)
    with pytest.raises(ValueError):
        cb.SolverConfig(lam=0.1, delta_tol=0.0)
    with pytest.raises(ValueError):
        cb.SolverConfig(lam=0.1, max_outer_iterations=0)
    with pytest.raises(ValueError):
        cb.SolverConfig(lam=0.1, workers=0)
    with pytest.raises(ValueError):
        cb.SolverConfig(lam=0.1, init="zeros")
    est = cb.PrecisionEstimate(np.eye(3) * 2.0)
    cfg = cb.SolverConfig(lam=0.1, init=est)
    w = cfg.initial_omega(3)
    w[0, 0] = 9.0
    assert est.omega[0, 0] == 2.0
    with pytest.raises(cb.DimensionError):
        cfg.initial_omega(4)


def test_soft_threshold_known_answers(golden):
    got = [cb.soft_threshold(float(v), 1.0) for v in golden["soft_x"]]
    assert np.array_equal(np.array(got), golden["soft_tau1"])
    with pytest.raises(ValueError):
        cb.soft_threshold(1.0, -0.1)


def test_synth_reproduces_reference_gram(golden):
    # make_golden.py asserted synth == reference generators bitwise; re-derive T here.
    x = synth.center(synth.sample_mvn(synth.ar2_precision(100), 50, seed=0))
    assert np.array_equal(x, golden["ar2_p100_n50_l0.3_x"])


def test_objective_and_edges_host(golden):
    t = golden["ar2_p100_n50_l0.3_t"]
    om = golden["ar2_p100_n50_l0.3_omega"]
    g = cb.GramMatrix(t, 50)
    est = cb.PrecisionEstimate(om)
    assert cb.edge_count(est) == int(golden["ar2_p100_n50_l0.3_edges"])
    assert cb.objective(est, g, 0.3) == pytest.approx(float(golden["ar2_p100_n50_l0.3_obj"][-1]), rel=1e-12)


def test_cyclic_max_reduce_and_diff_vector():
    rng = np.random.default_rng(1)
    for m in (1, 2, 3, 31, 100):
        d = rng.standard_normal(m)
        assert cb.cyclic_max_reduce(d) == max(abs(float(v)) for v in d)
    with pytest.raises(cb.EmptyVector):
        cb.cyclic_max_reduce(np.zeros(0))
    a = cb.PrecisionEstimate(np.eye(4) * 2)
    b = cb.PrecisionEstimate(np.eye(4))
    assert cb.diff_vector(a, b).shape == (10,)


def test_banded_ar2_sampler_matches_dense_sampler():
    """synth.sample_mvn_ar2_banded (configs[3:], large p) draws the same samples as
    the reference sampler (datagen.py:135-154) up to rounding."""
    from paper_2106_09382_b200 import synth

    for p, n, seed in ((50, 30, 0), (301, 120, 7)):
        a = synth.sample_mvn(synth.ar2_precision(p), n, seed=seed)
        b = synth.sample_mvn_ar2_banded(p, n, seed=seed)
        np.testing.assert_allclose(b, a, rtol=0, atol=1e-12 * np.abs(a).max())
