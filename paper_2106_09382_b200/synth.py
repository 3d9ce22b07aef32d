"""Synthetic CONCORD problems (host side; input generation for tests and bench).

Follows /root/reference/pkg/src/parconcord/datagen.py so that the same seeds
give the same matrices as the reference's generators (checked bitwise against
the reference in tests/golden/make_golden.py).  Not on the hot path.
"""

import numpy as np
from scipy.linalg import solve_triangular

MAX_HUB_DEGREE = 40  # datagen.py:37


class NotPositiveDefinite(ValueError):
    """datagen.py:32."""


def ar2_precision(p):
    """datagen.py:64-78: unit diagonal, first band 0.45, second band 0.40."""
    if p < 3:
        raise ValueError("ar2 truth needs p >= 3")
    om = np.eye(p)
    i = np.arange(p - 1)
    om[i, i + 1] = om[i + 1, i] = 0.45
    i = np.arange(p - 2)
    om[i, i + 2] = om[i + 2, i] = 0.40
    return om


def _attachment_edges(p, alpha, rng):
    """datagen.py:81-96."""
    a0 = alpha - 3.0
    deg = np.zeros(p)
    edges = [(0, 1)]
    deg[0] = deg[1] = 1.0
    for v in range(2, p):
        w = deg[:v] + a0
        w[deg[:v] >= MAX_HUB_DEGREE] = 0.0
        cum = np.cumsum(w)
        u = int(np.searchsorted(cum, rng.random() * cum[-1], side="right"))
        edges.append((u, v))
        deg[u] += 1.0
        deg[v] += 1.0
    return edges


def scale_free_precision(p, alpha=2.3, seed=0):
    """datagen.py:99-132."""
    if p < 3:
        raise ValueError("scale-free truth needs p >= 3")
    graph_seed, weight_seed = np.random.SeedSequence(seed).spawn(2)
    rng_graph = np.random.default_rng(graph_seed)
    rng_weight = np.random.default_rng(weight_seed)
    edges = _attachment_edges(p, alpha, rng_graph)
    u = np.zeros((p, p))
    mags = rng_weight.uniform(0.5, 1.0, size=len(edges))
    signs = rng_weight.choice([-1.0, 1.0], size=len(edges))
    for (i, j), m, s in zip(edges, mags, signs):
        u[i, j] = u[j, i] = m * s
    r = np.abs(u).sum(axis=1)
    b = u / (1.25 * np.sqrt(np.outer(r, r)))
    b = 0.5 * (b + b.T)
    support = u != 0.0
    small = support & (np.abs(b) < 0.1)
    b[small] = 0.1 * np.sign(b[small])
    np.fill_diagonal(b, 1.0)
    return b


def scale_free_tree(p, alpha=2.3, seed=0):
    """The scale-free truth of datagen.py:99-132 in O(p) memory: (parent, weight).

    The same attachment tree (datagen.py:81-96, the reference's RNG streams, so the
    same edges, magnitudes and signs bit for bit) and the same scaling
    u / (1.25 sqrt(r_i r_j)) with the 0.1 magnitude floor; vertex v >= 1 hangs
    off parent[v] < v with truth[v, parent[v]] = weight[v] (parent[0] = -1,
    unit diagonal).  The row sums r are accumulated edge by edge instead of as
    numpy's dense row sums, so a value may differ from scale_free_precision's
    in the last bit; the support is identical.  For p where the dense p x p
    truth does not fit (configs[4]).
    """
    if p < 3:
        raise ValueError("scale-free truth needs p >= 3")
    graph_seed, weight_seed = np.random.SeedSequence(seed).spawn(2)
    rng_graph = np.random.default_rng(graph_seed)
    rng_weight = np.random.default_rng(weight_seed)
    edges = np.asarray(_attachment_edges(p, alpha, rng_graph), dtype=np.int64)  # (u, v), u < v; edge k -> v = k+1
    mags = rng_weight.uniform(0.5, 1.0, size=len(edges))
    signs = rng_weight.choice([-1.0, 1.0], size=len(edges))
    u = mags * signs
    r = np.zeros(p)
    np.add.at(r, edges[:, 0], np.abs(u))
    np.add.at(r, edges[:, 1], np.abs(u))
    b = u / (1.25 * np.sqrt(r[edges[:, 0]] * r[edges[:, 1]]))
    small = np.abs(b) < 0.1
    b[small] = 0.1 * np.sign(b[small])
    parent = np.full(p, -1, dtype=np.int32)
    weight = np.zeros(p)
    parent[edges[:, 1]] = edges[:, 0]
    weight[edges[:, 1]] = b
    return parent, weight


def tree_cholesky(parent, weight):
    """Fill-free Cholesky of a tree truth (unit diagonal, truth[v, parent[v]] = weight[v]).

    With parent[v] < v, eliminating leaves first (decreasing v) creates no fill:
    L[v, v] = ldiag[v] and column v's only sub-diagonal entry is
    L[parent[v], v] = lpar[v]; truth = L L^T in that order.  Raises
    NotPositiveDefinite like sample_mvn (datagen.py:146-151).
    """
    p = parent.shape[0]
    d = np.ones(p)
    ldiag = np.zeros(p)
    lpar = np.zeros(p)
    for v in range(p - 1, -1, -1):
        if not d[v] > 0.0:
            raise NotPositiveDefinite("truth is not positive definite")
        ldiag[v] = np.sqrt(d[v])
        if parent[v] >= 0:
            lpar[v] = weight[v] / ldiag[v]
            d[parent[v]] -= lpar[v] * lpar[v]
    return lpar, ldiag


def tree_dense(parent, weight):
    """The dense p x p truth of a tree (small p, tests)."""
    p = parent.shape[0]
    om = np.eye(p)
    v = np.flatnonzero(parent >= 0)
    om[v, parent[v]] = om[parent[v], v] = weight[v]
    return om


def sample_scale_free_device(p, n, seed=0, alpha=2.3, truth_seed=None, device=0):
    """Centred N(0, inv(scale-free truth)) samples drawn on the GPU (csrc/datagen.cu tree sampler).

    Same distribution as center(sample_mvn(scale_free_precision(p, alpha, truth_seed), n, seed));
    a different (Philox) random stream, O(p n) work, no dense p x p Cholesky.
    """
    from . import _lib

    parent, weight = scale_free_tree(p, alpha, seed if truth_seed is None else truth_seed)
    lpar, ldiag = tree_cholesky(parent, weight)
    x = np.empty((n, p))
    _lib.check(_lib.load().concord_tree_data_f64(int(p), int(n), int(seed), _lib.ptr(parent), _lib.ptr(lpar),
                                                 _lib.ptr(ldiag), _lib.ptr(x), _lib.HOST, int(device)))
    return x


def sample_mvn(omega_true, n, seed=0):
    """datagen.py:135-154: n rows of N(0, inv(omega_true)), raw (uncentered)."""
    try:
        chol = np.linalg.cholesky(omega_true)
    except np.linalg.LinAlgError as exc:
        raise NotPositiveDefinite("truth is not positive definite") from exc
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((n, omega_true.shape[0]))
    x = solve_triangular(chol, z.T, lower=True, trans="T").T
    return np.ascontiguousarray(x)


def sample_mvn_ar2_banded(p, n, seed=0):
    """N(0, inv(ar2_precision(p))) samples in O(p*n) for large p (configs[3:], p >= 20000).

    Same distribution as sample_mvn(ar2_precision(p), n, seed) -- the same
    normal draws z and the same triangular system L^T x = z with L the
    (banded) Cholesky factor -- but solved with banded LAPACK routines, so the
    last bits differ from the dense path.  Used where the dense Cholesky of a
    p x p truth is the bottleneck and no CPU oracle exists.
    """
    from scipy.linalg import cholesky_banded, solve_banded

    ab = np.zeros((3, p))  # lower banded storage of the AR(2) truth
    ab[0] = 1.0
    ab[1, :-1] = 0.45
    ab[2, :-2] = 0.40
    lb = cholesky_banded(ab, lower=True)  # L in lower banded storage
    # L^T is upper triangular with 2 super-diagonals: upper banded storage u[2 + i - j, j] = L^T[i, j]
    ub = np.zeros((3, p))
    ub[2] = lb[0]
    ub[1, 1:] = lb[1, :-1]
    ub[0, 2:] = lb[2, :-2]
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((n, p))
    x = solve_banded((0, 2), ub, z.T).T
    return np.ascontiguousarray(x)


def sample_ar2_device(p, n, seed=0, device=0):
    """Centred N(0, inv(ar2_precision(p))) samples drawn on the GPU (csrc/datagen.cu).

    Same distribution as center(sample_mvn(ar2_precision(p), n, seed)), a
    different (Philox) random stream; O(p n) work on the device.
    """
    from . import _lib

    x = np.empty((n, p))
    _lib.check(_lib.load().concord_ar2_data_f64(int(p), int(n), int(seed), _lib.ptr(x), _lib.HOST, int(device)))
    return x


def center(x):
    """model.py:182-187 (center_columns on a raw array)."""
    return x - x.mean(axis=0)


def host_gram(x):
    """model.py:190-197 on the host: 0.5*(X^T X + (X^T X)^T)."""
    raw = x.T @ x
    return 0.5 * (raw + raw.T)


def quantize_exact_gram(x):
    """Round X to a 2^-s grid on which X^T X is EXACT in FP64, whatever the summation order.

    With |X| 2^s < 2^a and n < 2^b every product is an integer times 2^-2s below
    2^2a and every partial sum of n of them stays below 2^(2a+b) <= 2^53, so
    BLAS (any kernel, any thread count), the GPU's DMMA Gram and a scalar loop
    all produce the same bits -- T, and every result derived from it, is then
    portable between this container and the GPU box.  s is the largest such
    grid for the data (s = 18 for the p=5000, n=2000 AR(2) workload: a step of
    4e-6 on unit-scale data).
    """
    x = np.asarray(x, dtype=np.float64)
    b = int(np.ceil(np.log2(max(x.shape[0], 2))))
    a_data = int(np.floor(np.log2(max(float(np.max(np.abs(x))), 1e-300)))) + 1
    s = (53 - b) // 2 - a_data
    scale = float(2.0 ** s)
    return np.ascontiguousarray(np.round(x * scale) / scale), s


def portable_problem(kind, p, n, seed=0):
    """(X, T) with T = X^T X exact in FP64 on every machine (fixtures at configs[1]/[2]).

    X = the reference pipeline center(sample_mvn(truth, n, seed)) rounded onto
    the exact-Gram grid of `quantize_exact_gram`.  The draws run with one BLAS
    thread (OpenBLAS's triangular solve splits work by thread count).
    """
    from threadpoolctl import threadpool_limits

    truth = ar2_precision(p) if kind == "ar2" else scale_free_precision(p, seed=seed)
    with threadpool_limits(1):
        x = center(sample_mvn(truth, n, seed=seed))
    xq, _ = quantize_exact_gram(x)
    return xq, host_gram(xq)


def problem(kind, p, n, seed=0):
    """(centered X, T) for a truth kind in {"ar2", "scale_free"}."""
    truth = ar2_precision(p) if kind == "ar2" else scale_free_precision(p, seed=seed)
    x = center(sample_mvn(truth, n, seed=seed))
    return x, host_gram(x)
