"""CPU ORACLE -- test infrastructure only (the checker, never the product).

Restates the reference's CONCORD-PCD hot path on the CPU so the CUDA path can
be checked against it:

* sweeps: ``concord_oracle.c`` (bitwise restatement of
  /root/reference/pkg/src/parconcord/_ckernels.pyx), loaded from
  ``oracle/_build/liboracle.so``;
* optionally the reference's OWN compiled ``_ckernels`` from ``oracle/_ref``
  (built by ``make -C oracle ref`` from the .pyx where it lies under
  /root/reference; see :func:`load_ref`);
* the ``pcd_fit`` / ``cd_fit`` driver loops of solver.py:227-294, the
  objective of model.py:210-217, ``edge_count`` of model.py:249-253.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module.  Pinned against tests/golden/ (vectors produced by
the real reference package, tests/golden/make_golden.py) and against
oracle/_ref in tests/test_oracle.py.
"""

import ctypes
import glob
import importlib.util
import math
import os
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

_d = ctypes.c_double
_i64 = ctypes.c_int64
_pd = ctypes.POINTER(ctypes.c_double)
_pi = ctypes.POINTER(ctypes.c_int64)


def build():
    """Compile the C restatement (and oracle/_ref when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if os.path.isdir("/root/reference"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "_build", "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.oracle_cd_sweep.argtypes = [_pd, _pd, _i64, _d, _d]
        L.oracle_pcd_sweep.argtypes = [_pd, _pd, _i64, _d, _d, _pi, _pi, _pi, _i64, ctypes.c_int]
        L.oracle_u2_sweep.argtypes = [_pd, _pd, _i64, _d, _d, _pi, _pi, _i64]
        L.oracle_circle_flat.argtypes = [_i64, _pi, _pi, _pi]
        L.oracle_circle_flat.restype = _i64
        L.oracle_vech_max_abs_diff.argtypes = [_pd, _pd, _i64]
        L.oracle_vech_max_abs_diff.restype = _d
        _LIB = L
    return _LIB


def load_ref():
    """The reference's own compiled kernel module from oracle/_ref, or None."""
    global _REF
    if _REF is None:
        hits = glob.glob(os.path.join(HERE, "_ref", "_ckernels*.so"))
        if not hits:
            return None
        spec = importlib.util.spec_from_file_location("_ckernels", hits[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF = mod
    return _REF


def _dp(a):
    return a.ctypes.data_as(_pd)


def _ip(a):
    return a.ctypes.data_as(_pi)


def circle_flat(p):
    """schedule.py:68-88 + solver.py:166-178 -> (rs, ss, offsets), int64 0-based."""
    if p < 2:
        raise ValueError("schedule needs p >= 2")
    pe = p + (p % 2)
    npairs = p * (p - 1) // 2
    rs = np.empty(max(npairs, 1), np.int64)
    ss = np.empty(max(npairs, 1), np.int64)
    offsets = np.empty(pe, np.int64)
    lib().oracle_circle_flat(p, _ip(rs), _ip(ss), _ip(offsets))
    return rs[:npairs], ss[:npairs], offsets


def _check(om, t):
    assert om.dtype == np.float64 and om.flags.c_contiguous
    assert t.dtype == np.float64 and t.flags.c_contiguous
    assert om.shape == t.shape and om.shape[0] == om.shape[1]


def pcd_sweep(om, t, n, shrink, rs, ss, offsets, workers=1):
    """_ckernels.pyx:68-102 (in place)."""
    _check(om, t)
    rs = np.ascontiguousarray(rs, np.int64)
    ss = np.ascontiguousarray(ss, np.int64)
    offsets = np.ascontiguousarray(offsets, np.int64)
    lib().oracle_pcd_sweep(_dp(om), _dp(t), om.shape[0], float(n), float(shrink),
                           _ip(rs), _ip(ss), _ip(offsets), offsets.shape[0] - 1, int(workers))


def u2_sweep(om, t, n, shrink, rs, ss):
    """_ckernels.pyx:105-118 (in place)."""
    _check(om, t)
    rs = np.ascontiguousarray(rs, np.int64)
    ss = np.ascontiguousarray(ss, np.int64)
    lib().oracle_u2_sweep(_dp(om), _dp(t), om.shape[0], float(n), float(shrink),
                          _ip(rs), _ip(ss), rs.shape[0])


def cd_sweep(om, t, n, shrink):
    """_ckernels.pyx:53-65 (in place)."""
    _check(om, t)
    lib().oracle_cd_sweep(_dp(om), _dp(t), om.shape[0], float(n), float(shrink))


def vech_max_abs_diff(a, b):
    """solver.py:287: cyclic_max_reduce(_vech(a - b)) == linear max scan."""
    return lib().oracle_vech_max_abs_diff(_dp(a), _dp(b), a.shape[0])


_TRIU = {}


def vech(a):
    """solver.py:181-189 (`_vech`): the stacked upper triangle, by fancy indexing."""
    p = a.shape[0]
    if p not in _TRIU:
        _TRIU.clear()
        _TRIU[p] = np.triu_indices(p)
    rows, cols = _TRIU[p]
    return a[rows, cols]


def cyclic_max_reduce(d):
    """solver.py:141-163: max |d_j| by halving folds (numpy, as the reference runs it)."""
    work = np.array(d, dtype=np.float64, copy=True).ravel()
    m = work.shape[0]
    if m == 1:
        return float(abs(work[0]))
    z = (m - 1).bit_length()
    width = 1 << (z - 1)
    count = min(width, m - width)
    work[:count] = np.maximum(np.abs(work[:count]), np.abs(work[width:width + count]))
    for q in range(z - 2, -1, -1):
        width = 1 << q
        work[:width] = np.maximum(np.abs(work[:width]), np.abs(work[width:2 * width]))
    return float(work[0])


def objective(om, t, n, lam):
    """model.py:210-217, verbatim arithmetic."""
    diag = np.diag(om)
    logdet_part = -float(n) * float(np.sum(np.log(diag)))
    quad = 0.5 * float(np.einsum("ij,ij->", om @ t, om))
    penalty = float(n) * lam * float(np.sum(np.abs(om[np.triu_indices(om.shape[0], k=1)])))
    return logdet_part + quad + penalty


def edge_count(om):
    """model.py:249-253."""
    return int(np.count_nonzero(om[np.triu_indices(om.shape[0], k=1)]))


def pcd_fit(t, n, lam, delta_tol=1e-5, max_iter=200, workers=1, init=None,
            trace=True, sweeps=None, use_ref=False, numpy_delta=False):
    """solver.py:254-294 driver loop over the oracle (or oracle/_ref) sweep.

    Returns a dict mirroring FitReport.  ``sweeps`` (a list) receives a copy
    of the iterate after every sweep when given.  ``numpy_delta`` computes the
    convergence metric as the reference does, cyclic_max_reduce(_vech(om -
    snapshot)) in numpy (solver.py:287), instead of the C scan: the same value,
    and the reference's own cost inside wall_time_per_iteration.
    """
    t = np.ascontiguousarray(t, np.float64)
    p = t.shape[0]
    rs, ss, offsets = circle_flat(p)
    om = np.eye(p) if init is None else np.array(init, np.float64, copy=True, order="C")
    ref = load_ref() if use_ref else None
    if use_ref and ref is None:
        raise RuntimeError("oracle/_ref is not built")
    objs, times = [], []
    delta = math.inf
    converged = False
    it = 0
    for it in range(1, max_iter + 1):
        snap = om.copy()
        tic = time.perf_counter()
        if ref is not None:
            ref.pcd_sweep(om, t, float(n), float(n) * lam, rs.astype(np.intp),
                          ss.astype(np.intp), offsets.astype(np.intp), int(workers))
        else:
            pcd_sweep(om, t, n, float(n) * lam, rs, ss, offsets, workers)
        delta = cyclic_max_reduce(vech(om - snap)) if numpy_delta else vech_max_abs_diff(om, snap)
        times.append(time.perf_counter() - tic)
        if trace:
            objs.append(objective(om, t, n, lam))
        if sweeps is not None:
            sweeps.append(om.copy())
        if delta < delta_tol:
            converged = True
            break
    return dict(omega=om, iterations=it, final_delta=delta, converged=converged,
                objective_trace=tuple(objs), edge_count=edge_count(om),
                wall_time_per_iteration=tuple(times))


def cd_fit(t, n, lam, delta_tol=1e-5, max_iter=200):
    """solver.py:227-251 (serial CD; delta over the full matrix, model.py:243-246)."""
    t = np.ascontiguousarray(t, np.float64)
    p = t.shape[0]
    om = np.eye(p)
    delta = math.inf
    it = 0
    for it in range(1, max_iter + 1):
        snap = om.copy()
        cd_sweep(om, t, n, float(n) * lam)
        delta = float(np.max(np.abs(om - snap)))
        if delta < delta_tol:
            return dict(omega=om, iterations=it, final_delta=delta, converged=True,
                        edge_count=edge_count(om))
    return dict(omega=om, iterations=it, final_delta=delta, converged=False,
                edge_count=edge_count(om))
