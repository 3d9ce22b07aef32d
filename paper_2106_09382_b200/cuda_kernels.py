"""Sweep-level kernel module in the reference's backend protocol.

Same module contract as /root/reference/pkg/src/parconcord/_ckernels.pyx:
`name`, `cd_sweep(om, t, n, shrink)`, `pcd_sweep(om, t, n, shrink, rs, ss,
offsets, workers)` and `u2_sweep(om, t, n, shrink, rs, ss)`, mutating `om`
in place and keeping it exactly symmetric.  Each call runs one bit-exact
sweep on the GPU (csrc/pcd_exact.cu), so results equal the reference's
compiled backend bit for bit.  Buffer type errors raise ValueError, like the
typed memoryviews of the Cython module.
"""

import numpy as np

from . import _lib

name = "cuda"


def _mat(a, what, writable=False):
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.ndim != 2 or not a.flags.c_contiguous:
        raise ValueError(f"{what} must be a C-contiguous 2-d float64 array")
    if writable and not a.flags.writeable:
        raise ValueError(f"{what} must be writable")
    return a


def _idx(a, what):
    a = np.asarray(a)
    if a.ndim != 1 or a.dtype.kind not in "iu":
        raise ValueError(f"{what} must be a 1-d integer array")
    return np.ascontiguousarray(a, dtype=np.int64)


def _check_pair(om, t):
    _mat(om, "om", writable=True)
    _mat(t, "t")
    if om.shape != t.shape or om.shape[0] != om.shape[1]:
        raise ValueError("om and t must be square and of equal shape")


def pcd_sweep(om, t, n, shrink, rs, ss, offsets, workers=1, device=0):
    """_ckernels.pyx:68-102 -- rounds of concurrent pairs, then diagonals."""
    _check_pair(om, t)
    rs, ss, offsets = _idx(rs, "rs"), _idx(ss, "ss"), _idx(offsets, "offsets")
    L = _lib.load()
    _lib.check(L.concord_pcd_sweep_exact(_lib.ptr(om), _lib.ptr(t), om.shape[0], float(n), float(shrink),
                                         _lib.ptr(rs), _lib.ptr(ss), _lib.ptr(offsets), offsets.shape[0] - 1,
                                         device))


def u2_sweep(om, t, n, shrink, rs, ss, device=0):
    """_ckernels.pyx:105-118 -- serial replay with immediate writes, then diagonals."""
    _check_pair(om, t)
    rs, ss = _idx(rs, "rs"), _idx(ss, "ss")
    L = _lib.load()
    _lib.check(L.concord_u2_sweep_exact(_lib.ptr(om), _lib.ptr(t), om.shape[0], float(n), float(shrink),
                                        _lib.ptr(rs), _lib.ptr(ss), rs.shape[0], device))


def cd_sweep(om, t, n, shrink, device=0):
    """_ckernels.pyx:53-65 -- serial upper triangle row-major, then diagonals."""
    _check_pair(om, t)
    L = _lib.load()
    _lib.check(L.concord_cd_sweep_exact(_lib.ptr(om), _lib.ptr(t), om.shape[0], float(n), float(shrink), device))
