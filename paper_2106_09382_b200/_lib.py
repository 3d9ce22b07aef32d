"""ctypes binding of libconcord_b200.so (the C ABI in include/concord_pcd.h).

There is no CPU fallback: if the library cannot be loaded, or no CUDA device
is present, every solver entry point raises.
"""

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CONCORD_LIB_PATH") or os.path.join(PKG, "libconcord_b200.so")

CONCORD_OK = 0
CONCORD_YIELDED = 1
CONCORD_ERR_ARG = -1
CONCORD_NOT_CONVERGED = -2
CONCORD_ERR_CUDA = -3
CONCORD_ERR_ZERO_VARIANCE = -4
CONCORD_ERR_NO_DEVICE = -5
CONCORD_ERR_OOM = -6
HOST, DEVICE = 0, 1

# Every symbol include/concord_pcd.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "concord_abi_version", "concord_last_error", "concord_device_count",
    "concord_solver_create", "concord_solver_destroy", "concord_solver_set_stream",
    "concord_solver_stream", "concord_solver_set_gram", "concord_solver_gram_from_data",
    "concord_solver_get_gram", "concord_solver_fit", "concord_solver_get_omega",
    "concord_solver_edge_count", "concord_solver_sweep_stats", "concord_host_alloc",
    "concord_host_free", "concord_gram_f64", "concord_pcd_fit",
    "concord_pcd_sweep_exact", "concord_u2_sweep_exact", "concord_cd_sweep_exact",
    "concord_solver_create_sharded", "concord_solver_layout", "concord_shard_create",
    "concord_shard_ipc_handle", "concord_shard_open_peers", "concord_solver_objective_parts",
    "concord_solver_check_optimality", "concord_solver_estimate_entries",
    "concord_ar2_data_f64", "concord_solver_gram_from_ar2", "concord_blocked_plan", "concord_device_sm_count",
    "concord_solver_gram_from_raw_data", "concord_center_columns_f64",
    "concord_tree_data_f64", "concord_solver_gram_from_tree", "concord_solver_set_chain_warps",
    "concord_solver_request_yield", "concord_solver_export_state", "concord_solver_import_state",
    "concord_solver_take_state", "concord_solver_copy_gram",
    "concord_solver_reserve",
)

ABI_VERSION = 2
SHARD_HANDLE_BYTES = 64


class FitParams(ctypes.Structure):
    _fields_ = [
        ("lam", ctypes.c_double),
        ("delta_tol", ctypes.c_double),
        ("max_iter", ctypes.c_int32),
        ("want_trace", ctypes.c_int32),
        ("omega_init", ctypes.c_void_p),
        ("init_where", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class FitResult(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("converged", ctypes.c_int32),
        ("final_delta", ctypes.c_double),
        ("edge_count", ctypes.c_int64),
        ("kernel_ms", ctypes.c_double),
        ("setup_ms", ctypes.c_double),
        ("n_blocks", ctypes.c_int32),
        ("slab_width", ctypes.c_int32),
    ]


class Layout(ctypes.Structure):
    _fields_ = [
        ("p", ctypes.c_int64),
        ("slab_width", ctypes.c_int32),
        ("n_shards", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("blocks_per_shard", ctypes.c_int32),
        ("blocks_total", ctypes.c_int32),
        ("col0", ctypes.c_int64),
        ("ncols", ctypes.c_int64),
        ("lag_cap", ctypes.c_int32),
        ("kernel", ctypes.c_int32),
    ]


class BlockedPlan(ctypes.Structure):
    """concord_blocked_plan_t: the fit-kernel plan for a problem size (host-only query)."""
    _fields_ = [
        ("colours_per_barrier", ctypes.c_int32),
        ("cell_buffers", ctypes.c_int32),
        ("tdiag_in_smem", ctypes.c_int32),
        ("ring_stages", ctypes.c_int32),
        ("smem_bytes", ctypes.c_int64),
        ("slab_width", ctypes.c_int32),
        ("ctas", ctypes.c_int32),
        ("share", ctypes.c_int32),
    ]


class ConcordError(RuntimeError):
    """A failure reported by the CUDA library."""

    def __init__(self, code, message):
        self.code = code
        super().__init__(f"libconcord_b200 error {code}: {message}")


_lock = threading.Lock()
_lib = None


def load(build_if_missing=True):
    """Load (building first if needed) the CUDA library; raises if impossible."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if build_if_missing:
            from .build import _stale, build

            if _stale():
                build()
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA library {LIB_PATH} is missing; run python -m paper_2106_09382_b200.build")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        sig = {
            "concord_abi_version": ([], ctypes.c_int),
            "concord_last_error": ([], ctypes.c_char_p),
            "concord_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
            "concord_solver_create": ([i64, i32, i32, ctypes.POINTER(vp)], ctypes.c_int),
            "concord_solver_destroy": ([vp], ctypes.c_int),
            "concord_solver_set_stream": ([vp, vp], ctypes.c_int),
            "concord_solver_stream": ([vp], vp),
            "concord_solver_set_gram": ([vp, vp, d, i32], ctypes.c_int),
            "concord_solver_gram_from_data": ([vp, vp, i64, i32], ctypes.c_int),
            "concord_solver_gram_from_raw_data": ([vp, vp, i64, i32], ctypes.c_int),
            "concord_center_columns_f64": ([vp, i64, i64, i32, i32], ctypes.c_int),
            "concord_tree_data_f64": ([i64, i64, ctypes.c_uint64, vp, vp, vp, vp, i32, i32], ctypes.c_int),
            "concord_solver_gram_from_tree": ([vp, i64, ctypes.c_uint64, vp, vp, vp], ctypes.c_int),
            "concord_solver_set_chain_warps": ([vp, i32], ctypes.c_int),
            "concord_solver_request_yield": ([vp, i32], ctypes.c_int),
            "concord_solver_export_state": ([vp, vp, vp, i32], ctypes.c_int),
            "concord_solver_import_state": ([vp, vp, vp, i32], ctypes.c_int),
            "concord_solver_take_state": ([vp, vp], ctypes.c_int),
            "concord_solver_copy_gram": ([vp, vp], ctypes.c_int),
            "concord_solver_reserve": ([vp, i32], ctypes.c_int),
            "concord_solver_get_gram": ([vp, vp, i32], ctypes.c_int),
            "concord_solver_fit": ([vp, ctypes.POINTER(FitParams), ctypes.POINTER(FitResult), vp, vp, vp],
                                   ctypes.c_int),
            "concord_solver_get_omega": ([vp, vp, i32], ctypes.c_int),
            "concord_solver_edge_count": ([vp, ctypes.POINTER(i64)], ctypes.c_int),
            "concord_solver_sweep_stats": ([vp, vp, i32, ctypes.POINTER(i32)], ctypes.c_int),
            "concord_host_alloc": ([i64, ctypes.POINTER(vp)], ctypes.c_int),
            "concord_blocked_plan": ([i64, i32, ctypes.POINTER(BlockedPlan)], ctypes.c_int),
            "concord_device_sm_count": ([i32, ctypes.POINTER(i32)], ctypes.c_int),
            "concord_host_free": ([vp], ctypes.c_int),
            "concord_gram_f64": ([vp, i64, i64, vp, i32], ctypes.c_int),
            "concord_pcd_fit": ([vp, i64, d, ctypes.POINTER(FitParams), vp, ctypes.POINTER(FitResult), vp, vp,
                                 vp, i32], ctypes.c_int),
            "concord_pcd_sweep_exact": ([vp, vp, i64, d, d, vp, vp, vp, i64, i32], ctypes.c_int),
            "concord_u2_sweep_exact": ([vp, vp, i64, d, d, vp, vp, i64, i32], ctypes.c_int),
            "concord_cd_sweep_exact": ([vp, vp, i64, d, d, i32], ctypes.c_int),
            "concord_solver_create_sharded": ([i64, i32, i32, i32, ctypes.POINTER(vp)], ctypes.c_int),
            "concord_solver_layout": ([vp, ctypes.POINTER(Layout)], ctypes.c_int),
            "concord_shard_create": ([i64, i32, i32, i32, i32, ctypes.POINTER(vp)], ctypes.c_int),
            "concord_shard_ipc_handle": ([vp, vp], ctypes.c_int),
            "concord_shard_open_peers": ([vp, vp], ctypes.c_int),
            "concord_solver_objective_parts": ([vp, vp, i32], ctypes.c_int),
            "concord_solver_check_optimality": ([vp, d, ctypes.POINTER(d), ctypes.POINTER(i64), ctypes.POINTER(i64)],
                                                ctypes.c_int),
            "concord_solver_estimate_entries": ([vp, ctypes.POINTER(i64), vp, vp, vp, i64], ctypes.c_int),
            "concord_ar2_data_f64": ([i64, i64, ctypes.c_uint64, vp, i32, i32], ctypes.c_int),
            "concord_solver_gram_from_ar2": ([vp, i64, ctypes.c_uint64], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def last_error():
    return load().concord_last_error().decode(errors="replace")


def check(rc, allow=()):
    """Raise ConcordError for a non-zero return code not in `allow`."""
    if rc != CONCORD_OK and rc not in allow:
        if rc == CONCORD_ERR_ZERO_VARIANCE:
            from .model import ZeroVarianceColumn

            msg = last_error()
            col = [int(t) for t in msg.split() if t.isdigit()]
            raise ZeroVarianceColumn(col[0] if col else -1)
        raise ConcordError(rc, last_error())
    return rc


def device_count():
    c = ctypes.c_int(0)
    load().concord_device_count(ctypes.byref(c))
    return c.value


def require_device():
    if device_count() < 1:
        raise RuntimeError("paper_2106_09382_b200 needs a CUDA device (B200); none is visible. "
                           "There is no CPU fallback.")


def ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


class _PinnedOwner:
    """Keeps a cudaHostAlloc buffer alive for as long as a numpy view refers to it."""

    def __init__(self, addr):
        self.addr = addr

    def __del__(self):
        try:
            load().concord_host_free(ctypes.c_void_p(self.addr))
        except Exception:
            pass


class _PooledOwner:
    """A pooled page-locked block: returned to the pool (not freed) when the last view dies."""

    def __init__(self, addr, nbytes):
        self.addr = addr
        self.nbytes = nbytes

    def __del__(self):
        try:
            with _POOL_LOCK:
                free = _POOL.setdefault(self.nbytes, [])
                keep = (len(free) + 1) * self.nbytes <= _POOL_KEEP_BYTES or not free
                if keep:
                    free.append(self.addr)
            if not keep:
                load().concord_host_free(ctypes.c_void_p(self.addr))
        except Exception:
            pass


_POOL = {}  # nbytes -> free page-locked blocks
_POOL_LOCK = threading.Lock()  # lanes of a PathScheduler take and return blocks concurrently
_POOL_KEEP_BYTES = 4 << 30  # per block size (a lambda path keeps ten 200 MB results alive at p=5000)


def device_sm_count(device=0):
    n = ctypes.c_int32()
    check(load().concord_device_sm_count(int(device), ctypes.byref(n)))
    return n.value


def blocked_plan(p, n_sms=148):
    """Fit-kernel plan for a p x p problem on one device with n_sms SMs (no device needed)."""
    out = BlockedPlan()
    check(load().concord_blocked_plan(int(p), int(n_sms), ctypes.byref(out)))
    return {f: getattr(out, f) for f, _ in BlockedPlan._fields_}


def pooled_pinned_empty(shape, dtype=None):
    """numpy array in page-locked host memory, recycled through a pool.

    The result arrays of consecutive fits (200 MB at p=5000) then land in memory
    that is already pinned and faulted in: a device->host copy runs at DMA speed
    instead of paying page faults on fresh pageable memory (~45 ms per fit at
    p=5000).  The array owns its block until it is garbage collected.
    """
    import numpy as np

    dtype = np.dtype(dtype or np.float64)
    count = int(np.prod(shape))
    nbytes = max(count * dtype.itemsize, 1)
    if device_count() < 1:
        return np.empty(shape, dtype)
    with _POOL_LOCK:
        free = _POOL.get(nbytes)
        addr = free.pop() if free else None
    if addr is None:
        raw = ctypes.c_void_p()
        check(load().concord_host_alloc(nbytes, ctypes.byref(raw)))
        addr = raw.value
    buf = (ctypes.c_char * nbytes).from_address(addr)
    buf._owner = _PooledOwner(addr, nbytes)
    return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)


def pinned_empty(shape, dtype=None):
    """numpy array in page-locked host memory (cudaHostAlloc); plain memory if no device."""
    import numpy as np

    dtype = np.dtype(dtype or np.float64)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    if device_count() < 1:
        return np.empty(shape, dtype)
    raw = ctypes.c_void_p()
    check(load().concord_host_alloc(nbytes, ctypes.byref(raw)))
    buf = (ctypes.c_char * max(nbytes, 1)).from_address(raw.value)
    buf._owner = _PinnedOwner(raw.value)
    arr = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
    return arr
