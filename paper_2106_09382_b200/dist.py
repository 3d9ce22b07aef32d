"""Multi-GPU CONCORD-PCD: one process per GPU, column-sharded.

W = Omega*T, T and Omega are split by column block: GPU g owns slabs
[g*B, (g+1)*B) of the kernel's column slabs (B = blocks per shard).  The
fit runs the temporally blocked kernel (csrc/pcd_qblock.cu) on every GPU:
each CTA owns a range of pair indices and evaluates D=4 colours per grid
barrier, so the cross-GPU barrier is paid once per 4 colours.  Its data-path
exchange is the cells the colours read -- the slab owners' staged (W, Omega,
T) entries -- plus the per-row delta ring, the non-zero delta lists and the
diagonal step's (delta, new) vector.  It happens INSIDE the persistent
kernel: each writer stores into every GPU's copy of these buffers through
NVLink peer pointers (cudaIpc handles of one arena per GPU, opened here),
fences at system scope and arrives on every GPU's barrier counter; no host
NCCL call per colour.  T is replicated (the cells read T entries of every
column).  Every GPU evaluates identical arithmetic, so the estimate is
bitwise identical for any GPU count -- the analogue of the reference's
worker invariance (test_solver.py:222-230).  p < 256 uses the per-phase
kernel (csrc/pcd_wform.cu) with the same exchange per colour.

torch.distributed is the plumbing only: it all-gathers the 64-byte IPC
handles once, and at the end all-reduces the per-sweep objective partials /
edge counts and (optionally) gathers the column blocks of Omega.

    torchrun --nproc-per-node 8 ... :
        s = ShardedSolver(p)                 # one shard per rank
        s.set_gram(GramMatrix(t, n))         # full T on every rank
        rep = s.fit(lam=0.3)                 # FitReport (Omega gathered)
"""

import ctypes

import numpy as np

from . import _lib
from .model import GramMatrix, PrecisionEstimate
from .solver import FitReport, NotConverged

NSM = 148


# --------------------------------------------------------------- pure helpers


def partition(p, n_shards, n_blocks=0, nsm=NSM, rank=None):
    """Column split of the sharded solver (mirrors create_common in csrc/capi.cu).

    Returns the slab width, blocks per shard and each shard's column range
    (a shard may hold fewer columns -- or none -- at the end).
    """
    if n_blocks > 0:
        w = -(-p // n_blocks)
    else:
        tot = nsm * (n_shards if rank is not None else 1)
        w = max(8, -(-p // tot))
    w += w & 1
    w4 = (w + 3) & ~3  # default layout: whole 32-byte sectors when that keeps >= 90% of the slabs (capi.cu)
    if n_blocks <= 0 and w4 != w and 10 * -(-p // w4) >= 9 * -(-p // w):
        w = w4
    need = -(-p // w)
    per = -(-need // n_shards)
    ranges = []
    for g in range(n_shards):
        c0 = min(p, g * per * w)
        c1 = min(p, (g + 1) * per * w)
        ranges.append((c0, c1))
    return {"slab_width": w, "blocks_per_shard": per, "blocks_total": per * n_shards, "ranges": ranges}


def exchange_handles(handle, group=None):
    """All-gather one fixed-size handle per rank, in rank order."""
    import torch.distributed as dist

    if len(handle) != _lib.SHARD_HANDLE_BYTES:
        raise ValueError(f"handle must be {_lib.SHARD_HANDLE_BYTES} bytes")
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(handle), group=group)
    return b"".join(out)


def reduce_parts(parts, group=None):
    """Sum per-sweep objective partials / counts over ranks (float64, any shape)."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(np.ascontiguousarray(parts, dtype=np.float64)).clone()
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, group=group)
    return t.cpu().numpy()


def gather_columns(block, col0, p, group=None, dst=None):
    """Assemble the p x p matrix from every rank's p x ncols column block.

    dst=None: every rank gets the full matrix; dst=r: only rank r does (others get None).
    """
    import torch.distributed as dist

    item = (int(col0), np.ascontiguousarray(block))
    world = dist.get_world_size(group)
    if dst is None:
        parts = [None] * world
        dist.all_gather_object(parts, item, group=group)
    else:
        parts = [None] * world if dist.get_rank(group) == dst else None
        dist.gather_object(item, parts, dst=dst, group=group)
        if parts is None:
            return None
    full = np.empty((p, p))
    for c0, blk in parts:
        full[:, c0:c0 + blk.shape[1]] = blk
    return full


def objective_from_parts(parts, n, lam):
    """model.py:210-217 from the summed (<W,Omega>, sum_{i<j}|om|, sum log om_ii) of each sweep."""
    q, pen, lg = parts[:, 0], parts[:, 1], parts[:, 2]
    return -n * lg + 0.5 * q + n * lam * pen


# --------------------------------------------------------------- the solver


class ShardedSolver:
    """One column shard of a multi-GPU CONCORD-PCD problem (this process's GPU)."""

    def __init__(self, p, group=None, device=None, n_blocks=0):
        import torch
        import torch.distributed as dist

        L = _lib.load()
        _lib.require_device()
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.p = int(p)
        h = ctypes.c_void_p()
        _lib.check(L.concord_shard_create(self.p, self.world, self.rank, self.device, int(n_blocks),
                                          ctypes.byref(h)))
        self._h = h
        mine = (ctypes.c_char * _lib.SHARD_HANDLE_BYTES)()
        _lib.check(L.concord_shard_ipc_handle(h, mine))
        allh = exchange_handles(bytes(mine), group)
        buf = (ctypes.c_char * len(allh)).from_buffer_copy(allh)
        _lib.check(L.concord_shard_open_peers(h, buf))
        dist.barrier(group=group)  # every arena is zeroed and mapped before any kernel writes to it
        lay = _lib.Layout()
        _lib.check(L.concord_solver_layout(h, ctypes.byref(lay)))
        self.col0, self.ncols = int(lay.col0), int(lay.ncols)
        self.slab_width, self.blocks_total = int(lay.slab_width), int(lay.blocks_total)
        self.n = None

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().concord_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_gram(self, gram: GramMatrix):
        t = np.ascontiguousarray(gram.t, dtype=np.float64)
        _lib.check(_lib.load().concord_solver_set_gram(self._h, _lib.ptr(t), float(gram.n), _lib.HOST))
        self.n = gram.n

    def gram_from_data(self, x):
        _lib.check(_lib.load().concord_solver_gram_from_data(self._h, _lib.ptr(x.values), x.n, _lib.HOST))
        self.n = x.n

    def gram_from_ar2(self, n, seed=0):
        """T from n AR(2) samples drawn on this GPU (counter-based stream: every rank draws the same X)."""
        _lib.check(_lib.load().concord_solver_gram_from_ar2(self._h, int(n), int(seed)))
        self.n = int(n)

    def omega_block(self):
        out = np.empty((self.p, self.ncols))
        _lib.check(_lib.load().concord_solver_get_omega(self._h, _lib.ptr(out), _lib.HOST))
        return out

    def fit(self, lam, delta_tol=1e-5, max_iter=200, trace=True, gather=True, raise_on_cap=True):
        """Every rank calls this concurrently; returns a FitReport (Omega gathered when gather=True)."""
        import torch.distributed as dist

        L = _lib.load()
        prm = _lib.FitParams()
        prm.lam, prm.delta_tol, prm.max_iter, prm.want_trace = float(lam), float(delta_tol), int(max_iter), int(trace)
        res = _lib.FitResult()
        deltas, secs = np.zeros(max_iter), np.zeros(max_iter)
        dist.barrier(group=self.group)
        rc = L.concord_solver_fit(self._h, ctypes.byref(prm), ctypes.byref(res), _lib.ptr(deltas), None,
                                  _lib.ptr(secs))
        _lib.check(rc, allow=(_lib.CONCORD_NOT_CONVERGED,))
        k = int(res.iterations)
        parts = np.zeros((max(k, 1), 3))
        _lib.check(L.concord_solver_objective_parts(self._h, _lib.ptr(parts), k))
        tot = reduce_parts(np.concatenate([parts[:k].ravel(), [float(res.edge_count)]]), self.group)
        objs = objective_from_parts(tot[:-1].reshape(k, 3), float(self.n), lam) if trace else ()
        edges = int(round(tot[-1]))
        full = gather_columns(self.omega_block(), self.col0, self.p, self.group) if gather else None
        report = FitReport(
            estimate=PrecisionEstimate._trusted(full) if full is not None else None,
            iterations=k,
            final_delta=float(res.final_delta),
            converged=bool(res.converged),
            objective_trace=tuple(float(v) for v in objs),
            edge_count=edges,
            wall_time_per_iteration=tuple(float(v) for v in secs[:k]),
        )
        self.last_result = res
        if rc == _lib.CONCORD_NOT_CONVERGED and raise_on_cap:
            raise NotConverged(report)
        return report


def pcd_fit_sharded(gram: GramMatrix, lam, delta_tol=1e-5, max_outer_iterations=200, group=None):
    """pcd_fit over every rank of `group` (one GPU each); same FitReport on every rank."""
    s = ShardedSolver(gram.p, group=group)
    try:
        s.set_gram(gram)
        return s.fit(lam, delta_tol, max_outer_iterations)
    finally:
        s.close()


__all__ = ["ShardedSolver", "pcd_fit_sharded", "partition", "exchange_handles", "reduce_parts", "gather_columns",
           "objective_from_parts"]
