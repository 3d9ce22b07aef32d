"""The drop-in solver entry points: pcd_fit / cd_fit / FitReport on the GPU.

`pcd_fit(x_or_gram, config, schedule=None, backend=None)` keeps the signature,
arguments, return type and exceptions of the reference driver
(/root/reference/pkg/src/parconcord/solver.py:254-294).  With the default
backend ("cuda") the whole fit -- every colour of every sweep, the diagonal
step, the max |delta| convergence test and the objective trace -- runs in ONE
persistent cooperative kernel on a device-resident W = Omega*T (pcd_qblock.cu,
D colours per grid barrier; pcd_wform.cu for p < 256 and multi-GPU shards).
`pcd_path(..., concurrency=k)` runs a cold lambda path on k lanes of SMs
(`PathScheduler`).

backend="cuda-exact" instead runs the reference's own driver loop over GPU
sweeps that reproduce the compiled reference kernel bit for bit
(pcd_exact.cu); it is the parity hook, not the fast path.  There is no CPU
backend: without the CUDA library or a device every entry point raises.
"""

import contextlib
import ctypes
import math
import os
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .model import (
    DataMatrix,
    DimensionError,
    GramMatrix,
    PrecisionEstimate,
    SolverConfig,
    compute_gram,
)
from .schedule import (
    IndexPair,
    Schedule,
    flat_circle_schedule,
    flatten_schedule,
    is_circle_schedule,
    validate_schedule,
)

BACKENDS = ("cuda", "cuda-exact")


class NotConverged(RuntimeError):
    """Iteration cap hit; carries the partial FitReport (solver.py:46-54)."""

    def __init__(self, report):
        self.report = report
        super().__init__(
            f"no convergence after {report.iterations} outer iterations, "
            f"final delta {report.final_delta:.3e}"
        )


class ScheduleMismatch(ValueError):
    """Supplied schedule does not fit the problem (solver.py:57-58)."""


class EmptyVector(ValueError):
    """Reduction over zero elements (solver.py:61-62)."""


@dataclass(frozen=True)
class FitReport:
    """Everything a fit produced (solver.py:65-80).

    wall_time_per_iteration holds the device time of each sweep (all colours,
    the diagonal step and the fused max |delta|), measured in-kernel with the
    GPU global timer; objective bookkeeping is fused into the diagonal stream.
    """

    estimate: PrecisionEstimate
    iterations: int
    final_delta: float
    converged: bool
    objective_trace: tuple
    edge_count: int
    wall_time_per_iteration: tuple


# ----------------------------------------------------------------- backends


def available_backends():
    """Backends usable in this process (the CUDA library loads and a device is visible)."""
    try:
        _lib.load()
        return BACKENDS if _lib.device_count() > 0 else ()
    except Exception:
        return ()


def default_backend_name():
    env = os.environ.get("CONCORD_B200_BACKEND")
    if env:
        if env not in BACKENDS:
            raise ValueError(f"CONCORD_B200_BACKEND must be one of {BACKENDS}, got {env!r}")
        return env
    return "cuda"


def get_backend(name=None):
    """Sweep-level kernel module in the reference protocol (_backend.py:36-49).

    Both names resolve to the bit-exact GPU sweeps (`name`, `cd_sweep`,
    `pcd_sweep`, `u2_sweep`), so the reference's own driver loop and tests run
    against the GPU unchanged.
    """
    if name is None:
        name = default_backend_name()
    if name not in BACKENDS:
        raise ValueError(f"unknown backend {name!r}")
    from . import cuda_kernels

    _lib.require_device()
    return cuda_kernels


# ----------------------------------------------------------- host utilities


def cyclic_max_reduce(d) -> float:
    """max |d_j| (solver.py:141-163); the device fuses this into the sweep."""
    work = np.asarray(d, dtype=np.float64).ravel()
    if work.size == 0:
        raise EmptyVector("cannot reduce an empty vector")
    return float(np.max(np.abs(work)))


def diff_vector(a: PrecisionEstimate, b: PrecisionEstimate):
    """Stacked upper-triangle difference, length p(p+1)/2 (solver.py:192-200)."""
    if a.p != b.p:
        raise DimensionError(f"shapes differ: p={a.p} vs p={b.p}")
    iu = np.triu_indices(a.p)
    return (a.omega - b.omega)[iu]


def _as_gram(x_or_gram, device=0):
    if isinstance(x_or_gram, GramMatrix):
        return x_or_gram
    if isinstance(x_or_gram, DataMatrix):
        return compute_gram(x_or_gram, device=device)
    raise TypeError("expected a DataMatrix or GramMatrix")


# ------------------------------------------------------- device-resident solver


class Solver:
    """A device-resident CONCORD-PCD problem of size p on one GPU.

    Holds T, W = Omega*T and Omega in column-slab layout in HBM.  Use it to
    keep T resident across many fits (e.g. a lambda path); `pcd_fit` uses a
    transient one.
    """

    def __init__(self, p, device=0, n_blocks=0, n_shards=1):
        L = _lib.load()
        _lib.require_device()
        h = ctypes.c_void_p()
        if n_shards == 1:
            _lib.check(L.concord_solver_create(int(p), int(device), int(n_blocks), ctypes.byref(h)))
        else:
            # columns split over n_shards virtual shards with replicated exchange
            # buffers: the multi-GPU data flow (dist.py) on one device
            _lib.check(L.concord_solver_create_sharded(int(p), int(device), int(n_blocks), int(n_shards),
                                                       ctypes.byref(h)))
        self._h = h
        self._nblk = int(n_blocks)
        self.p = int(p)
        self.device = int(device)
        self.n = None
        self.last_result = None

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().concord_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def layout(self):
        """Column partition: slab width, shards, CTAs, this solver's column range."""
        lay = _lib.Layout()
        _lib.check(_lib.load().concord_solver_layout(self._h, ctypes.byref(lay)))
        return {f: getattr(lay, f) for f, _ in _lib.Layout._fields_}

    def set_chain_warps(self, chain_warps):
        """Kernel variant for this solver's fits: 6 chain warps (default), 4 (apply-heavy: dense
        fits) or 8 (chain-heavy: sparse fits on a small lane).  4 and 8 align the roles to warp
        groups and move registers between them (setmaxnreg); results are bitwise identical."""
        _lib.check(_lib.load().concord_solver_set_chain_warps(self._h, int(chain_warps)))
        self.chain_warps = int(chain_warps)

    def set_stream(self, stream_ptr):
        _lib.check(_lib.load().concord_solver_set_stream(self._h, ctypes.c_void_p(stream_ptr or None)))

    def set_gram(self, gram: GramMatrix):
        if gram.p != self.p:
            raise DimensionError(f"solver has p={self.p} but gram has p={gram.p}")
        t = np.ascontiguousarray(gram.t, dtype=np.float64)
        _lib.check(_lib.load().concord_solver_set_gram(self._h, _lib.ptr(t), float(gram.n), _lib.HOST))
        self.n = gram.n

    def set_gram_device(self, t_dev_ptr, n):
        """T already in device memory (row-major p x p float64 at t_dev_ptr)."""
        _lib.check(_lib.load().concord_solver_set_gram(self._h, ctypes.c_void_p(t_dev_ptr), float(n),
                                                      _lib.DEVICE))
        self.n = n

    def gram_from_data(self, x: DataMatrix, center=False):
        """compute_gram (model.py:190-197) of X as given, like the reference (callers own centering);
        center=True first runs center_columns on the device (bitwise numpy's, model.py:182-187) unless
        the DataMatrix is marked centred -- the CLI's load path (cli.py:101-102) without a host pass."""
        if x.p != self.p:
            raise DimensionError(f"solver has p={self.p} but data has p={x.p}")
        center = bool(center) and not x.centered
        fn = _lib.load().concord_solver_gram_from_raw_data if center else _lib.load().concord_solver_gram_from_data
        _lib.check(fn(self._h, _lib.ptr(x.values), x.n, _lib.HOST))
        self.n = x.n

    def gram_from_ar2(self, n, seed=0):
        """T of n centred AR(2) samples generated on the device (no host copy of X)."""
        _lib.check(_lib.load().concord_solver_gram_from_ar2(self._h, int(n), int(seed)))
        self.n = int(n)

    def gram_from_scale_free(self, n, seed=0, alpha=2.3, truth_seed=None):
        """T of n centred samples of the scale-free truth (datagen.py:99-132), drawn on the device
        through the truth's fill-free tree Cholesky factor (no dense p x p truth, no host copy of X)."""
        from .synth import scale_free_tree, tree_cholesky

        parent, weight = scale_free_tree(self.p, alpha, seed if truth_seed is None else truth_seed)
        lpar, ldiag = tree_cholesky(parent, weight)
        _lib.check(_lib.load().concord_solver_gram_from_tree(self._h, int(n), int(seed), _lib.ptr(parent),
                                                             _lib.ptr(lpar), _lib.ptr(ldiag)))
        self.n = int(n)

    def gram(self) -> GramMatrix:
        t = np.empty((self.p, self.p))
        _lib.check(_lib.load().concord_solver_get_gram(self._h, _lib.ptr(t), _lib.HOST))
        return GramMatrix._trusted(t, self.n)

    def fit_raw(self, lam, delta_tol=1e-5, max_iter=200, init=None, trace=True):
        """Run the persistent fit; returns (code, FitResult, deltas, objectives, sweep_seconds)."""
        L = _lib.load()
        prm = _lib.FitParams()
        prm.lam = float(lam)
        prm.delta_tol = float(delta_tol)
        prm.max_iter = int(max_iter)
        prm.want_trace = 1 if trace else 0
        keep = None
        if init is not None:
            keep = np.ascontiguousarray(init, dtype=np.float64)
            if keep.shape != (self.p, self.p):
                raise DimensionError(f"init has p={keep.shape[0]} but the problem has p={self.p}")
            prm.omega_init = keep.ctypes.data
            prm.init_where = _lib.HOST
        res = _lib.FitResult()
        deltas = np.zeros(max_iter)
        objs = np.zeros(max_iter)
        secs = np.zeros(max_iter)
        rc = L.concord_solver_fit(self._h, ctypes.byref(prm), ctypes.byref(res), _lib.ptr(deltas),
                                  _lib.ptr(objs), _lib.ptr(secs))
        _lib.check(rc, allow=(_lib.CONCORD_NOT_CONVERGED, _lib.CONCORD_YIELDED))
        self.last_result = res
        k = res.iterations
        return rc, res, deltas[:k], objs[:k], secs[:k]

    def request_yield(self, on=True):
        """Ask the blocked fit running on this solver (or its next one) to stop at the end of its
        current sweep unless that sweep converged or hit the cap: fit_raw then returns
        CONCORD_YIELDED and `take_state` on another solver continues it.  Thread-safe; stays set
        until request_yield(False)."""
        _lib.check(_lib.load().concord_solver_request_yield(self._h, 1 if on else 0))

    def take_state(self, src):
        """Continue src's yielded fit here: Omega and W = Omega T move slab layout to slab layout on
        the device; the next fit_raw resumes from them (bitwise the uninterrupted fit)."""
        _lib.check(_lib.load().concord_solver_take_state(self._h, src._h))

    def reserve(self, max_iter):
        """Allocate the scratch and the records of fits up to max_iter sweeps now (a solver that
        joins a running path must not allocate on the way: that can wait for the other kernels)."""
        _lib.check(_lib.load().concord_solver_reserve(self._h, int(max_iter)))

    def copy_gram(self, src):
        """T and n from another solver of the same p on the same device (device to device)."""
        _lib.check(_lib.load().concord_solver_copy_gram(self._h, src._h))
        self.n = src.n

    def export_state(self):
        """(Omega, W) of the last fit as host arrays (p x p each)."""
        om, w = np.empty((self.p, self.p)), np.empty((self.p, self.p))
        _lib.check(_lib.load().concord_solver_export_state(self._h, _lib.ptr(om), _lib.ptr(w), _lib.HOST))
        return om, w

    def import_state(self, om, w):
        """The next fit continues from (Omega, W) (host p x p arrays, e.g. from export_state)."""
        om = np.ascontiguousarray(om, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        if om.shape != (self.p, self.p) or w.shape != (self.p, self.p):
            raise DimensionError(f"state must be {self.p} x {self.p}")
        _lib.check(_lib.load().concord_solver_import_state(self._h, _lib.ptr(om), _lib.ptr(w), _lib.HOST))

    def omega(self, out=None):
        if out is None:
            out = _lib.pooled_pinned_empty((self.p, self.p))
        _lib.check(_lib.load().concord_solver_get_omega(self._h, _lib.ptr(out), _lib.HOST))
        return out

    def moving_fraction(self):
        """Fraction of the p(p-1)/2 pairs that moved per sweep in the last fit (device counters)."""
        it = int(self.last_result.iterations) if self.last_result is not None else 0
        if it <= 0:
            return 0.0
        nnz = np.zeros(it, dtype=np.int64)
        cnt = ctypes.c_int32()
        _lib.check(_lib.load().concord_solver_sweep_stats(self._h, _lib.ptr(nnz), it, ctypes.byref(cnt)))
        return float(nnz.sum()) / (it * (self.p * (self.p - 1) / 2))

    def check_optimality(self, lam, eps=1e-6):
        """check_optimality (model.py:256-289) of the last fit, on the device (M = W)."""
        from .model import OptimalityReport

        worst, i, j = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.load().concord_solver_check_optimality(self._h, float(lam), ctypes.byref(worst),
                                                               ctypes.byref(i), ctypes.byref(j)))
        return OptimalityReport(worst_violation=worst.value, worst_coordinate=(i.value, j.value), eps=eps,
                                ok=worst.value <= eps)

    def estimate_entries(self):
        """(i, j, value) arrays, 0-based, of every diagonal and every exact non-zero i < j,
        in (i, j) order -- what fileio.write_estimate stores (fileio.py:87-95)."""
        L = _lib.load()
        cnt = ctypes.c_int64()
        _lib.check(L.concord_solver_estimate_entries(self._h, ctypes.byref(cnt), None, None, None, 0))
        k = cnt.value
        ii, jj, vv = np.empty(k, np.int32), np.empty(k, np.int32), np.empty(k)
        _lib.check(L.concord_solver_estimate_entries(self._h, ctypes.byref(cnt), _lib.ptr(ii), _lib.ptr(jj),
                                                     _lib.ptr(vv), k))
        return ii, jj, vv

    def fit(self, lam, delta_tol=1e-5, max_iter=200, init=None, trace=True, raise_on_cap=True) -> FitReport:
        return self.report([self.fit_raw(lam, delta_tol, max_iter, init, trace)], trace, raise_on_cap)

    def report(self, segments, trace=True, raise_on_cap=True) -> FitReport:
        """FitReport of the fit whose last segment ran here: `segments` are fit_raw results, one per
        solver the fit ran on (PathScheduler hand-over), traces concatenated in order."""
        rc, res = segments[-1][0], segments[-1][1]
        deltas = np.concatenate([sg[2] for sg in segments])
        objs = np.concatenate([sg[3] for sg in segments])
        secs = np.concatenate([sg[4] for sg in segments])
        om = self.omega()
        # A converged fit's estimate is exactly symmetric with a positive diagonal by construction
        # (both mirrored cells get the same value; the diagonal closed form is positive).  A fit
        # that hit the cap may have diverged (non-finite data): validate it the way the
        # reference's _finish does (solver.py:214-224 -> model.py:117-120), which raises.
        report = FitReport(
            estimate=PrecisionEstimate._trusted(om) if res.converged else PrecisionEstimate(om),
            iterations=int(sum(int(sg[1].iterations) for sg in segments)),
            final_delta=float(res.final_delta),
            converged=bool(res.converged),
            objective_trace=tuple(float(v) for v in objs) if trace else (),
            edge_count=int(res.edge_count),
            wall_time_per_iteration=tuple(float(v) for v in secs),
        )
        if rc == _lib.CONCORD_NOT_CONVERGED and raise_on_cap:
            raise NotConverged(report)
        return report


def pcd_path(x_or_gram, lams, delta_tol=1e-5, max_outer_iterations=200, warm_start=False, device=0,
             trace=True, concurrency=1):
    """Fit a lambda path with T resident on the device.

    Cold mode (default) fits every lambda from the identity, exactly like
    independent `pcd_fit` calls; warm mode starts each fit from the previous
    estimate (SolverConfig.init semantics).  Returns one FitReport per lambda
    (a non-converged fit is returned with converged=False, not raised).

    concurrency=k (cold mode) runs the fits on k lanes, each a solver on its
    own share of the SMs (k=3 on a B200: 66/41/41; k=4: 66/28/27/27, the bench's), densest lambda first,
    lanes that run dry handing their SMs to the fits still running (`PathScheduler.run_segmented`);
    the results are bitwise those of sequential fits.
    """
    if concurrency > 1:
        if warm_start:
            raise ValueError("warm starts chain the fits: concurrency must be 1")
        return _path_concurrent(x_or_gram, lams, delta_tol, max_outer_iterations, device, trace, int(concurrency))
    with _checkout((_gram_p(x_or_gram), int(device)), lambda: Solver(_gram_p(x_or_gram), device=device)) as s:
        # T resident for the whole path
        if isinstance(x_or_gram, DataMatrix):
            s.gram_from_data(x_or_gram)
        elif isinstance(x_or_gram, GramMatrix):
            s.set_gram(x_or_gram)
        else:
            raise TypeError("expected a DataMatrix or GramMatrix")
        reports, prev = [], None
        for lam in lams:
            rep = s.fit(lam, delta_tol, max_outer_iterations, init=prev if warm_start else None, trace=trace,
                        raise_on_cap=False)
            reports.append(rep)
            prev = rep.estimate.omega
    return reports


class PathScheduler:
    """Cold lambda path on one device: k lanes, each a solver on its own share of the SMs
    (k=3 on a B200: 66/41/41 SMs).

    A sparse fit is latency-bound: one fit leaves most of a B200 idle, and two fits on halves of
    the device (own solver, stream and host thread) finish ~1.6x sooner than one after the other
    on all of it; two dense fits still gain ~1.2x.  The fits of a path are independent, so the
    path is a scheduling problem: the lanes pull the next lambda from one queue, densest (smallest
    lambda) first -- longest job first, so the long dense fit overlaps with the many short sparse
    ones.  A single fit runs on a full-device solver.  Results are bitwise those of sequential
    fits: the slab count never changes the bits.
    """

    def __init__(self, p, device=0, k=2, lanes=None, variants=None):
        """k equal lanes of SMs/k slabs, or `lanes`: the SM count of every lane (largest first),
        e.g. (74, 37, 37) -- the densest fit on the largest lane, the sparse ones on the others.
        `variants`: the kernel's chain warps per lane (Solver.set_chain_warps; default 6 on all)."""
        nsm = _lib.device_sm_count(device)
        if lanes is None:
            # one large lane (9/20 of the device) for the densest fits, the rest split evenly:
            # the sparse fits are latency-bound, so smaller lanes lose little per fit and add
            # lanes (round 2, final kernel: 66/28/27/27 -> 2.34 s, 66/41/41 -> 2.40-2.43 s,
            # 66/21/21/20/20 -> 2.67 s, 70/26/26/26 -> 2.69 s; profiles/r02/lanes_k45.log.  Round 1:
            # p=5000 path on 148 SMs: 74/74 -> 3.15 s, 74/37/37 -> 2.67 s, 66/41/41 ->
            # 2.55 s, 60/30/30/28 -> 2.62 s; profiles/r01/v6/lane_split_sweep.log)
            if k <= 1:
                lanes = []
            elif k == 2:
                lanes = [nsm // 2, nsm // 2]
            else:
                big = nsm * 9 // 20
                rest = nsm - big  # split as evenly as possible over the other lanes
                lanes = [big] + [rest // (k - 1) + (1 if j < rest % (k - 1) else 0) for j in range(k - 1)]
        lanes = sorted((int(v) for v in lanes), reverse=True)
        if sum(lanes) > nsm or any(v < 1 for v in lanes):
            raise ValueError(f"lanes {lanes} do not fit the device's {nsm} SMs")
        self.shares = []
        if len(lanes) > 1:
            try:
                for v in lanes:
                    self.shares.append(Solver(p, device=device, n_blocks=v))
                    # records allocated now: a lane's first fit must not allocate (or free) device
                    # memory while the other lanes' kernels run -- that waits for them
                    self.shares[-1].reserve(self.RESERVE_SWEEPS)
                # kernel variant per lane (Solver.set_chain_warps).  Alone, an apply-heavy dense fit
                # and chain-heavy sparse fits are 6% / 11% faster, but running concurrently every
                # combination was slower than the default (profiles/r02/lanes_variants.log), so the
                # lanes keep 6 chain warps unless told otherwise
                for sv, cw in zip(self.shares, variants or []):
                    sv.set_chain_warps(cw)
            except _lib.ConcordError as e:
                # every lane holds its own T, W and Omega (3 x 8p^2 bytes): when they do not fit
                # (p=50000: 60 GB each), the path runs one fit at a time on all SMs
                for s in self.shares:
                    s.close()
                self.shares = []
                if getattr(e, "code", None) != _lib.CONCORD_ERR_OOM:
                    raise
                lanes = []
        self.p, self.device, self.k, self.lanes = int(p), int(device), len(lanes), lanes
        self._full = None  # all-SM solver, created when a path has a single fit (or k <= 1)
        self._gram = None
        self._spare = {}  # CTA count -> idle solvers that continue a fit on a lane grown by hand-over
        self._spare_lock = threading.Lock()
        self._gram_gen = 0
        self._spare_made = False
        self.handovers = 0  # fits moved to a larger solver (last run_segmented call)

    @property
    def full(self):
        if self._full is None:
            self._full = Solver(self.p, device=self.device)
            if self._gram is not None:
                self._full.set_gram(self._gram)
        return self._full

    @property
    def solvers(self):
        spare = [s for v in self._spare.values() for s in v]
        return self.shares + ([self._full] if self._full is not None else []) + spare

    def close(self):
        for s in self.solvers:
            s.close()

    SPARE_BYTES = 16 << 30  # device memory the hand-over solvers may take
    RESERVE_SWEEPS = 5000  # per-sweep records the hand-over solvers allocate up front

    def set_gram(self, gram):
        self._gram = gram
        self._gram_gen += 1  # the hand-over solvers copy T from a lane when next used
        # one host upload; the other lanes copy T device to device (each its own slab layout)
        own = self.shares + ([self._full] if self._full is not None else [])
        for i, s in enumerate(own):
            if i == 0:
                s.set_gram(gram)
            else:
                s.copy_gram(own[0])
        if self.k > 1 and not self._spare_made:
            self._make_spares()

    def _make_spares(self):
        """One solver for every SM count a lane can grow to by hand-over (sums of two or more
        lanes), largest first, within SPARE_BYTES: created once, so a hand-over costs a state move
        (~1 ms at p=5000), not an allocation."""
        import itertools

        self._spare_made = True
        sums = set()
        for r in range(2, self.k + 1):
            for c in itertools.combinations(self.lanes, r):
                sums.add(sum(c))
        per = 3 * 8 * self.p * self.p * 1.1
        budget = self.SPARE_BYTES
        try:
            for v in sorted(sums, reverse=True):
                if per > budget:
                    break
                sv = Solver(self.p, device=self.device, n_blocks=v)
                sv._gen = -1
                sv.reserve(self.RESERVE_SWEEPS)
                self._spare.setdefault(v, []).append(sv)
                budget -= per
        except _lib.ConcordError as e:
            if getattr(e, "code", None) != _lib.CONCORD_ERR_OOM:
                raise

    def run(self, lams, fit_one):
        """fit_one(solver, lam) -> result; returns the results in the order of `lams`."""
        import threading

        lams = list(lams)
        out = [None] * len(lams)
        if self.k <= 1 or len(lams) <= 1:
            for i, lam in enumerate(lams):
                out[i] = fit_one(self.full, lam)
            return out
        queue = sorted(range(len(lams)), key=lambda i: lams[i])  # densest first
        lock = threading.Lock()
        errors = []
        first = {j: queue.pop(0) for j in range(min(self.k, len(queue)))}  # the largest lane takes the densest

        def lane(j):
            try:
                i = first.get(j)
                while i is not None:
                    out[i] = fit_one(self.shares[j], lams[i])
                    with lock:
                        i = queue.pop(0) if queue and not errors else None
            except BaseException as e:  # re-raised in the caller's thread
                errors.append(e)

        threads = [threading.Thread(target=lane, args=(j,)) for j in range(self.k)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        return out

    def _take_spare(self, nblk):
        with self._spare_lock:
            idle = self._spare.get(nblk)
            return idle.pop() if idle else None

    def _return_spare(self, s):
        with self._spare_lock:
            self._spare.setdefault(s._nblk, []).append(s)

    def run_segmented(self, lams, fit_seg, finish, handover=True):
        """The lanes of `run`, plus hand-over: when the queue is empty, a lane that finishes gives
        its SMs to the lane running the densest remaining fit, which stops at its next sweep end
        (Solver.request_yield) and continues on an idle solver of its grown SM count (take_state;
        `_make_spares` holds one per reachable count).  The last fits of a path therefore end on
        most of the device instead of on their lanes.

        fit_seg(solver, lam, done) -> (rc, iterations, payload): one segment of a fit (done = sweeps
        run by its earlier segments); finish(solver, lam, payloads) -> result, called on the solver
        that ran the last segment before anything else uses it.  Results are bitwise those of
        uninterrupted fits (W is carried, and the slab count never changes the bits)."""
        import threading

        lams = list(lams)
        out = [None] * len(lams)
        self.handovers = 0
        if self.k <= 1 or len(lams) <= 1:
            for i, lam in enumerate(lams):
                rc, _, pl = fit_seg(self.full, lam, 0)
                out[i] = finish(self.full, lam, [pl])
            return out
        handover = bool(handover) and self._gram_gen > 0
        queue = sorted(range(len(lams)), key=lambda i: lams[i])  # densest first
        lock = threading.Lock()
        errors = []
        first = {j: queue.pop(0) for j in range(min(self.k, len(queue)))}
        grant = {j: self.lanes[j] for j in range(self.k)}  # SMs each lane may use
        free = [0]  # SMs of finished lanes that no running fit could take yet
        running = {}  # lane -> (lambda index, solver it runs on; None while moving)
        claim = {}  # lane -> the idle solver of its grown SM count it moves to at its next yield
        lib = _lib.load()

        def donate(j):  # under lock: lane j ran dry
            free[0] += grant[j]
            grant[j] = 0
            for r in sorted(running, key=lambda r: lams[running[r][0]]):  # densest first
                nxt = self._take_spare(grant[r] + free[0])
                if nxt is None:
                    continue
                if r in claim:
                    self._return_spare(claim.pop(r))
                claim[r] = nxt
                grant[r] += free[0]
                free[0] = 0
                if running[r][1] is not None:
                    running[r][1].request_yield(True)
                return

        def lane(j):
            cur = self.shares[j]
            stream = lib.concord_solver_stream(cur._h)
            try:
                i = first.get(j)
                while i is not None:
                    pls, done = [], 0
                    with lock:
                        running[j] = (i, cur)
                    while True:
                        rc, it, pl = fit_seg(cur, lams[i], done)
                        pls.append(pl)
                        done += it
                        with lock:
                            cur.request_yield(False)
                            nxt = claim.pop(j, None)
                            if rc == _lib.CONCORD_YIELDED:
                                running[j] = (i, None)  # moving: donors only re-claim
                        if rc != _lib.CONCORD_YIELDED:
                            if nxt is not None:  # the fit ended before it could move
                                self._return_spare(nxt)
                            break
                        if nxt is None:  # (not expected) continue in place
                            cur.take_state(cur)
                            continue
                        nxt.request_yield(False)
                        nxt.set_stream(stream)
                        if nxt._gen != self._gram_gen:
                            nxt.copy_gram(cur)
                            nxt._gen = self._gram_gen
                        nxt.take_state(cur)
                        if cur is not self.shares[j]:
                            self._return_spare(cur)
                        cur = nxt
                        with lock:
                            running[j] = (i, cur)
                            self.handovers += 1
                            if j in claim:  # grown again while moving
                                cur.request_yield(True)
                    out[i] = finish(cur, lams[i], pls)
                    with lock:
                        running.pop(j, None)
                        i = queue.pop(0) if queue and not errors else None
                        if i is None and handover:
                            donate(j)
            except BaseException as e:  # re-raised in the caller's thread
                errors.append(e)
            finally:
                if cur is not self.shares[j]:
                    self._return_spare(cur)
                with lock:
                    if j in claim:
                        self._return_spare(claim.pop(j))

        threads = [threading.Thread(target=lane, args=(j,)) for j in range(self.k)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        for s in self.shares:
            s.request_yield(False)
        if errors:
            raise errors[0]
        return out


def _path_concurrent(x_or_gram, lams, delta_tol, max_outer_iterations, device, trace, k):
    if isinstance(x_or_gram, DataMatrix):
        gram = compute_gram(x_or_gram, device=device)
    elif isinstance(x_or_gram, GramMatrix):
        gram = x_or_gram
    else:
        raise TypeError("expected a DataMatrix or GramMatrix")
    key = ("path", gram.p, int(device), int(k))
    with _checkout(key, lambda: PathScheduler(gram.p, device=device, k=k)) as sched:
        sched.set_gram(gram)

        def seg(s, lam, done):
            r = s.fit_raw(lam, delta_tol, max_outer_iterations - done, trace=trace)
            return r[0], int(r[1].iterations), r

        return sched.run_segmented(lams, seg, lambda s, lam, segs: s.report(segs, trace, raise_on_cap=False))


def _gram_p(x):
    if isinstance(x, (GramMatrix, DataMatrix)):
        return x.p
    raise TypeError("expected a DataMatrix or GramMatrix")


# Device solvers are reused across pcd_fit / pcd_path calls of the same size and device
# (allocating 3 x 8p^2 bytes per call would otherwise dominate small fits).  A call checks
# one out EXCLUSIVELY: concurrent callers of the same p get solvers of their own, so pcd_fit
# stays re-entrant like the reference's pure function (solver.py:254-294), and
# release_device_memory() never closes a solver in use (it is closed when returned).
_POOL_LOCK = threading.Lock()
_POOL = {}  # key -> idle Solver / PathScheduler objects
_POOL_KEYS = 2  # problem sizes kept resident
_POOL_GEN = [0]  # bumped by release_device_memory()


def _alive(obj):
    return all(s._h is not None for s in (obj.solvers if isinstance(obj, PathScheduler) else [obj]))


@contextlib.contextmanager
def _checkout(key, make):
    evict = []
    with _POOL_LOCK:
        idle = _POOL.get(key)
        obj = idle.pop() if idle else None
        if obj is None and key not in _POOL and len(_POOL) >= _POOL_KEYS:
            evict = [o for k in list(_POOL) for o in _POOL.pop(k)]  # free device memory for a new size
        gen = _POOL_GEN[0]
    for o in evict:
        o.close()
    if obj is not None and not _alive(obj):
        obj = None
    if obj is None:
        obj = make()
    try:
        yield obj
    finally:
        with _POOL_LOCK:
            keep = gen == _POOL_GEN[0] and _alive(obj)
            if keep:
                _POOL.setdefault(key, []).append(obj)
        if not keep:
            obj.close()


def release_device_memory():
    """Free the device buffers pcd_fit keeps for reuse (solvers in use are freed when returned)."""
    with _POOL_LOCK:
        _POOL_GEN[0] += 1
        objs = [o for v in _POOL.values() for o in v]
        _POOL.clear()
    for o in objs:
        o.close()


# --------------------------------------------------------------- the drivers


def _schedule_arrays(schedule, p):
    if schedule is None:
        return None
    if schedule.p != p:
        raise ScheduleMismatch(f"schedule is for p={schedule.p} but the problem has p={p}")
    rep = validate_schedule(schedule)
    if not rep.ok:
        raise ScheduleMismatch(f"invalid schedule: {rep.message}")
    if is_circle_schedule(schedule):
        return None
    return flatten_schedule(schedule)


def pcd_fit(x_or_gram, config: SolverConfig, schedule: Schedule = None, backend=None,
            device: int = 0) -> FitReport:
    """Parallel coordinate descent over the circle schedule (solver.py:254-294).

    Raises NotConverged (carrying the partial report) when
    config.max_outer_iterations is exhausted first.
    """
    name = default_backend_name() if backend is None else backend
    if name not in BACKENDS:
        raise ValueError(f"unknown backend {name!r}")
    gram = _as_gram(x_or_gram, device)
    p = gram.p
    custom = _schedule_arrays(schedule, p)
    init = None if isinstance(config.init, str) else config.init
    if init is not None and init.p != p:
        raise DimensionError(f"init has p={init.p} but the problem has p={p}")
    if name == "cuda" and custom is None:
        with _checkout((p, int(device)), lambda: Solver(p, device=device)) as s:
            s.set_gram(gram)
            return s.fit(config.lam, config.delta_tol, config.max_outer_iterations,
                         init=None if init is None else init.omega, trace=True)
    # Reference driver loop over the bit-exact GPU sweeps (also any non-circle schedule).
    from . import cuda_kernels

    rs, ss, offsets = custom if custom is not None else flat_circle_schedule(p)
    return _host_loop(gram, config, lambda om, t, n, shrink: cuda_kernels.pcd_sweep(
        om, t, n, shrink, rs, ss, offsets, config.workers, device=device), max_abs_vech=True)


def cd_fit(x_or_gram, config: SolverConfig, backend=None, device: int = 0) -> FitReport:
    """Serial cyclic coordinate descent (solver.py:227-251) on exact GPU sweeps.

    Kept for API completeness; it is inherently serial (one pair at a time) and
    meant for small p.
    """
    name = default_backend_name() if backend is None else backend
    if name not in BACKENDS:
        raise ValueError(f"unknown backend {name!r}")
    gram = _as_gram(x_or_gram, device)
    from . import cuda_kernels

    return _host_loop(gram, config, lambda om, t, n, shrink: cuda_kernels.cd_sweep(om, t, n, shrink,
                                                                                   device=device),
                      max_abs_vech=False)


def _objective_host(om, t, n, lam):
    from .model import objective

    return objective(PrecisionEstimate._trusted(om), GramMatrix._trusted(t, n), lam)


def _host_loop(gram, config, sweep, max_abs_vech):
    t, n, p = gram.t, float(gram.n), gram.p
    omega = config.initial_omega(p)
    trace, times = [], []
    delta = math.inf
    iu = np.triu_indices(p) if max_abs_vech else None
    for it in range(1, config.max_outer_iterations + 1):
        snapshot = omega.copy()
        tic = time.perf_counter()
        sweep(omega, t, n, n * config.lam)
        diff = omega - snapshot
        delta = float(np.max(np.abs(diff[iu] if iu is not None else diff)))
        times.append(time.perf_counter() - tic)
        trace.append(_objective_host(omega, t, n, config.lam))
        if delta < config.delta_tol:
            return _finish(omega, it, delta, True, trace, times)
    raise NotConverged(_finish(omega, config.max_outer_iterations, delta, False, trace, times))


def _finish(omega, iterations, delta, converged, trace, times):
    est = PrecisionEstimate(omega)
    return FitReport(
        estimate=est,
        iterations=iterations,
        final_delta=delta,
        converged=converged,
        objective_trace=tuple(trace),
        edge_count=int(np.count_nonzero(np.triu(omega, 1))),
        wall_time_per_iteration=tuple(times),
    )


# ----------------------------------------------- scalar inspectors (API parity)


def update_offdiagonal(estimate: PrecisionEstimate, gram: GramMatrix, r: int, s: int, lam: float) -> float:
    """New value of pair (r, s), 0-based, without mutating (solver.py:86-109)."""
    p = estimate.p
    if not (0 <= r < p and 0 <= s < p):
        raise IndexError(f"indices ({r}, {s}) out of range for p={p}")
    if r == s:
        raise ValueError("off-diagonal update needs r != s")
    if estimate.p != gram.p:
        raise DimensionError("estimate and gram sizes differ")
    om, t = estimate.omega, gram.t
    s1 = float(np.dot(om[r], t[s]))
    s2 = float(np.dot(om[s], t[r]))
    num = -(s1 + s2 - om[r, s] * (t[s, s] + t[r, r]))
    from .model import soft_threshold

    return soft_threshold(num, float(gram.n) * lam) / (t[r, r] + t[s, s])


def update_diagonal(estimate: PrecisionEstimate, gram: GramMatrix, i: int) -> float:
    """New value of diagonal entry i, 0-based, without mutating (solver.py:112-118)."""
    p = estimate.p
    if not 0 <= i < p:
        raise IndexError(f"index {i} out of range for p={p}")
    if estimate.p != gram.p:
        raise DimensionError("estimate and gram sizes differ")
    om, t = estimate.omega, gram.t
    a = float(np.dot(om[i], t[i])) - om[i, i] * t[i, i]
    return (-a + math.sqrt(a * a + 4.0 * gram.n * t[i, i])) / (2.0 * t[i, i])


def read_write_sets(p: int, pair: IndexPair):
    """Cells a pair update reads and writes, 1-based (solver.py:124-138)."""
    r, s = pair.r, pair.s
    if not (1 <= r < s <= p):
        raise IndexError(f"pair ({r}, {s}) out of range for p={p}")
    read = {(r, u) for u in range(1, p + 1) if u != s} | {(u, s) for u in range(1, p + 1) if u != r}
    return read, {(r, s), (s, r)}
