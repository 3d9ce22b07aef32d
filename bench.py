"""Benchmark: CONCORD-PCD on B200 vs the reference CPU path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode path|sharded]
                    [--concurrency k]

Workload (BASELINE.json configs[2], the paper workload): AR(2) truth,
p=5000, n=2000 synthetic samples (datagen.py restated in synth.py, seed 0),
the 10-value lambda path 0.55, 0.50, ..., 0.10.  One STEP = the whole path:
ten complete cold-start CONCORD-PCD fits (identity init, delta_tol 1e-5),
scheduled by the package's PathScheduler -- --concurrency k (default 4)
lanes, each a solver on its own share of the SMs (k=4: 66/28/27/27 on a B200;
own stream and host thread), pull the fits densest first (one latency-bound fit leaves
most of a B200 idle; longest job first balances the lanes).  --concurrency 1 runs every
fit on all SMs, one after the other.
The metric is sweeps/s (outer iterations per second, BASELINE "sweeps/sec"),
with seconds-to-converge per lambda reported beside it.

* value: device time (CUDA events on the solvers' streams, from one start
  event to the last stream's end) with T resident in HBM; the W/T/Omega
  working set (3 x 200 MB per solver) exceeds the 126 MB L2.
* e2e: the same metric through the public API -- `pcd_path(GramMatrix,
  lambdas, concurrency=k)` -- with T in pinned host memory: every step uploads
  T (H2D, once per solver) and reads every Omega back (D2H).
* roofline: the fit kernel's (pcd_qblock_kernel) algorithmic bytes of all
  fits / the device time of the steps (aggregate over the concurrent fits).
* cpu_baseline / --impl reference: the reference's own compiled sweep
  (oracle/_ref, built from /root/reference's _ckernels.pyx) on all host cores,
  timed on a bounded sample of rounds (sweep cost is data-independent).

Multi-GPU (torchrun, one rank per GPU):
* --mode path (default): every GPU runs the whole path (independent
  problems, no data-path collective; scaling "weak").
* --mode sharded: BASELINE configs[3] -- p=20000, n=5000 -- ONE problem
  column-sharded over all ranks (paper_2106_09382_b200.dist): every colour's
  published values are all-gathered in-kernel through NVLink peer stores
  (scaling "strong"; sweeps/s of the one problem).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

LAMS = [0.55, 0.50, 0.45, 0.40, 0.35, 0.30, 0.25, 0.20, 0.15, 0.10]
METRIC = "sweeps/s (CONCORD-PCD fits, p=5000 n=2000, 10-lambda path)"
DATA_PATH = ("synthetic: AR(2) truth (datagen.ar2_precision), X ~ N(0, inv(truth)) n=2000 seed 0 (datagen.sample_mvn), "
             "centred, on the exact-Gram grid of synth.quantize_exact_gram (the reference fixtures' data)")
UNIT = "sweeps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["path", "sharded"], default="path")
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--delta-tol", type=float, default=1e-5)
    ap.add_argument("--concurrency", type=int, default=4,
                    help="fits run at a time per GPU, each on SMs/k (path mode); 1 = one fit on all SMs")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-handover", action="store_true",
                    help="lanes keep their SMs to the end (no hand-over of idle lanes to running fits)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target length of the CPU sample")
    ap.add_argument("--cpu-validate", action="store_true",
                    help="also run one complete reference fit at lambda=0.3 on the host (minutes)")
    a = ap.parse_args()
    if a.p is None:
        a.p = 20000 if a.mode == "sharded" else 5000
    if a.n is None:
        a.n = 5000 if a.mode == "sharded" else 2000
    return a


# --------------------------------------------------------------- plumbing


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, backend="nccl", force=False):
        if self.world > 1 or force:
            import socket

            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if "MASTER_PORT" not in os.environ:
                with socket.socket() as sk:
                    sk.bind(("127.0.0.1", 0))
                    os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
            dist.init_process_group(backend, rank=self.rank, world_size=self.world,
                                    device_id=None if backend != "nccl" else __import__("torch").device(
                                        "cuda", self.local))
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, v):
        if not self.pg:
            return v
        import torch

        t = torch.tensor([float(v)], device=f"cuda:{self.local}", dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v):
        if not self.pg:
            return v
        import torch

        t = torch.tensor([float(v)], device=f"cuda:{self.local}", dtype=torch.float64)
        self.pg.all_reduce(t)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


class Clocks:
    """nvidia-smi samples of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peak_hbm():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload):
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        e = d.get(workload)
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


def make_problem(p, n):
    """Centred AR(2) samples.  p <= 8000: the reference pipeline rounded onto the exact-Gram grid
    (synth.portable_problem), so T -- device DMMA Gram included -- is bitwise the T of the
    reference fixtures in tests/golden/p5000/."""
    from paper_2106_09382_b200 import synth

    if p > 8000:  # configs[3:]: banded sampler (same distribution, O(p n))
        return synth.center(synth.sample_mvn_ar2_banded(p, n, seed=0))
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        x = synth.center(synth.sample_mvn(synth.ar2_precision(p), n, seed=0))
    return synth.quantize_exact_gram(x)[0]


def algorithmic_bytes(p, nnz_per_sweep, want_trace=True):
    """colour k moves 48*p*nnz_k + 24*p bytes, the diagonal step 24*p^2
    (+8*p^2 for the fused objective's Omega read)."""
    pe = p + (p % 2)
    per_sweep_fixed = 24.0 * p * (pe - 1) + 24.0 * p * p + (8.0 * p * p if want_trace else 0.0)
    return sum(48.0 * p * float(k) + per_sweep_fixed for k in nnz_per_sweep)


# --------------------------------------------------------------- CPU reference


def cpu_reference_rate(t, n, lam, target_s, workers):
    """Sweeps/s of the reference's own per-iteration work on a bounded sample.

    The compiled pcd_sweep (oracle/_ref: the reference's _ckernels.pyx built
    here) runs a bounded sample of colour rounds -- its cost is data- and
    lambda-independent (_ckernels.pyx:33-36) -- and the driver's per-iteration
    work inside the reference's timed region (solver.py:283-288: the snapshot
    copy and cyclic_max_reduce(_vech(omega - snapshot))) is timed once at the
    same p.  Per-sweep seconds = sample / fraction of rounds + that overhead.
    """
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as orc

    ref = orc.load_ref()
    kind = "reference" if ref is not None else "port"
    p = t.shape[0]
    rs, ss, off = orc.circle_flat(p)
    nrounds = off.shape[0] - 1

    def run(k0, k1):
        om = np.eye(p)
        sub = off[k0:k1 + 1]
        tic = time.perf_counter()
        if ref is not None:
            ref.pcd_sweep(om, t, float(n), n * lam, rs.astype(np.intp), ss.astype(np.intp), sub.astype(np.intp),
                          int(workers))
        else:
            orc.pcd_sweep(om, t, n, n * lam, rs, ss, sub, workers)
        return time.perf_counter() - tic

    probe = max(2, min(nrounds, 32))
    run(0, probe)  # warm (first touch of T, thread pool start)
    dt = run(0, probe)
    rounds = int(max(probe, min(nrounds, target_s / max(dt / probe, 1e-9))))
    el = run(0, rounds)
    om = np.eye(p)
    tic = time.perf_counter()
    snap = om.copy()
    orc.cyclic_max_reduce(orc.vech(om - snap))
    overhead = time.perf_counter() - tic
    # each call also runs the p diagonal updates (1/p of a sweep) -- counted as work done
    sweep_s = el * nrounds / rounds + overhead
    return 1.0 / sweep_s, kind, rounds, el, overhead


def cpu_full_fit(t, n, lam, workers):
    """One complete reference fit (the stock solver.py:254-294 loop over oracle/_ref's pcd_sweep with the
    reference's numpy convergence metric), timed the reference's way: sum of wall_time_per_iteration."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as orc

    tic = time.perf_counter()
    rep = orc.pcd_fit(t, n, lam, 1e-5, 5000, workers=workers, trace=False, use_ref=orc.load_ref() is not None,
                      numpy_delta=True)
    wall = time.perf_counter() - tic
    return {"lam": lam, "iterations": rep["iterations"], "edges": rep["edge_count"],
            "sum_wall_time_per_iteration_s": float(sum(rep["wall_time_per_iteration"])), "wall_s_incl_schedule": wall,
            "per_sweep_s": float(sum(rep["wall_time_per_iteration"])) / rep["iterations"], "workers": workers}


# --------------------------------------------------------------- our arm


def run_ours(args, d):
    import torch

    import paper_2106_09382_b200 as cb
    from paper_2106_09382_b200 import _lib

    torch.cuda.set_device(d.local)
    p, n, K, W = args.p, args.n, args.steps, args.warmup
    k = max(1, int(args.concurrency))
    x = make_problem(p, n)
    # One step = the whole cold lambda path, run by the package's PathScheduler: k lanes, each a
    # solver on its own share of the SMs (own stream and host thread), pull the fits densest first
    # (one latency-bound fit leaves most of a B200 idle).  k = 1: every fit on all SMs.
    sched = cb.PathScheduler(p, device=d.local, k=k)
    sv_all = sched.shares if k > 1 else [sched.full]
    streams = [torch.cuda.Stream() for _ in sv_all]
    for sv, st in zip(sv_all, streams):
        sv.set_stream(st.cuda_stream)
    s, stream = sv_all[0], streams[0]
    lay = s.layout()
    kernel = f"pcd_qblock_kernel (D={lay['kernel']})" if lay["kernel"] else "pcd_wform_kernel"
    g0 = time.perf_counter()
    s.gram_from_data(cb.DataMatrix(x))  # X is centred (then rounded to the exact-Gram grid)
    gram_s = time.perf_counter() - g0
    g = s.gram()
    sched.set_gram(g)  # every lane's solver (the full-device one is created on demand)
    lams = list(LAMS)

    def one_seg(sv, lam, done):
        # one launch of the fit kernel: the whole fit, or the part of it run on one lane size when
        # the scheduler hands a lane's SMs over to it (PathScheduler.run_segmented)
        rc, res, deltas, objs, secs = sv.fit_raw(lam, args.delta_tol, 5000 - done, trace=True)
        nnz = np.zeros(res.iterations, dtype=np.int64)
        cnt = ctypes_int()
        _lib.check(_lib.load().concord_solver_sweep_stats(sv._h, _lib.ptr(nnz), res.iterations, cnt))
        return rc, int(res.iterations), (int(res.n_blocks), int(res.iterations), float(res.kernel_ms), nnz,
                                         bool(res.converged), int(res.edge_count), int(res.slab_width))

    def finish(sv, lam, segs):
        last = segs[-1]
        return (lam, sum(g[1] for g in segs), sum(g[2] for g in segs), np.concatenate([g[3] for g in segs]),
                last[4], last[5], segs[0][0], segs[0][6], segs)

    def one_fit(sv, lam):
        rc, _, seg = one_seg(sv, lam, 0)
        return finish(sv, lam, [seg])

    def frac(sv, f):
        return float(f[3].sum()) / (f[1] * (p * (p - 1) / 2))

    def step(out):
        out.extend(sched.run_segmented(lams, one_seg, finish, handover=not args.no_handover))

    for i in range(W):
        step([])
    clocks = Clocks(d.local)
    d.barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = [torch.cuda.Event(enable_timing=True) for _ in streams]
    e0.record(stream)
    for st in streams[1:]:
        st.wait_event(e0)
    fits = []
    for i in range(K):
        step(fits)
    for ev, st in zip(e1, streams):
        ev.record(st)
    torch.cuda.synchronize()
    d.barrier()
    clk = clocks.stop()
    elapsed_ms = d.max(max(e0.elapsed_time(ev) for ev in e1))
    sweeps = d.sum(sum(f[1] for f in fits))
    value = sweeps / (elapsed_ms / 1e3)

    # roofline of the dominant kernel (the fit kernel, one persistent launch per fit).  The recipe's
    # figure: algorithmic bytes per launch / the average launch duration (CUDA events on the launching
    # stream).  With k lanes the launches overlap on disjoint SM sets, so the device-level HBM
    # utilisation (all fits' bytes / the steps' device time) is reported beside it, as is every
    # lambda's own launch (on its lane's SMs) and two fits alone on the full device.
    kern_ms = [g[2] for f in fits for g in f[8]]  # per launch (a handed-over fit has several)
    avg_ms = sum(kern_ms) / len(kern_ms)
    avg_bytes = sum(algorithmic_bytes(p, g[3]) for f in fits for g in f[8]) / len(kern_ms)
    bytes_per = [algorithmic_bytes(p, f[3]) for f in fits]
    n_launch = len(kern_ms)
    peak, peak_src = measured_peak_hbm()
    achieved = avg_bytes / (avg_ms / 1e3) / 1e9
    device_gbs = sum(bytes_per) / (elapsed_ms / 1e3) / 1e9
    per_lambda = {}
    for lam in lams:
        sel = [(f, b) for f, b in zip(fits, bytes_per) if f[0] == lam]
        ms = sum(f[2] for f, _ in sel) / len(sel)
        gbs = sel[0][1] / (ms / 1e3) / 1e9
        per_lambda[f"{lam:.2f}"] = {"ctas": sel[0][0][6], "ms": round(ms, 3), "algorithmic_gb": round(sel[0][1] / 1e9, 2),
                                    "gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
                                    "launches": [[[g[0], g[1]] for g in f[8]] for f, _ in sel][-1]}
    full = {}
    sf = sched.full
    sf.set_stream(streams[0].cuda_stream)
    for lam in (0.30, 0.10):
        f = one_fit(sf, lam)
        b = algorithmic_bytes(p, f[3])
        full[f"{lam:.2f}"] = {"ctas": f[6], "iterations": f[1], "seconds_to_converge": round(f[2] / 1e3, 6),
                              "gbs": round(b / (f[2] / 1e3) / 1e9, 1), "frac": round(b / (f[2] / 1e3) / 1e9 / peak, 4)}
    workload = f"ar2 p={p} n={n} lambda-path cold"
    traffic = ncu_traffic(workload)
    nnz_frac = [frac(None, f) for f in fits]
    nsm = _lib.device_sm_count(d.local)
    par = (f"PathScheduler: {k} lanes of {'/'.join(str(v) for v in sched.lanes)} of {nsm} SMs (own solver, "
           f"stream, host thread) pulling the path's fits densest first; each fit a persistent cooperative "
           f"kernel" if k > 1 else
           "one fit at a time on all SMs, persistent cooperative kernel")
    if d.world > 1:
        par = f"{d.world} GPU(s), each running the whole path (independent problems); " + par

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": d.world, "steps": K, "warmup": W,
        "ms_per_step": elapsed_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": DATA_PATH,
        "config": {"workload": workload, "source": "BASELINE.json configs[2] (paper workload)", "p": p, "n": n,
                   "lambdas": lams, "fits_per_step": len(lams), "concurrency": k, "delta_tol": args.delta_tol,
                   "init": "identity",
                   "l2": "inputs larger than L2 (T, W, Omega slabs 3 x %.0f MB > 126 MB)" % (8 * p * p / 1e6),
                   "parallelism": par, "kernel": kernel, "n_blocks": fits[0][6], "slab_width": fits[0][7]},
        "seconds_to_converge": {f"{f[0]:.2f}": round(f[2] / 1e3, 6) for f in fits},
        "iterations": {f"{f[0]:.2f}": f[1] for f in fits},
        "edges": {f"{f[0]:.2f}": f[5] for f in fits},
        "nonzero_pair_fraction": {f"{f[0]:.2f}": round(v, 6) for f, v in zip(fits, nnz_frac)},
        "gram_s_incl_h2d": round(gram_s, 4),
        "roofline": {"kernel": kernel, "bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": avg_bytes, "avg_launch_ms": avg_ms,
                     "device_aggregate": {"achieved": device_gbs, "frac": device_gbs / peak,
                                          "note": "all fits' bytes / the steps' device time (k concurrent launches "
                                                  "on disjoint SMs): HBM utilisation of the device"},
                     "per_lambda": per_lambda, "full_device_fits": full,
                     "note": "bytes = sum over sweeps of 48p*nnz_k per colour + 24p per colour + 32p^2 diag/objective"
                             "; achieved = bytes per launch / average launch duration (each launch on its lane's "
                             "SMs only; per_lambda.launches = [CTAs, sweeps] of each launch of the fit's last run)"},
        "handovers_per_step": (n_launch - len(fits)) / K,
        # per fit: identity, fit kernel, edge count; per hand-over: 2 x (unpack + pack) + fit + edge count
        "gpu_launches": 3 * len(fits) + 6 * (n_launch - len(fits)),
        "clocks": clk,
    }

    if not args.no_e2e:
        out["e2e"] = run_e2e(args, d, s, stream, lams, k)
    if not args.no_cpu and d.world == 1 and d.rank == 0:
        t_host = s.gram().t
        rate, kind, rounds, el, ovh = cpu_reference_rate(t_host, n, 0.3, args.cpu_seconds, os.cpu_count())
        path_iters = sum(f[1] for f in fits[:len(lams)])  # one step = one path
        cb_out = {"value": rate, "unit": UNIT, "cores": os.cpu_count(), "kind": kind,
                  "sample": f"{rounds} of {p + (p % 2) - 1} colour rounds of one pcd_sweep at p={p} "
                            f"(workers={os.cpu_count()}), {el:.1f} s, plus the driver's per-iteration snapshot + "
                            f"cyclic_max_reduce(_vech) ({ovh:.2f} s, solver.py:283-288); sweep cost is "
                            f"data-independent",
                  "path_iterations": path_iters,
                  "seconds_per_path_extrapolated": path_iters / rate}
        if args.cpu_validate:
            v = cpu_full_fit(t_host, n, 0.3, os.cpu_count())
            v["sampled_per_sweep_s"] = 1.0 / rate
            v["gpu_iterations"] = dict((f"{f[0]:.2f}", f[1]) for f in fits)["0.30"]
            cb_out["validation"] = v
        else:
            rec = os.path.join(REPO, "profiles", "r02", "cpu_full_fit.json")
            if os.path.exists(rec):
                with open(rec) as fh:
                    cb_out["validation"] = dict(json.load(fh), recorded_in="profiles/r02/cpu_full_fit.json")
        out["cpu_baseline"] = cb_out
    s.close()
    return out


def ctypes_int():
    import ctypes

    return ctypes.byref(ctypes.c_int32(0))


def run_e2e(args, d, s, stream, lams, k=1):
    """Same metric through the public API with T in pinned host memory, one step = the whole
    path: pcd_path(GramMatrix(pinned T), lambdas, concurrency=k) uploads T once (H2D; the other
    lanes copy it on the device) and returns every Omega (D2H)."""
    import torch

    import paper_2106_09382_b200 as cb
    from paper_2106_09382_b200 import _lib

    p, n, K, W = args.p, args.n, args.steps, args.warmup
    t_pinned = _lib.pinned_empty((p, p))
    t_pinned[...] = s.gram().t
    gram = cb.GramMatrix(t_pinned, n)  # validated once, as a user would construct it

    def one_step():
        reps = cb.pcd_path(gram, lams, delta_tol=args.delta_tol, max_outer_iterations=5000, device=d.local,
                           concurrency=k)
        return sum(r.iterations for r in reps)

    for i in range(min(W, 2)):
        one_step()
    d.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sweeps = 0
    for i in range(K):
        sweeps += one_step()
    e1.record()
    torch.cuda.synchronize()
    d.barrier()
    el = d.max(e0.elapsed_time(e1))
    total = d.sum(sweeps)
    # PathScheduler.set_gram uploads T once; the other lanes copy it device to device
    return {"value": total / (el / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * p * p,
            "d2h_bytes_per_step": 8 * p * p * len(lams), "ms_per_step": el / K,
            "path": f"paper_2106_09382_b200.pcd_path(GramMatrix(pinned T), {len(lams)} lambdas, concurrency={k}) "
                    "-> FitReports"}


def run_sharded(args, d):
    """One p=20000 problem column-sharded over all ranks; value = sweeps/s of that problem."""
    import torch

    import paper_2106_09382_b200 as cb
    from paper_2106_09382_b200 import dist as cdist

    torch.cuda.set_device(d.local)
    p, n, K, W = args.p, args.n, args.steps, args.warmup
    g0 = time.perf_counter()
    s = cdist.ShardedSolver(p, device=d.local)
    s.gram_from_ar2(n, seed=0)  # X drawn on every GPU (same counter-based stream), never crosses PCIe
    gram_s = time.perf_counter() - g0
    lams = LAMS[:6]  # 0.55 .. 0.30: the sparse end of the path at this size

    def one_fit(lam):
        rep = s.fit(lam, args.delta_tol, 5000, trace=True, gather=False, raise_on_cap=False)
        return rep, float(s.last_result.kernel_ms)

    for i in range(W):
        one_fit(lams[i % len(lams)])
    clocks = Clocks(d.local)
    d.barrier()
    torch.cuda.synchronize()
    clocks.start()
    fits, kern = [], 0.0
    for i in range(K):
        lam = lams[i % len(lams)]
        rep, ms = one_fit(lam)
        fits.append((lam, rep.iterations, ms, rep.edge_count))
        kern += ms
    torch.cuda.synchronize()
    d.barrier()
    clk = clocks.stop()
    elapsed_ms = d.max(kern)  # device time of the fits (CUDA events around each kernel), max over ranks
    sweeps = sum(f[1] for f in fits)  # one problem: every rank ran the same sweeps
    out = {
        "metric": f"sweeps/s (CONCORD-PCD fits, p={p} n={n}, column-sharded over {d.world} GPU(s))",
        "value": sweeps / (elapsed_ms / 1e3), "unit": UNIT, "n_gpus": d.world, "steps": K, "warmup": W,
        "ms_per_step": elapsed_ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": f"synthetic: AR(2) truth, X ~ N(0, inv(truth)) n={n}, drawn on the GPU (Philox, seed 0), centred",
        "config": {"workload": f"ar2 p={p} n={n} sharded", "source": "BASELINE.json configs[3]", "p": p, "n": n,
                   "lambdas": [f[0] for f in fits], "parallelism": f"column-sharded dp{d.world} (in-kernel NVLink exchange)",
                   "slab_width": s.slab_width, "blocks_total": s.blocks_total,
                   "l2": "inputs larger than L2 (T, W, Omega %.1f GB)" % (24 * p * p / 1e9)},
        "seconds_to_converge": {f"{f[0]:.2f}": round(f[2] / 1e3, 6) for f in fits},
        "iterations": {f"{f[0]:.2f}": f[1] for f in fits},
        "edges": {f"{f[0]:.2f}": f[3] for f in fits},
        "sample_and_gram_s": round(gram_s, 3),
        "gpu_launches": 3 * K,
        "clocks": clk,
    }
    s.close()
    return out


# --------------------------------------------------------------- reference arm


def run_reference(args, d):
    if d.rank != 0:
        return None
    from paper_2106_09382_b200 import synth

    p, n, K, W = args.p, args.n, args.steps, args.warmup
    p_run = p
    if args.mode == "sharded":  # the reference's O(p^2) schedule does not fit at p=20000: time p=5000, scale by p^3
        p_run, n = 5000, 2000
    t = synth.host_gram(make_problem(p_run, n))
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    per_step = max(1.0, min(args.cpu_seconds, 150.0 / max(K + W, 1)))
    rates = []
    kind = None
    info = None
    for i in range(W + K):
        rate, kind, rounds, el, ovh = cpu_reference_rate(t, n, LAMS[i % len(LAMS)], per_step, os.cpu_count())
        if i >= W:
            rates.append((rate, rounds, el, ovh))
        info = (rounds, el)
    m_run = p_run + (p_run % 2) - 1
    total_sweeps = sum(r[1] / m_run for r in rates)
    total_s = sum(r[2] + r[3] * r[1] / m_run for r in rates)
    value = total_sweeps / total_s
    sample = (f"each step = {info[0]} colour rounds of the reference pcd_sweep at p={p_run} "
              f"(compiled _ckernels, workers={os.cpu_count()}) plus the driver's snapshot + "
              f"cyclic_max_reduce(_vech) per sweep (solver.py:283-288); sweeps = rounds/{m_run}")
    if p_run != p:
        value *= (p_run / p) ** 3  # the sweep is 16 p^3 bytes of dense dots (_ckernels.pyx:33-36)
        sample += f"; extrapolated to p={p} by (p/{p_run})^3"
    metric = METRIC if args.mode == "path" else f"sweeps/s (CONCORD-PCD fits, p={p} n={args.n}, column-sharded over {d.world} GPU(s))"
    workload = f"ar2 p={p} n={args.n} lambda-path cold" if args.mode == "path" else f"ar2 p={p} n={args.n} sharded"
    return {"metric": metric, "value": value, "unit": UNIT, "n_gpus": d.world, "steps": K, "warmup": W,
            "ms_per_step": 1e3 * total_s / K, "higher_is_better": True,
            "scaling": "weak" if args.mode == "path" else "strong", "vs_baseline": None,
            "dtype": "f64", "impl": "reference",
            "data": DATA_PATH if args.mode == "path" else
                    f"synthetic: AR(2) truth, X ~ N(0, inv(truth)) n={n} seed 0, centred",
            "config": ({"workload": workload, "source": "BASELINE.json configs[2] (paper workload)", "p": p, "n": args.n,
                        "lambdas": list(LAMS), "fits_per_step": len(LAMS), "delta_tol": args.delta_tol,
                        "init": "identity"} if args.mode == "path" else
                       {"workload": workload, "source": "BASELINE.json configs[3]", "p": p, "n": args.n}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


def main():
    args = parse()
    d = Dist()
    if args.impl == "reference":
        out = run_reference(args, d)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    d.init("nccl", force=args.mode == "sharded")
    try:
        out = run_sharded(args, d) if args.mode == "sharded" else run_ours(args, d)
    finally:
        d.close()
    if d.rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
