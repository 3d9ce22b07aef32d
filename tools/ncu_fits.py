"""Fit the bench's lambda path once (for ncu; not a bench number).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:pcd_ \
        --csv --log-file gpurun_out/traffic.csv python tools/ncu_fits.py [--p 5000] [--lams 0.55,...]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_09382_b200 as cb  # noqa: E402
from paper_2106_09382_b200 import _lib, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=5000)
ap.add_argument("--n", type=int, default=2000)
ap.add_argument("--lams", default="0.55,0.50,0.45,0.40,0.35,0.30,0.25,0.20,0.15,0.10")
ap.add_argument("--out", default="gpurun_out/ncu_fits.json")
a = ap.parse_args()
x, t = synth.portable_problem("ar2", a.p, a.n, seed=0)  # the bench's (and the fixtures') exact Gram
s = cb.Solver(a.p)
s.set_gram(cb.GramMatrix(t, a.n))
rows = []
for lam in [float(v) for v in a.lams.split(",")]:
    rc, res, deltas, objs, secs = s.fit_raw(lam, 1e-5, 5000)
    nnz = np.zeros(res.iterations, dtype=np.int64)
    import ctypes
    cnt = ctypes.c_int32(0)
    _lib.check(_lib.load().concord_solver_sweep_stats(s._h, _lib.ptr(nnz), res.iterations, ctypes.byref(cnt)))
    rows.append({"lam": lam, "iterations": int(res.iterations), "nnz_per_sweep": nnz.tolist()})
    print(f"lam={lam} iters={res.iterations}", flush=True)
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump({"p": a.p, "n": a.n, "fits": rows}, open(a.out, "w"))
