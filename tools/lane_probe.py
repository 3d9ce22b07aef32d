"""Timeline of the PathScheduler lanes over the bench path (probe, not a bench number)."""
import sys, threading, time
sys.path.insert(0, ".")
import numpy as np
import paper_2106_09382_b200 as cb
from paper_2106_09382_b200 import synth
p, n = 5000, 2000
x = synth.center(synth.sample_mvn(synth.ar2_precision(p), n, seed=0))
import os
lanes = [int(v) for v in os.environ.get('LANES', '74,74').split(',')]
variants = [int(v) for v in os.environ["VARIANTS"].split(",")] if os.environ.get("VARIANTS") else None
sched = cb.PathScheduler(p, lanes=lanes, variants=variants)
sched.full.gram_from_data(cb.DataMatrix(x, centered=True))
g = sched.full.gram()
for s in sched.shares:
    s.set_gram(g)
lams = [0.55, 0.50, 0.45, 0.40, 0.35, 0.30, 0.25, 0.20, 0.15, 0.10]
log = []
t00 = [0.0]
def fit_one(s, lam):
    t0 = time.perf_counter() - t00[0]
    rc, res, d, o, secs = s.fit_raw(lam, 1e-5, 5000)
    t1 = time.perf_counter() - t00[0]
    log.append((threading.current_thread().name, lam, round(t0, 3), round(t1, 3), round(res.kernel_ms / 1e3, 3)))
    return res
for rep in range(2):
    log.clear()
    t00[0] = time.perf_counter()
    sched.run(lams, fit_one)
    tot = time.perf_counter() - t00[0]
    print(f"pass {rep}: {tot:.3f} s", flush=True)
    for e in sorted(log, key=lambda r: r[2]):
        print("   ", e, flush=True)
