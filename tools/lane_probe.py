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
sched.set_gram(g)
HANDOVER = os.environ.get("HANDOVER", "1") == "1"
lams = [0.55, 0.50, 0.45, 0.40, 0.35, 0.30, 0.25, 0.20, 0.15, 0.10]
log = []
t00 = [0.0]
def fit_seg(s, lam, done):
    t0 = time.perf_counter() - t00[0]
    rc, res, d, o, secs = s.fit_raw(lam, 1e-5, 5000 - done)
    t1 = time.perf_counter() - t00[0]
    log.append((threading.current_thread().name, lam, s._nblk, res.iterations, round(t0, 3), round(t1, 3),
                round(res.kernel_ms / 1e3, 3)))
    return rc, res.iterations, res
PASSES = int(os.environ.get('PASSES', '2'))
QUIET = os.environ.get('QUIET') == '1'
times = []
for rep in range(PASSES):
    log.clear()
    t00[0] = time.perf_counter()
    sched.run_segmented(lams, fit_seg, lambda s, lam, segs: segs, handover=HANDOVER)
    tot = time.perf_counter() - t00[0]
    print(f"pass {rep}: {tot:.3f} s", flush=True)
    if rep:
        times.append(tot)
    if QUIET:
        continue
    for e in sorted(log, key=lambda r: r[4]):
        print("   ", e, flush=True)
print(f"== lanes {','.join(map(str, lanes))} handover {int(HANDOVER)}: best {min(times):.3f} s, median {sorted(times)[len(times)//2]:.3f} s", flush=True)
