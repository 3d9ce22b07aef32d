"""Do two concurrent fits on half the SMs each beat one fit on all SMs? (probe, not a bench number)"""
import sys, threading, time
sys.path.insert(0, ".")
import numpy as np
import paper_2106_09382_b200 as cb
from paper_2106_09382_b200 import synth
p, n = 5000, 2000
x = synth.center(synth.sample_mvn(synth.ar2_precision(p), n, seed=0))
s_full = cb.Solver(p)
s_full.gram_from_data(cb.DataMatrix(x, centered=True))
g = s_full.gram()
import os
os.environ["CONCORD_KERNEL"] = "qblock"
os.environ["CONCORD_PLAIN_LAUNCH"] = "1"
halves = [cb.Solver(p, n_blocks=74) for _ in range(2)]
for s in halves:
    s.set_gram(g)
    print("half layout", s.layout(), flush=True)
for lam in (0.3, 0.2, 0.1):
    for rep in range(4):
        t0 = time.perf_counter()
        r1 = s_full.fit(lam, 1e-5, 5000); r2 = s_full.fit(lam, 1e-5, 5000)
        t1 = time.perf_counter()
        out = [None, None]
        def run(i):
            out[i] = halves[i].fit(lam, 1e-5, 5000)
        th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
        t2 = time.perf_counter()
        for t in th: t.start()
        for t in th: t.join()
        t3 = time.perf_counter()
        same = np.array_equal(out[0].estimate.omega, r1.estimate.omega) and out[0].iterations == r1.iterations
        print(f"lam={lam} two sequential full fits {1e3*(t1-t0):.0f} ms | two concurrent half fits {1e3*(t3-t2):.0f} ms "
              f"(iters {out[0].iterations},{out[1].iterations}; bitwise same as full: {same})", flush=True)
