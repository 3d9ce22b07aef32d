"""When does a cooperative fit launch start while another lane's fit holds some SMs?  A 27-CTA
fit runs (lambda=0.1, seconds); a second fit of X CTAs is launched beside it: its wall time vs
alone shows whether the launch waited for the first to end (probe, not a bench number)."""
import sys, threading, time
sys.path.insert(0, ".")
import paper_2106_09382_b200 as cb
from paper_2106_09382_b200 import synth

p, n = 5000, 2000
x = synth.center(synth.sample_mvn(synth.ar2_precision(p), n, seed=0))
a = cb.Solver(p, n_blocks=27)
a.gram_from_data(cb.DataMatrix(x, centered=True))
g = a.gram()
for X in [148 - 27, 148 - 28, 148 - 30, 148 - 34, 100]:
    b = cb.Solver(p, n_blocks=X)
    b.set_gram(g)
    t0 = time.perf_counter(); b.fit_raw(0.5, 1e-5, 5000); alone = time.perf_counter() - t0
    done = {}
    def run_a():
        t = time.perf_counter(); a.fit_raw(0.1, 1e-5, 6); done["a"] = time.perf_counter() - t
    th = threading.Thread(target=run_a); th.start(); time.sleep(0.3)
    t0 = time.perf_counter(); rc, res, *_ = b.fit_raw(0.5, 1e-5, 5000); beside = time.perf_counter() - t0
    th.join()
    print(f"X={X}: alone {alone:.3f} s, beside the 27-CTA fit {beside:.3f} s (kernel {res.kernel_ms/1e3:.3f}); a took {done['a']:.3f} s", flush=True)
    b.close()
