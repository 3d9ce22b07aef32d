"""Cost of the shard exchange on one device (probe, not a bench number): p=20000, n=5000, lambda=0.3,
the blocked kernel with G virtual shards -- every exchange write goes to G copies, and with
CONCORD_FORCE_SYS_SCOPE=1 the arrivals use the multi-GPU system-scope fences.

    python tools/shard_overhead.py [p] [n]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_09382_b200 as cb  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
base = None
with cb.Solver(p) as s0:
    s0.gram_from_ar2(n, seed=0)
    g = s0.gram()
for G in (1, 2, 4, 8):
    with cb.Solver(p, n_shards=G) as s:
        s.set_gram(g)
        for rep in range(2):
            rc, res, d, o, secs = s.fit_raw(0.3, 1e-5, 500)
        om_sha = None
        print(f"G={G} sys_scope={os.environ.get('CONCORD_FORCE_SYS_SCOPE', '0')} kernel={s.layout()['kernel']} "
              f"iters={res.iterations} edges={res.edge_count} fit={res.kernel_ms / 1e3:.3f}s "
              f"ms/sweep={np.median(secs) * 1e3:.1f}", flush=True)
