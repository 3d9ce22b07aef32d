"""Lane hand-over: a blocked fit stopped at a sweep end (Solver.request_yield) and continued on a
solver of another slab count (take_state / export_state + import_state) is bitwise the
uninterrupted fit; PathScheduler.run_segmented moves the densest fit onto the SMs of lanes that ran
out of work, with the same bits as sequential fits.  No reference counterpart (a scheduling
mechanism): the oracle is our own uninterrupted fit, itself pinned to the reference elsewhere
(test_gpu_parity, test_gpu_p5000)."""

import numpy as np
import pytest

import paper_2106_09382_b200 as cb
from paper_2106_09382_b200 import _lib, synth

pytestmark = pytest.mark.gpu


def _problem(p, n=400, seed=5):
    _, t = synth.problem("ar2", p, n, seed=seed)
    return cb.GramMatrix(t, n)


def _uninterrupted(g, lam, max_iter=300):
    s = cb.Solver(g.p)
    s.set_gram(g)
    rep = s.fit(lam, 1e-5, max_iter, raise_on_cap=False)
    om, w = s.export_state()
    s.close()
    return rep, om, w


@pytest.mark.parametrize("p,lam", [(1000, 0.1), (777, 0.2), (1001, 0.3)])
def test_yield_every_sweep_across_slab_counts(p, lam):
    """Yield after every sweep and continue on the next solver of a cycle of slab counts."""
    g = _problem(p)
    ref, om_ref, w_ref = _uninterrupted(g, lam)
    sizes = [40, 148, 23, 97]
    solvers = [cb.Solver(p, n_blocks=v) for v in sizes]
    for s in solvers:
        s.set_gram(g)
    cur, segs, done, k = solvers[0], [], 0, 0
    cur.request_yield(True)
    while True:
        seg = cur.fit_raw(lam, 1e-5, 300 - done)
        segs.append(seg)
        done += seg[1].iterations
        if seg[0] != _lib.CONCORD_YIELDED:
            break
        assert seg[1].iterations == 1 and not seg[1].converged
        k += 1
        nxt = solvers[k % len(solvers)]
        nxt.request_yield(True)
        nxt.take_state(cur)
        cur.request_yield(False)
        cur = nxt
    cur.request_yield(False)
    rep = cur.report(segs, raise_on_cap=False)
    assert len(segs) == ref.iterations  # one launch per sweep
    assert rep.iterations == ref.iterations and rep.converged == ref.converged
    assert rep.edge_count == ref.edge_count
    assert np.array_equal(rep.estimate.omega, ref.estimate.omega)
    assert rep.final_delta == ref.final_delta
    np.testing.assert_allclose(rep.objective_trace, ref.objective_trace, rtol=1e-12)
    om, w = cur.export_state()
    assert np.array_equal(om, om_ref) and np.array_equal(w, w_ref)  # W carried bitwise
    for s in solvers:
        s.close()


def test_export_import_host_round_trip():
    """Yield once mid-fit, move (Omega, W) through host arrays, continue on a different layout."""
    p, lam = 1000, 0.1
    g = _problem(p)
    ref, _, _ = _uninterrupted(g, lam)
    a, b = cb.Solver(p, n_blocks=66), cb.Solver(p)
    a.set_gram(g)
    b.set_gram(g)
    a.request_yield(True)
    s1 = a.fit_raw(lam, 1e-5, 300)
    a.request_yield(False)
    assert s1[0] == _lib.CONCORD_YIELDED and s1[1].iterations == 1
    om, w = a.export_state()
    b.import_state(om, w)
    s2 = b.fit_raw(lam, 1e-5, 299)
    rep = b.report([s1, s2], raise_on_cap=False)
    assert rep.iterations == ref.iterations
    assert np.array_equal(rep.estimate.omega, ref.estimate.omega)
    # an imported state is consumed by one fit: the next fit is cold again
    again = b.fit(lam, 1e-5, 300)
    assert np.array_equal(again.estimate.omega, ref.estimate.omega)
    with pytest.raises(_lib.ConcordError):  # a pending state and omega_init together
        b.import_state(om, w)
        b.fit_raw(lam, 1e-5, 300, init=np.eye(p))
    a.close()
    b.close()


def test_yield_does_not_override_convergence_or_cap():
    """A request that lands on the converging sweep (or the cap) reports that, not a yield."""
    p, lam = 600, 0.3
    g = _problem(p)
    ref, _, _ = _uninterrupted(g, lam)
    s = cb.Solver(p)
    s.set_gram(g)
    s.request_yield(True)
    rc, res, *_ = s.fit_raw(lam, 1e-5, 1)  # the cap is the first sweep: not a yield
    assert rc == _lib.CONCORD_NOT_CONVERGED and res.iterations == 1
    rc, res, *_ = s.fit_raw(lam, 1e3, 300)  # converges at the first sweep
    assert rc == _lib.CONCORD_OK and res.converged and res.iterations == 1
    s.request_yield(False)
    rep = s.fit(lam, 1e-5, 300)
    assert np.array_equal(rep.estimate.omega, ref.estimate.omega)
    s.close()


def test_scheduler_hands_idle_lanes_to_the_dense_fit():
    """Two lanes, one dense and two sparse fits: once the sparse lane runs dry it gives its SMs to
    the dense fit, which finishes on a larger solver -- bitwise the sequential fits."""
    p = 2000
    g = _problem(p, n=600, seed=3)
    lams = [0.1, 0.5, 0.45]
    seq = cb.pcd_path(g, lams, max_outer_iterations=500)
    sched = cb.PathScheduler(p, k=2, lanes=[74, 74])
    sched.set_gram(g)

    import threading
    import time

    sparse_done = threading.Event()

    def seg(s, lam, done):
        if lam == lams[0] and done == 0 and gate[0]:
            # the dense fit starts only after the sparse lane ran dry and handed its SMs over (the
            # donation follows the sparse lane's finish in the same thread): deterministic hand-over
            sparse_done.wait(60)
            time.sleep(0.2)
        r = s.fit_raw(lam, 1e-5, 500 - done)
        return r[0], int(r[1].iterations), (r, s.layout())

    nfin = []

    def fin(s, lam, pls):
        if lam != lams[0]:
            nfin.append(lam)
            if len(nfin) == 2:  # both sparse fits done (on the other lane): the queue is empty
                sparse_done.set()
        return s.report([x[0] for x in pls], raise_on_cap=False), [x[1] for x in pls]

    gate = [True]
    out = sched.run_segmented(lams, seg, fin)
    assert sched.handovers >= 1
    dense, lays = out[0]
    # yielded after its first sweep and finished on the full-device solver (narrower slabs)
    assert len(lays) >= 2 and lays[-1]["slab_width"] < lays[0]["slab_width"]
    gate[0] = False
    sparse_done.clear()
    for a, (b, _) in zip(seq, out):
        assert a.iterations == b.iterations
        assert np.array_equal(a.estimate.omega, b.estimate.omega)
        np.testing.assert_allclose(a.objective_trace, b.objective_trace, rtol=1e-12)
    # the handed-over solvers are reused (no new allocations) by the next run, same bits again
    n_solvers = len(sched.solvers)
    out2 = sched.run_segmented(lams, seg, fin)
    assert len(sched.solvers) <= n_solvers + 1
    for a, (b, _) in zip(seq, out2):
        assert np.array_equal(a.estimate.omega, b.estimate.omega)
    # hand-over off: the plain lanes
    out3 = sched.run_segmented(lams, seg, fin, handover=False)
    assert sched.handovers == 0 and all(len(l) == 1 for _, l in out3)
    sched.close()


def test_state_through_device_pointers():
    """concord_solver_export_state / import_state with CONCORD_DEVICE buffers (torch tensors)."""
    import torch

    p, lam = 800, 0.15
    g = _problem(p, seed=9)
    ref, _, _ = _uninterrupted(g, lam)
    a, b = cb.Solver(p, n_blocks=30), cb.Solver(p, n_blocks=120)
    a.set_gram(g)
    b.set_gram(g)
    a.request_yield(True)
    s1 = a.fit_raw(lam, 1e-5, 300)
    a.request_yield(False)
    assert s1[0] == _lib.CONCORD_YIELDED
    om = torch.empty((p, p), dtype=torch.float64, device="cuda")
    w = torch.empty((p, p), dtype=torch.float64, device="cuda")
    L = _lib.load()
    _lib.check(L.concord_solver_export_state(a._h, om.data_ptr(), w.data_ptr(), _lib.DEVICE))
    torch.cuda.synchronize()
    om_h, w_h = a.export_state()
    assert np.array_equal(om.cpu().numpy(), om_h) and np.array_equal(w.cpu().numpy(), w_h)
    _lib.check(L.concord_solver_import_state(b._h, om.data_ptr(), w.data_ptr(), _lib.DEVICE))
    s2 = b.fit_raw(lam, 1e-5, 300 - s1[1].iterations)
    rep = b.report([s1, s2], raise_on_cap=False)
    assert rep.iterations == ref.iterations
    assert np.array_equal(rep.estimate.omega, ref.estimate.omega)
    a.close()
    b.close()
