"""Host logic of the lambda-path scheduler (no GPU): the lanes pull the fits densest first, the
largest lane takes the densest fit, results come back in the caller's order, errors propagate."""
import threading
import time

import pytest

from paper_2106_09382_b200.solver import PathScheduler


def _sched(lanes):
    s = PathScheduler.__new__(PathScheduler)  # no device: lanes are plain labels here
    s.p, s.device, s.k, s.lanes = 10, 0, len(lanes), list(lanes)
    s.shares = [f"lane{j}" for j in range(len(lanes))] if len(lanes) > 1 else []
    s._full, s._gram = "full", None
    return s


def test_results_in_caller_order_and_densest_first_on_the_largest_lane():
    sched = _sched([74, 37, 37])
    lams = [0.55, 0.1, 0.3, 0.2, 0.45, 0.15]
    starts = []
    lock = threading.Lock()

    def fit_one(lane, lam):
        with lock:
            starts.append((lane, lam))
        time.sleep(0.02 if lam > 0.12 else 0.1)  # the dense fit is the long one
        return (lane, lam)

    out = sched.run(lams, fit_one)
    assert [o[1] for o in out] == lams
    first_per_lane = {}
    for lane, lam in starts:
        first_per_lane.setdefault(lane, lam)
    assert first_per_lane["lane0"] == 0.1  # the largest lane takes the densest fit
    assert sorted(first_per_lane.values()) == [0.1, 0.15, 0.2]  # then the next densest ones
    assert all(lane != "full" for lane, _ in starts)


def test_single_fit_and_single_lane_use_the_full_device_solver():
    for sched, lams in ((_sched([74, 37, 37]), [0.3]), (_sched([]), [0.3, 0.2])):
        out = sched.run(lams, lambda lane, lam: lane)
        assert out == ["full"] * len(lams)


def test_lane_errors_reach_the_caller():
    sched = _sched([74, 74])

    def fit_one(lane, lam):
        if lam == 0.2:
            raise RuntimeError("boom")
        return lam

    with pytest.raises(RuntimeError, match="boom"):
        sched.run([0.5, 0.2, 0.3, 0.1], fit_one)


def test_default_lane_splits(monkeypatch):
    """k lanes on a 148-SM B200: 9/20 of the SMs for the densest fits, the rest split as evenly as
    possible (k=4 is the bench's 66/28/27/27; profiles/r02/lanes_k45.log)."""
    from paper_2106_09382_b200 import solver

    made = []

    class FakeSolver:
        def __init__(self, p, device=0, n_blocks=0):
            made.append(n_blocks)

        def set_chain_warps(self, cw):
            pass

        def reserve(self, max_iter):
            pass

    monkeypatch.setattr(solver._lib, "device_sm_count", lambda device: 148)
    monkeypatch.setattr(solver, "Solver", FakeSolver)
    assert PathScheduler(5000, k=2).lanes == [74, 74]
    assert PathScheduler(5000, k=3).lanes == [66, 41, 41]
    assert PathScheduler(5000, k=4).lanes == [66, 28, 27, 27]
    assert PathScheduler(5000, k=5).lanes == [66, 21, 21, 20, 20]
    assert sum(PathScheduler(5000, k=4).lanes) == 148
    with pytest.raises(ValueError):
        PathScheduler(5000, lanes=[100, 60])


class _FakeSolver:
    """Host stand-in for a Solver: a fit is `sweeps` sleeps; a set yield flag stops it after the
    current sweep (the kernel's rule) and take_state carries the sweeps done."""

    def __init__(self, nblk):
        self._h, self._nblk, self._gen, self.flag = None, nblk, -1, False
        self.state = None  # (lam, sweeps done) imported by take_state
        self.moves_in = 0

    def request_yield(self, on=True):
        self.flag = bool(on)

    def set_stream(self, ptr):
        pass

    def copy_gram(self, src):
        pass

    def take_state(self, src):
        self.state = src.state
        self.moves_in += 1


def _seg_sched(lanes, sweeps):
    import threading as th

    from paper_2106_09382_b200 import _lib

    sched = _sched(lanes)
    sched.shares = [_FakeSolver(v) for v in lanes]
    sched._spare, sched._spare_lock, sched._gram_gen, sched.handovers = {}, th.Lock(), 1, 0
    for r in range(2, len(lanes) + 1):  # what _make_spares creates: every sum of >= 2 lanes
        import itertools

        for c in itertools.combinations(lanes, r):
            sched._spare.setdefault(sum(c), [_FakeSolver(sum(c))])

    def fit_seg(s, lam, done):
        # a sweep takes 1/SMs of a unit: the lanes' SMs matter, as on the device
        n = 0
        while True:
            time.sleep(0.4 / s._nblk)
            n += 1
            s.state = (lam, done + n)
            if done + n >= sweeps[lam]:
                return _lib.CONCORD_OK, n, (s._nblk, n)
            if s.flag:
                return _lib.CONCORD_YIELDED, n, (s._nblk, n)

    return sched, fit_seg


def test_handover_moves_the_long_fit_onto_idle_lanes():
    """run_segmented: when the queue runs dry the finished lanes' SMs go to the fit still running;
    it stops at a sweep end and continues on the solver of the grown SM count -- every sweep of
    every fit is run exactly once, results come back in the caller's order."""
    sweeps = {0.1: 60, 0.3: 8, 0.4: 8, 0.5: 6}
    sched, fit_seg = _seg_sched([20, 10, 10], sweeps)
    lams = [0.5, 0.1, 0.4, 0.3]
    out = sched.run_segmented(lams, fit_seg, lambda s, lam, segs: (lam, segs, s._nblk))
    assert [o[0] for o in out] == lams
    for lam, segs, _ in out:
        assert sum(n for _, n in segs) == sweeps[lam]
    dense = out[1]
    assert len(dense[1]) >= 2 and dense[2] == 40  # ended on all 40 SMs
    assert [b for b, _ in dense[1]][0] == 20
    assert sched.handovers >= 1
    # every spare is back in the pool, no yield flag left set
    assert all(len(v) == 1 for v in sched._spare.values())
    assert not any(s.flag for s in sched.shares)


def test_handover_off_and_missing_spare_keep_the_lanes():
    sweeps = {0.1: 30, 0.3: 4}
    sched, fit_seg = _seg_sched([20, 10], sweeps)
    out = sched.run_segmented([0.1, 0.3], fit_seg, lambda s, lam, segs: segs, handover=False)
    assert all(len(segs) == 1 for segs in out) and sched.handovers == 0
    sched._spare = {}  # no solver of the grown size: the fit stays on its lane
    out = sched.run_segmented([0.1, 0.3], fit_seg, lambda s, lam, segs: segs)
    assert all(len(segs) == 1 for segs in out) and sched.handovers == 0
