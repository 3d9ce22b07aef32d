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

    monkeypatch.setattr(solver._lib, "device_sm_count", lambda device: 148)
    monkeypatch.setattr(solver, "Solver", FakeSolver)
    assert PathScheduler(5000, k=2).lanes == [74, 74]
    assert PathScheduler(5000, k=3).lanes == [66, 41, 41]
    assert PathScheduler(5000, k=4).lanes == [66, 28, 27, 27]
    assert PathScheduler(5000, k=5).lanes == [66, 21, 21, 20, 20]
    assert sum(PathScheduler(5000, k=4).lanes) == 148
    with pytest.raises(ValueError):
        PathScheduler(5000, lanes=[100, 60])
