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
