"""bench.py's host-side helpers on CPU: the algorithmic-byte count and the reference
CPU legs (the oracle / oracle/_ref checker timing the reference's own per-iteration work)."""

import os
import sys

import numpy as np
import pytest

from conftest import REPO, case

sys.path.insert(0, REPO)
import bench  # noqa: E402


def test_algorithmic_bytes_per_sweep():
    p = 10
    pe = p
    per_sweep = 24.0 * p * (pe - 1) + 24.0 * p * p + 8.0 * p * p  # colours' fixed part, diagonal, objective
    assert bench.algorithmic_bytes(p, [0]) == per_sweep
    assert bench.algorithmic_bytes(p, [3, 0]) == 2 * per_sweep + 48.0 * p * 3
    assert bench.algorithmic_bytes(p, [0], want_trace=False) == per_sweep - 8.0 * p * p
    p = 11  # odd p: p + 1 - 1 colours
    assert bench.algorithmic_bytes(p, [0]) == 24.0 * p * 11 + 24.0 * p * p + 8.0 * p * p


def test_cpu_full_fit_follows_the_reference_loop(golden):
    c = case(golden, "ar2_p100_n50_l0.3")
    v = bench.cpu_full_fit(c["t"], c["n"], c["lam"], workers=2)
    assert v["iterations"] == c["iters"] and v["edges"] == c["edges"]
    assert v["per_sweep_s"] > 0 and v["sum_wall_time_per_iteration_s"] >= v["per_sweep_s"]


def test_cpu_reference_rate_is_a_positive_sweep_rate(golden):
    c = case(golden, "ar2_p100_n50_l0.3")
    rate, kind, rounds, el, ovh = bench.cpu_reference_rate(c["t"], c["n"], 0.3, 0.05, 2)
    assert kind in ("reference", "port")
    assert rate > 0 and 2 <= rounds <= 99 and el > 0 and ovh >= 0
