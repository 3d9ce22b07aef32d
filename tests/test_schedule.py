"""Host logic of the schedule: closed form == reference rotation (no GPU)."""

import dataclasses
import itertools

import numpy as np
import pytest

import paper_2106_09382_b200 as cb
from paper_2106_09382_b200.schedule import circle_round_pairs, flatten_schedule, is_circle_schedule


def _rotation(p):
    """The reference rotation (schedule.py:68-88), 1-based positions."""
    pe = p + (p % 2)
    j = list(range(1, pe + 1))
    rounds = []
    for _ in range(pe - 1):
        rounds.append([(j[q], j[pe - 1 - q]) for q in range(pe // 2)])
        j = [j[0], j[-1]] + j[1:-1]
    return rounds


@pytest.mark.parametrize("p", list(range(2, 70)) + [101, 1000, 1001])
def test_closed_form_partner_equals_rotation(p):
    pe = p + (p % 2)
    m = pe - 1
    for k, rnd in enumerate(_rotation(p)):
        part = cb.circle_partner(np.arange(pe), k, m)
        for a, b in rnd:
            assert part[a - 1] == b - 1 and part[b - 1] == a - 1
        r, s = circle_round_pairs(k, p)
        want = [(min(a, b) - 1, max(a, b) - 1) for a, b in rnd if max(a, b) <= p]
        assert list(zip(r.tolist(), s.tolist())) == want


def test_p6_rounds_known_answer():
    sched = cb.build_circle_schedule(6)
    got = [{(q.r, q.s) for q in rnd} for rnd in sched.rounds]
    assert got == [{(1, 6), (2, 5), (3, 4)}, {(1, 5), (4, 6), (2, 3)}, {(1, 4), (3, 5), (2, 6)},
                   {(1, 3), (2, 4), (5, 6)}, {(1, 2), (3, 6), (4, 5)}]


@pytest.mark.parametrize("p", range(2, 40))
def test_schedule_shape_and_coverage(p):
    sched = cb.build_circle_schedule(p)
    pe = p + (p % 2)
    assert sched.p_even == pe and len(sched.rounds) == pe - 1
    assert cb.validate_schedule(sched).ok
    real = {q for k in range(len(sched.rounds)) for q in sched.active_pairs(k)}
    assert real == {cb.IndexPair(r, s) for r, s in itertools.combinations(range(1, p + 1), 2)}
    assert is_circle_schedule(sched)


@pytest.mark.parametrize("p", list(range(2, 21)) + [101])
def test_flat_schedule_equals_reference_golden(golden, p):
    rs, ss, off = cb.flat_circle_schedule(p)
    assert np.array_equal(rs, golden[f"sched_{p}_rs"])
    assert np.array_equal(ss, golden[f"sched_{p}_ss"])
    assert np.array_equal(off, golden[f"sched_{p}_off"])
    frs, fss, foff = flatten_schedule(cb.build_circle_schedule(p))
    assert np.array_equal(frs, rs) and np.array_equal(fss, ss) and np.array_equal(foff, off)


def test_round_counts_minimal():
    assert {p: cb.build_circle_schedule(p).active_round_count() for p in (4, 5, 6, 7)} == {4: 3, 5: 5, 6: 5,
                                                                                          7: 7}


def test_validation_detects_corruption():
    sched = cb.build_circle_schedule(6)
    rounds = [list(r) for r in sched.rounds]

    def corrupt(rr):
        return dataclasses.replace(sched, rounds=tuple(tuple(r) for r in rr))

    dup = [list(r) for r in rounds]
    dup[1][0] = rounds[0][0]
    assert not cb.validate_schedule(corrupt(dup)).ok
    clash = [list(r) for r in rounds]
    clash[0][0] = cb.IndexPair(1, 5)
    assert not cb.validate_schedule(corrupt(clash)).ok
    assert not cb.validate_schedule(corrupt(rounds[:-1])).ok
    oob = [list(r) for r in rounds]
    oob[0][0] = cb.IndexPair(1, 9)
    assert not cb.validate_schedule(corrupt(oob)).ok
    # a valid colouring in another round order is valid but not the circle schedule
    perm = corrupt(rounds[::-1])
    assert cb.validate_schedule(perm).ok and not is_circle_schedule(perm)
    with pytest.raises(cb.DimensionError):
        cb.build_circle_schedule(1)


def test_index_pair_normalises():
    assert (cb.IndexPair(5, 2).r, cb.IndexPair(5, 2).s) == (2, 5)
    with pytest.raises(ValueError):
        cb.IndexPair(3, 3)


def test_read_write_sets_disjoint_within_rounds():
    for p in (5, 8, 13):
        sched = cb.build_circle_schedule(p)
        for k in range(len(sched.rounds)):
            pairs = sched.active_pairs(k)
            cells = [cb.read_write_sets(p, q) for q in pairs]
            for a in range(len(pairs)):
                for b in range(len(pairs)):
                    if a != b:
                        assert not (cells[b][1] & (cells[a][0] | cells[a][1]))
