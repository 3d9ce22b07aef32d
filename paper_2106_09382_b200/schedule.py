"""Round-robin edge colouring of K_p: the pair schedule of one PCD sweep.

Same schedule as the reference (schedule.py:68-88): index 1 pinned, the
others rotate one position per round, position q pairs with p_even-1-q, odd p
gets a phantom index p+1 whose pairs are skipped.  On the GPU the schedule is
never materialised: `circle_partner` is the closed form the kernels evaluate
(csrc/common.cuh), checked against the rotation in tests/test_schedule.py.
The Python objects below exist for API compatibility and for validating
caller-supplied schedules.
"""

from dataclasses import dataclass

import numpy as np

from .model import DimensionError


@dataclass(frozen=True, order=True)
class IndexPair:
    """Unordered 1-based pair normalised to r < s (schedule.py:21-34)."""

    r: int
    s: int

    def __post_init__(self):
        if self.r == self.s:
            raise ValueError(f"pair indices must differ, got ({self.r}, {self.s})")
        if self.r > self.s:
            lo, hi = self.s, self.r
            object.__setattr__(self, "r", lo)
            object.__setattr__(self, "s", hi)


@dataclass(frozen=True)
class Schedule:
    """All rounds of one outer iteration over indices 1..p_even (schedule.py:37-59)."""

    p: int
    p_even: int
    rounds: tuple

    def is_phantom(self, pair: IndexPair) -> bool:
        return pair.s > self.p

    def active_pairs(self, k):
        return tuple(q for q in self.rounds[k] if not self.is_phantom(q))

    def active_round_count(self) -> int:
        return sum(1 for k in range(len(self.rounds)) if self.active_pairs(k))


@dataclass(frozen=True)
class ValidationReport:
    ok: bool
    message: str = ""


def circle_partner(x, k, m):
    """0-based partner of id x in round k of the circle schedule with m = p_even-1 rounds.

    Vectorised over numpy arrays.  Id 0 is the pinned index.
    """
    x = np.asarray(x, dtype=np.int64)
    y = 1 + (3 * m - x - 1 - 2 * k) % m
    y = np.where(y == x, 0, y)
    return np.where(x == 0, 1 + (m - 1 - k) % m, y)


def circle_round_pairs(k, p):
    """0-based (r, s) arrays of round k in the reference's within-round order, phantoms dropped."""
    pe = p + (p % 2)
    m = pe - 1
    q = np.arange(pe // 2, dtype=np.int64)
    a = np.where(q == 0, 0, 1 + (q - 1 - k + m) % m)
    b = 1 + (2 * m - q - 1 - k) % m
    r, s = np.minimum(a, b), np.maximum(a, b)
    keep = s < p
    return r[keep], s[keep]


def flat_circle_schedule(p):
    """(rs, ss, offsets) as solver._flatten_schedule would return for build_circle_schedule(p)."""
    if p < 2:
        raise DimensionError("schedule needs p >= 2")
    pe = p + (p % 2)
    rs, ss, offsets = [], [], [0]
    for k in range(pe - 1):
        r, s = circle_round_pairs(k, p)
        rs.append(r)
        ss.append(s)
        offsets.append(offsets[-1] + r.size)
    return np.concatenate(rs), np.concatenate(ss), np.asarray(offsets, dtype=np.int64)


def build_circle_schedule(p: int) -> Schedule:
    """The reference schedule object (schedule.py:68-88), from the closed form."""
    if p < 2:
        raise DimensionError("schedule needs p >= 2")
    pe = p + (p % 2)
    m = pe - 1
    rounds = []
    for k in range(m):
        q = np.arange(pe // 2)
        a = np.where(q == 0, 0, 1 + (q - 1 - k + m) % m)
        b = 1 + (2 * m - q - 1 - k) % m
        rounds.append(tuple(IndexPair(int(u) + 1, int(v) + 1) for u, v in zip(a, b)))
    return Schedule(p=p, p_even=pe, rounds=tuple(rounds))


def validate_schedule(schedule: Schedule) -> ValidationReport:
    """Round shape, within-round disjointness and exact-once coverage (schedule.py:91-149)."""
    p, pe = schedule.p, schedule.p_even
    if p < 2:
        return ValidationReport(False, "p must be at least 2")
    if pe != p + (p % 2):
        return ValidationReport(False, f"p_even={pe} does not match p={p}")
    if len(schedule.rounds) != pe - 1:
        return ValidationReport(False, f"expected {pe - 1} rounds, got {len(schedule.rounds)}")
    seen = set()
    for k, rnd in enumerate(schedule.rounds):
        if len(rnd) != pe // 2:
            return ValidationReport(False, f"round {k} has {len(rnd)} pairs, expected {pe // 2}")
        used = set()
        for pair in rnd:
            if not isinstance(pair, IndexPair):
                return ValidationReport(False, f"round {k} holds a non-IndexPair entry")
            if not (1 <= pair.r < pair.s <= pe):
                return ValidationReport(False, f"pair ({pair.r}, {pair.s}) out of range in round {k}")
            if pair.r in used or pair.s in used:
                return ValidationReport(False, f"round {k} reuses an index in ({pair.r}, {pair.s})")
            used.update((pair.r, pair.s))
            if pair in seen:
                return ValidationReport(False, f"pair ({pair.r}, {pair.s}) appears twice")
            seen.add(pair)
    if len(seen) != pe * (pe - 1) // 2:
        return ValidationReport(False, "not every pair is covered")
    return ValidationReport(True)


def flatten_schedule(schedule: Schedule):
    """solver.py:166-178: non-phantom pairs round by round, 0-based int64 arrays."""
    rs, ss, offsets = [], [], [0]
    for k in range(len(schedule.rounds)):
        for pr in schedule.active_pairs(k):
            rs.append(pr.r - 1)
            ss.append(pr.s - 1)
        offsets.append(len(rs))
    return (np.asarray(rs, dtype=np.int64), np.asarray(ss, dtype=np.int64),
            np.asarray(offsets, dtype=np.int64))


def is_circle_schedule(schedule: Schedule) -> bool:
    """True when the schedule's rounds are the circle method's, round by round (order in a round is free)."""
    p = schedule.p
    if schedule.p_even != p + (p % 2) or len(schedule.rounds) != schedule.p_even - 1:
        return False
    for k in range(len(schedule.rounds)):
        r, s = circle_round_pairs(k, p)
        want = set(zip((r + 1).tolist(), (s + 1).tolist()))
        got = {(q.r, q.s) for q in schedule.active_pairs(k)}
        if want != got:
            return False
    return True
