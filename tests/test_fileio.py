"""Boundary formats (fileio.py) and check_optimality against the reference's own outputs."""

import os

import numpy as np
import pytest

import paper_2106_09382_b200 as cb
from paper_2106_09382_b200 import fileio
from conftest import REPO, case

IO = os.path.join(REPO, "tests", "golden", "reference_io_golden.npz")


@pytest.fixture(scope="module")
def io_golden():
    with np.load(IO) as z:
        return {k: z[k] for k in z.files}


def test_write_estimate_is_byte_identical_to_reference(golden, io_golden, tmp_path):
    for name in [str(s) for s in golden["case_names"]]:
        c = case(golden, name)
        path = tmp_path / "e.txt"
        fileio.write_estimate(str(path), cb.PrecisionEstimate(c["omega"]), c["lam"], c["iters"], c["delta"])
        assert path.read_bytes() == io_golden[f"{name}_estimate_txt"].tobytes(), name
        est, meta = fileio.read_estimate(str(path))
        assert np.array_equal(est.omega, c["omega"])
        assert meta == {"lam": c["lam"], "iterations": c["iters"], "delta": c["delta"]}


def test_write_estimate_from_entry_arrays(golden, io_golden, tmp_path):
    c = case(golden, "sf_p101_n50_l0.3")
    ents = fileio.estimate_entries(cb.PrecisionEstimate(c["omega"]))
    path = tmp_path / "e.txt"
    fileio.write_estimate(str(path), ents, c["lam"], c["iters"], c["delta"], p=c["p"])
    assert path.read_bytes() == io_golden["sf_p101_n50_l0.3_estimate_txt"].tobytes()


def test_problem_round_trip_is_byte_identical(golden, io_golden, tmp_path):
    c = case(golden, "ar2_p9_n70_l0.1")
    path = tmp_path / "x.txt"
    fileio.write_problem(str(path), cb.DataMatrix(c["x"], centered=True))
    assert path.read_bytes() == io_golden["ar2_p9_n70_l0.1_problem_txt"].tobytes()
    back = fileio.read_problem(str(path))
    assert np.array_equal(back.values, c["x"]) and back.centered


@pytest.mark.parametrize("text,msg", [
    ("", "empty"), ("3,1\n", "header"), ("2,2,5\n1,2\n3,4\n", "centered flag"), ("3,2,0\n1,2\n", "promises"),
    ("1,2,0\n1,x\n", "cannot parse"), ("1,3,0\n1,2\n", "expected 3"),
    ("2,2,0\n1,2\n3,oops\n", ":3: cannot parse value 2"),
])
def test_read_problem_rejects_malformed(tmp_path, text, msg):
    path = tmp_path / "bad.txt"
    path.write_text(text)
    with pytest.raises(fileio.FileFormatError, match=msg):
        fileio.read_problem(str(path))


@pytest.mark.parametrize("text,msg", [
    ("2,0.1,3\n", "header"), ("2,0.1,3,0\n1,1,1\n1,3,0.5\n2,2,1\n", "out of range"),
    ("2,0.1,3,0\n1,1,1\n1,1,1\n2,2,1\n", "duplicate"), ("2,0.1,3,0\n1,1,1\n", "diagonal entry 2"),
    ("2,0.1,3,0\n1,1\n", "expected 'i,j,value'"),
    ("2,0.1,3,0\n1,1,1\n1,2,x\n2,2,1\n", ":3: cannot parse value"),
    ("2,0.1,3,0\n1,1,1\n\n1,q,1\n2,2,1\n", ":4: cannot parse j"),
    ("2,0.1,3,0\n1,1,1\n2,2,1\n1,1,2\n", ":4: duplicate entry \\(1, 1\\)"),
])
def test_read_estimate_rejects_malformed(tmp_path, text, msg):
    path = tmp_path / "bad.txt"
    path.write_text(text)
    with pytest.raises(fileio.FileFormatError, match=msg):
        fileio.read_estimate(str(path))


def test_check_optimality_matches_reference(golden, io_golden):
    for name in [str(s) for s in golden["case_names"]]:
        c = case(golden, name)
        rep = cb.check_optimality(cb.PrecisionEstimate(c["omega"]), cb.GramMatrix(c["t"], c["n"]), c["lam"])
        worst, i, j = io_golden[f"{name}_opt"]
        assert rep.worst_violation == worst, name
        assert rep.worst_coordinate == (int(i), int(j)), name
