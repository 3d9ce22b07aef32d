"""Device centring and the problem-file -> T path.

center_columns on the GPU must give numpy's bits (model.py:182-187: the mean of
axis 0 is a sequential row-by-row sum divided by n), so the device load path
(read_problem -> centre -> Gram, cli.py:101-102) yields the same T as the host
centring followed by the device Gram.
"""

import numpy as np
import pytest

import paper_2106_09382_b200 as cb
from paper_2106_09382_b200 import fileio

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p", [(1, 3), (7, 2), (777, 33), (2000, 500), (513, 1001)])
def test_device_centering_is_bitwise_numpy(n, p):
    rng = np.random.default_rng(n * 7 + p)
    x = rng.standard_normal((n, p)) * 3.0 + rng.uniform(-5, 5, size=p)
    dm = cb.DataMatrix(x)
    host = cb.center_columns(dm)
    dev = cb.center_columns(dm, device=0)
    assert dev.centered and np.array_equal(dev.values, host.values)
    assert np.array_equal(x, dm.values)  # the input is not modified


def test_solver_gram_from_raw_data_centres_on_device():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((600, 300)) + 2.0
    want = cb.compute_gram(cb.center_columns(cb.DataMatrix(x)))
    s = cb.Solver(300)
    try:
        s.gram_from_data(cb.DataMatrix(x), center=True)
        assert np.array_equal(s.gram().t, want.t)
        s.gram_from_data(cb.DataMatrix(x))  # reference semantics: compute_gram never centres
        assert np.array_equal(s.gram().t, cb.compute_gram(cb.DataMatrix(x)).t)
    finally:
        s.close()


@pytest.mark.parametrize("centered", [False, True])
def test_read_problem_gram_matches_host_path(tmp_path, centered):
    rng = np.random.default_rng(11)
    x = rng.standard_normal((120, 40)) + 1.5
    if centered:
        x = x - x.mean(axis=0)
    path = tmp_path / "problem.txt"
    fileio.write_problem(str(path), cb.DataMatrix(x, centered=centered))
    g = fileio.read_problem_gram(str(path), device=0)
    want = cb.compute_gram(cb.center_columns(fileio.read_problem(str(path))))
    assert g.n == 120 and np.array_equal(g.t, want.t)
