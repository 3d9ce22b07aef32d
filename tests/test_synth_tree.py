"""The scale-free truth in tree form (synth.scale_free_tree / tree_cholesky), host side.

The device sampler (csrc/datagen.cu tree_sample_kernel) solves L^T x = z with the
fill-free factor these functions build; here the factor and the truth are checked
against the dense restatement of datagen.py:99-132 (synth.scale_free_precision,
itself bit-checked against the reference in tests/golden/make_golden.py).
"""

import numpy as np
import pytest

from paper_2106_09382_b200 import synth


@pytest.mark.parametrize("p,seed", [(3, 0), (50, 1), (301, 0), (1000, 7)])
def test_tree_truth_equals_dense_truth(p, seed):
    parent, weight = synth.scale_free_tree(p, seed=seed)
    assert parent[0] == -1 and np.all(parent[1:] >= 0) and np.all(parent[1:] < np.arange(1, p))
    dense = synth.scale_free_precision(p, seed=seed)
    tree = synth.tree_dense(parent, weight)
    assert np.array_equal(tree != 0.0, dense != 0.0)  # same support (a tree: p - 1 edges)
    np.testing.assert_allclose(tree, dense, rtol=2e-15, atol=0)  # row sums edge by edge: last bits


@pytest.mark.parametrize("p", [3, 64, 500])
def test_tree_cholesky_reconstructs_truth(p):
    parent, weight = synth.scale_free_tree(p, seed=2)
    lpar, ldiag = synth.tree_cholesky(parent, weight)
    L = np.diag(ldiag)
    v = np.flatnonzero(parent >= 0)
    L[parent[v], v] = lpar[v]  # column v: L[v, v] and L[parent[v], v]; parent < v
    # leaves-first elimination: the factor is "reverse lower": truth = L L^T with L upper in index order
    np.testing.assert_allclose(L @ L.T, synth.tree_dense(parent, weight), rtol=0, atol=1e-14)


def test_tree_cholesky_rejects_indefinite():
    parent = np.array([-1, 0, 0], dtype=np.int32)
    with pytest.raises(synth.NotPositiveDefinite):
        synth.tree_cholesky(parent, np.array([0.0, 0.9, 0.9]))
