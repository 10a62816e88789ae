"""Pins for the tree-prior oracle (CPU only).

oracle.tree builds V_G and evaluates Eq. 3 densely.  Pinned against
scipy.stats.matrix_normal (library density of Eq. 3), the paper's own v_ij
definition on a hand-built tree (root-to-MRCA times), and central finite
differences of the log-density.
"""
import numpy as np
import pytest
from scipy import stats

import workload
from oracle import tree


def test_cov_matches_paper_definition_on_a_hand_tree():
    # items 0..3; ((0:1, 1:2)4:0.5, (2:1.5, 3:0.25)5:1)6 root tau0 = 0.7; unsequenced item 7? no -- all in tree
    parent = np.array([4, 4, 5, 5, 6, 6, -1])
    t = np.array([1.0, 2.0, 1.5, 0.25, 0.5, 1.0, 0.7])
    V = tree.tree_cov(parent, t, 4)
    tau0 = 0.7
    expect = np.array([
        [tau0 + 1.5, tau0 + 0.5, tau0, tau0],
        [tau0 + 0.5, tau0 + 2.5, tau0, tau0],
        [tau0, tau0, tau0 + 2.5, tau0 + 1.0],
        [tau0, tau0, tau0 + 1.0, tau0 + 1.25],
    ])
    np.testing.assert_array_equal(V, expect)
    # an unsequenced item is its own root: v_ii = tau_e, no covariance with the rest
    parent2 = np.array([3, 3, -1, -1])
    V2 = tree.tree_cov(parent2, np.array([1.0, 1.0, 4.0, 0.5]), 3)
    np.testing.assert_array_equal(V2, [[1.5, 0.5, 0], [0.5, 1.5, 0], [0, 0, 4.0]])


def test_cov_is_sum_of_shared_increments():
    """tree_cov equals A diag(t) A' (A = item-by-ancestor-or-self indicator) on random forests."""
    for n, ntrees, fu in [(20, 1, 0.0), (40, 3, 0.2)]:
        parent, t = workload.coalescent_forest(n, ntrees, fu, seed=n)
        A = np.zeros((n, parent.size))
        for i in range(n):
            a = i
            while a >= 0:
                A[i, a] = 1.0
                a = parent[a]
        np.testing.assert_allclose(tree.tree_cov(parent, t, n), (A * t) @ A.T, rtol=1e-14, atol=0)


@pytest.mark.parametrize("n,d,ntrees,fu", [(12, 2, 1, 0.0), (30, 3, 3, 0.2), (25, 1, 2, 0.1)])
def test_logp_matches_scipy_matrix_normal(n, d, ntrees, fu):
    parent, t = workload.coalescent_forest(n, ntrees, fu, seed=n)
    rng = np.random.default_rng(n)
    x = rng.normal(size=(n, d))
    mu0 = rng.normal(size=d)
    B = rng.normal(size=(d, d))
    S = B @ B.T + d * np.eye(d)
    lp, _ = tree.tree_prior(parent, t, x, mu0, S)
    V = tree.tree_cov(parent, t, n)
    ref = stats.matrix_normal.logpdf(x, mean=np.outer(np.ones(n), mu0), rowcov=V, colcov=S)
    assert lp == pytest.approx(ref, rel=1e-11)


def test_gradient_finite_differences():
    n, d = 15, 2
    parent, t = workload.coalescent_forest(n, 2, 0.1, seed=4)
    rng = np.random.default_rng(1)
    x = rng.normal(size=(n, d))
    S = np.array([[1.0, 0.3], [0.3, 0.5]])
    _, g = tree.tree_prior(parent, t, x, None, S)
    h = 1e-5
    for i, k in [(0, 0), (3, 1), (14, 0), (7, 1)]:
        xp, xm = x.copy(), x.copy()
        xp[i, k] += h
        xm[i, k] -= h
        fd = (tree.tree_prior(parent, t, xp, None, S)[0] - tree.tree_prior(parent, t, xm, None, S)[0]) / (2 * h)
        assert g[i, k] == pytest.approx(fd, rel=1e-6, abs=1e-8)
