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


def test_leapfrog_tree_with_unsequenced_forest_is_the_iid_leapfrog():
    """A forest of n unsequenced items (each its own root, t = tau^2; Sigma = I,
    mu0 = 0) is V_G = tau^2 I, i.e. the iid N(0, tau^2) prior (PAPER.md:189,
    reading R20): leapfrog_tree must reproduce the C oracle's leapfrog with
    prior_sd = tau -- x, p, dH and log L."""
    import oracle
    w = workload.Workload(40, 2, p_missing=0.1, seed=3)
    y, x0 = w.y_packed(), w.x0
    p0 = w.normals(4, (40, 2))
    tau = 1.7
    parent = np.full(40, -1, dtype=np.int64)
    t = np.full(40, tau * tau)
    a = tree.leapfrog_tree(y, x0, p0, w.sigma, 0.003, 7, parent, t)
    b = oracle.leapfrog(y, x0, p0, w.sigma, 0.003, 7, 1, prior_sd=tau)
    np.testing.assert_allclose(a["x"], b["x"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(a["p"], b["p"], rtol=1e-11, atol=1e-12)
    # Eq. 3 is normalised; the iid prior of the C oracle's H drops its constant
    # n d/2 log(2 pi tau^2): the Hamiltonians differ by exactly that, dH agrees
    const = 0.5 * 40 * 2 * np.log(2 * np.pi * tau * tau)
    assert a["H0"] == pytest.approx(b["H0"] + const, rel=1e-12)
    assert a["H1"] == pytest.approx(b["H1"] + const, rel=1e-12)
    assert a["H1"] - a["H0"] == pytest.approx(b["H1"] - b["H0"], rel=1e-8, abs=1e-10)
    assert a["loglik"] == pytest.approx(b["loglik"], rel=1e-12)


def test_leapfrog_tree_prior_only_is_the_linear_leapfrog_map():
    """All pairs missing (log L = 0): the target is the Gaussian Eq. 3 prior with
    precision A = Sigma^-1 (x) V_G^-1, and one leapfrog step is the linear map
    p' = p - eps/2 A x, x' = x + eps p', p'' = p' - eps/2 A x' on the stacked
    vectors (standard leapfrog).  L steps = that map applied L
    times, with H = -log p + |p|^2/2 from the closed-form Gaussian density."""
    n, d = 18, 2
    parent, t = workload.coalescent_forest(n, 2, 0.2, seed=11, tau0=0.8, tau_e=2.0)
    S = np.array([[1.0, 0.4], [0.4, 0.7]])
    mu0 = np.array([0.3, -0.2])
    rng = np.random.default_rng(2)
    x0 = rng.normal(size=(n, d))
    p0 = rng.normal(size=(n, d))
    y = np.full(n * (n - 1) // 2, np.nan)
    eps, L = 0.01, 5
    V = tree.tree_cov(parent, t, n)
    Vi, Si = np.linalg.inv(V), np.linalg.inv(S)
    grad = lambda x: -Vi @ (x - mu0) @ Si                      # d log p / dX, matrix form
    x, p = x0.copy(), p0.copy()
    for _ in range(L):
        p = p + 0.5 * eps * grad(x)
        x = x + eps * p
        p = p + 0.5 * eps * grad(x)
    a = tree.leapfrog_tree(y, x0, p0, 1.0, eps, L, parent, t, mu0, S)
    np.testing.assert_allclose(a["x"], x, rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(a["p"], p, rtol=1e-9, atol=1e-11)
    lp = lambda z: stats.matrix_normal.logpdf(z, mean=np.outer(np.ones(n), mu0), rowcov=V, colcov=S)
    assert a["H0"] == pytest.approx(-lp(x0) + 0.5 * (p0 * p0).sum(), rel=1e-10)
    assert a["H1"] == pytest.approx(-lp(x) + 0.5 * (p * p).sum(), rel=1e-10)
    assert a["loglik"] == 0.0
