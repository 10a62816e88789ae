"""GPU parity of the phylogenetic Brownian-diffusion prior (
PAPER.md:147-202, Eq. 3) against the dense CPU oracle (oracle/tree.py),
through the C-ABI.

The device never forms V_G: log p and its gradient come from a post-order /
pre-order pass over the forest.  Tolerances: log p within 1e-10 relative; each
gradient entry within 1e-9 relative or 1e-11 of the row-scale max |g| (the
dense oracle's own Cholesky error grows with cond(V_G)).
"""
import numpy as np
import pytest

import oracle
import workload
from oracle import tree

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mds():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1905_04582_b200 as m
    return m


def multifurcate(parent, t, n, rng, frac=0.3):
    """Collapse a fraction of internal edges (child internal node merged into its
    parent) to get multifurcating nodes; renumber internal nodes densely."""
    parent, t = parent.copy(), t.copy()
    alive = np.ones(parent.size, bool)
    for k in range(n, parent.size):
        if parent[k] >= 0 and rng.random() < frac:
            pk = parent[k]
            kids = np.flatnonzero(parent == k)
            parent[kids] = pk
            t[kids] += t[k]
            alive[k] = False
    newid = -np.ones(parent.size, np.int64)
    newid[alive] = np.arange(alive.sum())
    p2 = np.where(parent[alive] >= 0, newid[np.maximum(parent[alive], 0)], -1)
    return p2, t[alive]


def sample_prior(parent, t, n, d, mu0, S, rng):
    """X drawn from the prior itself (Brownian motion down the forest): the
    regime HMC draws live in.  (iid X far from the prior makes the dense
    oracle's V_G solve, cond ~ 1e8 for coalescent trees, the inaccurate side.)"""
    L = np.linalg.cholesky(S)
    val = np.zeros((parent.size, d))
    order = []
    kids = [[] for _ in range(parent.size)]
    for k, p in enumerate(parent):
        if p >= 0:
            kids[p].append(k)
        else:
            order.append(k)
    for v in order:                       # breadth-first: parents before children
        base = mu0 if parent[v] < 0 else val[parent[v]]
        val[v] = base + np.sqrt(t[v]) * (L @ rng.normal(size=d))
        order.extend(kids[v])
    return val[:n].copy()


def check(lp, g, ref_lp, ref_g):
    assert lp == pytest.approx(ref_lp, rel=1e-10)
    scale = np.abs(ref_g).max()
    err = np.abs(g - ref_g)
    assert np.all(err <= np.maximum(1e-9 * np.abs(ref_g), 1e-11 * scale)), err.max()


@pytest.mark.parametrize("n,d,ntrees,fu,multi", [(64, 2, 1, 0.0, False), (500, 2, 1, 0.0, False),
                                                 (1200, 3, 4, 0.1, False), (800, 6, 2, 0.05, True),
                                                 (300, 8, 1, 0.0, True), (3, 1, 1, 0.0, False)])
def test_tree_prior_parity(mds, n, d, ntrees, fu, multi):
    parent, t = workload.coalescent_forest(n, ntrees, fu, seed=n + d)
    rng = np.random.default_rng(n)
    if multi:
        parent, t = multifurcate(parent, t, n, rng)
    mu0 = rng.normal(size=d) * 0.3
    B = rng.normal(size=(d, d)) * 0.3
    S = B @ B.T + np.eye(d)
    x = sample_prior(parent, t, n, d, mu0, S, rng)
    ref_lp, ref_g = tree.tree_prior(parent, t, x, mu0, S)
    w = workload.Workload(n, d, seed=3)
    with mds.MDS(n, d) as c:
        c.set_locations(x)
        c.set_tree_prior(parent, t, mu0, S)
        lp, g = c.tree_prior()
        lp2, g2 = c.tree_prior()
    check(lp, g, ref_lp, ref_g)
    assert lp == lp2 and np.array_equal(g, g2)        # deterministic


def test_tree_prior_high_arity(mds):
    """A star tree (one internal node with 400 children, short branches) and a
    caterpillar (depth n - 1): extreme arity and depth."""
    n, d = 400, 2
    rng = np.random.default_rng(9)
    star_p = np.array([n] * n + [-1])
    star_t = np.concatenate([1e-3 + 1e-2 * rng.random(n), [2.0]])
    cat_p = np.empty(2 * n - 1, np.int64)
    cat_t = 0.05 + rng.random(2 * n - 1)
    # internal node n + k joins item k + 1 and the subtree below n + k - 1 (n + 0 joins items 0, 1)
    cat_p[0] = n
    for k in range(n - 1):
        cat_p[k + 1] = n + k
        cat_p[n + k] = n + k + 1 if k < n - 2 else -1
    for parent, t in ((star_p, star_t), (cat_p, cat_t)):
        x = sample_prior(parent, t, n, d, np.zeros(d), np.eye(d), rng)
        ref_lp, ref_g = tree.tree_prior(parent, t, x)
        with mds.MDS(n, d) as c:
            c.set_locations(x)
            c.set_tree_prior(parent, t)
            lp, g = c.tree_prior()
        check(lp, g, ref_lp, ref_g)


def test_tree_prior_c2_size(mds):
    n, d = 5392, 2
    parent, t = workload.coalescent_forest(n, 1, 0.0, seed=11)
    x = sample_prior(parent, t, n, d, np.zeros(d), np.eye(d), np.random.default_rng(2))
    ref_lp, ref_g = tree.tree_prior(parent, t, x)
    with mds.MDS(n, d) as c:
        c.set_locations(x)
        c.set_tree_prior(parent, t)
        lp, g = c.tree_prior()
    check(lp, g, ref_lp, ref_g)


def test_hmc_trajectory_with_tree_prior(mds):
    n, d = 300, 2
    w = workload.Workload(n, d, p_missing=0.05, seed=31)
    y, x = w.y_packed(), w.x0
    parent, t = workload.coalescent_forest(n, 2, 0.1, seed=5, tau0=4.0)
    S = np.array([[1.0, 0.2], [0.2, 0.8]])
    p0 = w.normals(1, (n, d))
    ref = tree.leapfrog_tree(y, x, p0, w.sigma, 0.002, 12, parent, t, None, S)
    with mds.MDS(n, d) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(x)
        c.set_sigma(w.sigma)
        c.set_tree_prior(parent, t, None, S)
        out = c.hmc_trajectory(p0, 0.002, 12, prior_sd=123.0)     # prior_sd ignored under the tree prior
        # with a tree prior the pass kernel's last CTA walks the tree: the pair
        # schedule has one CTA less -- plain evaluations are unchanged
        ll_t, g_t = c.log_likelihood_and_gradient()
        # back to the iid prior
        c.clear_tree_prior()
        out2 = c.hmc_trajectory(p0, 0.002, 12, prior_sd=10.0)
    full = oracle.loglik_grad(y, x, w.sigma, 1)
    assert ll_t == pytest.approx(full["loglik"], rel=1e-10)
    np.testing.assert_allclose(g_t, full["grad"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["x"], ref["x"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["p"], ref["p"], rtol=1e-9, atol=1e-9)
    assert out["H0"] == pytest.approx(ref["H0"], rel=1e-10)
    assert out["H1"] == pytest.approx(ref["H1"], rel=1e-10)
    ref2 = oracle.leapfrog(y, x, p0, w.sigma, 0.002, 12, 1, prior_sd=10.0)
    np.testing.assert_allclose(out2["x"], ref2["x"], rtol=1e-9, atol=1e-12)


def test_hmc_run_with_tree_prior_chain(mds):
    """A short chain under the tree prior: final log L consistent with the oracle at the final X."""
    w = workload.config("C1")
    y = w.y_packed()
    parent, t = workload.coalescent_forest(w.n, 1, 0.0, seed=2, tau0=10.0)
    with mds.MDS(w.n, w.d) as c:
        c.set_dissimilarities_packed(y)
        c.set_sigma(w.sigma)
        c.set_tree_prior(parent, t)
        x, st = c.hmc_run(30, 10, 0.01, 0.0, seed=3, x0=w.x0)
        assert 0 < st["accepted"] <= 30
    assert st["final_loglik"] == pytest.approx(oracle.loglik_grad(y, x, w.sigma, 1)["loglik"], rel=1e-10)


def test_tree_prior_errors(mds):
    with mds.MDS(4, 2) as c:
        c.set_locations(np.zeros((4, 2)))
        with pytest.raises(mds.MDSError) as e:
            c.tree_prior()
        assert e.value.status == 2
        good_p = np.array([4, 4, 5, 5, 6, 6, -1])
        good_t = np.array([1.0, 2.0, 1.5, 0.25, 0.5, 1.0, 0.7])
        for p, t in [(np.array([4, 4, 5, 5, 6, 6, 5]), good_t),           # cycle 5 -> 6 -> 5
                     (np.array([1, 4, 5, 5, 6, 6, -1]), good_t),          # item with a child
                     (good_p, np.where(np.arange(7) == 2, 0.0, good_t)),  # zero branch
                     (np.array([4, 4, 5, 5, 6, 6, -1, -1]), np.ones(8))]:  # childless internal node
            with pytest.raises(mds.MDSError) as e:
                c.set_tree_prior(p, t)
            assert e.value.status == 1
        with pytest.raises(mds.MDSError):
            c.set_tree_prior(good_p, good_t, None, np.array([[1.0, 2.0], [2.0, 1.0]]))   # not SPD
        c.set_tree_prior(good_p, good_t)
        lp, g = c.tree_prior()
    ref_lp, _ = tree.tree_prior(good_p, good_t, np.zeros((4, 2)))
    assert lp == pytest.approx(ref_lp, rel=1e-12)


def test_fp32_leapfrog_with_tree_prior(mds):
    """fp32 storage/pair math (reading R15) with the tree walk fused into the
    leapfrog pass (pass_kernel<float, D, T, LEAPFROG_TREE>): trajectory vs the
    oracle on fp32-rounded inputs, fp32 tolerance."""
    import torch
    n, d = 350, 3
    w = workload.Workload(n, d, p_missing=0.05, seed=91)
    y = w.y_packed().astype(np.float32).astype(np.float64)
    x = w.x0.astype(np.float32).astype(np.float64)
    parent, t = workload.coalescent_forest(n, 2, 0.05, seed=4, tau0=4.0)
    p0 = w.normals(4, (n, d))
    ref = tree.leapfrog_tree(y, x, p0, w.sigma, 0.002, 6, parent, t)
    with mds.MDS(n, d, "f32") as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(x)
        c.set_sigma(w.sigma)
        c.set_tree_prior(parent, t)
        c.leapfrog_device(6, 0.002, 0.0, p0_dev=torch.from_numpy(p0).cuda())
        xs = c.get_locations()
        ll = c.log_likelihood()
    np.testing.assert_allclose(xs, ref["x"], rtol=1e-5, atol=1e-7)
    assert ll == pytest.approx(ref["loglik"], rel=1e-4)


def test_tree_leapfrog_bitwise_deterministic(mds):
    """The fused walk (tips pass and first level on the pair CTAs, a device counter
    between them) keeps the pass deterministic: two runs from the same state are
    bitwise identical."""
    import torch
    n, d = 2000, 2
    w = workload.Workload(n, d, p_missing=0.05, seed=5)
    parent, t = workload.coalescent_forest(n, 3, 0.05, seed=6, tau0=3.0)
    p0 = torch.from_numpy(w.normals(7, (n, d))).cuda()
    outs = []
    for _ in range(2):
        with mds.MDS(n, d) as c:
            c.set_dissimilarities_packed(w.y_packed())
            c.set_locations(w.x0)
            c.set_sigma(w.sigma)
            c.set_tree_prior(parent, t)
            c.leapfrog_device(9, 0.001, 0.0, p0_dev=p0)
            outs.append((c.get_locations(), c.get_momentum(), c.log_likelihood()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]
