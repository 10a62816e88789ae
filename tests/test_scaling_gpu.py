"""GPU parity across the scale of the data: the scaling identity of Eq. 1/2.

For a > 0, ell(a y, a d; a sigma) = ell(y, d; sigma) - log a for every pair
(the truncated-normal density of PAPER.md:78-83 is a location-scale family,
and Phi(d/sigma) is scale-free), so
    log L(aY, aX, a sigma) = log L(Y, X, sigma) - n_obs log a,
    grad(aY, aX, a sigma)  = grad(Y, X, sigma) / a.
The device pair math carries sigma-dependent constants (cg = 1/(sigma sqrt(2 pi))
folded into the exp table, q coefficients scaled by 1/cg): a large sigma pushes
E' = cg exp(-t^2/2) below the normal range for large t, the case reading R33
 covers.  Every kernel that uses the pair math is checked here at
a in {1e-3, 1, 1e3, 1e4, 1e6} on the sigma = 0.05 tail instance (t up to ~10^2):
the fused pass (log L + gradient and the likelihood-only pass), the row delta
and the cross-validation accumulator, each against the oracle evaluated at the
scaled inputs and against the identity.
"""
import math

import numpy as np
import pytest

import oracle
import workload

pytestmark = pytest.mark.gpu

SCALES = (1e-3, 1.0, 1e3, 1e4, 1e6)


@pytest.fixture(scope="module")
def mds():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1905_04582_b200 as m
    return m


def tail_instance(n=300, pm=0.05):
    w = workload.Workload(n, 2, p_missing=pm, seed=77)
    return w, w.y_packed(), w.x0 * 3.0, 0.05


def assert_fp64(ll, g, ref, tag):
    rl, G = ref["loglik"], ref["grad"]
    assert abs(ll - rl) <= 1e-10 * abs(rl), (tag, ll, rl)
    err = np.abs(g - G)
    tol = np.maximum(1e-9 * np.abs(G), 1e-12)
    assert np.all(err <= tol), (tag, float((err / tol).max()))


@pytest.mark.parametrize("a", SCALES)
def test_pass_scaling_identity(mds, a):
    w, y, x, sigma = tail_instance()
    ys, xs, ss = y * a, x * a, sigma * a
    ref = oracle.loglik_grad(ys, xs, ss, 1)
    ref1 = oracle.loglik_grad(y, x, sigma, 1)
    with mds.MDS(w.n, 2, "f64", True) as c:
        c.set_dissimilarities_packed(ys)
        c.set_locations(xs)
        c.set_sigma(ss)
        ll, g = c.log_likelihood_and_gradient()
        lik_only = c.log_likelihood_at_sigma(ss)        # the likelihood-only pass mode
        n_obs = c.observed_pairs()
    assert np.isfinite(ll) and np.all(np.isfinite(g))
    assert_fp64(ll, g, ref, "a=%g" % a)
    assert abs(lik_only - ref["loglik"]) <= 1e-10 * abs(ref["loglik"])
    # the identity, against the unscaled oracle (independent of the scaled run's constants)
    want = ref1["loglik"] - n_obs * math.log(a)
    assert abs(ll - want) <= 1e-10 * abs(want), (ll, want)
    G1 = ref1["grad"] / a
    assert np.all(np.abs(g - G1) <= np.maximum(1e-9 * np.abs(G1), 1e-12 / a))


@pytest.mark.parametrize("a", (1e3, 1e6))
def test_pass_scaling_fp32(mds, a):
    """fp32 storage/math at a large scale (reading R15 tolerances vs the oracle on
    fp32-rounded inputs)."""
    w, y, x, sigma = tail_instance(n=257)
    ys, xs, ss = y * a, x * a, sigma * a
    y32 = ys.astype(np.float32).astype(np.float64)
    x32 = xs.astype(np.float32).astype(np.float64)
    ref = oracle.loglik_grad(y32, x32, ss, 1)
    with mds.MDS(w.n, 2, "f32", True) as c:
        c.set_dissimilarities_packed(ys)
        c.set_locations(xs)
        c.set_sigma(ss)
        ll, g = c.log_likelihood_and_gradient()
    rl, G, S = ref["loglik"], ref["grad"], ref["absscale"]
    assert abs(ll - rl) <= 1e-4 * abs(rl)
    assert np.linalg.norm(g - G) <= 1e-4 * np.linalg.norm(G)
    assert np.all(np.abs(g - G) <= 1e-4 * np.abs(G) + 1e-6 * S)


def _row_scale(y, x, i, sigma):
    n = x.shape[0]
    s = 0.0
    for j in range(n):
        if j == i:
            continue
        hi, lo = max(i, j), min(i, j)
        yy = y[hi * (hi - 1) // 2 + lo]
        if not np.isnan(yy):
            s += abs(oracle.pair_term(yy, float(np.linalg.norm(x[i] - x[j])), sigma, 1)[0])
    return s


@pytest.mark.parametrize("a", SCALES)
def test_row_delta_scaling(mds, a):
    w, y, x, sigma = tail_instance()
    ys, xs, ss = y * a, x * a, sigma * a
    rng = np.random.default_rng(5)
    with mds.MDS(w.n, 2, "f64", True) as c:
        c.set_dissimilarities_packed(ys)
        c.set_locations(xs)
        c.set_sigma(ss)
        for i in (0, 17, 150, 299):
            xn = xs[i] + rng.normal(size=2) * 0.3 * a
            got = c.row_loglik_delta(i, xn)
            ref = oracle.row_delta(ys, xs, i, xn, ss, 1)
            assert np.isfinite(got)
            assert abs(got - ref) <= 1e-10 * _row_scale(ys, xs, i, ss), (a, i, got, ref)
            # Delta is scale-free: the -log a of the moved and the old terms cancel
            ref1 = oracle.row_delta(y, x, i, xn / a, sigma, 1)
            assert abs(got - ref1) <= 1e-10 * _row_scale(y, x, i, sigma), (a, i, got, ref1)


@pytest.mark.parametrize("a", SCALES)
def test_cv_scaling(mds, a):
    w, y, x, sigma = tail_instance(n=400, pm=0.0)
    rng = np.random.default_rng(9)
    obs = np.flatnonzero(~np.isnan(y))
    held = np.sort(rng.choice(obs, size=obs.size // 5, replace=False))
    hi = np.floor((1 + np.sqrt(1 + 8 * held.astype(np.float64))) / 2).astype(np.int64)
    hi -= (hi * (hi - 1) // 2 > held)
    hj = held - hi * (hi - 1) // 2
    hy = y[held] * a
    train = y * a
    train[held] = np.nan
    S = 4
    xs = np.stack([(x + 0.01 * rng.normal(size=x.shape)) * a for _ in range(S)])
    sig = sigma * a * (1 + 0.1 * rng.random(S))
    with mds.MDS(w.n, 2, "f64", True) as c:
        c.set_dissimilarities_packed(train)
        c.cv_set_heldout(hi, hj, hy)
        for s in range(S):
            c.set_locations(xs[s])
            c.set_sigma(sig[s])
            c.cv_accumulate()
        lpd, _ = c.cv_lpd()
    ref = oracle.cv_lpd(hi, hj, hy, xs, sig, 1)
    ref1 = oracle.cv_lpd(hi, hj, hy / a, xs / a, sig / a, 1) - hy.size * math.log(a)
    assert np.isfinite(lpd)
    assert lpd == pytest.approx(ref, rel=1e-10)
    assert lpd == pytest.approx(ref1, rel=1e-10)
