"""Pins for the CPU oracle against things other than itself (CPU only).

Each test fixes the oracle to an independent source: scipy's truncated-normal
and normal log-densities (library routines for Eq. 1's density), mpmath
brute force at 30+ digits, hand-derived closed forms (tests/golden), central
finite differences of a scipy-built log-likelihood, geometric invariants,
and the closed-form leapfrog map of a Gaussian target.
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest
from scipy import stats

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")


def scipy_loglik(y_full, x, sigma, truncation=1):
    """Sum over observed i>j of the truncated-normal (or normal) log-density of
    y_ij given delta_ij (Eq. 1), via scipy -- independent of the oracle."""
    n = x.shape[0]
    tot = 0.0
    for i in range(1, n):
        for j in range(i):
            y = y_full[i, j]
            if np.isnan(y):
                continue
            d = float(np.linalg.norm(x[i] - x[j]))
            if truncation:
                tot += stats.truncnorm.logpdf(y, a=(0.0 - d) / sigma, b=np.inf, loc=d, scale=sigma)
            else:
                tot += stats.norm.logpdf(y, loc=d, scale=sigma)
    return tot


def rand_instance(rng, n, d, sigma=0.8, missing=0.0):
    x = rng.normal(size=(n, d))
    y = np.full((n, n), np.nan)
    for i in range(1, n):
        for j in range(i):
            dd = np.linalg.norm(x[i] - x[j])
            v = -1.0
            while v <= 0:
                v = dd + sigma * rng.normal()
            if rng.random() >= missing:
                y[i, j] = y[j, i] = v
    return x, y


# ---------------------------------------------------------------- pair term
def test_pair_coincident_closed_form():
    g = json.load(open(GOLDEN))["pair_coincident"]
    ell, coef = oracle.pair_term(g["y"], g["d"], g["sigma"], g["truncation"])
    pi = math.pi
    assert ell == pytest.approx(eval(g["ell_formula"], {"log": math.log, "pi": pi}), rel=1e-15)
    assert coef == pytest.approx(eval(g["coef_formula"], {"sqrt": math.sqrt, "pi": pi}), rel=1e-15)


@pytest.mark.parametrize("trunc", [0, 1])
def test_pair_term_vs_scipy(trunc):
    rng = np.random.default_rng(1)
    for _ in range(300):
        sigma = float(rng.uniform(0.2, 3.0))
        d = float(rng.uniform(0.0, 12.0) * sigma / 2)
        y = float(abs(rng.normal(d, sigma))) + 1e-3
        ell, _ = oracle.pair_term(y, d, sigma, trunc)
        if trunc:
            ref = stats.truncnorm.logpdf(y, a=-d / sigma, b=np.inf, loc=d, scale=sigma)
        else:
            ref = stats.norm.logpdf(y, loc=d, scale=sigma)
        assert ell == pytest.approx(ref, rel=1e-12, abs=1e-13)


def test_pair_coef_is_minus_dell_dd_mpmath():
    """coef = -(d ell / d delta) -- the Eq. 6 chain rule factor -- against an
    mpmath derivative of the Eq. 1 truncated-normal log-density."""
    mp.mp.dps = 40
    rng = np.random.default_rng(2)

    def ell_mp(y, d, s):
        y, d, s = mp.mpf(y), mp.mpf(d), mp.mpf(s)
        Phi = 1 - mp.erfc(d / s / mp.sqrt(2)) / 2
        return -mp.log(2 * mp.pi * s * s) / 2 - (y - d) ** 2 / (2 * s * s) - mp.log(Phi)

    for _ in range(40):
        s = float(rng.uniform(0.3, 2.0))
        d = float(rng.uniform(0.01, 8.0) * s)
        y = float(rng.uniform(0.01, 10.0))
        _, coef = oracle.pair_term(y, d, s, 1)
        ref = -mp.diff(lambda dd: ell_mp(y, dd, s), d)
        assert coef == pytest.approx(float(ref), rel=1e-13, abs=1e-15)


def test_log_phi_vs_mpmath_and_tail():
    mp.mp.dps = 50
    for t in list(np.linspace(0, 8.3, 84)) + [10.0, 15.0, 20.0, 30.0]:
        ref = mp.log1p(-mp.erfc(mp.mpf(t) / mp.sqrt(2)) / 2)
        got = oracle.log_phi(t)
        assert abs(got - float(ref)) <= 2e-13 * abs(float(ref)) + 1e-300, t
    # survey App. A: log Phi(8.3) ~ -5.2055697448902853e-17 where log(Phi) rounds to 0
    ref83 = float(mp.log1p(-mp.erfc(mp.mpf("8.3") / mp.sqrt(2)) / 2))
    assert oracle.log_phi(8.3) == pytest.approx(ref83, rel=1e-12)
    assert oracle.log_phi(8.3) < 0.0


# ---------------------------------------------------------------- full sums
def test_triangle_345_T0_exact():
    g = json.load(open(GOLDEN))["triangle_345_T0"]
    x = np.array(g["x"])
    yp = np.array([g["y_lower"]["1,0"], g["y_lower"]["2,0"], g["y_lower"]["2,1"]])
    r = oracle.loglik_grad(yp, x, g["sigma"], g["truncation"])
    assert np.array_equal(r["grad"], np.array(g["grad"]))          # exact in binary
    ref = eval(g["loglik_formula"], {"log": math.log, "pi": math.pi})
    assert r["loglik"] == pytest.approx(ref, rel=1e-15)
    yf = np.full((3, 3), np.nan)
    yf[1, 0], yf[2, 0], yf[2, 1] = yp
    assert r["loglik"] == pytest.approx(scipy_loglik(yf, x, 2.0, 0), rel=1e-14)


def test_triangle_345_T1_vs_scipy_and_mpmath():
    x = np.array([[0.0, 0.0], [3.0, 0.0], [0.0, 4.0]])
    yf = np.full((3, 3), np.nan)
    yf[1, 0], yf[2, 0], yf[2, 1] = 2.5, 4.5, 5.0
    r = oracle.loglik_grad(oracle.pack_lower(yf), x, 2.0, 1)
    assert r["loglik"] == pytest.approx(scipy_loglik(yf, x, 2.0, 1), rel=1e-14)
    ll, g = mp_brute(yf, x, 2.0, 1)
    assert r["loglik"] == pytest.approx(ll, rel=1e-14)
    np.testing.assert_allclose(r["grad"], g, rtol=1e-13, atol=1e-16)


def test_two_point_mills_ratio():
    g = json.load(open(GOLDEN))["two_point_mills"]
    x = np.array(g["x"])
    r = oracle.loglik_grad(np.array([g["y"]]), x, g["sigma"], 1)
    mills = stats.norm.pdf(1.0) / stats.norm.cdf(1.0)
    assert r["grad"][0, 0] == pytest.approx(mills, rel=1e-14)
    assert r["grad"][0, 1] == 0.0
    np.testing.assert_array_equal(r["grad"][1], -r["grad"][0])


def mp_brute(y_full, x, sigma, truncation, dps=35):
    """mpmath brute force of Eq. 2 and Eq. 6 (tiny N only)."""
    mp.mp.dps = dps
    n, d = x.shape
    X = [[mp.mpf(float(v)) for v in row] for row in x]
    s = mp.mpf(sigma)
    L = mp.mpf(0)
    G = [[mp.mpf(0)] * d for _ in range(n)]
    for i in range(n):
        for j in range(n):
            yv = y_full[max(i, j), min(i, j)]     # lower triangle only (reading R9)
            if i == j or np.isnan(yv):
                continue
            y = mp.mpf(float(yv))
            diff = [X[i][k] - X[j][k] for k in range(d)]
            dist = mp.sqrt(sum(v * v for v in diff))
            t = dist / s
            Phi = 1 - mp.erfc(t / mp.sqrt(2)) / 2
            if i > j:
                L += -mp.log(2 * mp.pi * s * s) / 2 - (y - dist) ** 2 / (2 * s * s)
                if truncation:
                    L -= mp.log(Phi)
            c = (dist - y) / (s * s)
            if truncation:
                c += mp.exp(-t * t / 2) / mp.sqrt(2 * mp.pi) / (s * Phi)
            if dist > 0:
                for k in range(d):
                    G[i][k] -= c * diff[k] / dist
    return float(L), np.array([[float(v) for v in row] for row in G])


@pytest.mark.parametrize("n,d,missing", [(4, 2, 0.0), (6, 3, 0.2), (8, 2, 0.0), (7, 6, 0.3)])
def test_brute_force_mpmath(n, d, missing):
    rng = np.random.default_rng(10 + n)
    x, y = rand_instance(rng, n, d, sigma=0.7, missing=missing)
    for trunc in (0, 1):
        r = oracle.loglik_grad(oracle.pack_lower(y), x, 0.7, trunc)
        ll, g = mp_brute(y, x, 0.7, trunc)
        assert r["loglik"] == pytest.approx(ll, rel=1e-13, abs=1e-13)
        np.testing.assert_allclose(r["grad"], g, rtol=1e-12, atol=1e-13)


def test_missing_pair_drops_out():
    x = np.array([[0.0, 0.0], [3.0, 0.0], [0.0, 4.0]])
    yf = np.full((3, 3), np.nan)
    yf[1, 0], yf[2, 0] = 2.5, 4.5          # pair (2,1) missing
    r = oracle.loglik_grad(oracle.pack_lower(yf), x, 2.0, 1)
    assert r["n_obs"] == 2
    assert r["loglik"] == pytest.approx(scipy_loglik(yf, x, 2.0, 1), rel=1e-14)
    ll, g = mp_brute(yf, x, 2.0, 1)
    np.testing.assert_allclose(r["grad"], g, rtol=1e-13, atol=1e-16)


def test_all_missing_is_zero():
    rng = np.random.default_rng(3)
    x = rng.normal(size=(9, 2))
    r = oracle.loglik_grad(np.full(36, np.nan), x, 1.0, 1)
    assert r["loglik"] == 0.0 and r["n_obs"] == 0
    assert not r["grad"].any()


def test_coincident_observed_pair():
    """delta = 0 observed: likelihood term counts (log Phi(0) = -log 2), the
    gradient direction is zero, and the pair is counted (reading R10)."""
    x = np.array([[1.0, 2.0], [1.0, 2.0], [4.0, 6.0]])
    yf = np.full((3, 3), np.nan)
    yf[1, 0], yf[2, 0], yf[2, 1] = 0.5, 5.0, 5.0
    r = oracle.loglik_grad(oracle.pack_lower(yf), x, 1.0, 1)
    assert r["zero_pairs"] == 1
    assert r["loglik"] == pytest.approx(scipy_loglik(yf, x, 1.0, 1), rel=1e-14)
    r2 = oracle.loglik_grad(np.array([np.nan, 5.0, 5.0]), x, 1.0, 1)
    np.testing.assert_allclose(r["grad"], r2["grad"], rtol=0, atol=0)


@pytest.mark.parametrize("seed", range(6))
def test_gradient_matches_fd_of_scipy_loglik(seed):
    """Eq. 6 vs central differences (h=1e-5) of the scipy-built Eq. 2."""
    rng = np.random.default_rng(100 + seed)
    n, d = int(rng.integers(5, 12)), int(rng.choice([2, 3, 6]))
    x, y = rand_instance(rng, n, d, sigma=0.9, missing=0.1)
    r = oracle.loglik_grad(oracle.pack_lower(y), x, 0.9, 1)
    h = 1e-5
    fd = np.zeros_like(x)
    for i in range(n):
        for k in range(d):
            xp = x.copy(); xp[i, k] += h
            xm = x.copy(); xm[i, k] -= h
            fd[i, k] = (scipy_loglik(y, xp, 0.9) - scipy_loglik(y, xm, 0.9)) / (2 * h)
    err = np.abs(fd - r["grad"])
    assert np.all(err <= 1e-6 * np.maximum(np.abs(r["grad"]), 1.0)), err.max()


# ---------------------------------------------------------------- invariants
def _inst(seed=7, n=40, d=3, missing=0.1):
    rng = np.random.default_rng(seed)
    return rng, *rand_instance(rng, n, d, sigma=0.6, missing=missing)


def test_gradient_sums_to_zero():
    _, x, y = _inst()
    r = oracle.loglik_grad(oracle.pack_lower(y), x, 0.6, 1)
    assert np.all(np.abs(r["grad"].sum(0)) <= 1e-13 * r["absscale"].sum(0))


def test_translation_rotation_permutation_invariance():
    rng, x, y = _inst()
    base = oracle.loglik_grad(oracle.pack_lower(y), x, 0.6, 1)
    # translation: same loglik, same gradient
    sh = oracle.loglik_grad(oracle.pack_lower(y), x + np.array([5.0, -2.0, 0.5]), 0.6, 1)
    assert sh["loglik"] == pytest.approx(base["loglik"], rel=1e-13)
    np.testing.assert_allclose(sh["grad"], base["grad"], rtol=1e-8, atol=1e-10)
    # rotation: same loglik, gradient rotates
    qm, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    ro = oracle.loglik_grad(oracle.pack_lower(y), x @ qm.T, 0.6, 1)
    assert ro["loglik"] == pytest.approx(base["loglik"], rel=1e-13)
    np.testing.assert_allclose(ro["grad"], base["grad"] @ qm.T, rtol=1e-8, atol=1e-10)
    # permutation: rows permute
    perm = rng.permutation(x.shape[0])
    pe = oracle.loglik_grad(oracle.pack_lower(y[np.ix_(perm, perm)]), x[perm], 0.6, 1)
    assert pe["loglik"] == pytest.approx(base["loglik"], rel=1e-13)
    np.testing.assert_allclose(pe["grad"], base["grad"][perm], rtol=1e-9, atol=1e-11)


def test_scaling_identity():
    """ell(ay, ad; a sigma) = ell(y, d; sigma) - log a  =>  log L scales by
    -n_obs log a and the gradient by 1/a."""
    _, x, y = _inst(missing=0.2)
    a = 3.0
    b = oracle.loglik_grad(oracle.pack_lower(y), x, 0.6, 1)
    s = oracle.loglik_grad(oracle.pack_lower(a * y), a * x, a * 0.6, 1)
    assert s["loglik"] == pytest.approx(b["loglik"] - b["n_obs"] * math.log(a), rel=1e-13)
    np.testing.assert_allclose(s["grad"], b["grad"] / a, rtol=1e-9, atol=1e-12)


def test_grad_rows_agree_with_full():
    _, x, y = _inst(n=50, d=2)
    full = oracle.loglik_grad(oracle.pack_lower(y), x, 0.6, 1)
    rows = np.array([0, 7, 49, 23])
    yr = y[rows].copy()
    out = oracle.grad_rows(rows, yr, x, 0.6, 1)
    np.testing.assert_allclose(out["grad"], full["grad"][rows], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(out["absscale"], full["absscale"][rows], rtol=1e-12)
    # row shares of log L add up to the total
    allrows = oracle.grad_rows(np.arange(50), y, x, 0.6, 1)
    assert allrows["rowlik"].sum() == pytest.approx(full["loglik"], rel=1e-13)


def test_loglik_rows_streaming_pins():
    """The streaming row-range log L (used at C5, whose packed triangle is 40 GB):
    its chunks, added in row order, equal the scipy truncnorm/norm sum of Eq. 1
    densities over the same pairs, and each chunk is the scipy sum over its rows."""
    rng = np.random.default_rng(12)
    x, y = rand_instance(rng, 23, 3, sigma=0.7, missing=0.15)
    yp = oracle.pack_lower(y)
    for trunc in (0, 1):
        tot, nobs = 0.0, 0
        for i0, i1 in [(0, 1), (1, 5), (5, 6), (6, 17), (17, 23)]:
            lo, hi = i0 * (i0 - 1) // 2 if i0 else 0, i1 * (i1 - 1) // 2
            ll, no = oracle.loglik_rows(i0, i1, yp[lo:hi], x, 0.7, trunc)
            ych = np.full_like(y, np.nan)
            ych[i0:i1] = y[i0:i1]
            assert ll == pytest.approx(scipy_loglik(ych, x, 0.7, trunc), rel=1e-13, abs=1e-300)
            tot += ll
            nobs += no
        assert tot == pytest.approx(scipy_loglik(y, x, 0.7, trunc), rel=1e-13)
        assert nobs == int((~np.isnan(yp)).sum())


# ---------------------------------------------------------------- leapfrog
def test_leapfrog_gaussian_closed_form():
    """All-missing Y: target is the N(0, tau^2) prior; one leapfrog step is the
    textbook linear map x1 = (1-h2/2)x + eps p, p1 = -eps w2 (1-h2/4) x + (1-h2/2) p
    with w2 = 1/tau^2, h2 = eps^2 w2."""
    rng = np.random.default_rng(5)
    n, d, tau, eps = 6, 2, 1.7, 0.3
    x0, p0 = rng.normal(size=(n, d)), rng.normal(size=(n, d))
    out = oracle.leapfrog(np.full(n * (n - 1) // 2, np.nan), x0, p0, 1.0, eps, 1, prior_sd=tau)
    w2 = 1 / tau**2
    h2 = eps**2 * w2
    np.testing.assert_allclose(out["x"], (1 - h2 / 2) * x0 + eps * p0, rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(out["p"], -eps * w2 * (1 - h2 / 4) * x0 + (1 - h2 / 2) * p0,
                               rtol=1e-14, atol=1e-15)


def test_leapfrog_reversible_and_energy_scaling():
    rng, x, y = _inst(n=20, d=2, missing=0.0)
    yp = oracle.pack_lower(y)
    p0 = rng.normal(size=x.shape)
    fw = oracle.leapfrog(yp, x, p0, 0.6, 0.01, 10, prior_sd=5.0)
    bw = oracle.leapfrog(yp, fw["x"], -fw["p"], 0.6, 0.01, 10, prior_sd=5.0)
    np.testing.assert_allclose(bw["x"], x, atol=1e-8)
    np.testing.assert_allclose(-bw["p"], p0, atol=1e-8)
    # |dH| ~ eps^2 over a fixed trajectory length
    e1 = 0.004
    a = oracle.leapfrog(yp, x, p0, 0.6, e1, 20, prior_sd=5.0)
    b = oracle.leapfrog(yp, x, p0, 0.6, e1 / 2, 40, prior_sd=5.0)
    ratio = abs(a["H1"] - a["H0"]) / abs(b["H1"] - b["H0"])
    assert 3.5 <= ratio <= 4.5, ratio
