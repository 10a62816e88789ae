"""Pins for the oracle's cross-validated lpd (CPU only).

oracle.cv_lpd follows PAPER.md:381-395 (log pointwise predictive density of a
held-out fold, Monte Carlo over posterior draws; reading R29 drops the
posterior-density factor of the printed estimator).  Pinned against scipy's
truncated-normal log-density with scipy.special.logsumexp, and against the
identities S = 1 (lpd = held-out log-likelihood) and repeated draws.
"""
import math

import numpy as np
import pytest
from scipy import stats
from scipy.special import logsumexp

import oracle


def scipy_lpd(hi, hj, hy, xs, sigmas, trunc=1):
    tot = 0.0
    for q in range(len(hy)):
        ls = []
        for x, s in zip(xs, sigmas):
            d = float(np.linalg.norm(x[hi[q]] - x[hj[q]]))
            if trunc:
                ls.append(stats.truncnorm.logpdf(hy[q], a=-d / s, b=np.inf, loc=d, scale=s))
            else:
                ls.append(stats.norm.logpdf(hy[q], loc=d, scale=s))
        tot += logsumexp(ls) - math.log(len(ls))
    return tot


def fold(rng, n, m):
    pairs = set()
    while len(pairs) < m:
        i, j = rng.integers(0, n, size=2)
        if i != j:
            pairs.add((max(i, j), min(i, j)))
    hi, hj = np.array(sorted(pairs)).T
    return hi, hj


@pytest.mark.parametrize("trunc", [1, 0])
def test_cv_lpd_matches_scipy(trunc):
    rng = np.random.default_rng(trunc)
    n, d, S, m = 15, 2, 6, 20
    hi, hj = fold(rng, n, m)
    hy = np.abs(rng.normal(1.5, 0.7, size=m))
    xs = rng.normal(size=(S, n, d))
    sig = 0.5 + rng.random(S)
    got = oracle.cv_lpd(hi, hj, hy, xs, sig, trunc)
    assert got == pytest.approx(scipy_lpd(hi, hj, hy, xs, sig, trunc), rel=1e-12)


def test_cv_lpd_identities():
    rng = np.random.default_rng(7)
    n, d, m = 12, 3, 15
    hi, hj = fold(rng, n, m)
    hy = np.abs(rng.normal(1.0, 0.5, size=m))
    x = rng.normal(size=(1, n, d))
    # S = 1: the held-out log-likelihood (sum of Eq. 2 terms)
    ll = sum(oracle.pair_term(hy[q], float(np.linalg.norm(x[0, hi[q]] - x[0, hj[q]])), 0.8, 1)[0]
             for q in range(m))
    assert oracle.cv_lpd(hi, hj, hy, x, [0.8]) == pytest.approx(ll, rel=1e-14)
    # S identical draws average to the same value
    assert oracle.cv_lpd(hi, hj, hy, np.repeat(x, 5, axis=0), [0.8] * 5) == pytest.approx(ll, rel=1e-14)
    # far-apart draw values: the max shift keeps it finite (naive exp underflows)
    xs = np.concatenate([x, x * 200.0])
    v = oracle.cv_lpd(hi, hj, hy, xs, [0.8, 0.8])
    assert np.isfinite(v) and v == pytest.approx(ll - m * math.log(2), rel=1e-12)
