"""Pins for the oracle's sigma^2 update (CPU only).

oracle.sigma_mh_step follows PAPER.md:205-210 (sigma^-2 ~ Gamma(s_0, r_0)) and
the per-iteration sigma^2 update of PAPER.md:672 as a random walk on
log sigma^2 (reading R27).  Pinned against scipy's truncated-normal and gamma
log-densities (the log acceptance ratio) and against the stationary law of
the chain when Y carries no information (the Gamma prior itself).
"""
import math

import numpy as np
import pytest
from scipy import stats

import oracle
from tests.test_oracle_pins import rand_instance, scipy_loglik


def scipy_log_ratio(y_full, x, sigma0, sigma1, shape, rate, trunc=1):
    """log L(sigma1) - log L(sigma0) + log p(phi1) - log p(phi0), with the
    density of phi = log sigma^2 obtained from scipy's Gamma density of
    tau = 1/sigma^2 = e^-phi times |dtau/dphi| = tau."""
    def lprior(s):
        tau = 1.0 / (s * s)
        return stats.gamma.logpdf(tau, a=shape, scale=1.0 / rate) + math.log(tau)
    return (scipy_loglik(y_full, x, sigma1, trunc) - scipy_loglik(y_full, x, sigma0, trunc)
            + lprior(sigma1) - lprior(sigma0))


@pytest.mark.parametrize("trunc", [1, 0])
def test_log_ratio_matches_scipy(trunc):
    rng = np.random.default_rng(11)
    x, y = rand_instance(rng, 12, 2, sigma=0.7, missing=0.2)
    yp = oracle.pack_lower(y)
    sigma, shape, rate, step = 0.7, 2.0, 0.5, 0.3
    for z in (-1.3, 0.2, 2.1):
        out = oracle.sigma_mh_step(yp, x, sigma, shape, rate, step, z, 0.5, trunc)
        s1 = math.exp(0.5 * (math.log(sigma * sigma) + step * z))
        ref = scipy_log_ratio(y, x, sigma, s1, shape, rate, trunc)
        assert out["log_ratio"] == pytest.approx(ref, rel=1e-11, abs=1e-11)
        assert out["accepted"] == (math.log(0.5) < ref)
        assert out["sigma"] == (s1 if out["accepted"] else sigma)


def test_accept_reject_rule():
    rng = np.random.default_rng(3)
    x, y = rand_instance(rng, 8, 2, sigma=1.0)
    yp = oracle.pack_lower(y)
    out = oracle.sigma_mh_step(yp, x, 1.0, 2.0, 1.0, 0.2, 0.7, 1.0)
    lr = out["log_ratio"]
    # u = 1 accepts iff log r > 0; u just below / above e^{log r} decides exactly
    assert out["accepted"] == (lr > 0)
    if lr < 0:
        assert oracle.sigma_mh_step(yp, x, 1.0, 2.0, 1.0, 0.2, 0.7, math.exp(lr) * 0.999)["accepted"]
        assert not oracle.sigma_mh_step(yp, x, 1.0, 2.0, 1.0, 0.2, 0.7, math.exp(lr) * 1.001)["accepted"]


def test_prior_only_chain_samples_gamma():
    """All pairs missing: log L = 0, so the chain's tau = 1/sigma^2 must follow
    Gamma(shape, rate).  A dropped Jacobian would give Gamma(shape - 1, rate)
    (mean 1/rate instead of 2/rate here)."""
    n = 2
    y = np.array([np.nan])
    x = np.zeros((n, 1))
    shape, rate = 2.0, 1.5
    rng = np.random.default_rng(5)
    sigma = 1.0
    taus = []
    for k in range(40000):
        out = oracle.sigma_mh_step(y, x, sigma, shape, rate, 1.2, rng.normal(), 1.0 - rng.random())
        sigma = out["sigma"]
        if k >= 2000 and k % 10 == 0:
            taus.append(1.0 / sigma ** 2)
    t = np.array(taus)
    mean, var = shape / rate, shape / rate ** 2
    se = math.sqrt(var / (t.size / 3.0))          # ~3x inflation for residual autocorrelation
    assert abs(t.mean() - mean) < 4 * se, (t.mean(), mean)
    assert abs(t.var() / var - 1) < 0.15
