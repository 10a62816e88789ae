"""Pins for the oracle's single-location updates (CPU only).

oracle.row_delta / oracle.rw_sweep follow PAPER.md:258-263 (a single x_i
invalidates only N - 1 terms; the random-walk sampler of Bedford et al.).
Pinned against scipy-built full log-likelihood differences, the move-back
identity, and the stationary law of the sweep when Y carries no information.
"""
import math

import numpy as np
import pytest

import oracle
from tests.test_oracle_pins import rand_instance, scipy_loglik


@pytest.mark.parametrize("trunc,missing", [(1, 0.0), (1, 0.3), (0, 0.1)])
def test_row_delta_is_full_loglik_difference(trunc, missing):
    rng = np.random.default_rng(20 + trunc)
    x, y = rand_instance(rng, 10, 2, sigma=0.8, missing=missing)
    yp = oracle.pack_lower(y)
    for i in (0, 4, 9):
        xn = x[i] + rng.normal(size=2) * 0.4
        x2 = x.copy()
        x2[i] = xn
        ref = scipy_loglik(y, x2, 0.8, trunc) - scipy_loglik(y, x, 0.8, trunc)
        assert oracle.row_delta(yp, x, i, xn, 0.8, trunc) == pytest.approx(ref, rel=1e-10, abs=1e-12)


def test_row_delta_identities():
    rng = np.random.default_rng(2)
    x, y = rand_instance(rng, 15, 3, sigma=1.0)
    yp = oracle.pack_lower(y)
    i = 6
    assert oracle.row_delta(yp, x, i, x[i], 1.0) == 0.0          # no move, no change
    xn = x[i] + 0.3
    x2 = x.copy()
    x2[i] = xn
    fwd = oracle.row_delta(yp, x, i, xn, 1.0)
    back = oracle.row_delta(yp, x2, i, x[i], 1.0)
    assert fwd == pytest.approx(-back, rel=1e-13)


def test_rw_sweep_rule_against_row_delta():
    """Each update accepts exactly when log u < Delta + Delta log prior."""
    rng = np.random.default_rng(9)
    x, y = rand_instance(rng, 12, 2, sigma=0.7)
    yp = oracle.pack_lower(y)
    k = 40
    rows = rng.integers(0, 12, size=k)
    z = rng.normal(size=(k, 2))
    u = 1.0 - rng.random(k)
    xs, acc = oracle.rw_sweep(yp, x, 0.7, rows, z, u, 0.2, prior_sd=3.0)
    xr = x.copy()
    na = 0
    for q in range(k):
        i = rows[q]
        xn = xr[i] + 0.2 * z[q]
        lr = oracle.row_delta(yp, xr, i, xn, 0.7) - (xn @ xn - xr[i] @ xr[i]) / (2 * 9.0)
        if math.log(u[q]) < lr:
            xr[i] = xn
            na += 1
    assert acc == na and np.array_equal(xs, xr)


def test_rw_sweep_prior_only_stationarity():
    """All pairs missing: the sweep samples the iid N(0, tau^2) prior."""
    n, d, tau = 5, 2, 1.5
    y = np.full(n * (n - 1) // 2, np.nan)
    rng = np.random.default_rng(4)
    x = np.zeros((n, d))
    samples = []
    for blk in range(300):
        k = 200
        x, _ = oracle.rw_sweep(y, x, 1.0, rng.integers(0, n, size=k), rng.normal(size=(k, d)),
                               1.0 - rng.random(k), 2.0, prior_sd=tau)
        if blk >= 20:
            samples.append(x.copy())
    s = np.stack(samples)
    assert abs(s.mean()) < 0.1
    assert abs(s.var() / tau ** 2 - 1) < 0.1
