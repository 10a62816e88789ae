"""GPU parity of the single-location updates (
PAPER.md:258-263) against the CPU oracle, through the C-ABI.

Row delta: fp64 within 1e-10 relative of the row's log-likelihood scale
(sum over its terms of |ell|, as log L's own 1e-10 relative tolerance) --
the delta is a difference of two sums of N - 1 terms.  Sweep: each update's
decision is taken in fp64 on both sides; with the caller's uniforms the whole
chain must match the oracle's (X within 1e-12, same acceptance count).
"""
import numpy as np
import pytest

import oracle
import workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mds():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1905_04582_b200 as m
    return m


def row_scale(y, x, i, sigma, trunc):
    # |ell| summed over row i's terms: the conditioning scale of the delta
    n = x.shape[0]
    s = 0.0
    for j in range(n):
        if j == i:
            continue
        a, b = max(i, j), min(i, j)
        yy = y[a * (a - 1) // 2 + b]
        if np.isnan(yy):
            continue
        s += abs(oracle.pair_term(yy, float(np.linalg.norm(x[i] - x[j])), sigma, trunc)[0])
    return s


@pytest.mark.parametrize("n,d,pm,trunc", [(64, 2, 0.0, 1), (1000, 3, 0.1, 1), (777, 6, 0.0, 0), (2, 1, 0.0, 1),
                                          (5392, 2, 0.0, 1)])
def test_row_delta(mds, n, d, pm, trunc):
    w = workload.Workload(n, d, p_missing=pm, seed=n + 3)
    y, x = w.y_packed(), w.x0
    rng = np.random.default_rng(n)
    with mds.MDS(n, d, "f64", bool(trunc)) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(x)
        c.set_sigma(w.sigma)
        for i in sorted({0, n - 1, n // 2, min(63, n - 1), min(64, n - 1)}):
            xn = x[i] + rng.normal(size=d) * 0.2
            got = c.row_loglik_delta(i, xn)
            ref = oracle.row_delta(y, x, i, xn, w.sigma, trunc)
            tol = 1e-10 * max(row_scale(y, x, i, w.sigma, trunc), 1e-300) if n <= 1000 else 1e-10 * abs(ref) + 1e-6
            assert abs(got - ref) <= tol, (i, got, ref)
            assert c.row_loglik_delta(i, x[i]) == 0.0      # no move: every term cancels exactly


def test_row_delta_f32(mds):
    w = workload.Workload(500, 2, p_missing=0.1, seed=5)
    y32 = w.y_packed().astype(np.float32).astype(np.float64)
    x32 = w.x0.astype(np.float32).astype(np.float64)
    with mds.MDS(500, 2, "f32") as c:
        c.set_dissimilarities_packed(y32)
        c.set_locations(x32)
        c.set_sigma(w.sigma)
        xn = x32[7] + 0.3
        got = c.row_loglik_delta(7, xn)
    ref = oracle.row_delta(y32, x32, 7, xn, w.sigma, 1)
    assert abs(got - ref) <= 1e-4 * row_scale(y32, x32, 7, w.sigma, 1)


def test_rw_sweep_matches_oracle_chain(mds):
    n, d = 600, 2
    w = workload.Workload(n, d, p_missing=0.05, seed=41)
    y, x = w.y_packed(), w.x0
    rng = np.random.default_rng(8)
    k = 400
    rows = rng.integers(0, n, size=k)
    z = rng.normal(size=(k, d))
    u = 1.0 - rng.random(k)
    step = 0.05
    ref_x, ref_acc = oracle.rw_sweep(y, x, w.sigma, rows, z, u, step, prior_sd=10.0)
    with mds.MDS(n, d) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(x)
        c.set_sigma(w.sigma)
        acc = c.rw_sweep(rows, z, u, step, prior_sd=10.0)
        xs = c.get_locations()
        ll = c.log_likelihood()        # cache invalidated: a fresh pass at the new X
    assert acc == ref_acc and 0 < acc < k
    np.testing.assert_allclose(xs, ref_x, rtol=0, atol=1e-12)
    assert ll == pytest.approx(oracle.loglik_grad(y, ref_x, w.sigma, 1)["loglik"], rel=1e-10)


def test_rw_sweep_errors(mds):
    w = workload.Workload(50, 2, seed=1)
    with mds.MDS(50, 2) as c:
        c.set_dissimilarities_packed(w.y_packed())
        c.set_locations(w.x0)
        c.set_sigma(w.sigma)
        with pytest.raises(mds.MDSError):
            c.rw_sweep(np.array([50]), np.zeros((1, 2)), np.array([0.5]), 0.1)
        with pytest.raises(mds.MDSError):
            c.rw_sweep(np.array([1]), np.zeros((1, 2)), np.array([0.0]), 0.1)
        with pytest.raises(mds.MDSError):
            c.row_loglik_delta(-1, np.zeros(2))
        assert c.rw_sweep(np.zeros(0, dtype=np.int64), np.zeros((0, 2)), np.zeros(0), 0.1) == 0
    with mds.MDS(50, 2, rank=0, world=2) as c:
        # sharded without an exchange (no communicator, no callback): not ready
        c.set_dissimilarities_packed(w.y_packed())
        c.set_locations(w.x0)
        c.set_sigma(w.sigma)
        with pytest.raises(mds.MDSError) as e:
            c.row_loglik_delta(0, np.zeros(2))
        assert e.value.status == 2
