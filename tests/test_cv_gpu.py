"""GPU parity of the cross-validated lpd
against the CPU oracle, through the C-ABI.  fp64 tolerance 1e-10 relative
(as log L): the lpd is a sum of m log-mean-exp terms of Eq. 2 values."""
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


def split_fold(w, frac, seed):
    """Hold out a random fraction of the observed pairs of w: (train_packed, hi, hj, hy)."""
    y = w.y_packed()
    rng = np.random.default_rng(seed)
    obs = np.flatnonzero(~np.isnan(y))
    held = np.sort(rng.choice(obs, size=int(frac * obs.size), replace=False))
    i = np.floor((1 + np.sqrt(1 + 8 * held.astype(np.float64))) / 2).astype(np.int64)
    i -= (i * (i - 1) // 2 > held)
    j = held - i * (i - 1) // 2
    train = y.copy()
    train[held] = np.nan
    return train, i, j, y[held]


@pytest.mark.parametrize("n,d,trunc,S", [(500, 2, 1, 8), (1000, 6, 1, 5), (300, 3, 0, 4)])
def test_cv_lpd_parity(mds, n, d, trunc, S):
    w = workload.Workload(n, d, p_missing=0.05, seed=n)
    train, hi, hj, hy = split_fold(w, 0.2, seed=n + 1)
    assert np.all(hi > hj)
    rng = np.random.default_rng(3)
    xs = np.stack([w.x0 + 0.02 * rng.normal(size=w.x0.shape) for _ in range(S)])
    sig = w.sigma * (1 + 0.1 * rng.random(S))
    with mds.MDS(n, d, "f64", bool(trunc)) as c:
        c.set_dissimilarities_packed(train)
        c.cv_set_heldout(hi, hj, hy)
        for s in range(S):
            c.set_locations(xs[s])
            c.set_sigma(sig[s])
            c.cv_accumulate()
        lpd, draws = c.cv_lpd()
        # training log L excludes the held-out pairs
        ll = c.log_likelihood()
    assert draws == S
    ref = oracle.cv_lpd(hi, hj, hy, xs, sig, trunc)
    assert lpd == pytest.approx(ref, rel=1e-10)
    assert ll == pytest.approx(oracle.loglik_grad(train, xs[-1], sig[-1], trunc)["loglik"], rel=1e-10)


def test_cv_state_and_errors(mds):
    w = workload.Workload(100, 2, seed=2)
    with mds.MDS(100, 2) as c:
        with pytest.raises(mds.MDSError) as e:
            c.cv_accumulate()
        assert e.value.status == 2
        with pytest.raises(mds.MDSError):
            c.cv_set_heldout([3], [3], [1.0])              # diagonal
        with pytest.raises(mds.MDSError):
            c.cv_set_heldout([3], [100], [1.0])            # out of range
        with pytest.raises(mds.MDSError):
            c.cv_set_heldout([3], [1], [-1.0])             # y < 0
        c.cv_set_heldout([5, 9], [1, 2], [0.7, 1.1])
        with pytest.raises(mds.MDSError):
            c.cv_lpd()                                     # no draw yet
        c.set_locations(w.x0)
        c.set_sigma(w.sigma)
        c.cv_accumulate()
        lpd, s = c.cv_lpd()
        assert s == 1 and np.isfinite(lpd)
        ref = sum(oracle.pair_term(yy, float(np.linalg.norm(w.x0[i] - w.x0[j])), w.sigma, 1)[0]
                  for i, j, yy in ((5, 1, 0.7), (9, 2, 1.1)))
        assert lpd == pytest.approx(ref, rel=1e-13)
        c.cv_set_heldout([], [], [])                       # empty fold
        c.cv_accumulate()
        assert c.cv_lpd() == (0.0, 1)
