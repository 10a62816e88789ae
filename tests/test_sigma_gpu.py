"""GPU parity of the sigma side and the gradient-only leapfrog steps
 against the CPU oracle, through the C-ABI.

Tolerances as tests/test_parity_gpu.py (north_star): fp64 log L within 1e-10
relative; X after a trajectory within 1e-9 relative.  The MH decision is
taken on both sides in fp64 from log r; the test's uniforms stay well away
from the boundary so the same decision is required.
"""
import math

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


@pytest.mark.parametrize("n,d,pm,trunc,prec", [
    (64, 2, 0.0, 1, "f64"), (700, 3, 0.1, 1, "f64"), (1000, 6, 0.0, 0, "f64"), (333, 2, 0.2, 1, "f32"),
])
def test_loglik_at_sigma(mds, n, d, pm, trunc, prec):
    w = workload.Workload(n, d, p_missing=pm, seed=n + 7)
    y, x = w.y_packed(), w.x0
    with mds.MDS(n, d, prec, bool(trunc)) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(x)
        c.set_sigma(w.sigma)
        ll0, g0 = c.log_likelihood_and_gradient()
        for s in (0.3 * w.sigma, w.sigma, 2.5 * w.sigma):
            got = c.log_likelihood_at_sigma(s)
            if prec == "f64":
                ref = oracle.loglik_grad(y, x, s, trunc, want_absscale=False)["loglik"]
                assert got == pytest.approx(ref, rel=1e-10), s
            else:
                y32 = y.astype(np.float32).astype(np.float64)
                x32 = x.astype(np.float32).astype(np.float64)
                ref = oracle.loglik_grad(y32, x32, s, trunc, want_absscale=False)["loglik"]
                assert got == pytest.approx(ref, rel=1e-4), s
        # the context's sigma and cached result are untouched
        ll1, g1 = c.log_likelihood_and_gradient()
        assert ll1 == ll0 and np.array_equal(g0, g1)


def test_sigma_mh_steps_match_oracle(mds):
    w = workload.Workload(500, 2, p_missing=0.05, seed=12)
    y, x = w.y_packed(), w.x0
    shape, rate, step = 2.0, 0.5, 0.05
    rng = np.random.default_rng(1)
    sigma_ref = 1.3 * w.sigma          # start off the mode so both outcomes occur
    n_acc = 0
    with mds.MDS(500, 2) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(x)
        c.set_sigma(sigma_ref)
        for k in range(12):
            z = rng.normal()
            u = 1.0 - rng.random()
            ref = oracle.sigma_mh_step(y, x, sigma_ref, shape, rate, step, z, u)
            acc, lr = c.sigma_mh_step(shape, rate, step, z, u)
            scale = abs(oracle.loglik_grad(y, x, sigma_ref, 1, want_absscale=False)["loglik"])
            assert lr == pytest.approx(ref["log_ratio"], abs=1e-10 * scale), k
            if abs(math.log(u) - ref["log_ratio"]) > 1e-6 * scale:
                assert acc == ref["accepted"], k
            sigma_ref = ref["sigma"]
            n_acc += acc
        # the context's sigma moved with the chain: its log L is the oracle's at sigma_ref
        ll, _ = c.log_likelihood_and_gradient()
    assert ll == pytest.approx(oracle.loglik_grad(y, x, sigma_ref, 1)["loglik"], rel=1e-10)
    assert 0 < n_acc < 12


def test_sigma_mh_errors(mds):
    w = workload.Workload(100, 2, seed=3)
    with mds.MDS(100, 2) as c:
        c.set_dissimilarities_packed(w.y_packed())
        c.set_locations(w.x0)
        with pytest.raises(mds.MDSError) as e:
            c.sigma_mh_step(2.0, 1.0, 0.1, 0.0, 0.5)           # sigma not set
        assert e.value.status == 2
        c.set_sigma(w.sigma)
        for bad in ((0.0, 1.0, 0.1, 0.0, 0.5), (2.0, -1.0, 0.1, 0.0, 0.5), (2.0, 1.0, 0.0, 0.0, 0.5),
                    (2.0, 1.0, 0.1, float("nan"), 0.5), (2.0, 1.0, 0.1, 0.0, 0.0), (2.0, 1.0, 0.1, 0.0, 1.5)):
            with pytest.raises(mds.MDSError) as e:
                c.sigma_mh_step(*bad)
            assert e.value.status == 1
        with pytest.raises(mds.MDSError):
            c.log_likelihood_at_sigma(-1.0)
        assert np.isfinite(c.log_likelihood())


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_leapfrog_device_gradient_only_steps(mds, prec):
    """L = 7 device-resident leapfrog steps: steps 1..6 run the gradient-only
    pass, step 7 the full one; X, p and log L at the end vs the oracle."""
    import torch
    n, d = 400, 3
    w = workload.Workload(n, d, p_missing=0.1, seed=17)
    y, x = w.y_packed(), w.x0
    p0 = w.normals(3, (n, d))
    eps, L = 0.002, 7
    if prec == "f32":
        y = y.astype(np.float32).astype(np.float64)
        x = x.astype(np.float32).astype(np.float64)
    ref = oracle.leapfrog(y, x, p0, w.sigma, eps, L, 1, prior_sd=5.0)
    with mds.MDS(n, d, prec) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(x)
        c.set_sigma(w.sigma)
        c.leapfrog_device(L, eps, 5.0, p0_dev=torch.from_numpy(p0).cuda())
        xs, ps = c.get_locations(), c.get_momentum()
        ll = c.log_likelihood()
    if prec == "f64":
        np.testing.assert_allclose(xs, ref["x"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(ps, ref["p"], rtol=1e-9, atol=1e-10)
        assert ll == pytest.approx(ref["loglik"], rel=1e-10)
    else:
        np.testing.assert_allclose(xs, ref["x"], rtol=1e-5, atol=1e-7)
        assert ll == pytest.approx(ref["loglik"], rel=1e-4)


def test_mcmc_run_c1_chain(mds):
    """PAPER.md:672's sampler (HMC on X, then MH on sigma^2): the final state is
    consistent with the oracle (log L at the final X and sigma)."""
    w = workload.config("C1")
    y = w.y_packed()
    with mds.MDS(w.n, w.d) as c:
        c.set_dissimilarities_packed(y)
        c.set_sigma(w.sigma)
        x, st = c.mcmc_run(40, 10, 0.01, 10.0, 7, 2.0, 0.5, 0.1, x0=w.x0)
        ll = c.log_likelihood()
    assert st["grad_evals"] == 400
    assert 0 < st["accepted_x"] <= 40 and 0 < st["accepted_sigma"] < 40
    ref = oracle.loglik_grad(y, x, st["final_sigma"], 1)["loglik"]
    assert st["final_loglik"] == pytest.approx(ref, rel=1e-10)
    assert ll == pytest.approx(ref, rel=1e-10)


def test_mcmc_run_prior_only_sigma(mds):
    """All pairs missing: log L = 0, so sigma^-2 must follow its Gamma(shape, rate) prior."""
    n, d = 20, 2
    shape, rate = 3.0, 2.0
    y = np.full(n * (n - 1) // 2, np.nan)
    taus = []
    with mds.MDS(n, d) as c:
        c.set_dissimilarities_packed(y)
        c.set_sigma(1.0)
        x = np.random.default_rng(0).normal(size=(n, d))
        for k in range(60):
            x, st = c.mcmc_run(25, 3, 0.5, 2.0, 100 + k, shape, rate, 1.0, x0=x)
            if k >= 5:
                taus.append(1.0 / st["final_sigma"] ** 2)
    t = np.array(taus)
    mean, var = shape / rate, shape / rate ** 2
    assert abs(t.mean() - mean) < 4 * math.sqrt(var / t.size), (t.mean(), mean)
    assert 0.6 < t.var() / var < 1.5
