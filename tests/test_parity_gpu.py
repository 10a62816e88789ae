"""GPU parity: libmds (through the C-ABI) vs the CPU oracle, element by element.

Tolerances (BASELINE.json north_star):
  fp64: log L within 1e-10 relative; every gradient entry within 1e-9 relative
        or 1e-12 absolute.
  fp32: against the oracle on fp32-ROUNDED X and Y (reading R15), log L within
        1e-4 relative, ||dg||/||g|| <= 1e-4 and |dg_ik| <= 1e-4|g_ik| + 1e-6 S_ik
        (reading R17; S_ik = sum_j |v_ijk|, the conditioning scale).
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


def run_gpu(m, n, d, y_packed, x, sigma, trunc=1, prec="f64", world=1):
    """Evaluate through the C-ABI; for world > 1, emulate the shards on one GPU
    and combine the partials with mds_combine_partials_device."""
    if world == 1:
        with m.MDS(n, d, prec, bool(trunc)) as ctx:
            ctx.set_dissimilarities_packed(y_packed)
            ctx.set_locations(x)
            ctx.set_sigma(sigma)
            ll, g = ctx.log_likelihood_and_gradient()
            return ll, g
    import torch
    parts = []
    ctxs = [m.MDS(n, d, prec, bool(trunc), rank=r, world=world) for r in range(world)]
    for c in ctxs:
        c.set_dissimilarities_packed(y_packed)
        c.set_locations(x)
        c.set_sigma(sigma)
        p = torch.zeros(n * d + 1, dtype=torch.float64, device="cuda")
        c.evaluate_partial_device(p)
        parts.append(p)
    gathered = torch.stack(parts).contiguous()
    outs = []
    for c in ctxs:
        ll = torch.zeros(1, dtype=torch.float64, device="cuda")
        g = torch.zeros(n * d, dtype=torch.float64, device="cuda")
        c.combine_partials_device(gathered, world, ll, g)
        torch.cuda.synchronize()
        outs.append((float(ll.item()), g.cpu().numpy().reshape(n, d)))
    for c in ctxs:
        c.close()
    for o in outs[1:]:
        assert o[0] == outs[0][0] and np.array_equal(o[1], outs[0][1])   # bitwise identical on all ranks
    return outs[0]


def assert_fp64_parity(ll, g, ref, tag=""):
    rl = ref["loglik"]
    assert abs(ll - rl) <= 1e-10 * abs(rl) + 1e-300, (tag, ll, rl)
    G = ref["grad"]
    err = np.abs(g - G)
    tol = np.maximum(1e-9 * np.abs(G), 1e-12)
    bad = err > tol
    if bad.any():
        k = np.argmax(err / tol)
        S = ref["absscale"].ravel()[k]
        raise AssertionError("%s: %d entries off; worst |d|=%.3e g=%.3e |d|/(u S)=%.2f"
                             % (tag, bad.sum(), err.ravel()[k], G.ravel()[k], err.ravel()[k] / (2.2e-16 * S)))


def instance(n, d, p_missing=0.0, seed=1, kind="clustered"):
    w = workload.Workload(n, d, kind=kind, p_missing=p_missing, seed=seed)
    return w, w.y_packed(), w.x0


# ------------------------------------------------------------------ configs
def test_c1_parity(mds):
    w = workload.config("C1")
    y = w.y_packed()
    ref = oracle.loglik_grad(y, w.x0, w.sigma, 1)
    ll, g = run_gpu(mds, w.n, w.d, y, w.x0, w.sigma)
    assert_fp64_parity(ll, g, ref, "C1")


@pytest.mark.parametrize("n,d,pm,trunc", [
    (2, 2, 0.0, 1), (3, 1, 0.0, 1), (63, 2, 0.0, 1), (65, 3, 0.1, 1), (129, 2, 0.0, 0),
    (200, 6, 0.1, 1), (257, 8, 0.3, 1), (500, 4, 0.0, 0), (1000, 2, 0.05, 1), (777, 5, 0.0, 1),
    (130, 7, 1.0, 1),
])
def test_ragged_sizes_parity(mds, n, d, pm, trunc):
    w, y, x = instance(n, d, pm, seed=n + d)
    ref = oracle.loglik_grad(y, x, w.sigma, trunc)
    ll, g = run_gpu(mds, n, d, y, x, w.sigma, trunc)
    if pm == 1.0:
        assert ll == 0.0 and not g.any()
    else:
        assert_fp64_parity(ll, g, ref, "n=%d d=%d" % (n, d))


def test_c2_full_parity(mds):
    w = workload.config("C2")
    y = w.y_packed()
    ref = oracle.loglik_grad(y, w.x0, w.sigma, 1)
    ll, g = run_gpu(mds, w.n, w.d, y, w.x0, w.sigma)
    assert_fp64_parity(ll, g, ref, "C2")


def test_gaussian_workload_parity(mds):
    w, y, x = instance(3000, 2, 0.0, seed=9, kind="gaussian")
    ref = oracle.loglik_grad(y, x, w.sigma, 1)
    ll, g = run_gpu(mds, w.n, w.d, y, x, w.sigma)
    assert_fp64_parity(ll, g, ref, "gaussian")


def test_sharded_equals_oracle(mds):
    w, y, x = instance(700, 3, 0.1, seed=21)
    ref = oracle.loglik_grad(y, x, w.sigma, 1)
    for world in (2, 3, 8, 16):
        ll, g = run_gpu(mds, w.n, w.d, y, x, w.sigma, world=world)
        assert_fp64_parity(ll, g, ref, "world=%d" % world)


def test_c4_full_size_sampled_rows(mds):
    """C4 at full size (N=30000, D=6, 10% missing), fp64: sampled gradient rows
    against the per-row oracle, and the total log L against the full oracle."""
    w = workload.config("C4")
    y = w.y_packed()
    ll, g = run_gpu(mds, w.n, w.d, y, w.x0, w.sigma)
    rows = np.array([0, 1, 63, 64, 4095, 12345, 29936, 29999])
    ref = oracle.grad_rows(rows, w.y_full_rows(rows), w.x0, w.sigma, 1)
    err = np.abs(g[rows] - ref["grad"])
    assert np.all(err <= np.maximum(1e-9 * np.abs(ref["grad"]), 1e-12)), err.max()
    # gradient rows sum to zero (antisymmetric pair contributions)
    assert np.all(np.abs(g.sum(0)) <= 1e-12 * np.abs(g).sum(0))
    full = oracle.loglik_grad(y, w.x0, w.sigma, 1, want_absscale=False)
    assert abs(ll - full["loglik"]) <= 1e-10 * abs(full["loglik"])


# ------------------------------------------------------------------ special cases
def test_triangle_345_golden(mds):
    import json, os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))["triangle_345_T0"]
    x = np.array(gold["x"])
    y = np.array([gold["y_lower"]["1,0"], gold["y_lower"]["2,0"], gold["y_lower"]["2,1"]])
    ll, g = run_gpu(mds, 3, 2, y, x, gold["sigma"], 0)
    G = np.array(gold["grad"])
    # the exact binary values within 2 ulp of the terms they are summed from
    # (S = sum_j |v_ijk|; entries that are exactly 0 are sums of +-rounded terms)
    # nonzero exact values within 2 ulp; the exact zeros within 1e-15 (the device's
    # d_21 = 5(1 + O(eps)) turns c_21 = (d - y)/sigma^2 = 0 into O(eps)/sigma^2)
    nz = G != 0
    assert np.all(np.abs(g - G)[nz] <= 2 * np.spacing(np.abs(G[nz])))
    assert np.all(np.abs(g[~nz]) <= 1e-15)
    ref = eval(gold["loglik_formula"], {"log": math.log, "pi": math.pi})
    assert ll == pytest.approx(ref, rel=1e-14)
    # T = 1 on the same triangle vs the oracle
    ll1, g1 = run_gpu(mds, 3, 2, y, x, gold["sigma"], 1)
    assert_fp64_parity(ll1, g1, oracle.loglik_grad(y, x, gold["sigma"], 1), "345 T1")


def test_coincident_points_and_zero_y(mds):
    rng = np.random.default_rng(4)
    x = rng.normal(size=(90, 2))
    x[10] = x[3]
    x[50] = x[3]
    full = np.abs(rng.normal(1.0, 0.5, size=(90, 90)))
    full[5, 2] = 0.0
    y = oracle.pack_lower(full)
    ref = oracle.loglik_grad(y, x, 0.7, 1)
    assert ref["zero_pairs"] == 3
    with mds.MDS(90, 2) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(x)
        c.set_sigma(0.7)
        ll, g = c.log_likelihood_and_gradient()
        assert c.zero_distance_pairs() == 3
        assert c.observed_pairs() == ref["n_obs"]
    assert_fp64_parity(ll, g, ref, "coincident")


def test_tail_and_extreme_sigma(mds):
    """Large t (the log Phi tail underflows), tiny and large sigma."""
    for sigma in (0.05, 0.6, 40.0):
        w, y, x = instance(300, 2, 0.0, seed=77)
        x = x * 3.0
        ref = oracle.loglik_grad(y, x, sigma, 1)
        ll, g = run_gpu(mds, 300, 2, y, x, sigma)
        assert_fp64_parity(ll, g, ref, "sigma=%g" % sigma)


def test_deterministic_bitwise(mds):
    w, y, x = instance(1500, 3, 0.05, seed=5)
    with mds.MDS(1500, 3) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(x)
        c.set_sigma(w.sigma)
        a = c.log_likelihood_and_gradient()
        c.set_sigma(w.sigma)          # bump version -> recompute
        b = c.log_likelihood_and_gradient()
    assert a[0] == b[0] and np.array_equal(a[1], b[1])


def test_full_matrix_setter_matches_packed(mds):
    w, y, x = instance(333, 2, 0.1, seed=8)
    full = workload.unpack_lower(y, 333)
    full[np.triu_indices(333, 1)] = -5.0        # upper triangle is never read
    with mds.MDS(333, 2) as c:
        c.set_dissimilarities(full)
        c.set_locations(x)
        c.set_sigma(w.sigma)
        ll, g = c.log_likelihood_and_gradient()
    assert_fp64_parity(ll, g, oracle.loglik_grad(y, x, w.sigma, 1), "full setter")


def test_errors(mds):
    w, y, x = instance(100, 2)
    with mds.MDS(100, 2) as c:
        with pytest.raises(mds.MDSError) as e:
            c.log_likelihood()
        assert e.value.status == 2                      # MDS_E_STATE
        bad = y.copy()
        bad[17] = -1.0
        with pytest.raises(mds.MDSError) as e:
            c.set_dissimilarities_packed(bad)
        assert e.value.status == 1
        bad[17] = np.inf
        with pytest.raises(mds.MDSError):
            c.set_dissimilarities_packed(bad)
        c.set_locations(x)
        c.set_sigma(w.sigma)
        with pytest.raises(mds.MDSError) as e:
            c.log_likelihood()                          # Y rejected -> not set
        assert e.value.status == 2
        c.set_dissimilarities_packed(y)
        assert np.isfinite(c.log_likelihood())
        with pytest.raises(mds.MDSError):
            c.set_sigma(0.0)
        xb = x.copy()
        xb[3, 1] = np.nan
        with pytest.raises(mds.MDSError):
            c.set_locations(xb)
        assert np.isfinite(c.log_likelihood())          # context still usable


# ------------------------------------------------------------------ fp32
def fp32_check(ll, g, ref):
    rl, G, S = ref["loglik"], ref["grad"], ref["absscale"]
    assert abs(ll - rl) <= 1e-4 * abs(rl)
    assert np.linalg.norm(g - G) <= 1e-4 * np.linalg.norm(G)
    assert np.all(np.abs(g - G) <= 1e-4 * np.abs(G) + 1e-6 * S)


@pytest.mark.parametrize("n,d,pm", [(64, 2, 0.0), (1000, 2, 0.0), (3000, 6, 0.1), (517, 3, 0.2)])
def test_fp32_parity(mds, n, d, pm):
    w, y, x = instance(n, d, pm, seed=3 * n)
    y32 = y.astype(np.float32).astype(np.float64)
    x32 = x.astype(np.float32).astype(np.float64)
    ref = oracle.loglik_grad(y32, x32, w.sigma, 1)
    ll, g = run_gpu(mds, n, d, y, x, w.sigma, prec="f32")
    fp32_check(ll, g, ref)


def test_c4_fp32_full_size_sampled_rows(mds):
    w = workload.config("C4")
    y = w.y_packed()
    ll, g = run_gpu(mds, w.n, w.d, y, w.x0, w.sigma, prec="f32")
    rows = np.array([0, 77, 20000, 29999])
    yr = w.y_full_rows(rows).astype(np.float32).astype(np.float64)
    x32 = w.x0.astype(np.float32).astype(np.float64)
    ref = oracle.grad_rows(rows, yr, x32, w.sigma, 1)
    G, S = ref["grad"], ref["absscale"]
    assert np.all(np.abs(g[rows] - G) <= 1e-4 * np.abs(G) + 1e-6 * S)


# ------------------------------------------------------------------ HMC
def test_hmc_trajectory_matches_oracle_leapfrog(mds):
    w, y, x = instance(300, 2, 0.0, seed=31)
    p0 = w.normals(1, (300, 2))
    ref = oracle.leapfrog(y, x, p0, w.sigma, 0.002, 20, 1, prior_sd=10.0)
    with mds.MDS(300, 2) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(x)
        c.set_sigma(w.sigma)
        out = c.hmc_trajectory(p0, 0.002, 20, prior_sd=10.0)
        # the context's X is unchanged by a trajectory
        ll, _ = c.log_likelihood_and_gradient()
    assert ll == pytest.approx(oracle.loglik_grad(y, x, w.sigma, 1)["loglik"], rel=1e-10)
    np.testing.assert_allclose(out["x"], ref["x"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(out["p"], ref["p"], rtol=1e-9, atol=1e-10)
    assert out["H0"] == pytest.approx(ref["H0"], rel=1e-10)
    assert out["H1"] == pytest.approx(ref["H1"], rel=1e-10)


def test_hmc_reversible_and_energy_scaling(mds):
    w, y, x = instance(400, 2, 0.0, seed=32)
    p0 = w.normals(2, (400, 2))
    with mds.MDS(400, 2) as c:
        c.set_dissimilarities_packed(y)
        c.set_sigma(w.sigma)
        c.set_locations(x)
        fw = c.hmc_trajectory(p0, 0.001, 10, prior_sd=10.0)
        c.set_locations(fw["x"])
        bw = c.hmc_trajectory(-fw["p"], 0.001, 10, prior_sd=10.0)
        np.testing.assert_allclose(bw["x"], x, atol=1e-8)
        c.set_locations(x)
        # asymptotic regime checked with the oracle: eps 4e-4 -> 2e-4 gives ratio ~4.03
        a = c.hmc_trajectory(p0, 0.0004, 40, prior_sd=10.0)
        b = c.hmc_trajectory(p0, 0.0002, 80, prior_sd=10.0)
    ratio = abs(a["H1"] - a["H0"]) / abs(b["H1"] - b["H0"])
    assert 3.5 <= ratio <= 4.5, ratio


def test_hmc_prior_only_stationarity(mds):
    """All-missing Y: the chain must sample the N(0, tau^2 I) prior (SPEC.md:387 analogue)."""
    n, d, tau = 200, 2, 2.0
    y = np.full(n * (n - 1) // 2, np.nan)
    rng = np.random.default_rng(0)
    xs = []
    with mds.MDS(n, d) as c:
        c.set_dissimilarities_packed(y)
        c.set_sigma(1.0)
        x = rng.normal(size=(n, d)) * tau
        for k in range(40):
            x, st = c.hmc_run(5, 10, 0.3, tau, seed=1000 + k, x0=x)
            xs.append(x.copy())
    s = np.stack(xs[5:])
    m = s.mean()
    v = s.var()
    neff = s.size / 4
    assert abs(m) < 4 * tau / math.sqrt(neff)
    assert abs(v / tau**2 - 1) < 0.1
    assert st["accepted"] >= 3


def test_hmc_run_c1_chain(mds):
    w = workload.config("C1")
    y = w.y_packed()
    with mds.MDS(w.n, w.d) as c:
        c.set_dissimilarities_packed(y)
        c.set_sigma(w.sigma)
        x, st = c.hmc_run(50, 20, 0.01, 10.0, seed=7, x0=w.x0)
        assert st["grad_evals"] == 1000
        assert 0 < st["accepted"] <= 50
        ll, _ = c.log_likelihood_and_gradient()
    assert st["final_loglik"] == pytest.approx(oracle.loglik_grad(y, x, w.sigma, 1)["loglik"], rel=1e-10)
    assert ll == pytest.approx(st["final_loglik"], rel=1e-12)


# The HMC driver's momenta and accept draws come from a counter-based generator
# (splitmix64 finaliser + Box-Muller, PAPER.md:321-336 leaves the generator open):
# the same generator written out here, independently of libmds, so that an
# oracle-driven chain can be replayed transition by transition.
_M64 = (1 << 64) - 1


def _mix(z):
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _u01(h):
    return (float(h >> 11) + 1.0) * (1.0 / 9007199254740992.0)


def _normal(seed, it, q):
    h1 = _mix(seed ^ _mix(it ^ _mix(2 * q)))
    h2 = _mix(seed ^ _mix(it ^ _mix(2 * q + 1)))
    return math.sqrt(-2.0 * math.log(_u01(h1))) * math.cos(6.283185307179586 * _u01(h2))


def test_hmc_run_matches_oracle_chain(mds):
    """mds_hmc_run (momenta staged on the host while the previous transition runs,
    fused save / redrift / H0 and restore launches, one graph per trajectory) against
    the same chain driven by the oracle's leapfrog: every transition's Metropolis
    decision, the acceptance count and the final X."""
    w = workload.config("C1")
    y = w.y_packed()
    # eps 0.08: 8 of 15 accepted, every decision at least 0.06 away from its threshold
    n, d, seed, n_iter, L, eps, tau = w.n, w.d, 4242, 15, 10, 0.08, 10.0
    x = w.x0.copy()
    acc = 0
    for it in range(n_iter):
        p0 = np.array([_normal(seed, it, q) for q in range(n * d)]).reshape(n, d)
        ref = oracle.leapfrog(y, x, p0, w.sigma, eps, L, 1, prior_sd=tau)
        dh = ref["H1"] - ref["H0"]
        u = _u01(_mix(seed ^ _mix(0xACCE97 ^ _mix(it))))
        if math.isfinite(dh) and math.log(u) < -dh:
            x = ref["x"]
            acc += 1
    assert 0 < acc < n_iter          # both branches (accept and restore) were taken
    with mds.MDS(n, d) as c:
        c.set_dissimilarities_packed(y)
        c.set_sigma(w.sigma)
        xg, st = c.hmc_run(n_iter, L, eps, tau, seed=seed, x0=w.x0)
    assert st["accepted"] == acc
    np.testing.assert_allclose(xg, x, rtol=1e-9, atol=1e-12)
    assert st["final_loglik"] == pytest.approx(oracle.loglik_grad(y, x, w.sigma, 1)["loglik"], rel=1e-10)


def test_virtual_ranges_and_wide_d(mds):
    """Warp ranges split into several segment tables (forced small with
    MDS_DEBUG_MAXSEG), and the widest D in both precisions."""
    import os
    w, y, x = instance(2500, 2, 0.05, seed=44)
    ref = oracle.loglik_grad(y, x, w.sigma, 1)
    os.environ["MDS_DEBUG_MAXSEG"] = "1"
    try:
        ll, g = run_gpu(mds, w.n, w.d, y, x, w.sigma)
    finally:
        del os.environ["MDS_DEBUG_MAXSEG"]
    assert_fp64_parity(ll, g, ref, "maxseg=1")
    for d in (7, 8):
        w, y, x = instance(700, d, 0.1, seed=50 + d)
        ref = oracle.loglik_grad(y, x, w.sigma, 1)
        ll, g = run_gpu(mds, w.n, d, y, x, w.sigma)
        assert_fp64_parity(ll, g, ref, "d=%d" % d)
        y32 = y.astype(np.float32).astype(np.float64)
        x32 = x.astype(np.float32).astype(np.float64)
        ll, g = run_gpu(mds, w.n, d, y, x, w.sigma, prec="f32")
        fp32_check(ll, g, oracle.loglik_grad(y32, x32, w.sigma, 1))


@pytest.mark.skipif(bool(__import__("os").environ.get("MDS_SKIP_C5")), reason="MDS_SKIP_C5 set")
def test_c5_full_size_parity(mds):
    """C5 at full size on one GPU (N = 100000, D = 2, fp64, 5.0e9 pairs, 40 GB of
    tiled Y streamed from the generator in row chunks).  log L against the oracle's
    streaming row-range sum (oracle.loglik_rows over the same chunks, run in a
    thread pool while the next chunk is generated and uploaded, added in row
    order) within 1e-10 relative; sampled gradient rows against the per-row
    oracle; the gradient rows sum to zero."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    w = workload.config("C5")
    step = 250
    futs = []
    workers = max(2, os.cpu_count() or 2)
    with mds.MDS(w.n, w.d, "f64", True) as c, ThreadPoolExecutor(workers) as pool:
        for i0 in range(0, w.n, step):
            i1 = min(w.n, i0 + step)
            y = w.y_rows(i0, i1)
            c.set_dissimilarity_rows(i0, i1, y)
            futs.append(pool.submit(oracle.loglik_rows, i0, i1, y, w.x0, w.sigma, 1))
            del y
            if len(futs) > 2 * workers:          # bound the chunks held in host memory
                futs[-2 * workers - 1].result()
        c.set_locations(w.x0)
        c.set_sigma(w.sigma)
        ll, g = c.log_likelihood_and_gradient()
        n_obs = c.observed_pairs()
        parts = [f.result() for f in futs]
    ref_ll, ref_obs = 0.0, 0
    for v, no in parts:                          # fixed row order
        ref_ll += v
        ref_obs += no
    assert n_obs == ref_obs
    assert abs(ll - ref_ll) <= 1e-10 * abs(ref_ll), (ll, ref_ll)
    rows = np.array([0, 1, 64, 4095, 50000, 77777, 99999])
    ref = oracle.grad_rows(rows, w.y_full_rows(rows), w.x0, w.sigma, 1)
    err = np.abs(g[rows] - ref["grad"])
    assert np.all(err <= np.maximum(1e-9 * np.abs(ref["grad"]), 1e-12)), err.max()
    assert np.all(np.abs(g.sum(0)) <= 1e-12 * np.abs(g).sum(0))


def test_create_argument_errors(mds):
    """Degenerate shapes and options are refused at creation (n < 2, d outside
    1..MDS_D_MAX, unknown precision or truncation flag)."""
    import ctypes
    for n, d, prec, trunc in [(1, 2, 0, 1), (0, 2, 0, 1), (10, 0, 0, 1), (10, 9, 0, 1), (10, 2, 7, 1), (10, 2, 0, 2)]:
        h = ctypes.c_void_p()
        st = mds._abi.lib.mds_create(n, d, prec, trunc, ctypes.byref(h))
        assert st == 1, (n, d, prec, trunc, st)          # MDS_E_INVALID_ARG
    for rank, world in [(2, 2), (-1, 2), (0, 0)]:
        h = ctypes.c_void_p()
        assert mds._abi.lib.mds_create_sharded(10, 2, 0, 1, rank, world, None, ctypes.byref(h)) == 1
    # the smallest problem: one pair
    with mds.MDS(2, 1) as c:
        c.set_dissimilarities_packed(np.array([1.5]))
        c.set_locations(np.array([[0.0], [2.0]]))
        c.set_sigma(0.8)
        ll, g = c.log_likelihood_and_gradient()
    ref = oracle.loglik_grad(np.array([1.5]), np.array([[0.0], [2.0]]), 0.8, 1)
    assert ll == pytest.approx(ref["loglik"], rel=1e-12)
    np.testing.assert_allclose(g, ref["grad"], rtol=1e-12)
