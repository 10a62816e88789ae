"""The fused peer-memory exchange (SURVEY 8(e) "stage 2", include/mds.h
mds_p2p_*) on ONE GPU.

The pass kernel of a connected context pushes its partial into every rank's
window, raises its flag, waits for all ranks' flags and combines (fused with
the leapfrog update) -- no NCCL, no host call.  Here the ranks are host
threads of one process, each with its own context and stream on the same GPU;
their grids are capped (mds_set_grid_limit) so that all ranks' pass kernels
are co-resident, as they are on separate GPUs.  The results must be bitwise
identical on every rank and to the all-gather path of the same shards (the
same rank-ordered sum), and match the oracle.
"""
import threading

import numpy as np
import pytest

import oracle
import workload
from oracle import tree as otree
from tests.test_sharded_gpu import ThreadAllgather

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mds():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1905_04582_b200 as m
    return m


def run_world(mds, world, n, d, body, exchange="p2p", ctas=None):
    """body(ctx, rank, sync) on `world` threads; exchange = "p2p" (windows connected
    by address) or "callback" (the stream-ordered in-process all-gather).

    sync() = this rank's stream drained + a host barrier: the bodies call it after
    their setup (setters may wait for the whole device, e.g. cudaFree in a tree
    prior's setup, which on ONE shared GPU would also wait for a peer's pass kernel
    that is waiting for this rank -- with a GPU per rank they wait only for their
    own device)."""
    import torch
    ctas = ctas or max(1, torch.cuda.get_device_properties(0).multi_processor_count // world)
    bar = threading.Barrier(world, timeout=120)
    wins = [None] * world
    ag = ThreadAllgather(world, n * d + 1) if exchange == "callback" else None
    out, errs = [None] * world, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            torch.cuda.set_stream(st)
            ctx = mds.MDS(n, d, "f64", True, rank=r, world=world, stream=st)
            ctx.set_grid_limit(ctas)
            if exchange == "p2p":
                wins[r], _ = ctx.p2p_window()
                bar.wait()
                ctx.p2p_connect(wins)
                assert ctx.p2p_connected()
            else:
                cb = ag.callback(mds, r)
                mds._abi.mds_set_allgather(ctx.ctx, cb, None)
            bar.wait()
            def sync():
                st.synchronize()
                bar.wait()

            out[r] = body(ctx, r, sync)
            st.synchronize()            # (not the device: a peer may still be queueing)
            bar.wait()
            ctx.close()
        except Exception as e:
            errs.append((r, repr(e)))
            bar.abort()
            if ag:
                ag.barrier.abort()

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    return out


def _same(a, b):
    if isinstance(a, dict):
        return all(_same(a[k], b[k]) for k in a)
    if isinstance(a, (tuple, list)):
        return all(_same(u, v) for u, v in zip(a, b))
    if isinstance(a, np.ndarray):
        return np.array_equal(a, b)
    return a == b or (a != a and b != b)


def test_p2p_world1_matches_direct(mds):
    """A world-1 context connected to its own window (push -> flag -> wait ->
    combine in one launch) reproduces the direct pass bitwise: evaluation,
    leapfrog steps, the likelihood-only pass and the row delta."""
    import torch
    n, d = 700, 2
    w = workload.Workload(n, d, p_missing=0.05, seed=81)
    y, x = w.y_packed(), w.x0
    p0 = torch.from_numpy(w.normals(1, (n, d))).cuda()
    res = []
    for p2p in (False, True):
        with mds.MDS(n, d, "f64", True) as ctx:
            ctx.set_grid_limit(100)
            if p2p:
                a, _ = ctx.p2p_window()
                ctx.p2p_connect([a])
            ctx.set_dissimilarities_packed(y)
            ctx.set_locations(x)
            ctx.set_sigma(w.sigma)
            ll, g = ctx.log_likelihood_and_gradient()
            ls = ctx.log_likelihood_at_sigma(0.8 * w.sigma)
            dl = ctx.row_loglik_delta(5, x[5] + 0.01)
            ctx.leapfrog_device(5, 0.002, 10.0, p0_dev=p0)
            torch.cuda.synchronize()
            res.append((ll, g, ls, dl, ctx.get_locations(), ctx.get_momentum(), ctx.log_likelihood()))
    assert _same(res[0], res[1])
    ref = oracle.loglik_grad(y, x, w.sigma, 1)
    assert res[1][0] == pytest.approx(ref["loglik"], rel=1e-10)
    np.testing.assert_allclose(res[1][1], ref["grad"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_sharded_matches_allgather(mds, world):
    """world ranks sharing the GPU: evaluation, an HMC trajectory (graph-captured
    leapfrog steps through the fused exchange), the sigma MH step (likelihood-only
    pass) and a single-location delta (one-CTA peer all-gather) are bitwise equal
    across ranks and to the all-gather path, and match the oracle."""
    n, d = 500, 2
    w = workload.Workload(n, d, p_missing=0.05, seed=90 + world)
    y, x = w.y_packed(), w.x0
    p0 = w.normals(1, (n, d))

    def body(ctx, r, sync):
        ctx.set_dissimilarities_packed(y)
        ctx.set_locations(x)
        ctx.set_sigma(w.sigma)
        sync()
        ll, g = ctx.log_likelihood_and_gradient()
        traj = ctx.hmc_trajectory(p0, 0.002, 8, prior_sd=10.0)
        ctx.set_locations(x)
        acc, lr = ctx.sigma_mh_step(2.0, 0.5, 0.05, 0.7, 0.5)
        dl = ctx.row_loglik_delta(3, x[3] + 0.02)
        return ll, g, traj["x"], traj["H1"], acc, lr, dl

    outs = run_world(mds, world, n, d, body, "p2p")
    ref_cb = run_world(mds, world, n, d, body, "callback")
    for o in outs[1:]:
        assert _same(o, outs[0])
    assert _same(outs[0], ref_cb[0])
    ll, g, xs, h1, acc, lr, dl = outs[0]
    ref = oracle.loglik_grad(y, x, w.sigma, 1)
    assert ll == pytest.approx(ref["loglik"], rel=1e-10)
    np.testing.assert_allclose(g, ref["grad"], rtol=1e-9, atol=1e-12)
    lf = oracle.leapfrog(y, x, p0, w.sigma, 0.002, 8, 1, prior_sd=10.0)
    np.testing.assert_allclose(xs, lf["x"], rtol=1e-9, atol=1e-12)


def test_p2p_tree_prior_leapfrog(mds):
    """Device-resident leapfrog steps under the tree prior through the fused
    exchange (the pass walks the tree and combines + updates in one launch)."""
    import torch
    n, d, world = 300, 2, 2
    w = workload.Workload(n, d, p_missing=0.0, seed=72)
    y, x = w.y_packed(), w.x0
    parent, t = workload.coalescent_forest(n, 1, 0.1, seed=4, tau0=4.0)
    p0 = w.normals(2, (n, d))

    def body(ctx, r, sync):
        ctx.set_dissimilarities_packed(y)
        ctx.set_locations(x)
        ctx.set_sigma(w.sigma)
        ctx.set_tree_prior(parent, t)
        pd = torch.from_numpy(p0).cuda()
        sync()
        ctx.leapfrog_device(6, 0.002, 0.0, p0_dev=pd)
        return ctx.get_locations(), ctx.log_likelihood()

    outs = run_world(mds, world, n, d, body, "p2p")
    assert _same(outs[0], outs[1])
    lf = otree.leapfrog_tree(y, x, p0, w.sigma, 0.002, 6, parent, t)
    np.testing.assert_allclose(outs[0][0], lf["x"], rtol=1e-9, atol=1e-12)
    assert outs[0][1] == pytest.approx(lf["loglik"], rel=1e-10)


def test_p2p_many_steps_double_buffer(mds):
    """Many back-to-back fused exchanges queued at once on both ranks (the
    receive slots alternate by exchange count): 40 leapfrog steps equal the
    all-gather path bitwise."""
    import torch
    n, d, world = 400, 2, 2
    w = workload.Workload(n, d, p_missing=0.0, seed=73)
    y, x = w.y_packed(), w.x0
    p0 = w.normals(3, (n, d))

    def body(ctx, r, sync):
        ctx.set_dissimilarities_packed(y)
        ctx.set_locations(x)
        ctx.set_sigma(w.sigma)
        pd = torch.from_numpy(p0).cuda()
        sync()
        ctx.leapfrog_device(40, 0.001, 10.0, p0_dev=pd)
        return ctx.get_locations(), ctx.get_momentum(), ctx.log_likelihood()

    a = run_world(mds, world, n, d, body, "p2p")
    b = run_world(mds, world, n, d, body, "callback")
    assert _same(a[0], a[1]) and _same(a[0], b[0])
