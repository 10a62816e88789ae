"""The sharded (world > 1) path end to end on ONE GPU.

Each rank is a host thread with its own libmds context (rank r of W, its own
CUDA stream) and the exchange registered through mds_set_allgather is an
in-process, stream-ordered all-gather: every rank copies its partial into a
shared device buffer on its stream and records an event; after a host
barrier each rank's stream waits on all ranks' events and copies the gathered
buffer out -- the same contract NCCL's all-gather fulfils across GPUs.  This
drives the library's own sharded orchestration (local pass -> exchange ->
rank-ordered combine -> leapfrog update, and the count-1 exchange of the
likelihood-only pass) with no second GPU.  Results must equal the oracle and
be bitwise identical on every rank.
"""
import threading

import numpy as np
import pytest

import oracle
import workload
from oracle import tree as otree

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mds():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1905_04582_b200 as m
    return m


class ThreadAllgather:
    """Stream-ordered all-gather among `world` threads on one device."""

    def __init__(self, world, max_count, max_calls=400):
        import torch
        self.world = world
        self.barrier = threading.Barrier(world, timeout=120)
        # one buffer per exchange (never reused: no cross-stream reuse hazards)
        self.bufs = [torch.zeros(world, max_count, dtype=torch.float64, device="cuda") for _ in range(max_calls)]
        self.events = [[None] * world for _ in range(max_calls)]
        self.calls = [0] * world
        torch.cuda.synchronize()

    def callback(self, mds, rank):
        import torch
        from paper_1905_04582_b200 import _wrap_dev

        def cb(user, send, recv, count, stream):
            try:
                k = self.calls[rank]
                self.calls[rank] += 1
                s = torch.cuda.ExternalStream(stream)
                dev = torch.device("cuda", torch.cuda.current_device())
                buf = self.bufs[k]
                with torch.cuda.stream(s):
                    buf[rank, :count].copy_(_wrap_dev(send, count, dev))
                    ev = torch.cuda.Event()
                    ev.record(s)
                    self.events[k][rank] = ev
                self.barrier.wait()
                with torch.cuda.stream(s):
                    for r in range(self.world):
                        s.wait_event(self.events[k][r])
                    _wrap_dev(recv, count * self.world, dev).copy_(buf[:, :count].reshape(-1))
                return 0
            except Exception as e:  # reported by the library as MDS_E_COMM
                print("allgather callback failed:", repr(e))
                return 1

        return mds._abi.ALLGATHER_FN(cb)


def run_ranks(mds, world, n, d, body):
    """Run body(ctx, rank) on `world` threads, one sharded context each."""
    import torch
    ag = ThreadAllgather(world, n * d + 1)
    out, errs = [None] * world, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            torch.cuda.set_stream(st)
            ctx = mds.MDS(n, d, "f64", True, rank=r, world=world, stream=st)
            cb = ag.callback(mds, r)
            mds._abi.mds_set_allgather(ctx.ctx, cb, None)
            out[r] = body(ctx, r)
            torch.cuda.synchronize()
            ctx.close()
        except Exception as e:
            errs.append((r, repr(e)))
            ag.barrier.abort()

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_eval_and_trajectory(mds, world):
    n, d = 400, 2
    w = workload.Workload(n, d, p_missing=0.05, seed=60 + world)
    y, x = w.y_packed(), w.x0
    p0 = w.normals(1, (n, d))

    def body(ctx, r):
        ctx.set_dissimilarities_packed(y)
        ctx.set_locations(x)
        ctx.set_sigma(w.sigma)
        ll, g = ctx.log_likelihood_and_gradient()
        traj = ctx.hmc_trajectory(p0, 0.002, 8, prior_sd=10.0)
        return ll, g, traj

    outs = run_ranks(mds, world, n, d, body)
    for o in outs[1:]:                       # bitwise identical on every rank
        assert o[0] == outs[0][0] and np.array_equal(o[1], outs[0][1])
        assert np.array_equal(o[2]["x"], outs[0][2]["x"]) and o[2]["H1"] == outs[0][2]["H1"]
    ll, g, traj = outs[0]
    ref = oracle.loglik_grad(y, x, w.sigma, 1)
    assert ll == pytest.approx(ref["loglik"], rel=1e-10)
    np.testing.assert_allclose(g, ref["grad"], rtol=1e-9, atol=1e-12)
    lf = oracle.leapfrog(y, x, p0, w.sigma, 0.002, 8, 1, prior_sd=10.0)
    np.testing.assert_allclose(traj["x"], lf["x"], rtol=1e-9, atol=1e-12)
    assert traj["H1"] == pytest.approx(lf["H1"], rel=1e-10)


def test_sharded_leapfrog_tree_prior_and_sigma_step(mds):
    """Device-resident leapfrog under the tree prior (standalone walk on the
    sharded path) and the sigma MH step (count-1 exchange of the likelihood-only
    pass), world = 2."""
    import torch
    n, d, world = 300, 2, 2
    w = workload.Workload(n, d, p_missing=0.0, seed=71)
    y, x = w.y_packed(), w.x0
    parent, t = workload.coalescent_forest(n, 1, 0.1, seed=3, tau0=4.0)
    p0 = w.normals(2, (n, d))

    def body(ctx, r):
        ctx.set_dissimilarities_packed(y)
        ctx.set_locations(x)
        ctx.set_sigma(w.sigma)
        acc, lr = ctx.sigma_mh_step(2.0, 0.5, 0.05, 0.7, 0.5)
        ctx.set_sigma(w.sigma)
        ctx.set_tree_prior(parent, t)
        ctx.leapfrog_device(6, 0.002, 0.0, p0_dev=torch.from_numpy(p0).cuda())
        return acc, lr, ctx.get_locations(), ctx.log_likelihood()

    outs = run_ranks(mds, world, n, d, body)
    assert outs[0][1] == outs[1][1] and np.array_equal(outs[0][2], outs[1][2]) and outs[0][3] == outs[1][3]
    acc, lr, xs, ll = outs[0]
    ref = oracle.sigma_mh_step(y, x, w.sigma, 2.0, 0.5, 0.05, 0.7, 0.5)
    assert lr == pytest.approx(ref["log_ratio"], abs=1e-10 * abs(oracle.loglik_grad(y, x, w.sigma, 1)["loglik"]))
    assert acc == ref["accepted"]
    lf = otree.leapfrog_tree(y, x, p0, w.sigma, 0.002, 6, parent, t)
    np.testing.assert_allclose(xs, lf["x"], rtol=1e-9, atol=1e-12)
    assert ll == pytest.approx(lf["loglik"], rel=1e-10)
