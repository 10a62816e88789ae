"""The library-owned exchange (SURVEY 8(e) stage 1; PAPER.md:440-446's c1) and
several processes on one GPU.

1. A context created with an NCCL unique id owns its communicator: even at
   world = 1 it runs the sharded sequence (local partial -> ncclAllGather on
   the context stream -> rank-ordered combine [+ leapfrog update]), which is
   then captured in the HMC driver's CUDA graph.  Results must match the
   oracle, and the unsharded context exactly (the combine of one partial adds
   it to 0.0; the fused update uses the same expressions as phase B, so
   trajectories agree to rounding).
2. Two PROCESSES sharing the one GPU, each a rank of a world-2 sharded
   context, exchanging through a host-staged gloo all-gather registered with
   mds_set_allgather: evaluation, HMC trajectory, the likelihood-only
   (sigma) pass and the single-location updates match the oracle and are
   bitwise identical across ranks.
"""
import os
import socket

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


def _assert_parity(ll, g, ref):
    assert abs(ll - ref["loglik"]) <= 1e-10 * abs(ref["loglik"])
    G = ref["grad"]
    assert np.all(np.abs(g - G) <= np.maximum(1e-9 * np.abs(G), 1e-12))


def test_world1_communicator_eval_and_sigma_pass(mds):
    w = workload.Workload(900, 3, p_missing=0.1, seed=5)
    y, x = w.y_packed(), w.x0
    nid = mds.mds_nccl_unique_id()
    assert len(nid) == 128
    with mds.MDS(w.n, w.d, rank=0, world=1, nccl_unique_id=nid) as c, mds.MDS(w.n, w.d) as u:
        assert c.has_communicator() and not u.has_communicator()
        for k in (c, u):
            k.set_dissimilarities_packed(y)
            k.set_locations(x)
            k.set_sigma(w.sigma)
        ll, g = c.log_likelihood_and_gradient()
        ll_u, g_u = u.log_likelihood_and_gradient()
        l2 = c.log_likelihood_at_sigma(0.9 * w.sigma)
        l2_u = u.log_likelihood_at_sigma(0.9 * w.sigma)
    _assert_parity(ll, g, oracle.loglik_grad(y, x, w.sigma, 1))
    assert ll == ll_u and np.array_equal(g, g_u)
    assert l2 == l2_u


def test_world1_communicator_hmc_graph_matches_unsharded(mds):
    """mds_hmc_run captures the L-step trajectory, ncclAllGather included, in one graph."""
    w = workload.Workload(500, 2, p_missing=0.0, seed=8)
    y = w.y_packed()
    out = []
    for nid in (mds.mds_nccl_unique_id(), None):
        with mds.MDS(w.n, w.d, rank=0, world=1, nccl_unique_id=nid) as c:
            c.set_dissimilarities_packed(y)
            c.set_sigma(w.sigma)
            x, st = c.hmc_run(6, 8, 0.004, 10.0, seed=3, x0=w.x0)
            out.append((x, st))
    (xa, sa), (xb, sb) = out
    assert sa["accepted"] == sb["accepted"] > 0
    np.testing.assert_allclose(xa, xb, rtol=1e-12, atol=1e-14)
    assert sa["final_loglik"] == pytest.approx(sb["final_loglik"], rel=1e-13)
    assert sa["final_loglik"] == pytest.approx(oracle.loglik_grad(y, xa, w.sigma, 1)["loglik"], rel=1e-10)


def test_world1_communicator_tree_prior_trajectory(mds):
    """Sharded steps under the tree prior: the pass kernel's last CTA walks the tree
    (EVAL_TREE modes) and the update follows the exchange; vs the oracle's
    tree leapfrog (pinned in tests/test_oracle_tree.py)."""
    n, d = 300, 2
    w = workload.Workload(n, d, p_missing=0.05, seed=19)
    y = w.y_packed()
    parent, t = workload.coalescent_forest(n, 3, 0.1, seed=4)
    p0 = w.normals(7, (n, d))
    ref = otree.leapfrog_tree(y, w.x0, p0, w.sigma, 0.002, 6, parent, t)
    with mds.MDS(n, d, rank=0, world=1, nccl_unique_id=mds.mds_nccl_unique_id()) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(w.x0)
        c.set_sigma(w.sigma)
        c.set_tree_prior(parent, t)
        out = c.hmc_trajectory(p0, 0.002, 6)
    np.testing.assert_allclose(out["x"], ref["x"], rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(out["p"], ref["p"], rtol=1e-8, atol=1e-9)
    assert out["H1"] - out["H0"] == pytest.approx(ref["H1"] - ref["H0"], rel=1e-6, abs=1e-8)


def test_world1_communicator_single_location_updates(mds):
    """Sharded single-location updates: the row delta as this
    rank's share + exchange + rank-ordered sum, and the random-walk sweep as
    propose -> share -> exchange -> decide per update, through the NCCL path."""
    n, d = 500, 2
    w = workload.Workload(n, d, p_missing=0.05, seed=43)
    y, x = w.y_packed(), w.x0
    rng = np.random.default_rng(3)
    k = 120
    rows = rng.integers(0, n, size=k)
    z = rng.normal(size=(k, d))
    u = 1.0 - rng.random(k)
    ref_x, ref_acc = oracle.rw_sweep(y, x, w.sigma, rows, z, u, 0.05, prior_sd=10.0)
    with mds.MDS(n, d, rank=0, world=1, nccl_unique_id=mds.mds_nccl_unique_id()) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(x)
        c.set_sigma(w.sigma)
        for i in (0, 77, 499):
            xn = x[i] + 0.1
            got = c.row_loglik_delta(i, xn)
            ref = oracle.row_delta(y, x, i, xn, w.sigma, 1)
            assert got == pytest.approx(ref, rel=1e-10, abs=1e-9)
        acc = c.rw_sweep(rows, z, u, 0.05, prior_sd=10.0)
        xs = c.get_locations()
    assert acc == ref_acc and 0 < acc < k
    np.testing.assert_allclose(xs, ref_x, rtol=0, atol=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_proc(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1905_04582_b200 as m
        w = workload.Workload(640, 2, p_missing=0.05, seed=77)
        y = w.y_packed()
        st = torch.cuda.Stream()
        torch.cuda.set_stream(st)
        c = m.MDS(w.n, w.d, rank=rank, world=world, stream=st)
        c.use_torch_allgather(host_staged=True)
        c.set_dissimilarities_packed(y)
        c.set_locations(w.x0)
        c.set_sigma(w.sigma)
        ll, g = c.log_likelihood_and_gradient()
        l2 = c.log_likelihood_at_sigma(1.1 * w.sigma)
        p0 = w.normals(3, (w.n, w.d))
        tr = c.hmc_trajectory(p0, 0.002, 5, prior_sd=10.0)
        rd = c.row_loglik_delta(100, w.x0[100] + 0.1)
        rng = np.random.default_rng(5)
        rows = rng.integers(0, w.n, size=40)
        acc = c.rw_sweep(rows, rng.normal(size=(40, w.d)), 1.0 - rng.random(40), 0.05, prior_sd=10.0)
        xs = c.get_locations()
        c.close()
        q.put((rank, ll, g, l2, tr["x"], tr["H0"], tr["H1"], rd, acc, xs))
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_two_processes_share_the_gpu_hoststaged_exchange(mds):
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_proc, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    assert all(len(r) == 10 for r in res), res
    (_, ll0, g0, l20, x0, h00, h10, rd0, a0, xs0), (_, ll1, g1, l21, x1, h01, h11, rd1, a1, xs1) = res
    # bitwise identical on both ranks
    assert ll0 == ll1 and np.array_equal(g0, g1) and l20 == l21
    assert np.array_equal(x0, x1) and h00 == h01 and h10 == h11
    w = workload.Workload(640, 2, p_missing=0.05, seed=77)
    y = w.y_packed()
    _assert_parity(ll0, g0, oracle.loglik_grad(y, w.x0, w.sigma, 1))
    assert l20 == pytest.approx(oracle.loglik_grad(y, w.x0, 1.1 * w.sigma, 1)["loglik"], rel=1e-10)
    ref = oracle.leapfrog(y, w.x0, w.normals(3, (w.n, w.d)), w.sigma, 0.002, 5, 1, prior_sd=10.0)
    np.testing.assert_allclose(x0, ref["x"], rtol=1e-9, atol=1e-12)
    assert h00 == pytest.approx(ref["H0"], rel=1e-10) and h10 == pytest.approx(ref["H1"], rel=1e-10)
    # single-location updates across the two ranks' shares
    assert rd0 == rd1 and a0 == a1 and np.array_equal(xs0, xs1)
    assert rd0 == pytest.approx(oracle.row_delta(y, w.x0, 100, w.x0[100] + 0.1, w.sigma, 1), rel=1e-10, abs=1e-9)
    rng = np.random.default_rng(5)
    rows = rng.integers(0, w.n, size=40)
    rx, racc = oracle.rw_sweep(y, w.x0, w.sigma, rows, rng.normal(size=(40, w.d)), 1.0 - rng.random(40), 0.05,
                               prior_sd=10.0)
    assert a0 == racc
    np.testing.assert_allclose(xs0, rx, rtol=0, atol=1e-12)


def _cb_proc(q):
    """The binding's torch.distributed exchange callback on an NCCL process group
    (world 1: the all_gather_into_tensor path libmds calls through
    mds_set_allgather), driven with device buffers on a side stream."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        import paper_1905_04582_b200 as m
        cb = m.allgather_callback(1)
        st = torch.cuda.Stream()
        send = torch.arange(1000, dtype=torch.float64, device="cuda")
        recv = torch.zeros(1000, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        rc = cb(None, send.data_ptr(), recv.data_ptr(), 1000, st.cuda_stream)
        st.synchronize()
        q.put((rc, bool(torch.equal(send, recv))))
    except Exception as e:
        q.put((repr(e), False))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_torch_nccl_exchange_callback(mds):
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_cb_proc, args=(q,))
    p.start()
    rc, ok = q.get(timeout=300)
    p.join(timeout=60)
    assert rc == 0 and ok, rc
