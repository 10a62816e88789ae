"""Host-side logic of the sharded path, on CPU (no GPU needed).

mds_plan exposes the work split the library uses (tile-row ownership, the
persistent kernel's warp ranges and segments, the fixed-order reduction lists)
and checks its invariants.  The world_size-2 test runs two gloo processes that
each plan their shard, exchange over torch.distributed (the same all-gather the
GPU path uses through mds_set_allgather) and verify the shards partition the
triangle and that a rank-ordered combine gives identical results on both ranks.
"""
import os
import socket

import numpy as np
import pytest

import paper_1905_04582_b200 as mds


@pytest.mark.parametrize("n", [2, 3, 63, 64, 65, 1000, 5392, 30000])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shards_partition_the_triangle(n, world):
    cover = np.zeros(n, dtype=np.int64)
    total = 0
    for r in range(world):
        own = np.zeros(n, dtype=np.uint8)
        info = mds.mds_plan(n, r, world, 148, 12, own)
        cover += own
        total += info["pairs"]
        assert info["slabs"] == info["segments"] + info["tiles"]
        assert info["max_units_per_warp"] - info["min_units_per_warp"] <= 1   # balanced warps
    assert total == n * (n - 1) // 2
    assert np.all(cover == 1)


@pytest.mark.parametrize("ctas,wpc", [(147, 12), (147, 8), (147, 24), (1, 12), (73, 16)])
def test_plan_for_any_pair_cta_count(ctas, wpc):
    """With a tree prior the pass kernel plans its pairs on G - 1 CTAs (the last
    walks the tree); any CTA count must still tile the triangle, balanced."""
    for n in (65, 5392):
        info = mds.mds_plan(n, 0, 1, ctas, wpc)
        assert info["pairs"] == n * (n - 1) // 2
        assert info["max_units_per_warp"] - info["min_units_per_warp"] <= 1


def test_plan_scales_to_c5():
    info = mds.mds_plan(100000, 0, 1, 148, 12)
    assert info["pairs"] == 100000 * 99999 // 2
    assert info["pair_slots"] >= info["pairs"]
    assert info["pair_slots"] / info["pairs"] < 1.002       # padding overhead ~0.1%


def test_plan_rejects_bad_arguments():
    for args in [(1, 0, 1, 148, 12), (100, 2, 2, 148, 12), (100, 0, 1, 0, 12), (100, 0, 0, 148, 12)]:
        with pytest.raises(mds.MDSError):
            mds.mds_plan(*args)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1905_04582_b200 as m
        own = np.zeros(n, dtype=np.uint8)
        info = m.mds_plan(n, rank, world, 148, 12, own)
        # this rank's "partial": per row, the number of pairs (i, j<i) it owns,
        # plus a trailing scalar (its pair total) -- the n*d + 1 layout of the GPU partial
        part = torch.zeros(n + 1, dtype=torch.float64)
        rows = torch.from_numpy(own.astype(np.float64))
        part[:n] = rows * torch.arange(n, dtype=torch.float64)
        part[n] = float(info["pairs"])
        gathered = torch.empty(world * (n + 1), dtype=torch.float64)
        dist.all_gather_into_tensor(gathered, part)
        g = gathered.view(world, n + 1)
        combined = g[0].clone()
        for r in range(1, world):            # rank-ordered sum, as combine_kernel
            combined += g[r]
        ok = bool(torch.all(combined[:n] == torch.arange(n, dtype=torch.float64))) and \
            combined[n].item() == n * (n - 1) // 2
        # identical on every rank
        chk = torch.tensor([combined.sum().item()], dtype=torch.float64)
        allv = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allv, chk)
        same = all(v.item() == allv[0].item() for v in allv)
        q.put((rank, ok and same))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1000, 5392])
def test_gloo_world2_partition_and_combine(n):
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _ in res) == [0, 1]
    assert all(ok for _, ok in res)


def _oracle_worker(rank, world, port, n, d, q):
    """One rank of the N > 1 path's host logic with libmds replaced by the oracle:
    this rank's partial = the Eq. 2 / Eq. 6 sums over the pairs of ITS tile-rows
    (mds_plan's ownership; the oracle on Y with every other row missing), gathered
    through the binding's exchange callback (allgather_callback, the function
    libmds calls through mds_set_allgather) over gloo in host memory, then the
    rank-ordered combine -- equal to the full oracle and identical on every rank."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import workload
        import paper_1905_04582_b200 as m
        w = workload.Workload(n, d, p_missing=0.1, seed=n + world)
        y = w.y_packed()
        own = np.zeros(n, dtype=np.uint8)
        m.mds_plan(n, rank, world, 148, 12, own)
        rows = np.repeat(np.arange(n), np.arange(n))          # row i of each packed entry
        ymine = np.where(own[rows] == 1, y, np.nan)
        r = oracle.loglik_grad(ymine, w.x0, w.sigma, 1, want_absscale=False)
        cnt = n * d + 1
        send = np.empty(cnt)
        send[:-1] = r["grad"].ravel()
        send[-1] = r["loglik"]
        recv = np.empty(world * cnt)
        cb = m.allgather_callback(world, device="cpu")
        assert cb(None, send.ctypes.data, recv.ctypes.data, cnt, None) == 0
        g = recv.reshape(world, cnt)
        comb = g[0].copy()
        for k in range(1, world):                              # rank order, as combine_kernel
            comb += g[k]
        full = oracle.loglik_grad(y, w.x0, w.sigma, 1, want_absscale=False)
        ok = abs(comb[-1] - full["loglik"]) <= 1e-10 * abs(full["loglik"])
        G = full["grad"].ravel()
        ok = ok and bool(np.all(np.abs(comb[:-1] - G) <= np.maximum(1e-9 * np.abs(G), 1e-12)))
        digest = torch.tensor([float(np.frombuffer(comb.tobytes(), dtype=np.uint64).sum() % (1 << 52))])
        allv = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allv, digest.double())
        q.put((rank, ok and all(v.item() == allv[0].item() for v in allv)))
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,d,world", [(300, 2, 2), (517, 3, 3)])
def test_gloo_oracle_partials_exchange_and_combine(n, d, world):
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_oracle_worker, args=(r, world, port, n, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _ in res) == list(range(world))
    assert all(ok is True for _, ok in res), res
