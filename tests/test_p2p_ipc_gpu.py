"""The fused peer-memory exchange through IPC handles, as multi-GPU runs use it:
one PROCESS per rank, windows connected with mds_p2p_connect_ipc after an
all-gather of the cudaIpcMemHandle bytes over torch.distributed (gloo here,
127.0.0.1), MDS.use_p2p_exchange.

On the one GPU of a test box both processes' contexts share the device, so their
kernels are time-sliced rather than concurrent: a rank's pass kernel waits in the
exchange until the GPU switches to the other process, whose pass raises its flag
(compute preemption).  Slow, but it drives the real cross-process path: IPC
handles, peer windows of another process, system-scope release/acquire flags.
Results must be bitwise identical on both ranks and match the oracle.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, D = 300, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      MDS_P2P_TIMEOUT_S="30")
    try:
        import torch
        import torch.distributed as dist
        import paper_1905_04582_b200 as mds
        import workload
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        w = workload.Workload(N, D, p_missing=0.05, seed=111)
        st = torch.cuda.Stream()
        torch.cuda.set_stream(st)
        ctx = mds.MDS(N, D, "f64", True, rank=rank, world=world, stream=st)
        ctx.set_grid_limit(148 // world)
        ctx.set_dissimilarities_packed(w.y_packed())
        ctx.set_locations(w.x0)
        ctx.set_sigma(w.sigma)
        st.synchronize()
        ctx.use_p2p_exchange()
        assert ctx.p2p_connected()
        ll, g = ctx.log_likelihood_and_gradient()
        p0 = torch.from_numpy(w.normals(1, (N, D))).cuda()
        st.synchronize()
        dist.barrier()
        ctx.leapfrog_device(3, 0.002, 10.0, p0_dev=p0)
        x = ctx.get_locations()
        st.synchronize()
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()
        q.put((rank, ll, g, x, None))
    except Exception as e:  # reported to the parent
        q.put((rank, None, None, None, repr(e)))


def test_p2p_ipc_two_processes():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    import oracle
    import workload
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r, ll, g, x, err = q.get(timeout=400)
        assert err is None, (r, err)
        res[r] = (ll, g, x)
    for p in ps:
        p.join(timeout=60)
    assert res[0][0] == res[1][0] and np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])
    w = workload.Workload(N, D, p_missing=0.05, seed=111)
    ref = oracle.loglik_grad(w.y_packed(), w.x0, w.sigma, 1)
    assert res[0][0] == pytest.approx(ref["loglik"], rel=1e-10)
    np.testing.assert_allclose(res[0][1], ref["grad"], rtol=1e-9, atol=1e-12)
    lf = oracle.leapfrog(w.y_packed(), w.x0, w.normals(1, (N, D)), w.sigma, 0.002, 3, 1, prior_sd=10.0)
    np.testing.assert_allclose(res[0][2], lf["x"], rtol=1e-9, atol=1e-12)
