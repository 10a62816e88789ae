"""B200-native hot path of Bayesian MDS (Holbrook et al., arXiv 1905.04582).

The product is ``libmds.so`` (sm_100a CUDA, C-ABI declared in include/mds.h).
This package is its thin Python binding: ``_abi`` exposes every C entry point
under the same name; ``MDS`` below only bundles a context handle with numpy /
torch argument marshalling.  All arithmetic runs in the CUDA kernels; there
is no CPU path.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from ._abi import *  # noqa: F401,F403  (mds_* same-name wrappers)
from ._abi import MDS_F32, MDS_F64, HmcConfig, HmcStats, MDSError

__all__ = ["MDS", "MDSError", "HmcConfig", "HmcStats", "MDS_F64", "MDS_F32"] + _abi.EXPORTS

def _wrap_dev(ptr: int, count: int, dev):
    """A torch float64 view of `count` doubles of device memory at ptr (no copy)."""
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                    "version": 3, "strides": None, "stream": None}

    return torch.as_tensor(_CAI(), device=dev)


def _device_f64(t, numel: int, what: str):
    """A torch tensor handed to a *_device entry point must be CUDA fp64,
    contiguous and of the expected size (the C side reads raw doubles)."""
    if not getattr(t, "is_cuda", False):
        raise TypeError("%s: expected a CUDA tensor (got device %s)" % (what, getattr(t, "device", "?")))
    import torch
    if t.dtype != torch.float64:
        raise TypeError("%s: expected torch.float64 (got %s)" % (what, t.dtype))
    if not t.is_contiguous():
        raise ValueError("%s: expected a contiguous tensor" % what)
    if t.numel() != numel:
        raise ValueError("%s: expected %d values (got %d)" % (what, numel, t.numel()))
    return t


def allgather_callback(world: int, group=None, host_staged: bool = False, owner=None, device=None):
    """The mds_allgather_fn of a torch.distributed exchange: gather `count` doubles
    at send from every rank into recv[world][count], rank order, stream-ordered
    on the stream libmds passes (marshalling only).

    host_staged=False: send/recv are device pointers, all_gather_into_tensor on
    the passed stream (NCCL).  host_staged=True: device -> host copy, all_gather
    through the (gloo) group, host -> device copy, all on that stream; with
    device="cpu" the pointers are host memory (CPU tests of the exchange logic)."""
    import torch
    import torch.distributed as dist

    def _host(ptr, count):
        buf = (ctypes.c_double * int(count)).from_address(int(ptr))
        return torch.frombuffer(buf, dtype=torch.float64)

    def _ag(user, send, recv, count, stream):
        try:
            if device == "cpu":
                s, r = _host(send, count), _host(recv, count * world)
                parts = list(r.view(world, count).unbind(0))
                dist.all_gather(parts, s, group=group)
                return 0
            dev = torch.device("cuda", torch.cuda.current_device())
            st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
            with torch.cuda.stream(st):
                s = _wrap_dev(send, count, dev)
                r = _wrap_dev(recv, count * world, dev)
                if not host_staged:
                    dist.all_gather_into_tensor(r, s, group=group)
                else:
                    hs = s.cpu()                       # synchronises the passed stream
                    parts = [torch.empty_like(hs) for _ in range(world)]
                    dist.all_gather(parts, hs, group=group)
                    r.copy_(torch.cat(parts).to(dev, non_blocking=False))
            return 0
        except Exception as e:  # reported as MDS_E_COMM
            if owner is not None:
                owner.last_exchange_error = repr(e)
            return 1

    return _ag


_PREC = {"f64": MDS_F64, "fp64": MDS_F64, "float64": MDS_F64, MDS_F64: MDS_F64,
         "f32": MDS_F32, "fp32": MDS_F32, "float32": MDS_F32, MDS_F32: MDS_F32}


class MDS:
    """One libmds context (marshalling only)."""

    def __init__(self, n: int, d: int, precision="f64", truncation: bool = True,
                 rank: int = 0, world: int = 1, stream=None, nccl_unique_id: bytes | None = None):
        """world > 1 (or a unique id): a row-sharded context owning tile-rows r mod world == rank.
        With nccl_unique_id (mds_nccl_unique_id() on one rank, the same bytes on all) creation is
        collective and the context owns its NCCL communicator; without, register an exchange
        (use_torch_allgather / mds_set_allgather)."""
        self.n, self.d = int(n), int(d)
        self.precision = _PREC[precision]
        self.rank, self.world = int(rank), int(world)
        if world == 1 and nccl_unique_id is None:
            self.ctx = _abi.mds_create(n, d, self.precision, int(bool(truncation)))
        else:
            self.ctx = _abi.mds_create_sharded(n, d, self.precision, int(bool(truncation)), rank, world,
                                               nccl_unique_id)
        if stream is not None:
            self.set_stream(stream)

    # lifetime
    def close(self):
        if getattr(self, "ctx", None):
            _abi.mds_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_stream(self, stream):
        """stream: a torch.cuda.Stream, a raw cudaStream_t int, or None."""
        h = getattr(stream, "cuda_stream", stream)
        _abi.mds_set_stream(self.ctx, h)

    # inputs
    def set_dissimilarities(self, y_full: np.ndarray):
        y = np.ascontiguousarray(y_full, dtype=np.float64)
        _abi.mds_set_dissimilarities(self.ctx, y, y.shape[1])

    def set_dissimilarity_rows(self, i0: int, i1: int, y_lower):
        if hasattr(y_lower, "data_ptr"):
            lo = i0 * (i0 - 1) // 2 if i0 > 0 else 0
            _device_f64(y_lower, i1 * (i1 - 1) // 2 - lo, "set_dissimilarity_rows")
            _abi.mds_set_dissimilarity_rows_device(self.ctx, i0, i1, y_lower)
        else:
            _abi.mds_set_dissimilarity_rows(self.ctx, i0, i1, np.ascontiguousarray(y_lower, dtype=np.float64))

    def set_dissimilarities_packed(self, y_packed):
        self.set_dissimilarity_rows(0, self.n, y_packed)

    def set_locations(self, x):
        if hasattr(x, "data_ptr"):
            _abi.mds_set_locations_device(self.ctx, _device_f64(x, self.n * self.d, "set_locations"))
        else:
            _abi.mds_set_locations(self.ctx, np.ascontiguousarray(x, dtype=np.float64))

    def set_sigma(self, sigma: float):
        _abi.mds_set_sigma(self.ctx, sigma)

    # evaluation
    def log_likelihood_and_gradient(self):
        ll = np.zeros(1)
        g = np.zeros((self.n, self.d))
        _abi.mds_log_likelihood_and_gradient(self.ctx, ll, g)
        return float(ll[0]), g

    def log_likelihood(self) -> float:
        ll = np.zeros(1)
        _abi.mds_log_likelihood(self.ctx, ll)
        return float(ll[0])

    def gradient(self) -> np.ndarray:
        g = np.zeros((self.n, self.d))
        _abi.mds_gradient(self.ctx, g)
        return g

    def evaluate_device(self, loglik_dev, grad_dev):
        if loglik_dev is not None:
            _device_f64(loglik_dev, 1, "evaluate_device(loglik)")
        if grad_dev is not None:
            _device_f64(grad_dev, self.n * self.d, "evaluate_device(grad)")
        _abi.mds_evaluate_device(self.ctx, loglik_dev, grad_dev)

    def evaluate_partial_device(self, part_dev):
        _abi.mds_evaluate_partial_device(self.ctx, _device_f64(part_dev, self.n * self.d + 1, "evaluate_partial"))

    def combine_partials_device(self, gathered_dev, world, loglik_dev, grad_dev):
        _device_f64(gathered_dev, int(world) * (self.n * self.d + 1), "combine_partials(gathered)")
        if loglik_dev is not None:
            _device_f64(loglik_dev, 1, "combine_partials(loglik)")
        if grad_dev is not None:
            _device_f64(grad_dev, self.n * self.d, "combine_partials(grad)")
        _abi.mds_combine_partials_device(self.ctx, gathered_dev, world, loglik_dev, grad_dev)

    # diagnostics / timing
    def observed_pairs(self) -> int:
        return _abi.mds_observed_pairs(self.ctx)

    def zero_distance_pairs(self) -> int:
        return _abi.mds_zero_distance_pairs(self.ctx)

    def set_timing(self, on: bool = True):
        _abi.mds_set_timing(self.ctx, on)

    def l2_flush(self, buf):
        """Overwrite the device tensor `buf` (> L2) with the pass kernel's launch
        shape (timing utility, mds_l2_flush)."""
        _abi.mds_l2_flush(self.ctx, buf.data_ptr(), buf.numel() * buf.element_size())

    def l2_flush_clean(self, buf):
        """Write the first half of `buf`, read the second half (each > L2): a cold and
        clean L2 for the next kernel (timing utility, mds_l2_flush_clean)."""
        _abi.mds_l2_flush_clean(self.ctx, buf.data_ptr(), buf.numel() * buf.element_size())

    def last_timing(self):
        return _abi.mds_last_timing(self.ctx)

    @staticmethod
    def shared_nccl_id(group=None) -> bytes:
        """A fresh NCCL unique id made on rank 0 of torch.distributed and broadcast to every
        rank (for MDS(..., nccl_unique_id=...))."""
        import torch.distributed as dist
        obj = [_abi.mds_nccl_unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return obj[0]

    def has_communicator(self) -> bool:
        return _abi.mds_has_communicator(self.ctx)

    def use_torch_allgather(self, group=None, host_staged: bool = False):
        """Register a torch.distributed all-gather as the exchange of this sharded
        context (mds_set_allgather; only for contexts created without an NCCL id).
        host_staged: stage through host memory (gloo process groups, e.g. several
        ranks sharing one GPU in tests); else all_gather_into_tensor on device (NCCL)."""
        self._ag_cb = _abi.ALLGATHER_FN(allgather_callback(self.world, group, host_staged, owner=self))
        _abi.mds_set_allgather(self.ctx, self._ag_cb, None)

    def p2p_window(self):
        """(device address, IPC handle bytes) of this context's peer-memory exchange window."""
        return _abi.mds_p2p_window(self.ctx)

    def p2p_connect(self, windows):
        """Same-process ranks: the world's window addresses in rank order."""
        _abi.mds_p2p_connect(self.ctx, windows)

    def use_p2p_exchange(self, group=None):
        """Multi-process ranks (one per GPU): all-gather the windows' IPC handles
        through torch.distributed and connect the fused peer-memory exchange
        (mds_p2p_connect_ipc).  Collective over the group."""
        import torch.distributed as dist
        _, h = self.p2p_window()
        hs = [None] * self.world
        dist.all_gather_object(hs, h, group=group)
        err = None
        try:
            _abi.mds_p2p_connect_ipc(self.ctx, hs)
        except MDSError as e:           # (its handshake failed: the context stays on its other exchange)
            err = e
        oks = [None] * self.world
        dist.all_gather_object(oks, err is None, group=group)
        if not all(oks):                # every rank leaves together, or none would match
            if err is None:
                _abi.mds_p2p_disconnect(self.ctx)
            raise err or MDSError(5, "peer-memory exchange: another rank's handshake failed")

    def p2p_connected(self) -> bool:
        return _abi.mds_p2p_connected(self.ctx)

    def set_grid_limit(self, ctas: int):
        _abi.mds_set_grid_limit(self.ctx, ctas)

    def get_locations(self) -> np.ndarray:
        x = np.zeros((self.n, self.d))
        _abi.mds_get_locations(self.ctx, x)
        return x

    def get_momentum(self) -> np.ndarray:
        p = np.zeros((self.n, self.d))
        _abi.mds_get_momentum(self.ctx, p)
        return p

    def leapfrog_device(self, n_steps: int, step_size: float, prior_sd: float = 0.0, p0_dev=None):
        cfg = HmcConfig(0, int(n_steps), float(step_size), float(prior_sd), 0)
        if p0_dev is not None:
            _device_f64(p0_dev, self.n * self.d, "leapfrog_device(p0)")
        _abi.mds_leapfrog_device(self.ctx, cfg, p0_dev)

    # sigma side
    def log_likelihood_at_sigma(self, sigma: float) -> float:
        return _abi.mds_log_likelihood_at_sigma(self.ctx, sigma)

    def sigma_mh_step(self, shape: float, rate: float, step: float, z: float, u: float):
        """One MH update of sigma^2 (random walk on log sigma^2, caller-drawn z, u).
        Returns (accepted, log_ratio); the context's sigma moves on acceptance."""
        return _abi.mds_sigma_mh_step(self.ctx, shape, rate, step, z, u)

    def mcmc_run(self, n_iter: int, n_leapfrog: int, step_size: float, prior_sd: float, seed: int,
                 shape: float, rate: float, sigma_step: float, x0: np.ndarray | None = None):
        """PAPER.md:672's sampler: per iteration one HMC transition of X, then one MH
        update of sigma^2 (prior sigma^-2 ~ Gamma(shape, rate)).  Returns (x, stats)."""
        cfg = HmcConfig(int(n_iter), int(n_leapfrog), float(step_size), float(prior_sd), int(seed))
        x = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64).copy()
        st = _abi.mds_mcmc_run(self.ctx, cfg, shape, rate, sigma_step, x)
        return x, dict(accepted_x=st.accepted_x, accepted_sigma=st.accepted_sigma, grad_evals=st.grad_evals,
                       seconds=st.seconds, final_loglik=st.final_loglik, final_sigma=st.final_sigma)

    # phylogenetic prior
    def set_tree_prior(self, parent, t, mu0=None, sigma_cov=None):
        f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
        _abi.mds_set_tree_prior(self.ctx, np.ascontiguousarray(parent, dtype=np.int64), f(t), f(mu0), f(sigma_cov))

    def clear_tree_prior(self):
        _abi.mds_set_tree_prior(self.ctx, np.zeros(0, dtype=np.int64), np.zeros(0))

    def tree_prior(self):
        """(log p(X), d log p / dX) under the tree prior at the current X."""
        g = np.zeros((self.n, self.d))
        lp = _abi.mds_tree_prior(self.ctx, g)
        return lp, g

    # cross-validation
    def cv_set_heldout(self, i, j, y):
        _abi.mds_cv_set_heldout(self.ctx, np.ascontiguousarray(i, dtype=np.int64),
                                np.ascontiguousarray(j, dtype=np.int64), np.ascontiguousarray(y, dtype=np.float64))

    def cv_accumulate(self):
        _abi.mds_cv_accumulate(self.ctx)

    def cv_lpd(self):
        """(lpd, draws) of the held-out fold over the draws accumulated."""
        return _abi.mds_cv_lpd(self.ctx)

    # single-location updates
    def row_loglik_delta(self, i: int, x_new_i) -> float:
        return _abi.mds_row_loglik_delta(self.ctx, i, np.ascontiguousarray(x_new_i, dtype=np.float64))

    def rw_sweep(self, rows, z, u, step: float, prior_sd: float = 0.0) -> int:
        """Sequential random-walk Metropolis updates of single locations (caller-drawn
        rows, z, u); X moves in place.  Returns the number accepted."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        z = np.ascontiguousarray(z, dtype=np.float64).reshape(rows.size, self.d)
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(rows.size)
        return _abi.mds_rw_sweep(self.ctx, rows, z, u, step, prior_sd)

    # HMC
    def hmc_trajectory(self, p0: np.ndarray, step_size: float, n_leapfrog: int, prior_sd: float = 0.0):
        cfg = HmcConfig(0, int(n_leapfrog), float(step_size), float(prior_sd), 0)
        x = np.zeros((self.n, self.d))
        p = np.zeros((self.n, self.d))
        h0, h1 = _abi.mds_hmc_trajectory(self.ctx, cfg, np.ascontiguousarray(p0, dtype=np.float64), x, p)
        return dict(x=x, p=p, H0=h0, H1=h1)

    def hmc_run(self, n_iter: int, n_leapfrog: int, step_size: float, prior_sd: float, seed: int,
                x0: np.ndarray | None = None):
        cfg = HmcConfig(int(n_iter), int(n_leapfrog), float(step_size), float(prior_sd), int(seed))
        x = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64).copy()
        st = _abi.mds_hmc_run(self.ctx, cfg, x)
        return x, dict(accepted=st.accepted, grad_evals=st.grad_evals, mean_abs_dH=st.mean_abs_dH,
                       seconds=st.seconds, final_loglik=st.final_loglik)
