"""ctypes binding of libmds (include/mds.h): the same names, argument marshalling only.

Every function here forwards to the C-ABI entry point of the same name and
raises MDSError on a non-OK status.  No arithmetic of the method happens in
Python; there is no fallback: if libmds.so is missing or fails to load, import
fails loudly.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MDS_LIB_PATH overrides the in-tree library (A/B builds of the same sources)
LIB_PATH = os.environ.get("MDS_LIB_PATH") or os.path.join(HERE, "libmds.so")

MDS_F64, MDS_F32 = 0, 1
STATUS = {0: "MDS_OK", 1: "MDS_E_INVALID_ARG", 2: "MDS_E_STATE", 3: "MDS_E_OOM", 4: "MDS_E_CUDA",
          5: "MDS_E_COMM", 6: "MDS_E_UNSUPPORTED"}

# every symbol include/mds.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "mds_create", "mds_create_sharded", "mds_nccl_unique_id", "mds_has_communicator", "mds_destroy",
    "mds_set_stream",
    "mds_set_dissimilarities", "mds_set_dissimilarity_rows", "mds_set_dissimilarity_rows_device",
    "mds_set_locations", "mds_set_locations_device", "mds_set_sigma",
    "mds_log_likelihood", "mds_gradient", "mds_log_likelihood_and_gradient", "mds_evaluate_device",
    "mds_evaluate_partial_device", "mds_combine_partials_device",
    "mds_observed_pairs", "mds_zero_distance_pairs", "mds_set_timing", "mds_last_timing",
    "mds_hmc_trajectory", "mds_hmc_run", "mds_leapfrog_device", "mds_get_locations", "mds_get_momentum",
    "mds_set_allgather", "mds_plan",
    "mds_p2p_window", "mds_p2p_connect", "mds_p2p_connect_ipc", "mds_p2p_disconnect", "mds_p2p_connected",
    "mds_set_grid_limit",
    "mds_log_likelihood_at_sigma", "mds_sigma_mh_step", "mds_mcmc_run", "mds_row_loglik_delta", "mds_rw_sweep",
    "mds_cv_set_heldout", "mds_cv_accumulate", "mds_cv_lpd", "mds_set_tree_prior", "mds_tree_prior",
    "mds_last_error", "mds_status_string", "mds_version", "mds_device_info", "mds_measure_fma_peaks", "mds_l2_flush", "mds_l2_flush_clean",
]


class MDSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("tile_rows", "tiles", "pair_slots", "pairs", "segments", "slabs",
                                              "max_slabs_per_block", "min_units_per_warp", "max_units_per_warp",
                                              "ranges_per_warp")]


class HmcConfig(ctypes.Structure):
    _fields_ = [("n_iter", ctypes.c_int32), ("n_leapfrog", ctypes.c_int32), ("step_size", ctypes.c_double),
                ("prior_sd", ctypes.c_double), ("seed", ctypes.c_uint64)]


class HmcStats(ctypes.Structure):
    _fields_ = [("accepted", ctypes.c_int64), ("grad_evals", ctypes.c_int64), ("mean_abs_dH", ctypes.c_double),
                ("seconds", ctypes.c_double), ("final_loglik", ctypes.c_double)]


class SigmaPrior(ctypes.Structure):
    _fields_ = [("shape", ctypes.c_double), ("rate", ctypes.c_double)]


class McmcStats(ctypes.Structure):
    _fields_ = [("accepted_x", ctypes.c_int64), ("accepted_sigma", ctypes.c_int64), ("grad_evals", ctypes.c_int64),
                ("seconds", ctypes.c_double), ("final_loglik", ctypes.c_double), ("final_sigma", ctypes.c_double)]


# int (*)(void* user, const double* send_dev, double* recv_dev, int64_t count, void* stream)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_int64, ctypes.c_void_p)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError("libmds.so not built at %s -- run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)" % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    P = ctypes.POINTER
    sig = {
        "mds_create": [i64, i32, i32, i32, P(vp)],
        "mds_create_sharded": [i64, i32, i32, i32, i32, i32, vp, P(vp)],
        "mds_nccl_unique_id": [vp],
        "mds_has_communicator": [vp, P(i32)],
        "mds_set_stream": [vp, vp],
        "mds_set_dissimilarities": [vp, dp, i64],
        "mds_set_dissimilarity_rows": [vp, i64, i64, dp],
        "mds_set_dissimilarity_rows_device": [vp, i64, i64, dp],
        "mds_set_locations": [vp, dp],
        "mds_set_locations_device": [vp, dp],
        "mds_set_sigma": [vp, ctypes.c_double],
        "mds_log_likelihood": [vp, dp],
        "mds_gradient": [vp, dp],
        "mds_log_likelihood_and_gradient": [vp, dp, dp],
        "mds_evaluate_device": [vp, dp, dp],
        "mds_evaluate_partial_device": [vp, dp],
        "mds_combine_partials_device": [vp, dp, i32, dp, dp],
        "mds_observed_pairs": [vp, P(i64)],
        "mds_zero_distance_pairs": [vp, P(i64)],
        "mds_set_timing": [vp, i32],
        "mds_last_timing": [vp, P(ctypes.c_float), P(ctypes.c_float)],
        "mds_hmc_trajectory": [vp, P(HmcConfig), dp, dp, dp, P(ctypes.c_double), P(ctypes.c_double)],
        "mds_hmc_run": [vp, P(HmcConfig), dp, P(HmcStats)],
        "mds_leapfrog_device": [vp, P(HmcConfig), dp],
        "mds_get_locations": [vp, dp],
        "mds_get_momentum": [vp, dp],
        "mds_set_allgather": [vp, ALLGATHER_FN, vp],
        "mds_p2p_window": [vp, P(vp), vp],
        "mds_p2p_connect": [vp, P(vp)],
        "mds_p2p_connect_ipc": [vp, vp],
        "mds_p2p_connected": [vp, P(i32)],
        "mds_p2p_disconnect": [vp],
        "mds_set_grid_limit": [vp, i32],
        "mds_plan": [i64, i32, i32, i32, i32, P(PlanInfo), vp],
        "mds_device_info": [P(i32), P(i32), P(i32)],
        "mds_measure_fma_peaks": [P(ctypes.c_double), P(ctypes.c_double)],
        "mds_l2_flush": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t],
        "mds_l2_flush_clean": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t],
        "mds_log_likelihood_at_sigma": [vp, ctypes.c_double, P(ctypes.c_double)],
        "mds_cv_set_heldout": [vp, i64, dp, dp, dp],
        "mds_set_tree_prior": [vp, i64, dp, dp, dp, dp],
        "mds_tree_prior": [vp, dp, dp],
        "mds_cv_accumulate": [vp],
        "mds_cv_lpd": [vp, P(ctypes.c_double), P(i64)],
        "mds_row_loglik_delta": [vp, i64, dp, P(ctypes.c_double)],
        "mds_rw_sweep": [vp, i64, dp, dp, dp, ctypes.c_double, ctypes.c_double, P(i64)],
        "mds_mcmc_run": [vp, P(HmcConfig), P(SigmaPrior), ctypes.c_double, dp, P(McmcStats)],
        "mds_sigma_mh_step": [vp, P(SigmaPrior), ctypes.c_double, ctypes.c_double, ctypes.c_double, P(i32),
                              P(ctypes.c_double)],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.mds_destroy.argtypes = [vp]
    lib.mds_destroy.restype = None
    lib.mds_last_error.argtypes = [vp]
    lib.mds_last_error.restype = ctypes.c_char_p
    lib.mds_status_string.argtypes = [ctypes.c_int]
    lib.mds_status_string.restype = ctypes.c_char_p
    lib.mds_version.argtypes = []
    lib.mds_version.restype = ctypes.c_char_p
    return lib


lib = _load()


def _check(st: int, ctx=None):
    if st != 0:
        msg = lib.mds_last_error(ctx).decode() if ctx else lib.mds_status_string(st).decode()
        raise MDSError(st, msg)


def _ptr(a):
    """Pointer of a numpy array (host) or a torch tensor / int (device)."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


# ---- same-name wrappers ---------------------------------------------------
def mds_create(n, d, precision=MDS_F64, truncation=1):
    h = ctypes.c_void_p()
    _check(lib.mds_create(int(n), int(d), int(precision), int(truncation), ctypes.byref(h)))
    return h


MDS_NCCL_ID_BYTES = 128


def mds_create_sharded(n, d, precision, truncation, rank, world, nccl_unique_id: bytes | None = None):
    """nccl_unique_id: the MDS_NCCL_ID_BYTES bytes of mds_nccl_unique_id() (same on every rank; the call is
    then collective and the context owns an NCCL communicator), or None (exchange via mds_set_allgather)."""
    h = ctypes.c_void_p()
    idbuf = None
    if nccl_unique_id is not None:
        if len(nccl_unique_id) != MDS_NCCL_ID_BYTES:
            raise ValueError("nccl_unique_id must be %d bytes" % MDS_NCCL_ID_BYTES)
        idbuf = ctypes.create_string_buffer(bytes(nccl_unique_id), MDS_NCCL_ID_BYTES)
    _check(lib.mds_create_sharded(int(n), int(d), int(precision), int(truncation), int(rank), int(world),
                                  idbuf, ctypes.byref(h)))
    return h


def mds_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(MDS_NCCL_ID_BYTES)
    _check(lib.mds_nccl_unique_id(buf))
    return buf.raw


def mds_has_communicator(ctx) -> bool:
    v = ctypes.c_int32()
    _check(lib.mds_has_communicator(ctx, ctypes.byref(v)), ctx)
    return bool(v.value)


def mds_destroy(ctx):
    lib.mds_destroy(ctx)


def mds_set_stream(ctx, stream):
    _check(lib.mds_set_stream(ctx, stream), ctx)


def mds_set_dissimilarities(ctx, y, ld):
    _check(lib.mds_set_dissimilarities(ctx, _ptr(y), int(ld)), ctx)


def mds_set_dissimilarity_rows(ctx, i0, i1, y_lower):
    _check(lib.mds_set_dissimilarity_rows(ctx, int(i0), int(i1), _ptr(y_lower)), ctx)


def mds_set_dissimilarity_rows_device(ctx, i0, i1, y_dev):
    _check(lib.mds_set_dissimilarity_rows_device(ctx, int(i0), int(i1), _ptr(y_dev)), ctx)


def mds_set_locations(ctx, x):
    _check(lib.mds_set_locations(ctx, _ptr(x)), ctx)


def mds_set_locations_device(ctx, x_dev):
    _check(lib.mds_set_locations_device(ctx, _ptr(x_dev)), ctx)


def mds_set_sigma(ctx, sigma):
    _check(lib.mds_set_sigma(ctx, float(sigma)), ctx)


def mds_log_likelihood(ctx, out):
    _check(lib.mds_log_likelihood(ctx, _ptr(out)), ctx)


def mds_gradient(ctx, grad):
    _check(lib.mds_gradient(ctx, _ptr(grad)), ctx)


def mds_log_likelihood_and_gradient(ctx, loglik, grad):
    _check(lib.mds_log_likelihood_and_gradient(ctx, _ptr(loglik), _ptr(grad)), ctx)


def mds_evaluate_device(ctx, loglik_dev, grad_dev):
    _check(lib.mds_evaluate_device(ctx, _ptr(loglik_dev), _ptr(grad_dev)), ctx)


def mds_evaluate_partial_device(ctx, part_dev):
    _check(lib.mds_evaluate_partial_device(ctx, _ptr(part_dev)), ctx)


def mds_combine_partials_device(ctx, gathered_dev, world, loglik_dev, grad_dev):
    _check(lib.mds_combine_partials_device(ctx, _ptr(gathered_dev), int(world), _ptr(loglik_dev),
                                           _ptr(grad_dev)), ctx)


def mds_observed_pairs(ctx):
    v = ctypes.c_int64()
    _check(lib.mds_observed_pairs(ctx, ctypes.byref(v)), ctx)
    return v.value


def mds_zero_distance_pairs(ctx):
    v = ctypes.c_int64()
    _check(lib.mds_zero_distance_pairs(ctx, ctypes.byref(v)), ctx)
    return v.value


def mds_set_timing(ctx, enable):
    _check(lib.mds_set_timing(ctx, int(bool(enable))), ctx)


def mds_l2_flush(ctx, dev_ptr, nbytes):
    _check(lib.mds_l2_flush(ctx, ctypes.c_void_p(dev_ptr), ctypes.c_size_t(nbytes)), ctx)


def mds_l2_flush_clean(ctx, dev_ptr, nbytes):
    _check(lib.mds_l2_flush_clean(ctx, ctypes.c_void_p(dev_ptr), ctypes.c_size_t(nbytes)), ctx)


def mds_last_timing(ctx):
    a, b = ctypes.c_float(), ctypes.c_float()
    _check(lib.mds_last_timing(ctx, ctypes.byref(a), ctypes.byref(b)), ctx)
    return a.value, b.value


def mds_hmc_trajectory(ctx, cfg: HmcConfig, p0, x_out=None, p_out=None):
    h0, h1 = ctypes.c_double(), ctypes.c_double()
    _check(lib.mds_hmc_trajectory(ctx, ctypes.byref(cfg), _ptr(p0), _ptr(x_out), _ptr(p_out),
                                  ctypes.byref(h0), ctypes.byref(h1)), ctx)
    return h0.value, h1.value


def mds_hmc_run(ctx, cfg: HmcConfig, x_inout=None):
    st = HmcStats()
    _check(lib.mds_hmc_run(ctx, ctypes.byref(cfg), _ptr(x_inout), ctypes.byref(st)), ctx)
    return st


def mds_leapfrog_device(ctx, cfg: HmcConfig, p0_dev=None):
    _check(lib.mds_leapfrog_device(ctx, ctypes.byref(cfg), _ptr(p0_dev)), ctx)


def mds_get_locations(ctx, x):
    _check(lib.mds_get_locations(ctx, _ptr(x)), ctx)


def mds_get_momentum(ctx, p):
    _check(lib.mds_get_momentum(ctx, _ptr(p)), ctx)


def mds_set_allgather(ctx, fn, user=None):
    """fn: an ALLGATHER_FN instance (keep a reference alive while ctx lives)."""
    _check(lib.mds_set_allgather(ctx, fn, user), ctx)


MDS_IPC_HANDLE_BYTES = 64


def mds_p2p_window(ctx):
    """-> (window device address, cudaIpcMemHandle_t bytes) of this context's exchange window."""
    addr = ctypes.c_void_p()
    h = ctypes.create_string_buffer(MDS_IPC_HANDLE_BYTES)
    _check(lib.mds_p2p_window(ctx, ctypes.byref(addr), h), ctx)
    return addr.value, h.raw


def mds_p2p_connect(ctx, windows):
    """windows: the world's window device addresses (ints), rank order."""
    arr = (ctypes.c_void_p * len(windows))(*[int(w) for w in windows])
    _check(lib.mds_p2p_connect(ctx, arr), ctx)


def mds_p2p_connect_ipc(ctx, handles):
    """handles: the world's IPC handle bytes (MDS_IPC_HANDLE_BYTES each), rank order."""
    buf = ctypes.create_string_buffer(b"".join(bytes(h) for h in handles))
    _check(lib.mds_p2p_connect_ipc(ctx, buf), ctx)


def mds_p2p_disconnect(ctx):
    _check(lib.mds_p2p_disconnect(ctx), ctx)


def mds_p2p_connected(ctx) -> bool:
    v = ctypes.c_int32()
    _check(lib.mds_p2p_connected(ctx, ctypes.byref(v)), ctx)
    return bool(v.value)


def mds_set_grid_limit(ctx, ctas):
    _check(lib.mds_set_grid_limit(ctx, int(ctas)), ctx)


def mds_plan(n, rank, world, ctas, warps_per_cta, owned_rows=None):
    """Host-only work plan (no GPU needed).  owned_rows: optional uint8 array of n."""
    info = PlanInfo()
    _check(lib.mds_plan(int(n), int(rank), int(world), int(ctas), int(warps_per_cta), ctypes.byref(info),
                        _ptr(owned_rows)))
    return {f: getattr(info, f) for f, _ in PlanInfo._fields_}


def mds_log_likelihood_at_sigma(ctx, sigma):
    v = ctypes.c_double()
    _check(lib.mds_log_likelihood_at_sigma(ctx, float(sigma), ctypes.byref(v)), ctx)
    return v.value


def mds_sigma_mh_step(ctx, shape, rate, step, z, u):
    """Returns (accepted: bool, log_ratio: float)."""
    pr = SigmaPrior(float(shape), float(rate))
    acc, lr = ctypes.c_int32(), ctypes.c_double()
    _check(lib.mds_sigma_mh_step(ctx, ctypes.byref(pr), float(step), float(z), float(u), ctypes.byref(acc),
                                 ctypes.byref(lr)), ctx)
    return bool(acc.value), lr.value


def mds_row_loglik_delta(ctx, i, x_new_i):
    v = ctypes.c_double()
    _check(lib.mds_row_loglik_delta(ctx, int(i), _ptr(x_new_i), ctypes.byref(v)), ctx)
    return v.value


def mds_rw_sweep(ctx, rows, z, u, step, prior_sd):
    """rows: int64 (k,), z: float64 (k, d), u: float64 (k,).  Returns the acceptance count."""
    acc = ctypes.c_int64()
    _check(lib.mds_rw_sweep(ctx, int(rows.size), _ptr(rows), _ptr(z), _ptr(u), float(step), float(prior_sd),
                            ctypes.byref(acc)), ctx)
    return acc.value


def mds_set_tree_prior(ctx, parent, t, mu0=None, sigma_cov=None):
    """parent: int64 (n_nodes,), t: float64 (n_nodes,); mu0 (d,), sigma_cov (d, d) or None.
    An empty parent array removes the tree prior."""
    _check(lib.mds_set_tree_prior(ctx, int(parent.size), _ptr(parent), _ptr(t), _ptr(mu0), _ptr(sigma_cov)), ctx)


def mds_tree_prior(ctx, grad=None):
    """Returns log p(X); fills grad (n x d float64) if given."""
    v = ctypes.c_double()
    _check(lib.mds_tree_prior(ctx, ctypes.byref(v), _ptr(grad)), ctx)
    return v.value


def mds_cv_set_heldout(ctx, i, j, y):
    """i, j: int64 arrays (m,), y: float64 (m,)."""
    _check(lib.mds_cv_set_heldout(ctx, int(y.size), _ptr(i), _ptr(j), _ptr(y)), ctx)


def mds_cv_accumulate(ctx):
    _check(lib.mds_cv_accumulate(ctx), ctx)


def mds_cv_lpd(ctx):
    """Returns (lpd, draws)."""
    v, s = ctypes.c_double(), ctypes.c_int64()
    _check(lib.mds_cv_lpd(ctx, ctypes.byref(v), ctypes.byref(s)), ctx)
    return v.value, s.value


def mds_mcmc_run(ctx, cfg: HmcConfig, shape, rate, sigma_step, x_inout=None):
    pr = SigmaPrior(float(shape), float(rate))
    st = McmcStats()
    _check(lib.mds_mcmc_run(ctx, ctypes.byref(cfg), ctypes.byref(pr), float(sigma_step), _ptr(x_inout),
                            ctypes.byref(st)), ctx)
    return st


def mds_last_error(ctx):
    return lib.mds_last_error(ctx).decode()


def mds_status_string(s):
    return lib.mds_status_string(int(s)).decode()


def mds_version():
    return lib.mds_version().decode()


def mds_device_info():
    a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib.mds_device_info(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value


def mds_measure_fma_peaks():
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(lib.mds_measure_fma_peaks(ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value
