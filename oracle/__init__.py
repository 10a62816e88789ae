"""CPU oracle for the Bayesian-MDS hot path (arXiv 1905.04582).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_1905_04582_b200`` never imports it; the
two share no code.

The arithmetic lives in ``mds_oracle.c`` (plain serial C, fp64, libm,
Neumaier sums, ``-O2 -fno-fast-math -ffp-contract=off``); this module only
builds it with gcc and marshals numpy arrays through ctypes.  See the C file's
header for the passages each function follows (Eq. 1, 2, 5, 6 and
App. B).

Pins (tests/test_oracle_pins.py): scipy truncnorm / norm log-densities,
closed-form 3-4-5 triangle values (tests/golden/closed_forms.json), mpmath
brute force, central finite differences, invariants, and the closed-form
leapfrog map of a Gaussian target.  Every function here is pinned; none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mds_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11"]

_lib = None


def build(force: bool = False) -> str:
    """Compile mds_oracle.c -> liboracle.so with gcc (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        d_p = P(ctypes.c_double)
        i64 = ctypes.c_int64
        i32 = ctypes.c_int32
        lib.oracle_pair_term.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_int, d_p, d_p]
        lib.oracle_log_phi.argtypes = [ctypes.c_double]
        lib.oracle_log_phi.restype = ctypes.c_double
        lib.oracle_loglik_grad.argtypes = [i64, i32, d_p, d_p, ctypes.c_double, i32,
                                           d_p, d_p, d_p, P(i64), P(i64)]
        lib.oracle_loglik_rows.argtypes = [i64, i32, i64, i64, d_p, d_p, ctypes.c_double, i32, d_p, P(i64)]
        lib.oracle_grad_rows.argtypes = [i64, i32, i64, P(i64), d_p, d_p, ctypes.c_double, i32,
                                         d_p, d_p, d_p]
        lib.oracle_leapfrog.argtypes = [i64, i32, d_p, d_p, d_p, ctypes.c_double, i32,
                                        ctypes.c_double, ctypes.c_double, i32, d_p, d_p, d_p]
        lib.oracle_sigma_mh_step.argtypes = [i64, i32, d_p, d_p, ctypes.c_double, i32, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                             d_p, P(i32), d_p]
        lib.oracle_row_delta.argtypes = [i64, i32, d_p, d_p, i64, d_p, ctypes.c_double, i32, d_p]
        lib.oracle_rw_sweep.argtypes = [i64, i32, d_p, d_p, ctypes.c_double, i32, i64, P(i64), d_p, d_p,
                                        ctypes.c_double, ctypes.c_double, P(i64)]
        lib.oracle_cv_lpd.argtypes = [i64, i32, i64, P(i64), P(i64), d_p, i64, d_p, d_p, i32, d_p]
        _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def pack_lower(y_full: np.ndarray) -> np.ndarray:
    """Full n x n matrix -> packed strict lower triangle (row i: y_i0..y_i,i-1)."""
    n = y_full.shape[0]
    il, jl = np.tril_indices(n, -1)
    return _f64(y_full[il, jl])


def pair_term(y: float, d: float, sigma: float, truncation: int = 1):
    """(ell, coef) of one pair: Eq. 2 term and Eq. 6 coefficient."""
    lib = _load()
    e = ctypes.c_double()
    c = ctypes.c_double()
    if lib.oracle_pair_term(float(y), float(d), float(sigma), int(truncation),
                            ctypes.byref(e), ctypes.byref(c)):
        raise ValueError("invalid pair_term arguments")
    return e.value, c.value


def log_phi(t: float) -> float:
    return _load().oracle_log_phi(float(t))


def loglik_grad(y_packed: np.ndarray, x: np.ndarray, sigma: float, truncation: int = 1,
                want_absscale: bool = True):
    """Serial oracle over the packed lower triangle.

    Returns dict(loglik, grad (n,d), absscale (n,d) or None, n_obs, zero_pairs).
    """
    lib = _load()
    x = _f64(x)
    n, d = x.shape
    y_packed = _f64(y_packed)
    if y_packed.size != n * (n - 1) // 2:
        raise ValueError("y_packed must hold n(n-1)/2 entries")
    ll = ctypes.c_double()
    g = np.zeros((n, d))
    s = np.zeros((n, d)) if want_absscale else None
    nobs = ctypes.c_int64()
    nz = ctypes.c_int64()
    rc = lib.oracle_loglik_grad(n, d, _dp(y_packed), _dp(x), float(sigma), int(truncation),
                                ctypes.byref(ll), _dp(g), _dp(s) if s is not None else None,
                                ctypes.byref(nobs), ctypes.byref(nz))
    if rc:
        raise ValueError("invalid oracle arguments")
    return dict(loglik=ll.value, grad=g, absscale=s, n_obs=nobs.value, zero_pairs=nz.value)


def loglik_rows(i0: int, i1: int, y_rows: np.ndarray, x: np.ndarray, sigma: float, truncation: int = 1):
    """(log L over the pairs (i, j < i), i0 <= i < i1, n_obs of the range) from the
    packed rows i0..i1-1 (streaming form of loglik_grad's Eq. 2 sum for sizes whose
    packed triangle does not fit host memory; add chunk results in row order)."""
    lib = _load()
    x = _f64(x)
    n, d = x.shape
    y_rows = _f64(y_rows)
    lo = i0 * (i0 - 1) // 2 if i0 > 0 else 0
    if y_rows.size != i1 * (i1 - 1) // 2 - lo:
        raise ValueError("y_rows must hold rows i0..i1-1 of the packed triangle")
    ll = ctypes.c_double()
    nobs = ctypes.c_int64()
    if lib.oracle_loglik_rows(n, d, int(i0), int(i1), _dp(y_rows), _dp(x), float(sigma), int(truncation),
                              ctypes.byref(ll), ctypes.byref(nobs)):
        raise ValueError("invalid oracle arguments")
    return ll.value, nobs.value


def grad_rows(rows, yrows: np.ndarray, x: np.ndarray, sigma: float, truncation: int = 1):
    """Gradient rows (Eq. 6) for selected i, given y_ij for all j (yrows[r, j])."""
    lib = _load()
    x = _f64(x)
    n, d = x.shape
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    yrows = _f64(yrows)
    m = rows.size
    if yrows.shape != (m, n):
        raise ValueError("yrows must be (len(rows), n)")
    g = np.zeros((m, d))
    s = np.zeros((m, d))
    rl = np.zeros(m)
    rc = lib.oracle_grad_rows(n, d, m, rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                              _dp(yrows), _dp(x), float(sigma), int(truncation), _dp(g), _dp(s), _dp(rl))
    if rc:
        raise ValueError("invalid oracle arguments")
    return dict(grad=g, absscale=s, rowlik=rl)


def leapfrog(y_packed: np.ndarray, x0: np.ndarray, p0: np.ndarray, sigma: float, eps: float,
             n_steps: int, truncation: int = 1, prior_sd: float = 0.0):
    """n_steps leapfrog steps (Eq. 5 dynamics, M = I). Returns dict(x, p, H0, H1, loglik)."""
    lib = _load()
    x = _f64(x0).copy()
    p = _f64(p0).copy()
    n, d = x.shape
    H0 = ctypes.c_double()
    H1 = ctypes.c_double()
    ll = ctypes.c_double()
    rc = lib.oracle_leapfrog(n, d, _dp(_f64(y_packed)), _dp(x), _dp(p), float(sigma), int(truncation),
                             float(prior_sd), float(eps), int(n_steps),
                             ctypes.byref(H0), ctypes.byref(H1), ctypes.byref(ll))
    if rc:
        raise ValueError("invalid oracle arguments")
    return dict(x=x, p=p, H0=H0.value, H1=H1.value, loglik=ll.value)


def sigma_mh_step(y_packed: np.ndarray, x: np.ndarray, sigma: float, shape: float, rate: float, step: float,
                  z: float, u: float, truncation: int = 1):
    """One MH step on log sigma^2 (prior sigma^-2 ~ Gamma(shape, rate)).
    Returns dict(sigma, accepted, log_ratio)."""
    lib = _load()
    x = _f64(x)
    n, d = x.shape
    so = ctypes.c_double()
    acc = ctypes.c_int32()
    lr = ctypes.c_double()
    rc = lib.oracle_sigma_mh_step(n, d, _dp(_f64(y_packed)), _dp(x), float(sigma), int(truncation), float(shape),
                                  float(rate), float(step), float(z), float(u), ctypes.byref(so),
                                  ctypes.byref(acc), ctypes.byref(lr))
    if rc:
        raise ValueError("invalid oracle arguments")
    return dict(sigma=so.value, accepted=bool(acc.value), log_ratio=lr.value)


def row_delta(y_packed: np.ndarray, x: np.ndarray, i: int, x_new, sigma: float, truncation: int = 1) -> float:
    """Change of log L when x_i alone moves to x_new."""
    lib = _load()
    x = _f64(x)
    n, d = x.shape
    xn = _f64(x_new).reshape(d)
    out = ctypes.c_double()
    if lib.oracle_row_delta(n, d, _dp(_f64(y_packed)), _dp(x), int(i), _dp(xn), float(sigma), int(truncation),
                            ctypes.byref(out)):
        raise ValueError("invalid oracle arguments")
    return out.value


def rw_sweep(y_packed: np.ndarray, x0: np.ndarray, sigma: float, rows, z, u, step: float, prior_sd: float = 0.0,
             truncation: int = 1):
    """Sequential single-location random-walk Metropolis updates.  Returns (x, accepted)."""
    lib = _load()
    x = _f64(x0).copy()
    n, d = x.shape
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    z = _f64(z).reshape(rows.size, d)
    u = _f64(u).reshape(rows.size)
    acc = ctypes.c_int64()
    if lib.oracle_rw_sweep(n, d, _dp(_f64(y_packed)), _dp(x), float(sigma), int(truncation), rows.size,
                           rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(z), _dp(u), float(step),
                           float(prior_sd), ctypes.byref(acc)):
        raise ValueError("invalid oracle arguments")
    return x, acc.value


def cv_lpd(hi, hj, hy, xs, sigmas, truncation: int = 1) -> float:
    """Held-out log pointwise predictive density over S draws.
    xs: (S, n, d) posterior draws of X; sigmas: (S,)."""
    lib = _load()
    xs = _f64(xs)
    S, n, d = xs.shape
    hi = np.ascontiguousarray(hi, dtype=np.int64)
    hj = np.ascontiguousarray(hj, dtype=np.int64)
    hy = _f64(hy)
    sg = _f64(sigmas).reshape(S)
    out = ctypes.c_double()
    P = ctypes.POINTER(ctypes.c_int64)
    if lib.oracle_cv_lpd(n, d, hy.size, hi.ctypes.data_as(P), hj.ctypes.data_as(P), _dp(hy), S, _dp(xs), _dp(sg),
                         int(truncation), ctypes.byref(out)):
        raise ValueError("invalid oracle arguments")
    return out.value
