"""Seeded synthetic MDS workloads, shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic (that lives separately in ``oracle/``
and in ``paper_1905_04582_b200/csrc``); it only simulates inputs from the data
model of PAPER.md:78-83 (Eq. 1).  See ``gen.c`` for the recipe.

Configs follow BASELINE.json ``configs`` (C1..C5); base seed
S = 1905045820 + config index.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libworkload.so")
_lib = None

BASE_SEED = 1905045820
N_CLUSTERS = 189  # 189 countries

# name -> (index, n, d, kind, p_missing); BASELINE.json configs[0..4]
CONFIGS = {
    "C1": (0, 64, 2, "clustered", 0.0),
    "C2": (1, 5392, 2, "clustered", 0.0),
    "C3": (2, 5392, 2, "clustered", 0.0),
    "C4": (3, 30000, 6, "clustered", 0.10),
    "C5": (4, 100000, 2, "clustered", 0.0),
}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        d_p = P(ctypes.c_double)
        i64, i32, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        lib.wl_latent.argtypes = [i64, i32, i32, u64, ctypes.c_double, i32, d_p, d_p]
        lib.wl_dissim_rows.argtypes = [i64, i32, d_p, u64, ctypes.c_double, ctypes.c_double, i64, i64, d_p]
        lib.wl_dissim_full_rows.argtypes = [i64, i32, d_p, u64, ctypes.c_double, ctypes.c_double, i64,
                                            P(i64), d_p]
        lib.wl_normals.argtypes = [u64, u64, i64, d_p]
        lib.wl_set_threads.argtypes = [i32]
        _lib = lib
    return _lib


def set_threads(n: int) -> None:
    """Threads of the row generators (0 = OpenMP default)."""
    _load().wl_set_threads(int(n))


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def sigma_star(d: int, kind: str = "clustered") -> float:
    """Generating residual scale: 0.6 sqrt(D/2) (clustered) or 1 (gaussian)."""
    return 0.6 * math.sqrt(d / 2.0) if kind == "clustered" else 1.0


class Workload:
    """Latent truth, evaluation state and generator handles for one config."""

    def __init__(self, n: int, d: int, kind: str = "clustered", p_missing: float = 0.0,
                 seed: int = BASE_SEED, sigma: float | None = None):
        self.n, self.d, self.kind, self.p_missing, self.seed = int(n), int(d), kind, float(p_missing), int(seed)
        self.sigma = float(sigma) if sigma is not None else sigma_star(d, kind)
        lib = _load()
        self.x_true = np.zeros((n, d))
        self.x0 = np.zeros((n, d))
        rc = lib.wl_latent(n, d, 0 if kind == "clustered" else 1, self.seed, self.sigma, N_CLUSTERS,
                           _dp(self.x_true), _dp(self.x0))
        if rc:
            raise ValueError("bad workload arguments")

    @property
    def n_pairs(self) -> int:
        return self.n * (self.n - 1) // 2

    def y_rows(self, i0: int, i1: int) -> np.ndarray:
        """Packed lower-triangle rows [i0, i1) (row i has i entries)."""
        lo = i0 * (i0 - 1) // 2 if i0 > 0 else 0
        hi = i1 * (i1 - 1) // 2
        out = np.empty(hi - lo)
        rc = _load().wl_dissim_rows(self.n, self.d, _dp(self.x_true), self.seed, self.sigma,
                                    self.p_missing, i0, i1, _dp(out))
        if rc:
            raise ValueError("bad row range")
        return out

    def y_packed(self) -> np.ndarray:
        return self.y_rows(0, self.n)

    def y_full_rows(self, rows) -> np.ndarray:
        """y_ij for every j, for each i in rows (NaN at j == i)."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty((rows.size, self.n))
        _load().wl_dissim_full_rows(self.n, self.d, _dp(self.x_true), self.seed, self.sigma, self.p_missing,
                                    rows.size, rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(out))
        return out

    def normals(self, stream: int, shape) -> np.ndarray:
        out = np.empty(int(np.prod(shape)))
        _load().wl_normals(self.seed, stream, out.size, _dp(out))
        return out.reshape(shape)


def config(name: str, **over) -> Workload:
    idx, n, d, kind, pm = CONFIGS[name]
    kw = dict(n=n, d=d, kind=kind, p_missing=pm, seed=BASE_SEED + idx)
    kw.update(over)
    return Workload(**kw)


def unpack_lower(y_packed: np.ndarray, n: int) -> np.ndarray:
    """Packed lower triangle -> full symmetric n x n (NaN diagonal)."""
    full = np.full((n, n), np.nan)
    il, jl = np.tril_indices(n, -1)
    full[il, jl] = y_packed
    full[jl, il] = y_packed
    return full


def coalescent_forest(n: int, n_trees: int = 1, frac_unsequenced: float = 0.0, seed: int = BASE_SEED,
                      tau0: float = 1.0, tau_e: float = 4.0, theta: float = 1.0):
    """Synthetic phylogeny input for the Brownian-diffusion prior:
    the n items are split into n_trees Kingman-coalescent trees plus a fraction of
    unsequenced items.  Node k < n is item k (a tip); internal nodes are numbered
    from n up.  Returns (parent, t): parent[k] = -1 for roots; t[k] = branch length
    to the parent, or the root's prior variance factor for roots (tau0 for tree
    roots, tau_e for unsequenced items).  Input generation only (no method
    arithmetic); every tree is binary with strictly positive branch lengths."""
    rng = np.random.default_rng(seed)
    items = rng.permutation(n)
    n_un = int(round(frac_unsequenced * n))
    unseq, seq = items[:n_un], items[n_un:]
    groups = [g for g in np.array_split(seq, n_trees) if g.size > 0]
    parent = list(np.full(n, -1, dtype=np.int64))
    t = list(np.zeros(n))
    height = list(np.zeros(n))
    for i in unseq:
        t[i] = tau_e
    for g in groups:
        lineages = [int(v) for v in g]
        time = 0.0
        while len(lineages) > 1:
            k = len(lineages)
            time += rng.exponential(theta / (k * (k - 1) / 2.0)) + 1e-9
            a, b = rng.choice(k, size=2, replace=False)
            ca, cb = lineages[a], lineages[b]
            node = len(parent)
            parent.append(-1)
            t.append(0.0)
            height.append(time)
            for c in (ca, cb):
                parent[c] = node
                t[c] = time - height[c]
            lineages = [v for q, v in enumerate(lineages) if q not in (a, b)] + [node]
        t[lineages[0]] = tau0
    return np.array(parent, dtype=np.int64), np.array(t, dtype=np.float64)
