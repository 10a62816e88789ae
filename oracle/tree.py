"""CPU oracle for the phylogenetic Brownian-diffusion prior (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; the product path never does, and nothing is shared with
the CUDA implementation (which never forms V_G).

Plain dense numpy fp64, written from the paper's definition:

  PAPER.md:157-186 (Eq. 3)  X ~ MN(mu0, V_G, Sigma):
      log p(X) = -1/2 tr[Sigma^-1 (X - mu0)' V_G^-1 (X - mu0)]
                 - (N D / 2) log 2 pi - (N / 2) log|Sigma| - (D / 2) log|V_G|
  PAPER.md:189-200          V_G: block diagonal; v_ii = tau_e for an unsequenced
      item; within a tree, v_ij = tau_0 + (elapsed time from the root to the
      most recent common ancestor of i and j), v_ii = tau_0 + (root-to-tip time).

Forest encoding (as mds_set_tree_prior): node k < n is item k; parent[k] = -1
for a root; t[k] = branch length to the parent, or the root's prior variance
factor (tau_0 / tau_e).  Then V_G = A diag(t) A' with A[i, a] = 1 iff node a
is item i or one of its ancestors: the covariance of a sum of independent
increments, which is the paper's v_ij entry by entry (shared root-to-MRCA
path + root variance); tree_cov forms it block by block.  Gradient: d log p / dX = -V_G^-1 (X - mu0) Sigma^-1.
"""
from __future__ import annotations

import numpy as np


def tree_cov(parent, t, n: int, dtype=np.float64) -> np.ndarray:
    """V_G (n x n) of PAPER.md:189-200 for the forest (parent, t).

    V_G = sum over nodes a of t_a 1_{S_a} 1_{S_a}', S_a = the items at or below
    node a: every increment (branch, or a root's prior variance) is shared by
    exactly the tips below it.  With the tips in depth-first order each S_a is
    a contiguous block, so the sum is formed block by block (in `dtype`)."""
    parent = np.asarray(parent, dtype=np.int64)
    t = np.asarray(t, dtype=np.float64)
    N = parent.size
    kids = [[] for _ in range(N)]
    roots = []
    for k in range(N):
        (kids[parent[k]] if parent[k] >= 0 else roots).append(k)
    lo = np.zeros(N, dtype=np.int64)
    hi = np.zeros(N, dtype=np.int64)
    order = []                                   # items in depth-first order
    for r in roots:
        stack = [(r, False)]
        while stack:
            v, done = stack.pop()
            if done:
                hi[v] = len(order)
                continue
            lo[v] = len(order)
            if v < n:
                order.append(v)
            stack.append((v, True))
            for c in reversed(kids[v]):
                stack.append((c, False))
    Vp = np.zeros((n, n), dtype=dtype)
    for a in range(N):
        if hi[a] > lo[a]:
            Vp[lo[a]:hi[a], lo[a]:hi[a]] += dtype(t[a])
    pos = np.empty(n, dtype=np.int64)
    pos[np.array(order, dtype=np.int64)] = np.arange(n)
    return Vp[np.ix_(pos, pos)]


def tree_prior(parent, t, x, mu0=None, sigma_cov=None):
    """(log p(X), d log p / dX) of Eq. 3, dense."""
    x = np.asarray(x, dtype=np.float64)
    n, d = x.shape
    mu0 = np.zeros(d) if mu0 is None else np.asarray(mu0, dtype=np.float64)
    S = np.eye(d) if sigma_cov is None else np.asarray(sigma_cov, dtype=np.float64)
    V = tree_cov(parent, t, n)
    Y = x - mu0
    Lv = np.linalg.cholesky(V)
    VinvY = np.linalg.solve(Lv.T, np.linalg.solve(Lv, Y))
    # iterative refinement with V_G and the residual in extended precision:
    # coalescent trees have branches ~1e-7 under root paths ~1, so V_G rounded
    # to fp64 already perturbs sibling differences v_ii - v_ij = t_i by ~1e-10
    # relative, and cond(V_G) ~ 1e9 would leave ~cond*u in V_G^-1 Y
    Vl, Yl = tree_cov(parent, t, n, np.longdouble), Y.astype(np.longdouble)
    for _ in range(3):
        R = (Yl - Vl @ VinvY.astype(np.longdouble)).astype(np.float64)
        VinvY = VinvY + np.linalg.solve(Lv.T, np.linalg.solve(Lv, R))
    Sinv = np.linalg.inv(S)
    quad = np.trace(Sinv @ Y.T @ VinvY)
    logdetV = 2.0 * np.log(np.diag(Lv)).sum()
    _, logdetS = np.linalg.slogdet(S)
    logp = -0.5 * quad - 0.5 * n * d * np.log(2 * np.pi) - 0.5 * n * logdetS - 0.5 * d * logdetV
    grad = -VinvY @ Sinv
    return float(logp), grad


def leapfrog_tree(y_packed, x0, p0, sigma, eps, n_steps, parent, t, mu0=None, sigma_cov=None, truncation=1):
    """Leapfrog (Eq. 5, M = I) on log pi = log L + log p_tree,
    composed from the oracle's log L/gradient (mds_oracle.c) and tree_prior above.
    Returns dict(x, p, H0, H1, loglik)."""
    from . import loglik_grad

    def logpi(x):
        r = loglik_grad(y_packed, x, sigma, truncation, want_absscale=False)
        lp, gp = tree_prior(parent, t, x, mu0, sigma_cov)
        return r["loglik"] + lp, r["grad"] + gp, r["loglik"]

    x = np.array(x0, dtype=np.float64)
    p = np.array(p0, dtype=np.float64)
    lpi, g, _ = logpi(x)
    H0 = -lpi + 0.5 * float((p * p).sum())
    ll = None
    for _ in range(n_steps):
        p = p + 0.5 * eps * g
        x = x + eps * p
        lpi, g, ll = logpi(x)
        p = p + 0.5 * eps * g
    H1 = -lpi + 0.5 * float((p * p).sum())
    return dict(x=x, p=p, H0=H0, H1=H1, loglik=ll)
