#!/usr/bin/env python
"""Small problems through every libmds kernel, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck) -- tools/sanitize.sh runs this under each tool.

Covers the pass kernel in all 9 modes (EVAL, EVAL_NOLIK via the sharded
gradient-only step, LEAPFROG, LEAPFROG_NOLIK, LIK, LEAPFROG[_NOLIK]_TREE,
EVAL[_NOLIK]_TREE), fp64 and fp32, the combine / combine-update kernels, the
standalone tree walk, the row (single-location) kernels, the CV kernels, the
HMC driver (graph) and the sigma MH step.  Exits non-zero on any library error.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1905_04582_b200 as mds  # noqa: E402
import workload  # noqa: E402


def run(n=130, d=2, prec="f64"):
    w = workload.Workload(n, d, p_missing=0.1, seed=n)
    y = w.y_packed()
    parent, t = workload.coalescent_forest(n, 2, 0.1, seed=3)
    p0 = w.normals(2, (n, d))
    with mds.MDS(n, d, prec) as c:
        c.set_dissimilarities_packed(y)
        c.set_locations(w.x0)
        c.set_sigma(w.sigma)
        c.log_likelihood_and_gradient()                      # EVAL
        c.log_likelihood_at_sigma(1.1 * w.sigma)             # LIK
        c.hmc_trajectory(p0, 0.002, 3, prior_sd=5.0)         # LEAPFROG_NOLIK + LEAPFROG
        c.hmc_run(2, 3, 0.002, 5.0, seed=1)                  # graph replay
        c.sigma_mh_step(2.0, 1.0, 0.1, 0.3, 0.5)
        c.zero_distance_pairs()
        c.row_loglik_delta(5, w.x0[5] + 0.1)                 # row kernel (cluster)
        c.rw_sweep(np.array([1, 7, 7, 64]), np.full((4, d), 0.1), np.full(4, 0.5), 0.2, 3.0)
        c.cv_set_heldout(np.array([3, 9]), np.array([1, 2]), np.array([0.5, 1.5]))
        c.cv_accumulate()
        c.cv_accumulate()
        c.cv_lpd()
        c.set_tree_prior(parent, t)
        c.tree_prior()                                       # standalone walk
        c.hmc_trajectory(p0, 0.002, 3)                       # LEAPFROG_NOLIK_TREE + LEAPFROG_TREE
        c.mcmc_run(2, 2, 0.002, 0.0, 3, 2.0, 1.0, 0.1)
    if prec == "f64":
        # library-owned communicator at world 1: EVAL partial -> ncclAllGather -> combine
        with mds.MDS(n, d, prec, rank=0, world=1, nccl_unique_id=mds.mds_nccl_unique_id()) as c:
            c.set_dissimilarities_packed(y)
            c.set_locations(w.x0)
            c.set_sigma(w.sigma)
            c.log_likelihood_and_gradient()
            c.hmc_trajectory(p0, 0.002, 3, prior_sd=5.0)     # EVAL_NOLIK/EVAL + combine_update
            c.set_tree_prior(parent, t)
            c.hmc_trajectory(p0, 0.002, 3)                   # EVAL_NOLIK_TREE / EVAL_TREE
        # fused peer-memory exchange at world 1 (own window): push, flags, wait,
        # combine + leapfrog update in the pass kernel (plain launch, own grid barrier),
        # and the one-CTA peer all-gather of the small exchanges
        with mds.MDS(n, d, prec) as c:
            a, _ = c.p2p_window()
            c.p2p_connect([a])
            c.set_dissimilarities_packed(y)
            c.set_locations(w.x0)
            c.set_sigma(w.sigma)
            c.log_likelihood_and_gradient()
            c.log_likelihood_at_sigma(1.1 * w.sigma)
            c.row_loglik_delta(5, w.x0[5] + 0.1)
            c.hmc_trajectory(p0, 0.002, 3, prior_sd=5.0)
            c.set_tree_prior(parent, t)
            c.hmc_trajectory(p0, 0.002, 3)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    run(130, 2, "f64")
    run(70, 3, "f32")
    torch.cuda.synchronize()
    print("sanitize_run ok")
