#!/usr/bin/env python
"""Measure the SURVEY 8(f) "next" rows on one GPU (C2 data: N = 5392, D = 2, fp64).

  NEXT-1  likelihood-only pass at another sigma (mds_log_likelihood_at_sigma),
          one sigma MH step, and the gradient-only leapfrog step (per-step time
          of a 20-step device-resident trajectory: 19 gradient-only + 1 full
          pass) vs the full leapfrog step.
  NEXT-2  tree-prior kernel (coalescent tree over the C2 items): extra time per
          leapfrog step with the prior on vs off.
  NEXT-3  cross-validation accumulate per posterior draw (20% held-out fold).
  NEXT-4  row delta and the random-walk single-location sweep (per update).

Timing: CUDA events on the context stream, warm-up first.  One JSON object per row.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def ev_time(fn, reps, stream):
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    w = workload.config("C2")
    n, d = w.n, w.d
    P = n * (n - 1) // 2
    y = w.y_packed()
    ctx = mds.MDS(n, d, "f64", True, stream=s)
    ctx.set_dissimilarities_packed(y)
    ctx.set_locations(w.x0)
    ctx.set_sigma(w.sigma)
    out = []

    # ---- NEXT-1
    t_lik = ev_time(lambda: ctx.log_likelihood_at_sigma(1.1 * w.sigma), 50, s)
    rng = np.random.default_rng(0)
    t_mh = ev_time(lambda: ctx.sigma_mh_step(2.0, 0.5, 0.01, rng.normal(), 1.0 - rng.random()), 50, s)
    ctx.set_sigma(w.sigma)
    p0 = torch.zeros((n, d), dtype=torch.float64, device="cuda")
    ctx.leapfrog_device(1, 2e-5, 10.0, p0_dev=p0)
    t_full = ev_time(lambda: ctx.leapfrog_device(1, 2e-5, 10.0), 200, s)
    t_traj = ev_time(lambda: ctx.leapfrog_device(20, 2e-5, 10.0), 20, s) / 20
    t_go = (20 * t_traj - t_full) / 19
    out.append({"row": "NEXT-1", "config": "C2", "lik_only_pass_ms": t_lik, "lik_only_pair_evals_per_s": P / (t_lik * 1e-3),
                "sigma_mh_step_ms": t_mh,
                "full_leapfrog_step_ms": t_full, "grad_only_leapfrog_step_ms": t_go,
                "grad_only_pair_evals_per_s": P / (t_go * 1e-3),
                "trajectory_L20_step_ms": t_traj,
                "note": "sigma_mh_step includes a host sync; 1 lik-only pass when log L at the current sigma is cached"})

    # ---- NEXT-2
    parent, t = workload.coalescent_forest(n, 1, 0.0, seed=11)
    ctx.set_tree_prior(parent, t)
    ctx.leapfrog_device(1, 2e-5, 10.0, p0_dev=p0)
    t_tree_step = ev_time(lambda: ctx.leapfrog_device(1, 2e-5, 10.0), 200, s)
    t_tree_eval = ev_time(lambda: ctx.tree_prior(), 50, s)
    ctx.clear_tree_prior()
    out.append({"row": "NEXT-2", "config": "C2 + coalescent tree (%d nodes)" % parent.size,
                "leapfrog_step_with_tree_ms": t_tree_step, "leapfrog_step_iid_ms": t_full,
                "tree_prior_kernel_ms_est": t_tree_step - t_full, "tree_prior_call_ms": t_tree_eval,
                "note": "tree_prior_call includes a D2H copy + host sync"})

    # ---- NEXT-3
    obs = np.flatnonzero(~np.isnan(y))
    held = np.sort(np.random.default_rng(1).choice(obs, size=obs.size // 5, replace=False))
    i = np.floor((1 + np.sqrt(1 + 8 * held.astype(np.float64))) / 2).astype(np.int64)
    i -= (i * (i - 1) // 2 > held)
    j = held - i * (i - 1) // 2
    ctx.cv_set_heldout(i, j, y[held])
    t_cv = ev_time(lambda: ctx.cv_accumulate(), 200, s)
    m = held.size
    bytes_per_pair = 8 + 8 + 2 * 8 + 2 * 8       # (i, j) int2 + y + read (max, sum) + write (max, sum)
    out.append({"row": "NEXT-3", "config": "C2, 20%% fold (%d held-out pairs)" % m, "accumulate_ms": t_cv,
                "heldout_pairs_per_s": m / (t_cv * 1e-3),
                "hbm_gbs_algorithmic": m * bytes_per_pair / (t_cv * 1e-3) / 1e9,
                "bytes_per_pair": bytes_per_pair})

    # ---- NEXT-4
    xn = w.x0[100] + 0.01
    t_row = ev_time(lambda: ctx.row_loglik_delta(100, xn), 50, s)
    K = n
    rows = rng.integers(0, n, size=K)
    z = rng.normal(size=(K, d))
    u = 1.0 - rng.random(K)
    ctx.set_locations(w.x0)
    t0 = time.perf_counter()
    t_sweep = ev_time(lambda: ctx.rw_sweep(rows, z, u, 0.01, 10.0), 3, s)
    acc = ctx.rw_sweep(rows, z, u, 0.01, 10.0)
    out.append({"row": "NEXT-4", "config": "C2", "row_delta_call_ms": t_row, "sweep_updates": K,
                "sweep_ms": t_sweep, "us_per_update": t_sweep * 1e3 / K,
                "pair_terms_per_s": 2 * (n - 1) * K / (t_sweep * 1e-3), "accepted_last": acc,
                "note": "row_delta_call includes H2D/D2H + host sync; sweep = one launch of K sequential updates"})
    for o in out:
        print(json.dumps(o), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
