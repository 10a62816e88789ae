#!/usr/bin/env python
"""Measure the non-headline BASELINE.json configs on one GPU (not bench lines).

  C3: the C2 data as an HMC chain, 1000 transitions x 20 leapfrog steps
      (mds_hmc_run: one CUDA graph per transition; step size from a short
      pilot targeting 0.65-0.85 acceptance).
  C4: N = 30000, D = 6, 10% missing, fp64 and fp32: one fused pass (leapfrog
      step) timed like bench.py.
  C5 at P = 1 (N = 100000, D = 2; 40 GB of fp64 Y generated on the GPU side
      from the host generator in row chunks) when --c5 is given.

Prints one JSON object per config.  Timing: CUDA events on the context stream.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def step_rate(ctx, n, d, steps, warmup, eps=2e-5, tau=10.0):
    import torch
    s = torch.cuda.current_stream()
    p0 = torch.zeros((n, d), dtype=torch.float64, device="cuda")
    ctx.leapfrog_device(1, eps, tau, p0_dev=p0)
    for _ in range(warmup):
        ctx.leapfrog_device(1, eps, tau)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        a.record(s)
        ctx.leapfrog_device(1, eps, tau)
        b.record(s)
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(b) for a, b in ev])
    return float(ms.mean()), float(np.median(ms))


def run_c4(prec):
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    w = workload.config("C4")
    t0 = time.time()
    ctx = mds.MDS(w.n, w.d, prec, True, stream=torch.cuda.current_stream())
    for i0 in range(0, w.n, 5000):
        ctx.set_dissimilarity_rows(i0, min(w.n, i0 + 5000), w.y_rows(i0, min(w.n, i0 + 5000)))
    ctx.set_locations(w.x0)
    ctx.set_sigma(w.sigma)
    setup = time.time() - t0
    mean_ms, med_ms = step_rate(ctx, w.n, w.d, 20, 3)
    P = w.n * (w.n - 1) // 2
    ctx.close()
    return {"config": "C4", "precision": prec, "n": w.n, "d": w.d, "missing": w.p_missing,
            "ms_per_step": mean_ms, "ms_p50": med_ms, "pair_evals_per_s": P / (mean_ms * 1e-3),
            "setup_s": setup}


def run_c3(n_iter, L):
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    w = workload.config("C3")
    ctx = mds.MDS(w.n, w.d, "f64", True, stream=torch.cuda.current_stream())
    ctx.set_dissimilarities_packed(w.y_packed())
    ctx.set_sigma(w.sigma)
    # pilot: adapt eps to 0.65-0.85 acceptance over 50 transitions
    eps, x = 2e-3, w.x0.copy()
    for _ in range(8):
        x, st = ctx.hmc_run(50, L, eps, 10.0, seed=1905045922, x0=x)
        acc = st["accepted"] / 50
        if 0.65 <= acc <= 0.85:
            break
        eps *= 1.4 if acc > 0.85 else 0.6
    torch.cuda.synchronize()
    t0 = time.time()
    x, st = ctx.hmc_run(n_iter, L, eps, 10.0, seed=1905045922 + 100, x0=x)
    wall = time.time() - t0
    P = w.n * (w.n - 1) // 2
    ctx.close()
    return {"config": "C3", "n": w.n, "d": w.d, "iterations": n_iter, "leapfrog": L, "step_size": eps,
            "acceptance": st["accepted"] / n_iter, "mean_abs_dH": st["mean_abs_dH"],
            "device_seconds": st["seconds"], "wall_seconds": wall, "grad_evals": st["grad_evals"],
            "evals_per_s": st["grad_evals"] / st["seconds"],
            "pair_evals_per_s": P * st["grad_evals"] / st["seconds"], "final_loglik": st["final_loglik"],
            "paper_context": "PAPER.md:672 -- 2e6 HMC states in ~48 h on a GP100 (86.4 ms/state) for the flu data"}


def run_c5(steps=5):
    """C5 at P = 1: N = 100000, D = 2, fp64 -- 5.0e9 pairs, 40 GB of tiled Y on one
    B200.  Y is streamed to the context in row chunks straight from the seeded
    generator (no host N x N matrix); the timed steps are device-resident
    leapfrog steps as in bench.py (Y is far larger than L2: no flush needed)."""
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    w = workload.config("C5")
    t0 = time.time()
    ctx = mds.MDS(w.n, w.d, "f64", True, stream=torch.cuda.current_stream())
    step = 1000
    for i0 in range(0, w.n, step):
        i1 = min(w.n, i0 + step)
        ctx.set_dissimilarity_rows(i0, i1, w.y_rows(i0, i1))
    ctx.set_locations(w.x0)
    ctx.set_sigma(w.sigma)
    torch.cuda.synchronize()
    setup = time.time() - t0
    mean_ms, med_ms = step_rate(ctx, w.n, w.d, steps, 1)
    P = w.n * (w.n - 1) // 2
    ll = ctx.log_likelihood()
    ctx.close()
    return {"config": "C5", "precision": "f64", "n": w.n, "d": w.d, "gpus": 1, "ms_per_step": mean_ms,
            "ms_p50": med_ms, "pair_evals_per_s": P / (mean_ms * 1e-3), "setup_s": setup, "loglik": ll}


def run_mcmc(n_iter=200, L=20):
    """The PAPER.md:672 sampler on the C3 data: per iteration one HMC transition of
    X (L = 20) and one MH update of sigma^2 (mds_mcmc_run)."""
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    w = workload.config("C3")
    ctx = mds.MDS(w.n, w.d, "f64", True, stream=torch.cuda.current_stream())
    ctx.set_dissimilarities_packed(w.y_packed())
    ctx.set_sigma(w.sigma)
    x, st = ctx.mcmc_run(20, L, 0.00235, 10.0, 5, 2.0, 0.5, 0.002, x0=w.x0)    # warm-up
    t0 = time.time()
    x, st = ctx.mcmc_run(n_iter, L, 0.00235, 10.0, 6, 2.0, 0.5, 0.002, x0=x)
    wall = time.time() - t0
    P = w.n * (w.n - 1) // 2
    ctx.close()
    return {"config": "C3 + sigma^2 MH (mds_mcmc_run)", "iterations": n_iter, "leapfrog": L,
            "device_seconds": st["seconds"], "wall_seconds": wall, "ms_per_iteration": st["seconds"] * 1e3 / n_iter,
            "accepted_x": st["accepted_x"], "accepted_sigma": st["accepted_sigma"], "final_sigma": st["final_sigma"],
            "grad_evals_per_s": st["grad_evals"] / st["seconds"]}


def run_sweep(ns=(5392, 10000, 20000, 30000, 50000, 100000), kinds=("clustered", "gaussian"), steps=5):
    """SURVEY 8(d) roofline N sweep (fig:time_by_N): D = 2, fp64,
    P = 1, both workloads; device-resident leapfrog steps as bench.py (no flush:
    Y exceeds L2 from N = 10000 on)."""
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    out = []
    for kind in kinds:
        for n in ns:
            w = workload.Workload(n, 2, kind=kind, seed=workload.BASE_SEED + 40 + n)
            ctx = mds.MDS(n, 2, "f64", True, stream=torch.cuda.current_stream())
            step = 2000
            for i0 in range(0, n, step):
                i1 = min(n, i0 + step)
                ctx.set_dissimilarity_rows(i0, i1, w.y_rows(i0, i1))
            ctx.set_locations(w.x0)
            ctx.set_sigma(w.sigma)
            mean_ms, med_ms = step_rate(ctx, n, 2, steps if n > 30000 else 20, 2)
            ctx.close()
            P = n * (n - 1) // 2
            out.append({"sweep": kind, "n": n, "d": 2, "ms_per_step": mean_ms, "pair_evals_per_s": P / (mean_ms * 1e-3)})
            print(json.dumps(out[-1]), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3-iter", type=int, default=1000)
    ap.add_argument("--leapfrog", type=int, default=20)
    ap.add_argument("--skip-c3", action="store_true")
    ap.add_argument("--skip-c4", action="store_true")
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="SURVEY 8(d) N sweep (D = 2, fp64, both workloads)")
    ap.add_argument("--mcmc", action="store_true", help="C3 data with the sigma^2 update (mds_mcmc_run)")
    a = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    if not a.skip_c4:
        for prec in ("f64", "f32"):
            print(json.dumps(run_c4(prec)), flush=True)
    if not a.skip_c3:
        print(json.dumps(run_c3(a.c3_iter, a.leapfrog)), flush=True)
    if a.c5:
        print(json.dumps(run_c5()), flush=True)
    if a.sweep:
        run_sweep()
    if a.mcmc:
        print(json.dumps(run_mcmc()), flush=True)


if __name__ == "__main__":
    main()
