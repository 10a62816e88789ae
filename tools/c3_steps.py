#!/usr/bin/env python
"""Where a C3 transition's time goes (C2 data, L2-resident): device time per leapfrog
step for (a) single LEAPFROG steps, (b) L = 20 steps per mds_leapfrog_device call
(steps 1..19 gradient-only), (c) hmc_run transitions (graph + energies + accept),
each event-timed on the context stream.  usage: python tools/c3_steps.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    w = workload.config("C3")
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx = mds.MDS(w.n, w.d, "f64", True, stream=st)
    ctx.set_dissimilarities_packed(w.y_packed())
    ctx.set_locations(w.x0)
    ctx.set_sigma(w.sigma)
    p0 = torch.from_numpy(w.normals(1, (w.n, w.d))).cuda()
    eps = 2e-4
    ctx.leapfrog_device(1, eps, 10.0, p0_dev=p0)
    out = {}
    for name, calls, L in (("single_leapfrog_step", 200, 1), ("leapfrog_device_L20", 10, 20)):
        for _ in range(3):
            ctx.leapfrog_device(L, eps, 10.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(calls):
            ctx.leapfrog_device(L, eps, 10.0)
        e1.record(st)
        torch.cuda.synchronize()
        out[name + "_us_per_step"] = e0.elapsed_time(e1) * 1e3 / (calls * L)
    x, s = ctx.hmc_run(50, 20, 2.35e-3, 10.0, seed=7, x0=w.x0.copy())
    out["hmc_run_us_per_step"] = s["seconds"] * 1e6 / (50 * 20)
    # per-transition vs per-step cost: transitions of L = 1, 20, 40 at a small step
    for L in (1, 20, 40):
        x, s = ctx.hmc_run(50, L, 2e-4, 10.0, seed=7, x0=w.x0.copy())
        out["hmc_run_L%d_us_per_transition" % L] = s["seconds"] * 1e6 / 50
    print(json.dumps(out))


if __name__ == "__main__":
    main()
