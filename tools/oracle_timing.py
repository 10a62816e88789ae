#!/usr/bin/env python
"""The oracle timed on the host at full size (SURVEY 8(d) "Oracle timing"):
C2 (median of 5 full evaluations), C4 (3 full evaluations, fp64 inputs) and C5
(ONE evaluation of log L, streamed: the packed triangle is generated row chunk
by row chunk and never held whole; 1 core).  A reported baseline, not
a target.  -> profiles/r02/oracle_timing.json"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workload  # noqa: E402


def host():
    model = "unknown"
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            model = line.split(":", 1)[1].strip()
            break
    return "%s, %d logical cores" % (model, os.cpu_count() or 0)


def full(name, reps):
    w = workload.config(name)
    y = w.y_packed()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.loglik_grad(y, w.x0, w.sigma, 1, want_absscale=False)
        ts.append(time.perf_counter() - t0)
    med = float(np.median(ts))
    return {"evals": reps, "seconds": ts, "median_s": med, "pairs": w.n_pairs,
            "pair_evals_per_s": w.n_pairs / med}


def c5_streamed():
    """log L by the streaming row-range oracle over 500-row chunks, serial, one
    evaluation (the gradient at C5 is timed on the GPU side only)."""
    w = workload.config("C5")
    t_gen = 0.0
    t_or = 0.0
    ll = 0.0
    for i0 in range(0, w.n, 500):
        i1 = min(w.n, i0 + 500)
        a = time.perf_counter()
        y = w.y_rows(i0, i1)
        t_gen += time.perf_counter() - a
        a = time.perf_counter()
        v, _ = oracle.loglik_rows(i0, i1, y, w.x0, w.sigma, 1)
        t_or += time.perf_counter() - a
        ll += v
    return {"evals": 1, "what": "log L (Eq. 2) over all 5.0e9 pairs, streamed in 500-row chunks",
            "oracle_s": t_or, "generator_s": t_gen, "pairs": w.n_pairs, "pair_evals_per_s": w.n_pairs / t_or,
            "loglik": ll}


if __name__ == "__main__":
    workload.set_threads(os.cpu_count() or 1)
    out = {"host_cpu": host(), "cores_used": 1}
    out["C2"] = full("C2", 5)
    print(json.dumps(out["C2"]), flush=True)
    out["C4"] = full("C4", 3)
    print(json.dumps(out["C4"]), flush=True)
    out["C5"] = c5_streamed()
    print(json.dumps(out["C5"]), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "oracle_timing.json"), "w"), indent=1)
