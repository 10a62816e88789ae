#!/usr/bin/env python
"""A short C3 chain (C2 data, L = 20 leapfrog steps per transition) for launch lists:
ncu --metrics gpu__time_duration.sum ... python tools/c3_short.py [n_iter]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    n_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    w = workload.config("C3")
    ctx = mds.MDS(w.n, w.d, "f64", True, stream=torch.cuda.current_stream())
    ctx.set_dissimilarities_packed(w.y_packed())
    ctx.set_sigma(w.sigma)
    x, st = ctx.hmc_run(n_iter, 20, 2e-3, 10.0, seed=1905045922, x0=w.x0.copy())
    torch.cuda.synchronize()
    print({k: st[k] for k in ("accepted", "seconds", "grad_evals")})
    ctx.close()


if __name__ == "__main__":
    main()
