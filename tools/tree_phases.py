#!/usr/bin/env python
"""Phase split of the leapfrog pass with the tree walk fused into its last CTA
(C2 data + coalescent tree); run with MDS_PROFILE_PHASES=2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    torch.cuda.set_device(0)
    w = workload.config("C2")
    parent, t = workload.coalescent_forest(w.n, 1, 0.0, seed=11)
    ctx = mds.MDS(w.n, w.d, "f64", True, stream=torch.cuda.current_stream())
    ctx.set_dissimilarities_packed(w.y_packed())
    ctx.set_locations(w.x0)
    ctx.set_sigma(w.sigma)
    ctx.set_tree_prior(parent, t)
    p0 = torch.zeros((w.n, w.d), dtype=torch.float64, device="cuda")
    ctx.leapfrog_device(1, 2e-5, 0.0, p0_dev=p0)
    for _ in range(50):
        ctx.leapfrog_device(1, 2e-5, 0.0)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.leapfrog_device(1, 2e-5, 0.0)
    ctx.last_timing()
    ctx.close()


if __name__ == "__main__":
    main()
