#!/usr/bin/env python
"""Per-CTA phase-A end times of the C2 leapfrog pass (MDS_PROFILE_PHASES=2), R repeats:
is the phase-A spread a property of the SM (reproducible per SM id) or noise?
usage: MDS_PROFILE_PHASES=2 python tools/cta_skew.py [repeats] 2> phases.txt"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    w = workload.config("C2")
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx = mds.MDS(w.n, w.d, "f64", True, stream=st)
    ctx.set_dissimilarities_packed(w.y_packed())
    ctx.set_locations(w.x0)
    ctx.set_sigma(w.sigma)
    p0 = torch.from_numpy(w.normals(1, (w.n, w.d))).cuda()
    ctx.leapfrog_device(1, 2e-5, 10.0, p0_dev=p0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(reps):
        ctx.l2_flush(flush)
        ctx.set_timing(True)
        ctx.leapfrog_device(1, 2e-5, 10.0)
        ctx.last_timing()
        ctx.set_timing(False)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
