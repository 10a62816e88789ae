"""Per-step overhead experiments for the leapfrog pass (GPU): back-to-back steps
vs per-step events, and the per-step L2 flush done by torch (FillFunctor) vs
mds_l2_flush (the pass kernel's launch shape) vs none.  Diagnostic only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1905_04582_b200 as mds
import workload

w = workload.config("C2")
s = torch.cuda.current_stream()
ctx = mds.MDS(w.n, w.d, "f64", True, stream=s)
ctx.set_dissimilarities_packed(w.y_packed())
ctx.set_locations(w.x0)
ctx.set_sigma(w.sigma)
p0 = torch.from_numpy(w.normals(1, (w.n, w.d))).cuda()
ctx.leapfrog_device(1, 2e-5, 10.0, p0_dev=p0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def ev():
    return torch.cuda.Event(enable_timing=True)


K = 300
for _ in range(20):
    ctx.leapfrog_device(1, 2e-5, 10.0)
torch.cuda.synchronize()
a, b = ev(), ev()
a.record(s)
ctx.leapfrog_device(K, 2e-5, 10.0)
b.record(s)
torch.cuda.synchronize()
print("one call x%d steps      : %.2f us/step" % (K, a.elapsed_time(b) * 1e3 / K))
for mode in ("none", "torch", "mds"):
    e0 = [ev() for _ in range(K)]
    e1 = [ev() for _ in range(K)]
    for k in range(K):
        if mode == "torch":
            flush.zero_()
        elif mode == "mds":
            ctx.l2_flush(flush)
        e0[k].record(s)
        ctx.leapfrog_device(1, 2e-5, 10.0)
        e1[k].record(s)
    torch.cuda.synchronize()
    t = np.array([x.elapsed_time(y) * 1e3 for x, y in zip(e0, e1)])
    print("flush=%-5s per-step events: med %.2f mean %.2f us" % (mode, np.median(t), t.mean()))
