"""Per-step overhead experiments for the leapfrog pass (GPU): back-to-back steps
in one call vs one call per step, timing mode on/off, with/without L2 flush."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workload, paper_1905_04582_b200 as mds

w = workload.config("C2")
s = torch.cuda.current_stream()
ctx = mds.MDS(w.n, w.d, "f64", True, stream=s)
ctx.set_dissimilarities_packed(w.y_packed()); ctx.set_locations(w.x0); ctx.set_sigma(w.sigma)
p0 = torch.from_numpy(w.normals(1, (w.n, w.d))).cuda()
ctx.leapfrog_device(1, 2e-5, 10.0, p0_dev=p0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def ev(): return torch.cuda.Event(enable_timing=True)
for timing in (False, True):
    ctx.set_timing(timing)
    torch.cuda.synchronize()
    a, b = ev(), ev(); a.record(s); ctx.leapfrog_device(200, 2e-5, 10.0); b.record(s); torch.cuda.synchronize()
    print("timing=%d one call x200 steps: %.2f us/step" % (timing, a.elapsed_time(b) * 1e3 / 200))
    a, b = ev(), ev(); a.record(s)
    for k in range(200): ctx.leapfrog_device(1, 2e-5, 10.0)
    b.record(s); torch.cuda.synchronize()
    print("timing=%d 200 calls: %.2f us/step" % (timing, a.elapsed_time(b) * 1e3 / 200))
    e0 = [ev() for _ in range(200)]; e1 = [ev() for _ in range(200)]
    for k in range(200):
        flush.zero_(); e0[k].record(s); ctx.leapfrog_device(1, 2e-5, 10.0); e1[k].record(s)
    torch.cuda.synchronize()
    t = [x.elapsed_time(y) * 1e3 for x, y in zip(e0, e1)]
    print("timing=%d flushed per-step events: med %.2f us" % (timing, np.median(t)))
    if timing:
        print("pass kernel ms (lib events):", ctx.last_timing())
