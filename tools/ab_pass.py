#!/usr/bin/env python
"""A/B timing of the leapfrog pass on one box: the same synthetic problem (clustered,
fp64, D = 2, N = --n; Y > L2 for N >= 6000 so no flush) through several libmds builds,
alternating rounds.  usage: ab_pass.py --n 30000 --steps 40 --rounds 3 lib1.so [lib2.so ...]
('cur' = the in-tree libmds.so).  One subprocess per (round, lib): prints ms/step and G pairs/s."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(n, d, steps, prec):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import workload
    import paper_1905_04582_b200 as mds
    w = workload.Workload(n, d, seed=12345)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    c = mds.MDS(n, d, prec, True, stream=st)
    for i0 in range(0, n, 2048):
        c.set_dissimilarity_rows(i0, min(n, i0 + 2048), w.y_rows(i0, min(n, i0 + 2048)))
    c.set_locations(w.x0)
    c.set_sigma(w.sigma)
    p0 = torch.from_numpy(w.normals(1, (n, d))).cuda()
    c.leapfrog_device(1, 2e-5, 10.0, p0_dev=p0)
    for _ in range(5):
        c.leapfrog_device(1, 2e-5, 10.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        c.leapfrog_device(1, 2e-5, 10.0)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ll = c.log_likelihood()
    print(json.dumps({"ms": ms, "gps": n * (n - 1) / 2 / (ms * 1e-3) / 1e9, "ll": ll}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30000)
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--prec", default="f64")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("libs", nargs="*")
    a = ap.parse_args()
    if a.child:
        child(a.n, a.d, a.steps, a.prec)
        return
    res = {l: [] for l in a.libs}
    for r in range(a.rounds):
        for l in a.libs:
            env = dict(os.environ)
            if l != "cur":
                env["MDS_LIB_PATH"] = os.path.abspath(l)
            out = subprocess.run([sys.executable, __file__, "--child", "--n", str(a.n), "--d", str(a.d),
                                  "--steps", str(a.steps), "--prec", a.prec], env=env, capture_output=True,
                                 text=True, timeout=600)
            try:
                v = json.loads(out.stdout.strip().splitlines()[-1])
            except Exception:
                v = {"error": out.stderr[-500:]}
            res[l].append(v)
            print(r, l, v, flush=True)
    for l, vs in res.items():
        g = [v["gps"] for v in vs if "gps" in v]
        if g:
            print("%-50s median %.2f G pairs/s  (%s)" % (l, sorted(g)[len(g) // 2], " ".join("%.2f" % x for x in g)))


if __name__ == "__main__":
    main()
