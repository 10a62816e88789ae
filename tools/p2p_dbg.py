"""Peer-memory exchange on ONE GPU with `world` threads (debug/timing aid):
python tools/p2p_dbg.py [world] [ctas]; prints each rank's progress and grid."""
import faulthandler
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(150, exit=True)
import torch  # noqa: E402

import paper_1905_04582_b200 as mds  # noqa: E402
import workload  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctas = int(sys.argv[2]) if len(sys.argv) > 2 else 148 // world
n, d = 500, 2
w = workload.Workload(n, d, p_missing=0.05, seed=92)
y, x = w.y_packed(), w.x0
p0 = w.normals(1, (n, d))
bar = threading.Barrier(world)
wins = [None] * world


def log(r, msg):
    print("%.3f r%d %s" % (time.time() % 1000, r, msg), flush=True)


def worker(r):
    try:
        torch.cuda.set_device(0)
        if os.environ.get("RAW_STREAM"):
            from cuda.bindings import runtime as rt
            err, h = rt.cudaStreamCreateWithFlags(1)
            st = torch.cuda.ExternalStream(int(h))
        else:
            st = torch.cuda.Stream()
        torch.cuda.set_stream(st)
        ctx = mds.MDS(n, d, "f64", True, rank=r, world=world, stream=st)
        ctx.set_grid_limit(ctas)
        wins[r], _ = ctx.p2p_window()
        bar.wait()
        ctx.p2p_connect(wins)
        ctx.set_dissimilarities_packed(y)
        ctx.set_locations(x)
        ctx.set_sigma(w.sigma)
        st.synchronize()
        bar.wait()
        log(r, "eval")
        ll, g = ctx.log_likelihood_and_gradient()
        log(r, "eval done %r" % ll)
        if os.environ.get("MDS_PROFILE_PHASES"):
            ctx.last_timing()
        tr = ctx.hmc_trajectory(p0, 0.002, 8, prior_sd=10.0)
        log(r, "traj done %r" % tr["H1"])
        a = ctx.sigma_mh_step(2.0, 0.5, 0.05, 0.7, 0.5)
        log(r, "sigma done %r" % (a,))
        dl = ctx.row_loglik_delta(3, x[3] + 0.02)
        log(r, "delta done %r" % dl)
        st.synchronize()
        bar.wait()
        ctx.close()
    except Exception as e:
        log(r, "ERROR %r" % e)
        if os.environ.get("MDS_PROFILE_PHASES"):
            try:
                ctx.last_timing()
            except Exception:
                pass
        bar.abort()


ths = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
[t.start() for t in ths]
[t.join() for t in ths]
print("done")
