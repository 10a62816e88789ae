#!/usr/bin/env python
"""bench.py -- MDS likelihood+gradient pair-evals/s on B200 (BASELINE.json metric).

One "step" = one HMC leapfrog step of the hot path:
half-kick + drift, one fused likelihood+gradient pass over every unordered pair
(pair kernel + fixed-order reduction [+ NCCL all-gather + rank-ordered combine
when sharded]), half-kick.  value = unordered pairs (all of them, observed or
not) x steps / device time (max over ranks).

Headline workload, the SAME at every N (strong scaling): BASELINE.json
configs[4] = C5, N = 100000, D = 2, fp64, clustered synthetic points (K = 189),
truncation on: 5.0e9 pairs per step, 40 GB of tiled Y (5 GB per rank at N = 8),
larger than the 126 MB L2, so no flush is needed between steps.  At N = 1 the
line also carries C2 (BASELINE configs[1], the paper's N = 5392; L2-flushed) and
C4 (configs[3], N = 30000, D = 6, 10% missing, fp64 and fp32) under "configs".

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--dry-run]

--gpus N > 1 without torchrun's environment re-launches this script under
torch.distributed.run (one rank per GPU, 127.0.0.1 rendezvous).  Each rank
owns the tile-rows r mod N, generates and uploads only those rows, and owns an
NCCL communicator inside libmds (unique id broadcast over torch.distributed).
The exchange (--exchange p2p, default) is the fused peer-memory exchange: the
pass kernel stores its partial into every rank's window over NVLink (IPC
handles all-gathered through torch.distributed), waits for the ranks' flags and
combines, one launch per step; --exchange nccl uses ncclAllGather of n*d + 1
doubles on the context stream instead (also the fallback if the windows cannot
be connected).  --exchange gloo-host registers a host-staged gloo all-gather (several
ranks sharing one GPU: a plumbing check, not a measurement).  --dry-run: plan
only (CPU, gloo): every rank reports its share of the pairs.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MDS likelihood+gradient pair-evals/s"
UNIT = "pair-evals/s"
PAPER_CONTEXT = ("PAPER.md:724 (Quadro GP100, OpenCL, fp64, N=5338): 4.5 ms likelihood + 4 ms gradient "
                 "per eval = 1.68e9 unordered pair-evals/s for the pair of calls; context only")
L2_BYTES = 126 << 20
SM_MAX_GHZ = 1.965
I64_REF = 160.0      # FP64 instructions per pair of the libdevice formulation (fixed reference)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--extra", default="auto",
                    help="extra configs at N = 1 (comma list of C2, C3, C4, C4f32; 'none'); auto = all at N = 1")
    ap.add_argument("--step-size", type=float, default=2e-5)
    ap.add_argument("--prior-sd", type=float, default=10.0)
    ap.add_argument("--e2e-seconds", type=float, default=2.0)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", choices=["p2p", "nccl", "torch", "gloo-host"], default="p2p",
                    help="sharded exchange: libmds-owned NCCL communicator (default), torch.distributed NCCL "
                         "callback, or host-staged gloo callback (ranks sharing a GPU)")
    ap.add_argument("--flush", choices=["auto", "mds", "none"], default="auto",
                    help="L2 flush between timed steps: auto = when the rank's Y fits 2x L2")
    ap.add_argument("--graph", type=int, default=0, help="1: replay the K timed steps from one CUDA graph")
    ap.add_argument("--dry-run", action="store_true", help="plan only (CPU): per-rank pair shares")
    return ap.parse_args()


# ----------------------------------------------------------------------------- launcher
def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 outside torchrun: one rank per GPU on this node (the driver's own
    launch line, run for the user)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
    cmd += [a for a in sys.argv[1:]]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        load = [v for v in sm if smax and v > 0.3 * smax] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers
def host_cpu() -> str:
    """CPU model and logical core count of the host running the oracle."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return "%s, %d logical cores" % (model, os.cpu_count() or 0)


def sass_counts(prec: str, d: int, mode: int = 2) -> dict | None:
    """Per-pair instruction counts of the pass kernel's loop (static SASS count,
    profiles/sass_counts.json, written by tools/count_sass.py); mode 2 = LEAPFROG."""
    path = os.path.join(ROOT, "profiles", "sass_counts.json")
    try:
        tab = json.load(open(path))
        key = "%s_d%d_t1" % (prec, d) if mode == 2 else "%s_d%d_t1_m%d" % (prec, d, mode)
        # the rotation loop (every whole unit) is the one that runs; a warp range's partial
        # first / last unit goes through the group-mode loop
        r = dict(tab[key + "_rot"]) if key + "_rot" in tab else dict(tab[key])
        r["count_source"] = ("static SASS count of the rotation loop (MDS_ROT_COUNT build, "
                             "tools/count_sass.py)" if key + "_rot" in tab else "static SASS count of the loop")
        return r
    except Exception:
        return None


def profile_json(name: str) -> dict:
    try:
        return json.load(open(os.path.join(ROOT, "profiles", name)))
    except Exception:
        return {}


def hbm_peak():
    """(GB/s, source): MEASURED_PEAKS.json (driver-written) else the B200_PROFILING.md fallback."""
    try:
        v = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs (of measured)"
    except Exception:
        return 6650.0, "B200_PROFILING.md fallback 6.65 TB/s (of fallback)"


def t_quantiles(w, samples: int = 200000) -> dict:
    """Quantiles of t = delta*_ij / sigma over random pairs of the workload's evaluation
    state (reported with every benchmark; tail t > 8.3 is the cheap part)."""
    rng = np.random.default_rng(1)
    i = rng.integers(0, w.n, samples)
    j = rng.integers(0, w.n, samples)
    keep = i != j
    dd = np.linalg.norm(w.x0[i[keep]] - w.x0[j[keep]], axis=1) / w.sigma
    q = np.quantile(dd, [0.1, 0.5, 0.9])
    return {"p10": float(q[0]), "p50": float(q[1]), "p90": float(q[2]), "frac_gt_8.3": float((dd > 8.3).mean()),
            "pairs_sampled": int(keep.sum())}


def owned_row_ranges(mds, n, rank, world, chunk_rows):
    """Contiguous row ranges of the tile-rows this rank owns (cyclic I mod world),
    cut into pieces of at most chunk_rows rows."""
    own = np.zeros(n, dtype=np.uint8)
    mds.mds_plan(n, rank, world, 148, 12, own)
    out, i = [], 0
    while i < n:
        if not own[i]:
            i += 1
            continue
        j = i
        while j < n and own[j] and j - i < chunk_rows:
            j += 1
        out.append((i, j))
        i = j
    return out


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle as it stands (serial C, 1 core) on this arm's workload/metric:
    each step is a bounded sample (the leading n_s x n_s sub-problem, one full
    evaluation) sized so that K + W steps take about two minutes."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    import workload
    w = workload.config(args.workload)
    budget = 120.0
    n_probe = min(w.n, 2000)
    y_probe = w.y_rows(0, n_probe)
    t0 = time.perf_counter()
    oracle.loglik_grad(y_probe, w.x0[:n_probe], w.sigma, 1, want_absscale=False)
    t_probe = max(time.perf_counter() - t0, 1e-6)
    per_pair = t_probe / (n_probe * (n_probe - 1) / 2)
    per_step = budget / max(1, args.steps + args.warmup)
    ns = int(min(w.n, max(64, math.sqrt(2.0 * per_step / per_pair))))
    ys = w.y_rows(0, ns)
    xs = w.x0[:ns]
    for _ in range(args.warmup):
        oracle.loglik_grad(ys, xs, w.sigma, 1, want_absscale=False)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.loglik_grad(ys, xs, w.sigma, 1, want_absscale=False)
    el = time.perf_counter() - t0
    pairs = ns * (ns - 1) // 2
    v = pairs * args.steps / el
    sample = "leading %d x %d block of %s (%d pairs) per step, serial C oracle, 1 core" % (ns, ns, args.workload, pairs)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": "%s (oracle sample)" % args.workload, "n": ns, "d": w.d},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "host_cpu": host_cpu()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline(w, budget_s: float, tag: str):
    """The oracle as it stands (serial C, 1 core) on a bounded sample of the same
    workload: whole evaluations of its leading n_s x n_s sub-problem."""
    import oracle
    ns = min(w.n, 4000)
    y = w.y_rows(0, ns)
    x = w.x0[:ns]
    evals, tot = 0, 0.0
    while tot < budget_s or evals == 0:
        t0 = time.perf_counter()
        oracle.loglik_grad(y, x, w.sigma, 1, want_absscale=False)
        tot += time.perf_counter() - t0
        evals += 1
    pairs = ns * (ns - 1) // 2
    return {"value": pairs * evals / tot, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": "%d full evaluations (log L + gradient) of the leading %d x %d block of %s (%d pairs "
                      "each), serial C oracle, %.1f s" % (evals, ns, ns, tag, pairs, tot),
            "host_cpu": host_cpu()}


# ----------------------------------------------------------------------------- dry run (CPU)
def run_dry(args):
    """Launcher + rendezvous + ownership plan, no GPU: each rank reports the pairs
    of its tile-rows; rank 0 checks they partition the triangle."""
    import torch
    import torch.distributed as dist
    import workload
    import paper_1905_04582_b200 as mds
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    idx, n, d, kind, pm = workload.CONFIGS[args.workload]
    info = mds.mds_plan(n, rank, world, 148, 12)
    ranges = owned_row_ranges(mds, n, rank, world, 1 << 30)
    t = torch.tensor([float(info["pairs"]), float(info["tiles"]), float(len(ranges))], dtype=torch.float64)
    allv = [torch.zeros_like(t) for _ in range(world)] if world > 1 else [t]
    if world > 1:
        dist.all_gather(allv, t)
    if rank == 0:
        pairs = [float(v[0]) for v in allv]
        print(json.dumps({"dry_run": True, "n_gpus": world, "workload": args.workload, "n": n,
                          "pairs_per_rank": pairs, "total_pairs": sum(pairs), "expected_pairs": n * (n - 1) // 2,
                          "tiles_per_rank": [float(v[1]) for v in allv],
                          "balance_max_over_mean": max(pairs) / (sum(pairs) / world)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- our arm
class Rank:
    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world, self.local = dist_env()
        self.args = args
        # more ranks than GPUs (one test box): ranks share GPU 0 over a gloo group
        # (a plumbing run -- time-sliced, not a measurement); NCCL needs a GPU per rank
        self.shared = args.exchange == "gloo-host" or (self.world > 1 and self.world > torch.cuda.device_count())
        torch.cuda.set_device(self.local if not self.shared else 0)
        if self.world > 1:
            if self.shared:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, vals):
        if self.world == 1:
            return [float(v) for v in vals]
        t = self.torch.tensor([float(v) for v in vals], dtype=self.torch.float64,
                              device="cpu" if self.shared else "cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(v) for v in t.cpu()]

    def nccl_id(self):
        if self.args.exchange not in ("nccl", "p2p") or self.shared:
            return None
        import paper_1905_04582_b200 as mds
        if self.world == 1:
            return None
        obj = [mds.mds_nccl_unique_id() if self.rank == 0 else None]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]


def build_ctx(R, mds, w, prec, stream):
    """A context for workload w on this rank: its tile-rows only, generated and
    uploaded row chunk by row chunk (the full triangle never exists on one host)."""
    t0 = time.perf_counter()
    ctx = mds.MDS(w.n, w.d, prec, True, rank=R.rank, world=R.world, stream=stream, nccl_unique_id=R.nccl_id())
    if R.world > 1 and R.args.exchange == "p2p":
        # the fused peer-memory exchange over the windows' IPC handles; the context's
        # NCCL communicator stays as the fallback if the windows cannot be connected
        try:
            ctx.use_p2p_exchange()
        except Exception as e:  # noqa: BLE001 (reported in the JSON line)
            R.p2p_error = repr(e)
        R.dist.barrier()
    elif R.world > 1 and not ctx.has_communicator():
        ctx.use_torch_allgather(host_staged=R.args.exchange == "gloo-host")
    t_gen = 0.0
    for i0, i1 in owned_row_ranges(mds, w.n, R.rank, R.world, 512):
        a = time.perf_counter()
        y = w.y_rows(i0, i1)
        t_gen += time.perf_counter() - a
        ctx.set_dissimilarity_rows(i0, i1, y)
        del y
    ctx.set_locations(w.x0)
    ctx.set_sigma(w.sigma)
    R.torch.cuda.synchronize()
    return ctx, {"setup_s": time.perf_counter() - t0, "generate_s": t_gen}


# C3's step size: the 50-transition pilot of tools/run_configs.py (acceptance 0.65-0.85)
# settles at 2.352e-3 on this workload (acceptance 0.67 over the 1000 transitions)
C3_STEP_SIZE = 2.352e-3


def run_c3_chain(R, mds, workload, stream):
    """BASELINE configs[2]: the C2 data as a full HMC chain, 1000 transitions x 20
    leapfrog steps through the library's own driver (mds_hmc_run: one CUDA graph of
    the 20 fused passes per transition, momenta drawn on the host, one host sync per
    transition for the accept/reject).  Device time between the chain's first and last
    event (mds_hmc_run's own)."""
    w = workload.config("C3")
    ce, su = build_ctx(R, mds, w, "f64", stream)
    ce.hmc_run(5, 20, C3_STEP_SIZE, 10.0, seed=1905045922, x0=w.x0.copy())       # warm-up (graph, buffers)
    n_iter, L = 1000, 20
    _, st = ce.hmc_run(n_iter, L, C3_STEP_SIZE, 10.0, seed=1905045922 + 100, x0=w.x0.copy())
    ce.close()
    P = w.n * (w.n - 1) // 2
    return {"workload": "C3: N=%d D=%d f64, HMC chain of %d transitions x %d leapfrog steps (prior sd 10, "
                        "step %.4g)" % (w.n, w.d, n_iter, L, C3_STEP_SIZE),
            "value": P * st["grad_evals"] / st["seconds"], "unit": UNIT, "chain_seconds": st["seconds"],
            "us_per_leapfrog_step": st["seconds"] * 1e6 / (n_iter * L), "grad_evals": st["grad_evals"],
            "acceptance": st["accepted"] / n_iter, "l2": "no flush: the chain runs back to back (Y, 120 MB tiled, stays largely in the 126 MB L2)",
            "setup_s": su["setup_s"]}


def time_steps(R, ctx, w, steps, warmup, flush_buf, graph=False, clocks=None):
    """W untimed warm-up leapfrog steps, then K timed ones, each bracketed by CUDA
    events on the context's stream; barrier + synchronize on both sides; optional
    untimed L2 flush before every timed step.  Returns (per-step ms [K], pass-kernel
    mean ms or None)."""
    torch = R.torch
    stream = torch.cuda.current_stream()
    n, d = w.n, w.d
    p0 = torch.from_numpy(w.normals(1, (n, d))).cuda()
    ctx.leapfrog_device(1, R.args.step_size, R.args.prior_sd, p0_dev=p0)
    for _ in range(max(0, warmup - 1)):
        ctx.leapfrog_device(1, R.args.step_size, R.args.prior_sd)
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True, external=graph) for _ in range(steps)]
    ev1 = [torch.cuda.Event(enable_timing=True, external=graph) for _ in range(steps)]

    def body():
        for k in range(steps):
            if flush_buf is not None:
                ctx.l2_flush(flush_buf)
            ev0[k].record(stream)
            ctx.leapfrog_device(1, R.args.step_size, R.args.prior_sd)
            ev1[k].record(stream)

    g = None
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            body()
        torch.cuda.synchronize()
    # sharded: events around the pass kernel inside the library (its share of the step)
    ctx.set_timing(R.world > 1)
    R.barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
        time.sleep(0.2)
    R.barrier()
    torch.cuda.synchronize()
    if g is not None:
        g.replay()
    else:
        body()
    torch.cuda.synchronize()
    R.barrier()
    clk = clocks.stop() if clocks else None
    step_ms = np.array([a.elapsed_time(b) for a, b in zip(ev0, ev1)])
    kern_ms = None
    if R.world > 1:
        kern_ms, _ = ctx.last_timing()
    ctx.set_timing(False)
    if os.environ.get("MDS_PROFILE_PHASES") in ("1", "2"):
        ctx.set_timing(True)
        ctx.leapfrog_device(1, R.args.step_size, R.args.prior_sd)
        ctx.last_timing()
        ctx.set_timing(False)
    return step_ms, kern_ms, clk


def roofline_of(prec, d, pairs_per_launch, kern_ms, clk_mhz, traffic, cfg=None):
    """Roofline of the pass kernel.  fp64: ALU-bound on the FP64
    pipe -- FP64 lane-instructions per pair (static SASS count of the loop) x pairs per
    launch / launch time vs 148 x 64 lanes x clock.  fp32: issue-bound -- issued
    lane-instructions per pair (ncu's dynamic count of the kernel when captured, else the
    static loop count) vs 148 SM x 4 schedulers x 32 lanes x clock."""
    sc = sass_counts(prec, d)
    if sc is None or not kern_ms:
        return None
    nc = profile_json("ncu_summary.json").get("%s_%s" % (cfg, prec)) if cfg else None
    if prec == "f64":
        lanes, bound, ipp = 64, "alu", sc["fp64_per_pair"]
        unit, src = "T fp64-lane-op/s", "148 SM x 64 FP64 lanes/clk x 1.965 GHz max SM clock (B200_PROFILING.md)"
    else:
        lanes, bound = 128, "issue"
        ipp = nc["issued_inst_per_pair_dynamic"] if nc and "issued_inst_per_pair_dynamic" in nc \
            else sc["issued_per_pair"]
        unit = "T issued lane-instr/s"
        src = ("148 SM x 4 schedulers x 1 warp-instruction/clk x 32 lanes x 1.965 GHz (B200_PROFILING.md); "
               "instructions per pair: %s" % ("ncu dynamic count (profiles/ncu_summary.json)"
                                              if nc else "static loop count (profiles/sass_counts.json)"))
    peak = 148 * lanes * SM_MAX_GHZ * 1e9
    achieved = ipp * pairs_per_launch / (kern_ms * 1e-3)
    hbm, hbm_src = hbm_peak()
    bpp = 8.0 if prec == "f64" else 4.0
    rf = {"bound": bound, "achieved": achieved / 1e12, "peak": peak / 1e12,
          "unit": unit, "frac": achieved / peak,
          "traffic": traffic,
          "kernel": "pass_kernel<%s,D=%d,T=1,LEAPFROG>" % (prec, d),
          "ops_per_pair": ipp, "issued_per_pair": sc.get("issued_per_pair"),
          "ops_source": sc.get("count_source"),
          "pass_kernel_ms": kern_ms,
          "peak_source": src,
          "hbm_gbs": bpp * pairs_per_launch / (kern_ms * 1e-3) / 1e9,
          "hbm_frac": bpp * pairs_per_launch / (kern_ms * 1e-3) / (hbm * 1e9), "hbm_peak_source": hbm_src}
    if clk_mhz:
        rf["frac_at_measured_clock"] = achieved / (148 * lanes * clk_mhz * 1e6)
    if prec == "f32":
        rf["fp32_lane_frac"] = sc["fp32_per_pair"] * pairs_per_launch / (kern_ms * 1e-3) / peak
    if prec == "f64":
        # pair-evals/s against R_ALU with the FIXED libdevice reference
        # I64_ref = 160 FP64 instructions per pair (independent of this kernel's count)
        rf["frac_fixed_I64_ref"] = (pairs_per_launch / (kern_ms * 1e-3)) / (148 * 64 * SM_MAX_GHZ * 1e9 / I64_REF)
    return rf


def run_ours(args):
    import torch
    import workload
    import paper_1905_04582_b200 as mds

    R = Rank(args)
    rank, world = R.rank, R.world
    # torch.distributed.run sets OMP_NUM_THREADS=1 per rank: give the input generator
    # this rank's share of the host cores instead
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    workload.set_threads(max(1, (os.cpu_count() or 1) // max(1, local_world)))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    w = workload.config(args.workload)
    n, d = w.n, w.d
    P_N = n * (n - 1) // 2
    ctx, setup = build_ctx(R, mds, w, args.precision, stream)

    y_rank_bytes = (8 if args.precision == "f64" else 4) * P_N / world
    flush = None
    if args.flush == "mds" or (args.flush == "auto" and y_rank_bytes < 2 * L2_BYTES):
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    clocks = ClockSampler(torch.cuda.current_device())
    step_ms, kern_ms, clk = time_steps(R, ctx, w, args.steps, args.warmup, flush,
                                       graph=bool(args.graph), clocks=clocks)
    tot_ms = float(step_ms.sum())
    if kern_ms is None:
        kern_ms = float(step_ms.mean())        # unsharded: a step IS one pass-kernel launch
    tot_ms, kern_ms = R.max_over_ranks([tot_ms, kern_ms])
    ms_per_step = tot_ms / args.steps
    value = P_N * args.steps / (tot_ms * 1e-3)

    # ---- end to end through the public API with host buffers (per step: H2D X, one
    # fused pass [+ exchange], D2H log L + gradient)
    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        return t.numpy()

    xs = [pinned(w.x0), pinned(w.x0 + 1e-6)]
    ll = pinned(np.zeros(1))
    g = pinned(np.zeros((n, d)))
    e2e_steps = int(max(3, min(200, args.e2e_seconds / max(ms_per_step * 1e-3, 1e-6))))
    for q in range(2):
        ctx.set_locations(xs[q % 2])
        mds.mds_log_likelihood_and_gradient(ctx.ctx, ll, g)
    R.barrier()
    torch.cuda.synchronize()
    e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_a.record(stream)
    for q in range(e2e_steps):
        ctx.set_locations(xs[q % 2])
        mds.mds_log_likelihood_and_gradient(ctx.ctx, ll, g)
    e_b.record(stream)
    torch.cuda.synchronize()
    e2e_ms = R.max_over_ranks([e_a.elapsed_time(e_b)])[0]
    e2e = {"value": P_N * e2e_steps / (e2e_ms * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": n * d * 8, "d2h_bytes_per_step": (n * d + 1) * 8, "steps": e2e_steps,
           "api": "mds_set_locations(host X) + mds_log_likelihood_and_gradient(host log L, host grad)"}
    ctx.close()
    del ctx

    # ---- extra configs at N = 1 (the paper's size and BASELINE's "1/2/4/8" config)
    extras = {}
    want = [] if world > 1 else (["C2", "C3", "C4", "C4f32"] if args.extra == "auto" else
                                 [e for e in args.extra.split(",") if e and e != "none"])
    for name in want:
        if name == "C3":
            extras[name] = run_c3_chain(R, mds, workload, stream)
            continue
        cfg = name.replace("f32", "")
        prec = "f32" if name.endswith("f32") else "f64"
        we = workload.config(cfg)
        ce, su = build_ctx(R, mds, we, prec, stream)
        yb = (8 if prec == "f64" else 4) * we.n_pairs
        fb = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if yb < 2 * L2_BYTES else None
        k = max(args.steps, 20)
        sm, _, _ = time_steps(R, ce, we, k, max(args.warmup, 3), fb)
        ce.close()
        del ce, fb
        kms = float(sm.mean())
        rf = roofline_of(prec, we.d, we.n_pairs, kms, clk.get("sm_mhz") if clk else None,
                         profile_json("traffic.json").get("%s_%s" % (cfg, prec)), cfg)
        extras[name] = {"workload": "%s: N=%d D=%d %s, %.0f%% missing" % (cfg, we.n, we.d, prec, 100 * we.p_missing),
                        "value": we.n_pairs / (kms * 1e-3), "unit": UNIT, "ms_per_step": kms, "steps": k,
                        "step_ms_p50": float(np.median(sm)),
                        "l2": "flushed between timed steps (mds_l2_flush, 256 MiB)" if yb < 2 * L2_BYTES
                        else "Y (%.1f GB) > L2, no flush" % (yb / 1e9),
                        "setup_s": su["setup_s"],
                        "roofline_frac": rf["frac"] if rf else None,
                        "roofline_bound": rf["bound"] if rf else None,
                        "frac_fixed_I64_ref": rf.get("frac_fixed_I64_ref") if rf else None}

    if rank != 0:
        if world > 1:
            R.dist.destroy_process_group()
        return

    traffic = profile_json("traffic.json").get("%s_%s" % (args.workload, args.precision))
    roofline = roofline_of(args.precision, d, P_N / world, kern_ms, clk.get("sm_mhz") if clk else None, traffic,
                           args.workload)
    if roofline is not None:
        roofline["pass_kernel_share_of_step"] = kern_ms / ms_per_step
        nc = profile_json("ncu_summary.json").get("%s_%s" % (args.workload, args.precision))
        if nc:
            roofline["ncu"] = nc
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(w, args.cpu_seconds, args.workload)

    if world == 1:
        par = "single GPU"
    else:
        par = "tile-row shards x %d (rank r owns tile-rows I mod %d == r); exchange: %s" % (
            world, world, {"p2p": ("fused peer-memory exchange: the pass kernel stores its partial into every "
                                   "rank's window over NVLink and combines after the flags (one launch per step)"
                                   if not getattr(R, "p2p_error", None) else
                                   "ncclAllGather (peer-memory windows failed: %s)" % R.p2p_error),
                           "nccl": "ncclAllGather of n*d+1 doubles per step by the libmds-owned communicator",
                           "torch": "torch.distributed all_gather_into_tensor (NCCL) callback",
                           "gloo-host": "host-staged gloo all-gather callback (ranks share one GPU)"}[args.exchange])
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": "%s: N=%d D=%d %s clustered (K=189) sigma=%.4f, truncation on; one leapfrog step "
                               "(fused lik+grad pass) per step" % (args.workload, n, d, args.precision, w.sigma),
                   "n": n, "d": d, "pairs_per_step": P_N, "observed_fraction": 1.0 - w.p_missing,
                   "l2": ("flushed between timed steps (untimed mds_l2_flush, 256 MiB write)" if flush is not None
                          else "no flush: the rank's Y (%.1f GB) exceeds the 126 MB L2" % (y_rank_bytes / 1e9)),
                   "launch": "one CUDA graph of the K steps" if args.graph else "stream launches",
                   "parallelism": par, "t_quantiles": t_quantiles(w), **setup},
        "evals_per_s": 1e3 / ms_per_step,
        "step_ms_p50": float(np.median(step_ms)), "step_ms_min": float(step_ms.min()),
        "gpu_launches": (1 if world == 1 else 2) * args.steps,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clk,
        "configs": extras,
        "paper_context": PAPER_CONTEXT,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        R.dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(a))
    if a.impl == "reference":
        run_reference(a)
    elif a.dry_run:
        run_dry(a)
    else:
        run_ours(a)
