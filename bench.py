#!/usr/bin/env python
"""bench.py -- MDS likelihood+gradient pair-evals/s on B200 (BASELINE.json metric).

One "step" = one HMC leapfrog step of the hot path:
half-kick + drift, one fused likelihood+gradient pass over every unordered pair
(pair kernel + fixed-order reduction [+ NCCL all-gather + combine when sharded]),
half-kick.  Workload (N=1): BASELINE.json configs[1] = C2, N = 5392, D = 2, fp64,
clustered synthetic points (K = 189), truncation on.  value = unordered pairs
(all of them, observed or not) x steps / device time.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun (N > 1) every rank owns the tile-rows r mod N and the exchange
is torch.distributed all_gather_into_tensor over NCCL; timing is CUDA events
on the launching stream, max over ranks.  L2 is flushed (256 MiB write)
between timed steps because C2's tiled Y (120 MB) would otherwise sit in the
126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import math
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--step-size", type=float, default=2e-5)
    ap.add_argument("--prior-sd", type=float, default=10.0)
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", type=int, default=0,
                    help="1: capture the K timed steps (flush + step, with external timing events) in one CUDA "
                         "graph and replay it (N = 1 only)")
    ap.add_argument("--flush", choices=["torch", "mds", "mds-clean"], default="mds",
                    help="L2 flush between timed steps: torch fill, or mds_l2_flush (same write, launched "
                         "with the pass kernel's grid/block/smem shape)")
    return ap.parse_args()


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
def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def cpu_baseline(w, budget_s: float):
    """The oracle as it stands (serial C, 1 core) on a bounded sample of the
    same workload: the leading n_s x n_s sub-problem, whole evaluations."""
    import oracle
    n = w.n
    y = w.y_rows(0, n)
    # time one full evaluation; if too slow for the budget, shrink to a leading block
    ns = n
    t0 = time.perf_counter()
    oracle.loglik_grad(y, w.x0, w.sigma, 1, want_absscale=False)
    t1 = time.perf_counter() - t0
    evals, tot = 1, t1
    while tot < budget_s:
        t0 = time.perf_counter()
        oracle.loglik_grad(y, w.x0, w.sigma, 1, want_absscale=False)
        tot += time.perf_counter() - t0
        evals += 1
    pairs = ns * (ns - 1) // 2
    return {"value": pairs * evals / tot, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": "%d full %s evaluations (N=%d, %d pairs each), serial C oracle, %.1f s" % (
                evals, "C2" if n == 5392 else "workload", ns, pairs, tot),
            "host_cpu": host_cpu()}


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


def sass_fp64_per_pair(prec: str, d: int) -> float | None:
    """FP64-pipe instructions per evaluated pair slot in the pair kernel's loop
    (static SASS count, profiles/sass_counts.json, written by tools/count_sass.py)."""
    path = os.path.join(ROOT, "profiles", "sass_counts.json")
    try:
        tab = json.load(open(path))
        return tab["%s_d%d_t1" % (prec, d)]["fp64_per_pair"]
    except Exception:
        return None


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    import workload
    w = workload.config(args.workload)
    budget = 120.0
    # per-step sample: leading n_s items so that (K + W) steps take ~budget seconds
    ns_full = w.n
    y_all = w.y_rows(0, ns_full)
    t0 = time.perf_counter()
    oracle.loglik_grad(y_all, w.x0, w.sigma, 1, want_absscale=False)
    t_full = time.perf_counter() - t0
    per_step = budget / max(1, args.steps + args.warmup)
    frac = min(1.0, per_step / max(t_full, 1e-9))
    ns = max(64, int(ns_full * math.sqrt(frac)))
    ys = y_all[: ns * (ns - 1) // 2]
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
    }))


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import workload
    import paper_1905_04582_b200 as mds

    w = workload.config(args.workload)
    n, d = w.n, w.d
    P_N = n * (n - 1) // 2
    # a dedicated stream (graph capture needs a non-default stream)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = mds.MDS(n, d, args.precision, True, rank=rank, world=world, stream=stream)
    if world > 1:
        ctx.use_torch_allgather()
    t0 = time.perf_counter()
    y = w.y_packed()
    ctx.set_dissimilarities_packed(y)
    del y
    ctx.set_locations(w.x0)
    ctx.set_sigma(w.sigma)
    t_setup = time.perf_counter() - t0
    p0 = torch.from_numpy(w.normals(1, (n, d))).cuda()
    # our kernels per leapfrog step: the persistent pass kernel (phase A pairs +
    # phase B reduction/leapfrog update); sharded: + combine + update kernels
    launches_per_step = 1 if world == 1 else 3

    # > 126 MB L2 (mds-clean: two halves of 256 MiB, written then read)
    flush = torch.empty((512 if args.flush == "mds-clean" else 256) << 20, dtype=torch.uint8, device="cuda")
    # warm-up (also primes grad log pi)
    ctx.leapfrog_device(1, args.step_size, args.prior_sd, p0_dev=p0)
    for _ in range(max(0, args.warmup - 1)):
        ctx.leapfrog_device(1, args.step_size, args.prior_sd)
    torch.cuda.synchronize()

    clocks = ClockSampler(torch.cuda.current_device())
    use_graph = bool(args.graph) and world == 1
    ev0 = [torch.cuda.Event(enable_timing=True, external=use_graph) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True, external=use_graph) for _ in range(args.steps)]

    def timed_steps():
        for k in range(args.steps):
            if args.flush == "mds":        # untimed L2 flush before every timed step
                ctx.l2_flush(flush)
            elif args.flush == "mds-clean":
                ctx.l2_flush_clean(flush)
            else:
                flush.zero_()
            ev0[k].record(stream)
            ctx.leapfrog_device(1, args.step_size, args.prior_sd)
            ev1[k].record(stream)

    graph = None
    if use_graph:
        # launch mechanics only: the same K (flush, step) pairs, captured once on
        # the context's stream and replayed; events are external (timed) nodes
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            timed_steps()
        torch.cuda.synchronize()
    # the library's timing mode (events around every launch) perturbs
    # back-to-back cooperative launches by ~8 us/step; unsharded, a step IS one
    # pass-kernel launch, so the per-step events below are the kernel's launch
    # duration.  Sharded steps have several kernels + NCCL: timing mode is on.
    ctx.set_timing(world > 1)
    clocks.start()
    time.sleep(0.2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if graph is not None:
        graph.replay()
    else:
        timed_steps()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = np.array([a.elapsed_time(b) for a, b in zip(ev0, ev1)])
    if os.environ.get("MDS_PROFILE_PHASES") in ("1", "2"):
        ctx.last_timing()                  # prints the last pass's phase split to stderr
    if world > 1:
        pair_ms, red_ms = ctx.last_timing()
    else:
        pair_ms, red_ms = float(step_ms.mean()), 0.0
    ctx.set_timing(False)
    tot_ms = float(step_ms.sum())
    if world > 1:
        t = torch.tensor([tot_ms, pair_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms, pair_ms = float(t[0]), float(t[1])
    ms_per_step = tot_ms / args.steps
    value = P_N * args.steps / (tot_ms * 1e-3)

    # ---- end to end through the public API with host buffers (per step: H2D X, pass, D2H log L + grad)
    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        return t.numpy()

    xs = [pinned(w.x0), pinned(w.x0 + 1e-6)]
    ll = pinned(np.zeros(1))
    g = pinned(np.zeros((n, d)))
    for q in range(3):
        ctx.set_locations(xs[q % 2])
        mds.mds_log_likelihood_and_gradient(ctx.ctx, ll, g)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_a.record(stream)
    for q in range(args.e2e_steps):
        ctx.set_locations(xs[q % 2])
        mds.mds_log_likelihood_and_gradient(ctx.ctx, ll, g)
    e_b.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e_a.elapsed_time(e_b)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    e2e = {"value": P_N * args.e2e_steps / (e2e_ms * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": n * d * 8, "d2h_bytes_per_step": (n * d + 1) * 8,
           "steps": args.e2e_steps,
           "api": "mds_set_locations(host X) + mds_log_likelihood_and_gradient(host log L, host grad)"}

    if rank != 0:
        ctx.close()
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline: FP64 pipe (ALU-bound path)
    fp64_rate, fp32_rate = mds.mds_measure_fma_peaks()
    sms, _, _ = mds.mds_device_info()
    peak_derived = sms * 64 * 1.965e9          # 64 FP64 lanes/SM/clk x max SM clock
    ipp = sass_fp64_per_pair(args.precision, d)
    roofline = None
    if ipp is not None and pair_ms > 0:
        pairs_per_launch = P_N / world
        achieved = ipp * pairs_per_launch / (pair_ms * 1e-3)
        roofline = {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_derived / 1e12,
                    "unit": "T fp64-lane-op/s", "frac": achieved / peak_derived,
                    "traffic": None, "kernel": "pass_kernel<%s,D=%d,T=1,LEAPFROG>" % (args.precision, d),
                    "fp64_ops_per_pair": ipp, "pass_kernel_ms": pair_ms, "post_kernel_ms": red_ms,
                    "peak_source": "148 SM x 64 FP64 lanes/clk x 1.965 GHz (B200_PROFILING.md SM count/clock); "
                                   "dfma microbenchmark on this GPU: %.2f T lane-op/s" % (fp64_rate / 1e12),
                    "hbm_frac": (8.0 * pairs_per_launch / (pair_ms * 1e-3)) / 6543.7e9}
        tr = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tr):
            try:
                roofline["traffic"] = json.load(open(tr)).get("%s_%s" % (args.workload, args.precision))
            except Exception:
                pass

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(w, args.cpu_seconds)

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": "%s: N=%d D=%d %s clustered (K=189) sigma=%.4f, truncation on; "
                               "one leapfrog step (fused lik+grad pass) per step" % (args.workload, n, d,
                                                                                    args.precision, w.sigma),
                   "n": n, "d": d, "pairs_per_step": P_N, "observed_fraction": 1.0 - w.p_missing,
                   "l2": "flushed between timed steps (untimed, %s)" % (
                       {"torch": "256 MiB torch fill", "mds": "256 MiB write, mds_l2_flush",
                        "mds-clean": "256 MiB write + 256 MiB read, mds_l2_flush_clean"}[args.flush]),
                   "launch": "one CUDA graph of the K (flush, step) pairs" if graph is not None
                   else "stream launches",
                   "parallelism": "tile-row shards x %d" % world if world > 1 else "single GPU",
                   "setup_s": t_setup},
        "evals_per_s": 1e3 / ms_per_step,
        "step_ms_p50": float(np.median(step_ms)), "step_ms_min": float(step_ms.min()),
        "gpu_launches": launches_per_step * args.steps,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clk,
        "paper_context": PAPER_CONTEXT,
        "fma_peaks_measured": {"fp64_lane_op_per_s": fp64_rate, "fp32_lane_op_per_s": fp32_rate},
    }
    print(json.dumps(out))
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
