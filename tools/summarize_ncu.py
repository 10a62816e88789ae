#!/usr/bin/env python
"""Summaries of ncu captures for profiles/ (run here, on the CPU side, after gpurun).

  python tools/summarize_ncu.py KEY=gpurun_out/<capture>.ncu-rep ... [--launches gpurun_out/<list>.csv]
      [--round r02]

KEY is the bench config key (e.g. C5_f64).  Writes/updates
  profiles/ncu_summary.json  key metrics of the one captured pass-kernel launch per KEY
  profiles/traffic.json      dram read + write bytes of that launch per KEY (bench's roofline "traffic")
  profiles/<round>/launches_<name>.txt  per-kernel launch counts / mean time / share of the list
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "sm__inst_executed_pipe_fp64.sum": "fp64_warp_inst",
    "sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fp32_fma_pipe_active_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_inst",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math_pipe_throttle",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio": "stall_not_selected",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio": "stall_dispatch",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_scoreboard",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
         "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9, "Ghz": 1e9, "GHz": 1e9, "cycle/second": 1.0,
         "cycle/nsecond": 1e9, "cycle/usecond": 1e6}


def raw(rep):
    txt = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2]


def summarize(rep, pairs):
    h, u, v = raw(rep)
    out = {"capture": os.path.relpath(rep, ROOT), "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None}
    for i, n in enumerate(h):
        if n in METRICS:
            try:
                x = float(v[i])
            except ValueError:
                continue
            x *= SCALE.get(u[i], 1.0)
            out[METRICS[n]] = x
    if pairs:
        out["pairs"] = pairs
        if "fp64_warp_inst" in out:
            out["fp64_inst_per_pair"] = out["fp64_warp_inst"] * 32 / pairs
        if "warp_inst" in out:
            out["issued_inst_per_pair_dynamic"] = out["warp_inst"] * 32 / pairs
        if "dram_read" in out:
            out["dram_bytes_per_pair"] = (out["dram_read"] + out.get("dram_write", 0.0)) / pairs
    return out


def launches(csv_path, name, rnd):
    per = defaultdict(list)
    with open(csv_path) as f:
        lines = [l for l in f if l.startswith('"')]
    for row in csv.DictReader(io.StringIO("".join(lines))):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = row["Kernel Name"].split("(")[0]
        per[k].append(float(row["Metric Value"]) * SCALE.get(row["Metric Unit"], 1.0))
    tot = sum(sum(v) for v in per.values())
    lines = ["# %s: %d launches (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised)"
             % (os.path.relpath(csv_path, ROOT), sum(len(v) for v in per.values())),
             "%-70s %6s %12s %8s" % ("kernel", "count", "mean_us", "share")]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append("%-70s %6d %12.2f %7.1f%%" % (k[:70], len(v), 1e6 * sum(v) / len(v), 100 * sum(v) / tot))
    d = os.path.join(PROF, rnd)
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, "launches_%s.txt" % name)
    open(path, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def main():
    args = sys.argv[1:]
    rnd = "r02"
    if "--round" in args:
        k = args.index("--round")
        rnd = args[k + 1]
        del args[k:k + 2]
    if "--launches" in args:
        k = args.index("--launches")
        p = args[k + 1]
        del args[k:k + 2]
        launches(p, os.path.splitext(os.path.basename(p))[0], rnd)
    pairs_of = {"C1": 2016, "C2": 14534136, "C4": 449985000, "C5": 4999950000}
    sj = os.path.join(PROF, "ncu_summary.json")
    tj = os.path.join(PROF, "traffic.json")
    summ = json.load(open(sj)) if os.path.exists(sj) else {}
    traf = json.load(open(tj)) if os.path.exists(tj) else {}
    for a in args:
        key, rep = a.split("=", 1)
        s = summarize(rep, pairs_of.get(key.split("_")[0]))
        summ[key] = s
        if "dram_read" in s:
            traf[key] = s["dram_read"] + s.get("dram_write", 0.0)
        print(key, json.dumps(s, indent=1))
    summ["_about"] = ("ncu --set full --clock-control none of ONE timed leapfrog pass (pass_kernel<T,D,1,LEAPFROG>) "
                      "per bench config; per-pair counts use all N(N-1)/2 pairs (tools/summarize_ncu.py)")
    traf["_about"] = ("dram__bytes_read.sum + dram__bytes_write.sum of one timed pass_kernel launch per bench config "
                      "(ncu --set full; profiles/ncu_summary.json)")
    json.dump(summ, open(sj, "w"), indent=1, sort_keys=True)
    json.dump(traf, open(tj, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
