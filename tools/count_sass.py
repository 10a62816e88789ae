#!/usr/bin/env python
"""Static SASS instruction mix of the pair kernel's inner loop -> profiles/sass_counts.json.

For every pass_kernel<T, D, TRUNC, MODE> instantiation in libmds.so: find the loop
(the backward branch of the column-group loop), count its instructions by
class, and divide by the pairs one loop trip evaluates per lane (its MUFU.RSQ count).  The
FP64 count per pair is the 'algorithmic' FP64 work of the roofline.
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1905_04582_b200", "libmds.so")
OUT = os.path.join(ROOT, "profiles", "sass_counts.json")

FP64 = {"DFMA", "DMUL", "DADD", "DSETP", "DMNMX"}
CSRC = os.path.join(ROOT, "paper_1905_04582_b200", "csrc")
FP32 = {"FFMA", "FMUL", "FADD", "FSETP", "FMNMX", "FSEL"}


def rotation_only_sass():
    """LEAPFROG pass kernels (mode 2) built with MDS_ROT_COUNT, whose only pair loop is
    the rotation's (it runs every whole unit; the group-mode loop of a warp range's
    partial first / last unit is compiled out there).  The libmds.so kernels hold
    both loops; the static count picks the smaller one."""
    out = []
    for prec in ("f64", "f32"):
        obj = "/tmp/mds_count_rot_m2_%s.o" % prec
        subprocess.check_call(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-I", os.path.join(ROOT, "include"), "-DMDS_ROT_COUNT", "-c", "-o", obj,
                               os.path.join(CSRC, "pass_m2_%s.cu" % prec)])
        out.append(subprocess.check_output(["cuobjdump", "-sass", obj], text=True))
    return "\n".join(out)


def main():
    sass = subprocess.check_output(["cuobjdump", "-sass", LIB], text=True)
    funcs = [("", f) for f in re.split(r"\n\s+Function : ", sass)[1:]]
    funcs += [("_rot", f) for f in re.split(r"\n\s+Function : ", rotation_only_sass())[1:]]
    res = {}
    for tag, f in funcs:
        name = f.split("\n", 1)[0].strip()
        m = re.match(r"_ZN4mdsk11pass_kernelI([fd])Li(\d)ELb([01])ELi(\d)EEEvNS_8PassArgsE", name)
        if not m:
            continue
        prec = "f64" if m.group(1) == "d" else "f32"
        d, t, mode = int(m.group(2)), int(m.group(3)), int(m.group(4))
        lines = re.findall(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", f)
        ins = [(int(a, 16), txt.strip()) for a, txt in lines]
        # backward branch of the group loop
        # the pair loop is the backward-branch loop with the most MUFU.RSQ ops
        loop, best = None, None
        for addr, txt in ins:
            # a loop's back edge: predicated, not a warp-uniform retry (BRA.U.ANY) or an
            # out-of-line wait path jumping back
            mm = re.match(r"@!?P\w+\s+BRA\s+(0x[0-9a-f]+)", txt)
            if mm and int(mm.group(1), 16) < addr:
                cand = (int(mm.group(1), 16), addr)
                # the pair loop: one reciprocal-sqrt seed per pair (the tree-prior walk
                # fused into the leapfrog modes has MUFU.RCP64H loops but no RSQ)
                nm = sum(1 for a2, t2 in ins if cand[0] <= a2 <= cand[1] and "MUFU.RSQ" in t2)
                # innermost loop among those with the most RSQ: the 4-column group loop
                # (8 pairs per lane per trip), not the unit / segment / step loops around it
                key = (nm, -(cand[1] - cand[0]))
                if best is None or key > best:
                    loop, best = cand, key
        if loop is None:
            continue
        body = [txt for addr, txt in ins if loop[0] <= addr <= loop[1]]
        ops = [re.sub(r"^@!?U?P\w+\s+", "", b).split()[0].split(".")[0] for b in body]
        # one reciprocal-sqrt seed per evaluated pair: the loop's pair count
        npairs = sum(1 for b in body if re.search(r"MUFU\.RSQ", b))
        n64 = sum(o in FP64 for o in ops)
        n32 = sum(o in FP32 for o in ops)
        nmufu = sum(o == "MUFU" for o in ops)
        # key: <prec>_d<D>_t<T> for the leapfrog pass (mode 2, the bench kernel),
        # + "_m<mode>" for the other modes (mds_pass.cuh "Mode")
        key = "%s_d%d_t%d" % (prec, d, t) + ("" if mode == 2 else "_m%d" % mode) + tag
        res[key] = {
            "kernel": name, "loop_instructions": len(ops),
            "pairs_per_trip": npairs,
            "fp64_per_pair": n64 / npairs, "fp32_per_pair": n32 / npairs,
            "mufu_per_pair": nmufu / npairs, "issued_per_pair": len(ops) / npairs,
        }
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    json.dump(res, open(OUT, "w"), indent=1, sort_keys=True)
    for k in sorted(res):
        r = res[k]
        print("%-10s fp64/pair %6.2f  fp32/pair %6.2f  mufu/pair %4.2f  issued/pair %6.2f" % (
            k, r["fp64_per_pair"], r["fp32_per_pair"], r["mufu_per_pair"], r["issued_per_pair"]))


if __name__ == "__main__":
    main()
