#!/usr/bin/env python
"""Summarise an `ncu --page source --csv --print-source sass` dump: stall samples by
reason over the whole kernel and over the hottest contiguous region, and the top
instructions by sample count.  usage: ncu_src_summary.py source.csv [top]"""
import csv
import sys
from collections import Counter


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    H = rows[hdr]
    data = [r for r in rows[hdr + 1:] if len(r) == len(H)]
    ix = {h: i for i, h in enumerate(H)}
    stall_cols = [h for h in H if h.startswith("stall_") and "Not Issued" not in h]
    tot = Counter()
    for r in data:
        for h in stall_cols:
            tot[h] += int(r[ix[h]] or 0)
    S = sum(tot.values())
    print("total samples", S)
    for h, v in tot.most_common():
        if v:
            print("  %-24s %6.2f%%" % (h, 100.0 * v / S))
    samp = [(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), k) for k, r in enumerate(data)]
    print("top instructions (samples, index, source, main stalls)")
    for v, k in sorted(samp, reverse=True)[:top]:
        r = data[k]
        st = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:3]
        print("%6d %5d %-60s %s" % (v, k, r[ix["Source"]].strip()[:60], " ".join("%s=%d" % (n, c) for c, n in st if c)))
    # opcode classes over all samples
    cls = Counter()
    for v, k in samp:
        op = data[k][ix["Source"]].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        cls[o.split(".")[0]] += v
    print("samples by opcode:", ", ".join("%s %.1f%%" % (o, 100.0 * v / S) for o, v in cls.most_common(20)))


if __name__ == "__main__":
    main()
