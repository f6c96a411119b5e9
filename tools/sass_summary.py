"""Aggregate an ncu `--page source --csv --print-source sass` export by SASS opcode.

usage: python tools/sass_summary.py SOURCE.csv [kernel-substring] > summary.txt
Only the sections of kernels whose name contains the substring (default escoin_jit_sconv) are
counted.  Prints executed warp-instructions per opcode (share of total) with the warp-stall
samples attributed to that opcode split by reason, then the 12 instructions with the most stall
samples — so a multi-MB per-instruction export becomes a few dozen lines (gpurun_out is capped).
"""
import collections
import csv
import re
import sys


def num(x):
    try:
        return float(x.replace(",", "") or 0)
    except ValueError:
        return 0.0


def main(path, want="escoin_jit_sconv"):
    agg = collections.Counter()
    stall = collections.defaultdict(collections.Counter)
    top = []
    hdr = None
    keep = False
    kernels = 0
    for r in csv.reader(open(path, errors="replace")):
        if r and r[0] == "Kernel Name":
            keep = want in (r[1] if len(r) > 1 else "")
            kernels += keep
            hdr = None
            continue
        if r and r[0] == "Address":
            hdr = r
            src, ex = r.index("Source"), r.index("Instructions Executed")
            scols = [(i, c) for i, c in enumerate(r) if c.startswith("stall_") and "Not Issued" not in c]
            continue
        if not keep or hdr is None or len(r) != len(hdr):
            continue
        s = r[src].strip()
        m = re.match(r"^(@!?U?P\w+\s+)?([A-Z0-9_]+)", s)
        if not m:
            continue
        op = m.group(2)
        agg[op] += num(r[ex])
        tot_s = 0.0
        for i, c in scols:
            v = num(r[i])
            stall[op][c[6:]] += v
            tot_s += v
        top.append((tot_s, s[:60], {c[6:]: num(r[i]) for i, c in scols if num(r[i]) > 0}))
    tot = sum(agg.values())
    print("kernels: %d  executed warp instructions: %.0f" % (kernels, tot))
    for op, v in agg.most_common(18):
        st = ", ".join("%s %d" % (k, n) for k, n in stall[op].most_common(3) if n > 0)
        print("%-10s %13.0f %6.2f%%   stalls: %s" % (op, v, 100.0 * v / max(tot, 1), st))
    print("instructions with the most stall samples:")
    for t, s, d in sorted(top, key=lambda x: -x[0])[:12]:
        print("  %7d  %-60s %s" % (t, s, ", ".join("%s %d" % kv for kv in sorted(d.items(), key=lambda x: -x[1])[:3])))


if __name__ == "__main__":
    main(*sys.argv[1:])
