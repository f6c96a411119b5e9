"""Aggregate an ncu `--page source --csv --print-source sass` export by SASS opcode.

usage: python tools/sass_summary.py SOURCE.csv > summary.txt
Prints, per kernel section, executed warp-instructions per opcode (share of total) and the
columns found, so a multi-MB per-instruction export becomes a few lines (gpurun_out is capped).
"""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path, errors="replace")))
    hdr_i = next(i for i, r in enumerate(rows) if any("Source" == c.strip() for c in r))
    hdr = [c.strip() for c in rows[hdr_i]]
    src = hdr.index("Source")
    cand = [i for i, c in enumerate(hdr) if re.search(r"Instructions Executed|inst_executed", c, re.I)
            and "Predicated" not in c]
    ex = cand[0] if cand else None
    stall_cols = [i for i, c in enumerate(hdr) if "Sampling" in c or "stall" in c.lower()]
    print("columns:", hdr)
    agg = collections.Counter()
    samp = collections.Counter()
    tot = 0.0
    for r in rows[hdr_i + 1:]:
        if len(r) <= src or ex is None:
            continue
        s = r[src].strip()
        m = re.match(r"^(@!?U?P\w+\s+)?([A-Z0-9_]+)", s)
        if not m:
            continue
        op = m.group(2)
        try:
            v = float(r[ex].replace(",", "") or 0)
        except ValueError:
            continue
        agg[op] += v
        tot += v
        for i in stall_cols[:1]:
            try:
                samp[op] += float(r[i].replace(",", "") or 0)
            except ValueError:
                pass
    print("total executed warp instructions: %.0f (column %s)" % (tot, hdr[ex] if ex is not None else None))
    for op, v in agg.most_common(25):
        print("%-12s %14.0f %6.2f%%  samples %8.0f" % (op, v, 100.0 * v / max(tot, 1), samp[op]))


if __name__ == "__main__":
    main(sys.argv[1])
