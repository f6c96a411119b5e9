"""Summarise an ncu --page source --csv (SASS) dump: stall reasons by instruction class / region."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {n: i for i, n in enumerate(h)}
reasons = [n for n in h if n.startswith("stall_") and "(Not Issued)" not in n]
data = []
for r in rows[2:]:
    try:
        data.append((int(r[0], 16), r[1].strip(), int(r[5] or 0), {k: int(r[idx[k]] or 0) for k in reasons}))
    except (ValueError, IndexError):
        pass
brx = [i for i, d in enumerate(data) if d[1].startswith("BRX")]
lo, hi = (brx[0] - 40, brx[-1] + 1) if brx else (0, 0)
regions = {"pre": data[:lo], "dispatch": data[lo:hi], "post": data[hi:]}
for name, seg in regions.items():
    tot = collections.Counter()
    for d in seg:
        tot.update(d[3])
    ins = sum(d[2] for d in seg)
    print("%-9s inst %7.1fM  samples %6d  %s" % (name, ins / 1e6, sum(tot.values()),
          " ".join("%s=%d" % (k[6:], v) for k, v in tot.most_common(8))))
# dispatch region by opcode
byop = collections.defaultdict(lambda: [0, collections.Counter()])
for d in regions["dispatch"]:
    op = d[1].split()[0] if not d[1].startswith("@") else d[1].split()[1]
    op = op.split(".")[0]
    byop[op][0] += d[2]
    byop[op][1].update(d[3])
print("dispatch region by opcode:")
for op, (ins, c) in sorted(byop.items(), key=lambda kv: -sum(kv[1][1].values())):
    print("  %-8s inst %7.1fM samples %6d  %s" % (op, ins / 1e6, sum(c.values()),
          " ".join("%s=%d" % (k[6:], v) for k, v in c.most_common(4))))
