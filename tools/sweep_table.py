"""Compare variant sweeps: best-7 per layer of one sweep json, or A/B of two."""
import json
import sys

a = json.load(open(sys.argv[1]))
b = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else None
for wl, layers in a.items():
    for L, row in layers.items():
        items = sorted([(v["tflops"], k) for k, v in row.items() if isinstance(v, dict)], reverse=True)
        if b is None:
            print(wl, L, " ".join("%s=%.1f" % (k, t) for t, k in items[:7]))
        else:
            rb = b.get(wl, {}).get(L, {})
            print(wl, L, " ".join("%s=%.1f/%s" % (k, t, rb[k]["tflops"] if isinstance(rb.get(k), dict) else "-")
                                  for t, k in items[:5]))
