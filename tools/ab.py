"""A/B timing of specialised-kernel tunings on chosen layers (flushed L2, CUDA events, median of reps).

usage: python tools/ab.py WORKLOAD layer[,layer...]|all "tun;tun;..." [reps] [batch]
       tun = Q,P,CC,NS,warps,minb,pf,mb,units (0 = the model pick)
Prints one JSON line per (layer, tuning) with the median/min ms, TFLOP/s and whether the output
is bitwise identical to the first tuning's.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("ESCOIN_JIT_CACHE", os.path.join(ROOT, "build", "jit_cache"))
os.makedirs(os.environ["ESCOIN_JIT_CACHE"], exist_ok=True)
from paper_1802_10280_b200 import escoin, inputs, workloads  # noqa: E402


def main():
    wl = workloads.workload(sys.argv[1])
    names = sys.argv[2]
    tunings = [[int(v) for v in t.split(",")] if t.strip() not in ("", "0") else [] for t in sys.argv[3].split(";")]
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    N = int(sys.argv[5]) if len(sys.argv) > 5 else wl.batch
    layers = wl.layers if names == "all" else [l for l in wl.layers if l.name in names.split(",")]
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream()
    from concurrent.futures import ThreadPoolExecutor
    handles = []
    for L in layers:
        w = (inputs.layer_weights_skewed if os.environ.get("AB_SKEW") else inputs.layer_weights)(
            wl.net, L, wl.sparsity_permille)
        b = torch.from_numpy(inputs.bias(wl.net, L.name, L.M)).to(dev)
        x = torch.from_numpy(inputs.activations(wl.net, L.name, 0, N, L.C, L.H, L.W)).to(dev)
        out = torch.empty((N, L.M, L.E, L.F), device=dev)
        hs = [escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad).to_device(0) for _ in tunings]
        handles.append((L, hs, x, out, b))
    t0 = time.time()

    def comp(job):
        h, tun = job
        try:
            h.jit(N, *tun)
            return True
        except escoin.EscoinError:
            return False
    jobs = [(h, t) for (_, hs, _, _, _) in handles for h, t in zip(hs, tunings)]
    with ThreadPoolExecutor(64) as ex:
        ok = list(ex.map(comp, jobs))
    print("# compiled %d kernels in %.1fs" % (sum(ok), time.time() - t0), flush=True)
    for L, hs, x, out, b in handles:
        ref = None
        for h, tun in zip(hs, tunings):
            if h.kernel() != escoin.KERNEL_JIT:
                print(json.dumps({"layer": L.name, "tuning": tun, "error": "unsupported"}))
                continue
            for _ in range(3):
                escoin.sconv_forward(N, L.C, L.H, L.W, L.M, L.K, L.stride, L.pad, h, x, out, b, True, s.cuda_stream)
            ts = []
            for _ in range(reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                escoin.sconv_forward(N, L.C, L.H, L.W, L.M, L.K, L.stride, L.pad, h, x, out, b, True, s.cuda_stream)
                e1.record(s)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            o = out.cpu().numpy().tobytes()
            if ref is None:
                ref = o
            flops = 2.0 * N * h.info()["nnz"] * L.E * L.F
            med = float(np.median(ts))
            print(json.dumps({"layer": L.name, "label": h.label(), "ms": round(med, 5), "ms_min": round(min(ts), 5),
                              "tflops": round(flops / med / 1e9, 2), "same_bits": o == ref}), flush=True)


if __name__ == "__main__":
    main()
