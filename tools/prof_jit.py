"""Run chosen layers of a workload once each through the specialised kernel (for ncu captures).

usage: python tools/prof_jit.py WORKLOAD [layer,layer,...|all] [tuning Q,P,CC,NS,warps,minb,pf,mb,units|0]
Every layer: stretch, compile (cubin cache ESCOIN_JIT_CACHE), one warm-up forward, then an L2
flush and one forward inside the NVTX range "prof" (ncu --nvtx --nvtx-include "prof/").
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("ESCOIN_JIT_CACHE", os.path.join(ROOT, "build", "jit_cache"))
os.makedirs(os.environ["ESCOIN_JIT_CACHE"], exist_ok=True)
from paper_1802_10280_b200 import escoin, inputs, workloads  # noqa: E402


def main():
    wl = workloads.workload(sys.argv[1])
    names = sys.argv[2] if len(sys.argv) > 2 else "all"
    tun = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 and sys.argv[3] != "0" else []
    layers = wl.layers if names == "all" else [l for l in wl.layers if l.name in names.split(",")]
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    runs = []
    for L in layers:
        w = inputs.layer_weights(wl.net, L, wl.sparsity_permille)
        b = torch.from_numpy(inputs.bias(wl.net, L.name, L.M)).to(dev)
        x = torch.from_numpy(inputs.activations(wl.net, L.name, 0, wl.batch, L.C, L.H, L.W)).to(dev)
        out = torch.empty((wl.batch, L.M, L.E, L.F), device=dev)
        csr = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad).to_device(0)
        t0 = time.time()
        csr.jit(wl.batch, *tun)
        print("%s %s compile %.1fs" % (L.name, csr.label(), time.time() - t0), flush=True)
        runs.append((L, csr, x, out, b))
    s = torch.cuda.current_stream().cuda_stream
    for L, csr, x, out, b in runs:
        escoin.sconv_forward(wl.batch, L.C, L.H, L.W, L.M, L.K, L.stride, L.pad, csr, x, out, b, True, s)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("prof")
    for L, csr, x, out, b in runs:
        flush.zero_()
        escoin.sconv_forward(wl.batch, L.C, L.H, L.W, L.M, L.K, L.stride, L.pad, csr, x, out, b, True, s)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
