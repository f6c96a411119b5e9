"""Per-layer timing of the pattern-specialised kernel against the autotuned interpreter kernels.

python tools/jit_probe.py WORKLOAD [tuning ...]   tuning = Q,P,CC,NS,warps,minb,prefetch (0 = default)
Prints one JSON line per (layer, candidate): ms, TFLOP/s, compile seconds, registers.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1802_10280_b200 import escoin, inputs, workloads  # noqa: E402


_flush = None


def timeit(fn, reps=10):
    """Mean ms over reps; FLUSH=1: a 256 MB write before every rep (outside the events), as bench.py."""
    global _flush
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    if os.environ.get("FLUSH") == "1":
        if _flush is None:
            _flush = torch.empty(64 * 1024 * 1024, device="cuda")
        tot = 0.0
        for _ in range(reps):
            _flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / reps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    wl = sys.argv[1]
    tunings = [tuple(int(v) for v in a.split(",")) for a in sys.argv[2:]] or [(0,) * 7]
    W = workloads.workload(wl)
    N = 128
    only = os.environ.get("LAYERS")
    for L in W.layers:
        if only and L.name not in only.split(","):
            continue
        x = torch.from_numpy(inputs.activations(W.net, L.name, 0, N, L.C, L.H, L.W)).cuda()
        w = inputs.layer_weights(W.net, L, W.sparsity_permille)
        b = torch.from_numpy(inputs.bias(W.net, L.name, L.M)).cuda()
        out = torch.empty((N, L.M, L.E, L.F), device="cuda")
        csr = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad).to_device(0)
        nnz = csr.info()["nnz"]
        flop = 2.0 * N * nnz * L.E * L.F
        st = torch.cuda.current_stream().cuda_stream
        if os.environ.get("NO_AUTOTUNE") != "1":
            kid, _ = csr.autotune(N, x, out, b, True, 3, st)
        else:
            kid = csr.kernel()
        ms = timeit(lambda: escoin.forward(csr, x, bias=b, relu=True, out=out))
        ref = out.clone()
        print(json.dumps(dict(layer=L.name, cand="auto:" + escoin.kernel_name(kid), ms=round(ms, 4),
                              tflops=round(flop / ms / 1e9, 2))), flush=True)
        for t in tunings:
            t0 = time.time()
            try:
                csr.jit(N, *t)
            except escoin.EscoinError as e:
                print(json.dumps(dict(layer=L.name, cand="jit" + str(t), error=str(e))), flush=True)
                continue
            ct = time.time() - t0
            ms = timeit(lambda: escoin.forward(csr, x, bias=b, relu=True, out=out))
            same = bool(torch.equal(out, ref))
            print(json.dumps(dict(layer=L.name, cand="jit" + str(t), ms=round(ms, 4),
                                  tflops=round(flop / ms / 1e9, 2), compile_s=round(ct, 1), bitwise=same,
                                  **csr.jit_info())), flush=True)
        csr.free()


if __name__ == "__main__":
    main()
