"""BASELINE configs[4]: density sweep 5-100% on the AlexNet conv3 shape, batch 128.

Direct sparse (escoin, autotuned) vs im2col+cuBLAS SGEMM vs im2col+cuSPARSE SpMM
vs cuDNN FP32 dense, plus the dense tensor-core references (cuDNN TF32 and our
tcgen05 3xTF32 kernel); reports ms per layer and the crossover densities.
Writes gpurun_out/density_sweep.json and gpurun_out/density_sweep.md.
"""
import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, ".")
import baselines as bl  # noqa: E402
from paper_1802_10280_b200 import escoin, inputs, workloads  # noqa: E402


def timeit(fn, flush, reps=5):
    for _ in range(2):
        flush.zero_()
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main(batch=128):
    L = workloads.sweep_layer()
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 * 1024 * 1024, device=dev)
    x = torch.from_numpy(inputs.activations("alexnet", L.name, 0, batch, L.C, L.H, L.W)).to(dev)
    b_np = inputs.bias("alexnet", L.name, L.M)
    bias = torch.from_numpy(b_np).to(dev)
    out = torch.empty((batch, L.M, L.E, L.F), device=dev)
    s = torch.cuda.current_stream().cuda_stream
    rows = []
    # pattern-specialised kernels: compiled for every density up front, in parallel host threads
    ws = {dpm: inputs.layer_weights("alexnet", L, 1000 - dpm) for dpm in workloads.SWEEP_DENSITIES_PERMILLE}
    jits = {dpm: escoin.Csr.stretch(ws[dpm], L.H, L.W, L.stride, L.pad).to_device(0) for dpm in ws}
    with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        list(ex.map(lambda c: c.jit(batch), jits.values()))
    for dpm in workloads.SWEEP_DENSITIES_PERMILLE:
        w = ws[dpm]
        csr = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad).to_device(0)
        nnz = csr.info()["nnz"]
        kid, _ = csr.autotune(batch, x, out, bias, True, 3, s)
        run = lambda c: escoin.sconv_forward(batch, L.C, L.H, L.W, L.M, L.K, L.stride, L.pad, c, x, out, bias,
                                             True, s)
        t_int = timeit(lambda: run(csr), flush)
        t_jit = timeit(lambda: run(jits[dpm]), flush)
        t_esc = min(t_int, t_jit)
        y = torch.empty_like(out)
        r = {"density": dpm / 1000.0, "nnz": nnz, "escoin_ms": t_esc,
             "escoin_kernel": "jit" if t_jit <= t_int else escoin.kernel_name(kid),
             "escoin_tflops": 2.0 * batch * nnz * L.E * L.F / t_esc / 1e9,
             "interpreter_ms": t_int, "interpreter_kernel": escoin.kernel_name(kid), "jit_ms": t_jit}
        for mode in ["cublas", "cusparse"]:
            op = bl.LoweredConv(L, w, b_np, dev, mode)
            r[mode + "_ms"] = timeit(lambda: op(x, y), flush)
            del op
        op = bl.CudnnConv(L, w, b_np, dev)
        r["cudnn_ms"] = timeit(lambda: op(x, y), flush)
        op = bl.CudnnConv(L, w, b_np, dev, "tf32")
        r["cudnn_tf32_ms"] = timeit(lambda: op(x, y), flush)
        wd = torch.from_numpy(w).to(dev)
        r["tcgen05_3xtf32_ms"] = timeit(lambda: escoin.bench_dense_tc_forward(wd, x, bias, L.stride, L.pad, True, 3,
                                                                             out=y), flush)
        rows.append(r)
        print(json.dumps(r), flush=True)
        csr.free()
        jits[dpm].free()
    def crossover(key):
        for r in rows:
            if r["escoin_ms"] > r[key]:
                return r["density"]
        return None
    res = {"layer": "AlexNet conv3 shape (C=256, 13x13, M=384, 3x3, pad 1), batch %d" % batch, "rows": rows,
           "escoin_slower_than_cublas_from_density": crossover("cublas_ms"),
           "escoin_slower_than_cusparse_from_density": crossover("cusparse_ms"),
           "escoin_slower_than_cudnn_from_density": crossover("cudnn_ms"),
           "escoin_slower_than_cudnn_tf32_from_density": crossover("cudnn_tf32_ms"),
           "escoin_slower_than_tcgen05_3xtf32_from_density": crossover("tcgen05_3xtf32_ms")}
    json.dump(res, open("gpurun_out/density_sweep.json", "w"), indent=1)
    md = ["# Density sweep — %s" % res["layer"], "",
          "| density | nnz | escoin ms (kernel) | escoin TFLOP/s | JIT ms | best interpreter ms (kernel) | im2col+cuBLAS ms | im2col+cuSPARSE ms | cuDNN FP32 ms "
          "| cuDNN TF32 ms | tcgen05 3xTF32 ms |",
          "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        md.append("| %.2f | %d | %.3f (%s) | %.2f | %.3f | %.3f (%s) | %.3f | %.3f | %.3f | %.3f | %.3f |" % (
            r["density"], r["nnz"], r["escoin_ms"], r["escoin_kernel"], r["escoin_tflops"], r["jit_ms"],
            r["interpreter_ms"], r["interpreter_kernel"], r["cublas_ms"],
            r["cusparse_ms"], r["cudnn_ms"], r["cudnn_tf32_ms"], r["tcgen05_3xtf32_ms"]))
    md += ["", "escoin slower than cuBLAS from density %s, than cuSPARSE from %s, than cuDNN FP32 from %s, "
           "than cuDNN TF32 from %s, than the tcgen05 3xTF32 kernel from %s (None = never)." % (
               res["escoin_slower_than_cublas_from_density"], res["escoin_slower_than_cusparse_from_density"],
               res["escoin_slower_than_cudnn_from_density"], res["escoin_slower_than_cudnn_tf32_from_density"],
               res["escoin_slower_than_tcgen05_3xtf32_from_density"])]
    open("gpurun_out/density_sweep.md", "w").write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
