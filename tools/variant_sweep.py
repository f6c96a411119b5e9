"""Time every applicable sconv variant on every layer of a workload (diagnostics for kernel customization)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1802_10280_b200 import escoin, inputs, workloads  # noqa: E402


def main(wl_name, batch=128, reps=5):
    W = workloads.workload(wl_name)
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 * 1024 * 1024, device=dev)
    res = {}
    for L in W.layers:
        w = inputs.layer_weights(W.net, L, W.sparsity_permille)
        b = torch.from_numpy(inputs.bias(W.net, L.name, L.M)).to(dev)
        x = torch.from_numpy(inputs.activations(W.net, L.name, 0, batch, L.C, L.H, L.W)).to(dev)
        out = torch.empty((batch, L.M, L.E, L.F), device=dev)
        csr = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad)
        csr.to_device(0)
        nnz = csr.info()["nnz"]
        row = {}
        for k in escoin.kernels():
            if not (k[0] == 0 or (k[2] == L.K and k[3] == L.stride)):
                continue
            try:
                csr.set_kernel(k[0])
            except escoin.EscoinError as e:
                row[k[1]] = str(e.status)
                continue
            s = torch.cuda.current_stream().cuda_stream
            escoin.sconv_forward(batch, L.C, L.H, L.W, L.M, L.K, L.stride, L.pad, csr, x, out, b, True, s)
            ts = []
            for _ in range(reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                escoin.sconv_forward(batch, L.C, L.H, L.W, L.M, L.K, L.stride, L.pad, csr, x, out, b, True, s)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            row[k[1]] = {"ms": round(ms, 4), "tflops": round(2.0 * batch * nnz * L.E * L.F / ms / 1e9, 2)}
        res[L.name] = row
        print(L.name, json.dumps(row), flush=True)
    return res


if __name__ == "__main__":
    r = {}
    for wl in sys.argv[1:] or ["alexnet"]:
        r[wl] = main(wl)
    json.dump(r, open("gpurun_out/variant_sweep.json", "w"), indent=1)
