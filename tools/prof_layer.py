"""Run one layer with one chosen sconv variant a few times (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1802_10280_b200 import escoin, inputs, workloads  # noqa: E402


def main(wl, layer, kname, batch=128, reps=2):
    W = workloads.workload(wl)
    L = [l for l in W.layers if l.name == layer][0]
    dev = torch.device("cuda", 0)
    w = inputs.layer_weights(W.net, L, W.sparsity_permille)
    b = torch.from_numpy(inputs.bias(W.net, L.name, L.M)).to(dev)
    x = torch.from_numpy(inputs.activations(W.net, L.name, 0, batch, L.C, L.H, L.W)).to(dev)
    out = torch.empty((batch, L.M, L.E, L.F), device=dev)
    csr = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad)
    kid = [k[0] for k in escoin.kernels() if k[1] == kname][0]
    csr.set_kernel(kid)
    csr.to_device(0)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(reps):
        escoin.sconv_forward(batch, L.C, L.H, L.W, L.M, L.K, L.stride, L.pad, csr, x, out, b, True, s)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
