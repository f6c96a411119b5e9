"""Per-rank parity of the batch-sharded driver (run under torchrun by tests/test_sconv_gpu.py).

Every rank runs bench.py's own setup (CSR stretched on rank 0 and broadcast, wrap_device on the
other ranks, specialised kernels compiled once per node through the cubin cache, autotune) on
its shard [n0, n0 + B) of the GLOBAL batch (strong scaling), then checks
  * its outputs against the fp64 oracle at sampled points, for the same GLOBAL image indices;
  * bitwise against a full-global-batch forward of the same handle sliced to [n0, n0 + B)
    (R#12: the result of an image does not depend on the batch it is computed in).
Rank 0 prints one JSON line with every rank's result.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import oracle  # noqa: E402
from paper_1802_10280_b200 import escoin, inputs, shard, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="alexnet")
    ap.add_argument("--layers", default="conv3,conv4")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--backend", default="gloo")
    a = ap.parse_args()
    rank, world, _ = shard.world()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group(a.backend)
    W = workloads.workload(a.workload)
    keep = a.layers.split(",")
    wl = workloads.Workload(W.name, W.net, [l for l in W.layers if l.name in keep], batch=W.batch)
    args = argparse.Namespace(batch=a.batch, weak=False, sparsity=800, kernel=-1, no_jit=False, no_autotune=False,
                              tune_variants=False, jit_tunings="0;16,1,0,0,16,2")
    flush = torch.empty(16 * 1024 * 1024, dtype=torch.float32, device=dev)
    runs, n0, B, GB, _ = bench.setup(args, wl, dev, rank, world, torch, escoin, flush)
    res = {"rank": rank, "range": [n0, n0 + B], "layers": []}
    rng = np.random.default_rng(1000 + rank)
    for r in runs:
        L = r.L
        s = torch.cuda.current_stream().cuda_stream
        bench.fwd(escoin, r, s)
        torch.cuda.synchronize()
        out = r.out.cpu().numpy()
        # oracle at sampled points of this shard, addressed by GLOBAL image index
        w = inputs.layer_weights(wl.net, L, 800)
        b = inputs.bias(wl.net, L.name, L.M)
        xs = inputs.activations(wl.net, L.name, n0, B, L.C, L.H, L.W)
        rp, ci, v = oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad)
        npts = 1500
        co = np.stack([rng.integers(0, B, npts), rng.integers(0, L.M, npts), rng.integers(0, L.E, npts),
                       rng.integers(0, L.F, npts)], 1)
        ref, scale = oracle.sconv_points(xs, rp, ci, v, L.M, L.K, L.stride, L.pad, co, bias=b, relu=True)
        got = out[co[:, 0], co[:, 1], co[:, 2], co[:, 3]].astype(np.float64)
        ok_oracle = bool(np.all(np.abs(got - ref) <= 1e-5 * (scale + np.abs(b[co[:, 1]]))))
        # bitwise against the full global batch through the same handle, sliced
        xf = torch.from_numpy(inputs.activations(wl.net, L.name, 0, GB, L.C, L.H, L.W)).to(dev)
        full = escoin.forward(r.csr, xf, bias=r.bias, relu=True)
        torch.cuda.synchronize()
        ok_slice = full[n0:n0 + B].cpu().numpy().tobytes() == out.tobytes()
        res["layers"].append({"layer": L.name, "oracle_ok": ok_oracle, "slice_bitwise": ok_slice,
                              "kernel": r.kernel})
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        print(json.dumps(allres), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
