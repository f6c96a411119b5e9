"""Measured comparison points for bench.py (NOT the product; not the method).

The paper's baselines are Caffe's lowering paths (P:230-288, P:348-352,
P:699-703): im2col followed by cuBLAS sgemm (dense pruned weights) or by
cuSPARSE csrmm (CSR weights).  Here:
  * im2col          torch.nn.functional.unfold (one CUDA kernel, all images)
  * cublas          torch.matmul -> cublasSgemmStridedBatched, FP32 compute,
                    TF32 disabled (same precision as the sparse path): one
                    [M x CRS] x [CRS x EF] GEMM per image (Caffe's per-image loop)
  * cublas_gemm     the same lowering as ONE GEMM per group over the whole
                    batch: [M x CRS] x [CRS x N*EF] (the lowered matrix is
                    re-laid out once; bigger GEMMs, the fairer dense baseline)
  * cusparse        torch.sparse CSR @ dense -> cusparseSpMM (the legacy
                    csrmm API no longer exists), on the [CRS x N*EF] lowered
                    matrix; the two layout permutes it needs are included
  * bias + ReLU     one fused elementwise pass (the sparse path fuses it)
Grouped layers (AlexNet conv2/4/5) run one GEMM/SpMM per group, as Caffe does.
"""
from __future__ import annotations

import numpy as np
import torch


class LoweredConv:
    def __init__(self, layer, w_dense: np.ndarray, bias: np.ndarray, device, mode: str):
        """w_dense: block-diagonal expanded pruned weights [M][C][K][K]."""
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False
        self.L = layer
        self.mode = mode
        g = layer.groups
        Mg, Cg = layer.M // g, layer.C // g
        K = layer.K
        self.w = []
        self.a = []
        for gi in range(g):
            wg = w_dense[gi * Mg:(gi + 1) * Mg, gi * Cg:(gi + 1) * Cg].reshape(Mg, Cg * K * K)
            t = torch.from_numpy(np.ascontiguousarray(wg)).to(device)
            self.w.append(t)
            if mode == "cusparse":
                self.a.append(t.to_sparse_csr())
        self.bias = torch.from_numpy(bias).to(device).view(1, -1, 1)

    def __call__(self, x: torch.Tensor, out: torch.Tensor):
        L = self.L
        N = x.shape[0]
        g = L.groups
        Mg, Cg = L.M // g, L.C // g
        EF = L.E * L.F
        o = out.view(N, L.M, EF)
        for gi in range(g):
            xg = x[:, gi * Cg:(gi + 1) * Cg]
            col = torch.nn.functional.unfold(xg, L.K, padding=L.pad, stride=L.stride)  # [N, CRS, EF]
            if self.mode == "cublas":
                torch.matmul(self.w[gi], col, out=o[:, gi * Mg:(gi + 1) * Mg])
            elif self.mode == "cublas_gemm":
                B = col.transpose(0, 1).reshape(col.shape[1], N * EF)
                Y = torch.mm(self.w[gi], B)                              # [Mg, N*EF], one SGEMM
                o[:, gi * Mg:(gi + 1) * Mg].copy_(Y.view(Mg, N, EF).transpose(0, 1))
            else:
                B = col.transpose(0, 1).reshape(col.shape[1], N * EF)
                Y = torch.sparse.mm(self.a[gi], B)                       # [Mg, N*EF]
                o[:, gi * Mg:(gi + 1) * Mg].copy_(Y.view(Mg, N, EF).transpose(0, 1))
        torch.relu_(o.add_(self.bias))
        return out


class CudnnConv:
    """Dense cuDNN convolution — extra reference points (not the method):
      precision "fp32": FP32 math, TF32 off (same precision as the sparse path);
      precision "tf32": TF32 tensor cores (tcgen05 on B200; ~1e-3 relative error);
      precision "bf16": BF16 tensor cores, channels-last, activations converted
                        to BF16 once outside the timed region (a BF16 network
                        would carry BF16 activations), output back to FP32.
    """

    def __init__(self, layer, w_dense: np.ndarray, bias: np.ndarray, device, precision: str = "fp32"):
        self.precision = precision
        L = layer
        g = L.groups
        Mg, Cg = L.M // g, L.C // g
        wg = np.concatenate([w_dense[i * Mg:(i + 1) * Mg, i * Cg:(i + 1) * Cg] for i in range(g)], 0)
        self.w = torch.from_numpy(np.ascontiguousarray(wg)).to(device)
        self.b = torch.from_numpy(bias).to(device)
        if precision == "bf16":
            self.w = self.w.to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
            self.b = self.b.to(torch.bfloat16)
        self.xc = None
        self.L = L

    def __call__(self, x, out):
        L = self.L
        torch.backends.cudnn.allow_tf32 = self.precision == "tf32"
        xin = x
        if self.precision == "bf16":
            if self.xc is None or self.xc[0] is not x:
                self.xc = (x, x.to(torch.bfloat16).contiguous(memory_format=torch.channels_last))
            xin = self.xc[1]
        y = torch.nn.functional.conv2d(xin, self.w, self.b, stride=L.stride, padding=L.pad, groups=L.groups)
        out.copy_(torch.relu_(y))
        torch.backends.cudnn.allow_tf32 = False
        return out
