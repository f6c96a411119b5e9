"""Instruction-fetch microbenchmark: straight-line FFMA (immediate weight) code of S instructions per pass,
executed by W warps per CTA, one or two CTAs per SM (148 SMs), repeated R passes (same code).  Prints
TFLOP/s per (code KB, warps, CTAs/SM, FFMA form) — how far a code stream larger than the L1.5 instruction
cache (32 KB) falls below the FFMA peak when every warp of the CTA runs the same stream.

usage: python tools/icache_bench.py   (needs a GPU; PTX JIT-compiled by the driver)"""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def ptx(S, pair, nacc=16, seed=1):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal(S).astype(np.float32).view(np.uint32)
    L = [".version 8.7", ".target sm_100a", ".address_size 64",
         ".visible .entry k(.param .u64 p_out, .param .u32 p_R)", "{",
         ".reg .pred %p<2>;", ".reg .b32 %r<8>;", ".reg .b64 %rd<4>;", ".reg .f32 %%a<%d>;" % nacc,
         ".reg .b64 %%A<%d>;" % (nacc // 2), ".reg .b64 %W;",
         "ld.param.u32 %r1, [p_R];", "mov.u32 %r2, %tid.x;", "cvt.rn.f32.u32 %a0, %r2;"]
    for i in range(1, nacc):
        L.append("add.f32 %%a%d, %%a0, 0f%08X;" % (i, np.float32(i).view(np.uint32)))
    if pair:
        for i in range(nacc // 2):
            L.append("mov.b64 %%A%d, {%%a%d, %%a%d};" % (i, 2 * i, 2 * i + 1))
    L += ["mov.u32 %r3, 0;", "LOOP:"]
    for s in range(S):
        if pair:
            i = s % (nacc // 2)
            L.append("mov.b64 %%W, 0x%08X%08X; fma.rn.f32x2 %%A%d, %%A%d, %%W, %%A%d;" % (w[s], w[s], i, (i + 1) % (nacc // 2), i))
        else:
            i = s % nacc
            L.append("fma.rn.f32 %%a%d, %%a%d, 0f%08X, %%a%d;" % (i, (i + 1) % nacc, w[s], i))
    L += ["add.u32 %r3, %r3, 1;", "setp.lt.u32 %p0, %r3, %r1;", "@%p0 bra LOOP;"]
    if pair:
        for i in range(nacc // 2):
            L.append("mov.b64 {%%a%d, %%a%d}, %%A%d;" % (2 * i, 2 * i + 1, i))
    for i in range(1, nacc):
        L.append("add.f32 %%a0, %%a0, %%a%d;" % i)
    L += ["setp.eq.f32 %p1, %a0, 0f3F800001;", "ld.param.u64 %rd0, [p_out];", "@%p1 st.global.f32 [%rd0], %a0;",
          "ret;", "}"]
    return "\n".join(L)


def main():
    import torch
    from cuda.bindings import driver as cu  # cuda-python
    torch.cuda.init()
    torch.empty(1, device="cuda")
    out = torch.zeros(1, device="cuda")
    res = []
    for pair in (0, 1):
        for kb in (8, 24, 48, 96, 192, 384):
            S = kb * 1024 // 16
            text = ptx(S, pair).encode()
            err, mod = cu.cuModuleLoadData(text)
            assert err == cu.CUresult.CUDA_SUCCESS, err
            err, fn = cu.cuModuleGetFunction(mod, b"k")
            for warps, ctas in ((8, 1), (16, 1), (24, 1), (32, 1), (16, 2), (8, 4)):
                R = max(2, int(2e6 // (S * (2 if pair else 1) * warps * ctas)) * 8)
                args = ((out.data_ptr(), R), (ctypes.c_void_p, ctypes.c_uint32))
                grid = 148 * ctas
                stream = cu.CUstream(torch.cuda.current_stream().cuda_stream)
                for it in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    err, = cu.cuLaunchKernel(fn, grid, 1, 1, warps * 32, 1, 1, 0, stream, args, 0)
                    assert err == cu.CUresult.CUDA_SUCCESS, err
                    e1.record()
                    e1.synchronize()
                    ms = e0.elapsed_time(e1)
                flops = 2.0 * S * (2 if pair else 1) * R * warps * 32 * grid
                r = {"ffma2": pair, "code_kb": kb, "warps": warps, "ctas_per_sm": ctas, "passes": R,
                     "tflops": round(flops / ms / 1e9, 2)}
                print(json.dumps(r), flush=True)
                res.append(r)
            cu.cuModuleUnload(mod)


if __name__ == "__main__":
    main()
