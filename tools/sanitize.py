"""Small forwards of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck).

usage: compute-sanitizer --tool TOOL python tools/sanitize.py
Runs the tiny config (C1) and a ragged multi-tile case through: the specialised kernel in barrier
and mbarrier pipeline modes, with 4-byte and vector staging, a multi-unit linked kernel, a
regrouped one, an 11x11/stride-4 one; every compiled interpreter variant that accepts the shape;
the paper mapping; the dense tcgen05 engine.  Prints one line per case (outputs are checked
against each other for identical bits; parity vs the oracle is the test suite's job).
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1802_10280_b200 import escoin, inputs, workloads  # noqa: E402


def run(csr, x, b, relu=True):
    out = escoin.forward(csr, x, bias=b, relu=relu)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def main():
    dev = torch.device("cuda", 0)
    L = workloads.TINY
    cases = [("tiny", inputs.layer_weights("tiny", L, 800), inputs.activations("tiny", "tiny", 0, 1, L.C, L.H, L.W),
              1, 1)]
    rng = np.random.default_rng(3)
    w = rng.standard_normal((40, 12, 3, 3)).astype(np.float32)
    w[rng.random(w.shape) >= 0.25] = 0.0
    cases.append(("ragged", w, rng.random((5, 12, 13, 16)).astype(np.float32), 1, 1))
    w11 = rng.standard_normal((8, 3, 11, 11)).astype(np.float32)
    w11[rng.random(w11.shape) >= 0.2] = 0.0
    cases.append(("k11s4", w11, rng.random((2, 3, 31, 31)).astype(np.float32), 4, 0))
    for name, w, xh, st, pad in cases:
        M, C, K, _ = w.shape
        N, _, H, W = xh.shape
        x = torch.from_numpy(xh).to(dev)
        b = torch.from_numpy((rng.random(M) * 0.2 - 0.1).astype(np.float32)).to(dev)
        ref = None
        tunings = [dict(), dict(mbarrier=1, NS=4), dict(vec=1), dict(Q=8, units=3), dict(Q=8, reorder=1),
                   dict(Q=16, warps=4, minb=2, P=2), dict(Q=8, perm=1, reorder=-1), dict(Q=8, P=2, warps=4, perm=1,
                                                                                      reorder=-1), dict(sws=-1),
                   dict(Q=8, pw=1), dict(Q=8, warps=2, pw=1, units=2), dict(Q=8, P=2, warps=2, pw=1),
                   dict(Q=8, P=2, warps=2, hp=1), dict(Q=8, P=4, warps=2, pair=1)]
        for tun in tunings:
            csr = escoin.Csr.stretch(w, H, W, st, pad).to_device(0)
            try:
                csr.jit(n_hint=N, **tun)
            except escoin.EscoinError as e:
                print(name, "jit", tun, "unsupported", e.status, flush=True)
                continue
            o = run(csr, x, b)
            ref = o if ref is None else ref
            print(name, csr.label(), "same" if o.tobytes() == ref.tobytes() else "DIFFERENT", flush=True)
        for kid, kname, kK, kS in escoin.kernels():
            if kid != 0 and (kK != K or kS != st):
                continue
            csr = escoin.Csr.stretch(w, H, W, st, pad).to_device(0)
            try:
                csr.set_kernel(kid)
            except escoin.EscoinError:
                continue
            o = run(csr, x, b)
            print(name, kname, "same" if ref is None or o.tobytes() == ref.tobytes() else "DIFFERENT", flush=True)
        csr = escoin.Csr.stretch(w, H, W, st, pad).to_device(0)
        csr.set_kernel(escoin.KERNEL_DENSE_TC)
        o = run(csr, x, b)
        print(name, csr.label(), "max|diff| %.3g" % float(np.max(np.abs(o - ref))) if ref is not None else "", flush=True)


if __name__ == "__main__":
    main()
