"""Print the host-side tiling plan of every applicable variant for each layer of a workload."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1802_10280_b200 import escoin, inputs, workloads  # noqa: E402

L = escoin.lib()
L.escoin_internal_plan.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
COLS = ["WM", "WP", "NB", "TR", "PR", "PC", "SR", "SCs", "plane", "CC", "smem", "recs", "PCs", "NS"]


def dump(wl, nmax=99):
    W = workloads.workload(wl)
    for lay in W.layers[:nmax]:
        w = inputs.layer_weights(W.net, lay, W.sparsity_permille)
        csr = escoin.Csr.stretch(w, lay.H, lay.W, lay.stride, lay.pad)
        for k in escoin.kernels():
            if k[2] == lay.K and k[3] == lay.stride:
                out = np.zeros(14, np.int64)
                rc = L.escoin_internal_plan(csr.handle, k[0], out.ctypes.data)
                print("%-10s %-22s %-14s rc=%d %s" % (wl, lay.name, k[1], rc,
                                                     " ".join("%s=%d" % (c, v) for c, v in zip(COLS, out))))


if __name__ == "__main__":
    for wl in sys.argv[1:] or ["alexnet"]:
        dump(wl)
