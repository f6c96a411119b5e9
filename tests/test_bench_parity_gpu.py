"""Full-size parity of exactly what bench.py times (BASELINE configs at batch 128).

For every layer of every workload the bench runs, this replays bench.setup() — the same
stretch, the same escoin_csr_jit tunings (bench.jit_tunings_for(workload)), the same flushed
autotune — then compares EVERY output element of the selected kernel with the fp64 oracle
(reading R#11: |gpu - ref| <= 1e-5 * (sum|w*x| + |bias|)), and checks that every other
compiled tuning of the layer gives bitwise the same tensor (R#12), so each kernel the
autotune could pick is covered.  Alg.2, weight stretching P:437-442.
"""
import argparse

import numpy as np
import pytest

import bench
import oracle
from paper_1802_10280_b200 import escoin, inputs, workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


def _setup(wl_name):
    W = workloads.workload(wl_name)
    args = argparse.Namespace(batch=None, weak=False, sparsity=800, kernel=-1, no_jit=False, no_autotune=False,
                              tune_variants=False, jit_tunings=bench.jit_tunings_for(wl_name))
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    runs, n0, B, GB, _ = bench.setup(args, W, dev, 0, 1, torch, escoin, flush)
    assert (n0, B, GB) == (0, 128, 128)
    return W, runs


@pytest.mark.parametrize("wl_name", ["alexnet", "resnet50", "googlenet", "googlenet_1x1", "resnet50_v15",
                                     "alexnet_conv1", "alexnet_convs"])
def test_bench_setup_every_output_vs_oracle(wl_name):
    W, runs = _setup(wl_name)
    tunings = [[int(v) for v in t.split(",")] if t.strip() not in ("", "0") else []
               for t in bench.jit_tunings_for(wl_name).split(";")]
    s = torch.cuda.current_stream().cuda_stream
    failures = []
    for r in runs:
        L = r.L
        bench.fwd(escoin, r, s)
        torch.cuda.synchronize()
        out = r.out.cpu().numpy()
        label = r.csr.label()
        w = inputs.layer_weights(W.net, L, 800 if L.sparse else 0)  # bench.setup's rule (R#25)
        b = inputs.bias(W.net, L.name, L.M)
        x = r.h_x.numpy()
        rp, ci, v = oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad)
        ref, scale = oracle.sconv(x, rp, ci, v, L.M, L.K, L.stride, L.pad, bias=b, relu=True)
        bound = TOL * (scale + np.abs(b.astype(np.float64))[None, :, None, None])

        def within(o):
            return not (np.abs(o.astype(np.float64) - ref) > bound).any()
        if not within(out):
            err = np.abs(out.astype(np.float64) - ref)
            failures.append("%s %s: max err/bound %.3g" % (L.name, label, float(np.max(err / bound))))
        # every other compiled tuning (re-selecting a compiled tuning compiles nothing): the one-range
        # kernels give the same bits as each other (R#12); split-channel ones (_k: a different summation
        # order, JitPlan::ks) are checked against the oracle instead
        if r.csr.kernel() == escoin.KERNEL_JIT:
            one_range = None if "_k" in label else out.tobytes()
            for tun in tunings:
                try:
                    r.csr.jit(128, *tun)
                except escoin.EscoinError:
                    continue
                bench.fwd(escoin, r, s)
                torch.cuda.synchronize()
                o = r.out.cpu().numpy()
                lab = r.csr.label()
                if "_k" in lab:
                    if not within(o):
                        failures.append("%s %s: outside the tolerance" % (L.name, lab))
                elif one_range is None:
                    one_range = o.tobytes()
                elif o.tobytes() != one_range:
                    failures.append("%s %s differs from the other one-range kernels" % (L.name, lab))
        del ref, scale, bound
    assert not failures, failures
