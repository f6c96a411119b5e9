"""GPU parity: the CUDA path (through the C-ABI) against the fp64 CPU oracle.

Tolerance (north_star; reading R#11), element by element:
    |gpu - ref| <= 1e-5 * (sum |w*x| + |bias[m]|)
Exact regime: integer weights/inputs keep every partial sum < 2^24, so the
GPU must equal the oracle bitwise.  Integer/index work (the stretch) is
bit-exact in tests/test_abi.py.
"""
import itertools

import numpy as np
import pytest

import oracle
from paper_1802_10280_b200 import escoin, inputs, workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


def kernel_ids(K, S):
    return [k[0] for k in escoin.kernels() if k[0] == 0 or (k[2] == K and k[3] == S)]


def run_gpu(w, x, bias, stride, pad, relu, kernel=escoin.KERNEL_AUTO, csr=None):
    """Forward through the C-ABI; returns (None, None) when the requested variant
    cannot tile this shape (ESCOIN_ERR_UNSUPPORTED is a legitimate answer)."""
    M, C, K, _ = w.shape
    N, _, H, W = x.shape
    if csr is None:
        csr = escoin.Csr.stretch(w, H, W, stride, pad)
        csr.set_kernel(kernel)
        try:
            csr.to_device(0)
        except escoin.EscoinError as e:
            if e.status == escoin.ERR_UNSUPPORTED and kernel != escoin.KERNEL_AUTO:
                return None, None
            raise
    dx = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    db = None if bias is None else torch.from_numpy(bias).cuda()
    out = escoin.forward(csr, dx, bias=db, relu=relu)
    torch.cuda.synchronize()
    return out.cpu().numpy(), csr


def check(out, ref, scale, bias):
    b = 0.0 if bias is None else np.abs(bias.astype(np.float64))[None, :, None, None]
    err = np.abs(out.astype(np.float64) - ref)
    bound = TOL * (scale + b)
    bad = err > bound
    assert not bad.any(), "max err ratio %.3g at %s" % (np.max(err / np.maximum(bound, 1e-300)),
                                                       np.argwhere(bad)[:3].tolist())
    return float(np.max(err / np.maximum(scale + b, 1e-300)))


def oracle_ref(w, x, bias, stride, pad, relu):
    M, C, K, _ = w.shape
    rp, ci, v = oracle.csr_stretch(w, x.shape[2], x.shape[3], stride, pad)
    return oracle.sconv(x, rp, ci, v, M, K, stride, pad, bias=bias, relu=relu)


# ------------------------------------------------------------------ C1 tiny
@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("with_bias", [False, True])
def test_tiny_all_kernels(relu, with_bias):
    L = workloads.TINY
    x = inputs.activations("tiny", "tiny", 0, 1, L.C, L.H, L.W)
    w = inputs.layer_weights("tiny", L, 800)
    b = inputs.bias("tiny", "tiny", L.M) if with_bias else None
    ref, scale = oracle_ref(w, x, b, L.stride, L.pad, relu)
    outs = []
    for k in kernel_ids(L.K, L.stride):
        out, _ = run_gpu(w, x, b, L.stride, L.pad, relu, kernel=k)
        if out is None:
            continue
        check(out, ref, scale, b)
        outs.append(out)
    assert len(outs) >= 2  # the paper mapping and at least one tiled variant
    for o in outs[1:]:  # every variant accumulates in the same order -> identical bits
        assert o.tobytes() == outs[0].tobytes()


# ------------------------------------------------------------------ random grid
GRID = [  # N, C, H, W, M, K, stride, pad, density
    (2, 5, 14, 14, 9, 3, 1, 1, 0.3), (3, 16, 13, 13, 40, 3, 1, 1, 0.2), (1, 7, 27, 27, 33, 5, 1, 2, 0.2),
    (2, 3, 9, 17, 5, 5, 1, 2, 0.5), (4, 20, 7, 7, 17, 3, 1, 1, 0.2), (2, 9, 28, 28, 12, 3, 1, 1, 0.2),
    (1, 12, 56, 56, 8, 3, 1, 1, 0.15), (3, 11, 10, 12, 13, 1, 1, 0, 0.3), (2, 6, 15, 11, 7, 3, 2, 1, 0.4),
    (2, 4, 16, 16, 6, 1, 2, 0, 0.5), (1, 3, 11, 11, 4, 5, 2, 0, 0.6), (5, 2, 5, 6, 3, 3, 1, 0, 1.0),
    (2, 33, 14, 14, 31, 3, 1, 1, 0.1), (1, 4, 8, 8, 70, 3, 1, 2, 0.2), (2, 8, 32, 30, 10, 5, 1, 2, 0.1),
    (1, 1, 4, 4, 1, 3, 1, 1, 1.0), (3, 18, 6, 6, 29, 1, 1, 0, 0.25),
    (3, 37, 7, 7, 26, 1, 1, 0, 0.2), (2, 70, 14, 14, 45, 1, 1, 0, 0.2), (1, 9, 5, 3, 7, 1, 1, 0, 0.5),
]


@pytest.mark.parametrize("case", GRID)
def test_parity_grid(case):
    N, C, H, W, M, K, s, p, d = case
    rng = np.random.default_rng(abs(hash(case)) % 2**32)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= d] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, s, p, True)
    outs = []
    for k in kernel_ids(K, s):
        out, _ = run_gpu(w, x, b, s, p, True, kernel=k)
        if out is None:
            continue
        check(out, ref, scale, b)
        outs.append(out)
    for o in outs[1:]:
        assert o.tobytes() == outs[0].tobytes()


# ------------------------------------------------------------------ mosaic tiling
MOSAIC_GRID = [  # N, C, H, W, M, K, pad — "same" padding, stride 1 (where mosaic applies)
    (5, 12, 13, 13, 40, 3, 1), (7, 9, 14, 14, 33, 3, 1), (3, 10, 7, 7, 20, 3, 1), (3, 6, 27, 27, 17, 5, 2),
    (1, 8, 13, 13, 16, 3, 1), (9, 5, 6, 9, 12, 3, 1),
]


@pytest.mark.parametrize("mos", [1, 2, 3, 4])
@pytest.mark.parametrize("case", MOSAIC_GRID)
def test_mosaic_tiling_parity(case, mos, monkeypatch):
    # the batch laid out as one super-image (mos images per super-row, shared
    # zero separators): same values, same bits as the per-image tiling
    N, C, H, W, M, K, p = case
    rng = np.random.default_rng(7 + mos)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= 0.25] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, 1, p, True)
    monkeypatch.setenv("ESCOIN_MOSAIC", "0")
    base = {k: run_gpu(w, x, b, 1, p, True, kernel=k)[0] for k in kernel_ids(K, 1) if k != 0}
    monkeypatch.setenv("ESCOIN_MOSAIC", str(mos))
    ran = 0
    for k, o0 in base.items():
        out, _ = run_gpu(w, x, b, 1, p, True, kernel=k)
        if out is None:
            continue
        check(out, ref, scale, b)
        if o0 is not None:
            assert out.tobytes() == o0.tobytes(), k
        ran += 1
    assert ran >= 1


def test_mosaic_full_batch_sampled(monkeypatch):
    monkeypatch.setenv("ESCOIN_MOSAIC", "2")
    test_full_batch_sampled("alexnet", "conv3")


# ------------------------------------------------------------------ exact regimes
@pytest.mark.parametrize("case", [(2, 16, 14, 14, 32, 3, 1, 1), (2, 24, 13, 13, 20, 5, 1, 2),
                                  (1, 32, 28, 28, 16, 3, 1, 1), (2, 40, 7, 7, 50, 1, 1, 0)])
def test_exact_integer_regime(case):
    N, C, H, W, M, K, s, p = case
    L = workloads.Layer("ex", C, H, W, M, K, s, p)
    x = inputs.activations("ex", "ex", 0, N, C, H, W, exact=True)
    w = inputs.layer_weights("ex", L, 700, exact=True)
    b = inputs.bias("ex", "ex", M, exact=True)
    ref, scale = oracle_ref(w, x, b, s, p, False)
    assert np.max(scale) < 2 ** 24
    for k in kernel_ids(K, s):
        out, _ = run_gpu(w, x, b, s, p, False, kernel=k)
        if out is None:
            continue
        assert np.array_equal(out.astype(np.float64), ref), "kernel %d not bit-exact" % k


@pytest.mark.parametrize("K,pad", [(3, 1), (5, 2), (1, 0), (3, 0)])
def test_one_hot_is_shifted_copy(K, pad):
    # one nonzero = 1.0 per output channel, bias 0 -> out is an exact shifted
    # copy of the zero-padded input: tests indexing and padding bit-exactly
    N, C, H, W = 2, 6, 13, 11
    taps = [(c, kh, kw) for c in range(C) for kh in range(K) for kw in range(K)]
    M = len(taps)
    w = np.zeros((M, C, K, K), np.float32)
    for m, (c, kh, kw) in enumerate(taps):
        w[m, c, kh, kw] = 1.0
    rng = np.random.default_rng(1)
    x = rng.random((N, C, H, W)).astype(np.float32)
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    E, F = H + 2 * pad - K + 1, W + 2 * pad - K + 1
    for k in kernel_ids(K, 1):
        out, _ = run_gpu(w, x, None, 1, pad, False, kernel=k)
        if out is None:
            continue
        for m, (c, kh, kw) in enumerate(taps):
            assert np.array_equal(out[:, m], xp[:, c, kh:kh + E, kw:kw + F]), (k, m)


def test_all_zero_weights_give_bias():
    rng = np.random.default_rng(2)
    x = rng.random((2, 8, 14, 14)).astype(np.float32)
    w = np.zeros((20, 8, 3, 3), np.float32)
    b = (rng.random(20) - 0.5).astype(np.float32)
    for k in kernel_ids(3, 1):
        out, _ = run_gpu(w, x, b, 1, 1, False, kernel=k)
        if out is None:
            continue
        assert np.array_equal(out, np.broadcast_to(b[None, :, None, None], out.shape))
        outr, _ = run_gpu(w, x, b, 1, 1, True, kernel=k)
        assert np.array_equal(outr, np.maximum(out, 0))


def test_empty_rows_and_ragged_m():
    rng = np.random.default_rng(3)
    x = rng.random((3, 10, 13, 13)).astype(np.float32)
    w = rng.standard_normal((23, 10, 3, 3)).astype(np.float32)
    w[rng.random(w.shape) > 0.2] = 0
    w[[0, 5, 6, 22]] = 0.0   # empty CSR rows
    b = rng.random(23).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, 1, 1, False)
    for k in kernel_ids(3, 1):
        out, _ = run_gpu(w, x, b, 1, 1, False, kernel=k)
        if out is None:
            continue
        check(out, ref, scale, b)
        assert np.array_equal(out[:, [0, 5, 6, 22]], np.broadcast_to(b[None, [0, 5, 6, 22], None, None],
                                                                    out[:, [0, 5, 6, 22]].shape))


# ------------------------------------------------------------------ determinism / batch invariance
def test_deterministic_and_batch_slice_invariant():
    L = workloads.alexnet_full()[2]  # conv3 shape
    x = inputs.activations("alexnet", "conv3", 0, 8, L.C, L.H, L.W)
    w = inputs.layer_weights("alexnet", L, 800)
    b = inputs.bias("alexnet", "conv3", L.M)
    full, csr = run_gpu(w, x, b, 1, 1, True)
    again, _ = run_gpu(w, x, b, 1, 1, True, csr=csr)
    assert full.tobytes() == again.tobytes()
    part, _ = run_gpu(w, x[5:7], b, 1, 1, True, csr=csr)
    assert part.tobytes() == full[5:7].tobytes()


# ------------------------------------------------------------------ config layers
def layer_case(wl, L, n0, n):
    W = workloads.workload(wl)
    x = inputs.activations(W.net, L.name, n0, n, L.C, L.H, L.W)
    w = inputs.layer_weights(W.net, L, W.sparsity_permille)
    b = inputs.bias(W.net, L.name, L.M)
    return x, w, b


@pytest.mark.parametrize("wl", ["alexnet", "resnet50", "googlenet", "resnet50_v15"])
def test_config_layers_small_batch(wl):
    # every sparse layer of the config, all outputs of N=2 images, default kernel
    for L in workloads.workload(wl).layers:
        x, w, b = layer_case(wl, L, 0, 2)
        ref, scale = oracle_ref(w, x, b, L.stride, L.pad, True)
        out, _ = run_gpu(w, x, b, L.stride, L.pad, True)
        check(out, ref, scale, b)


def test_googlenet_1x1_small_batch():
    for L in workloads.workload("googlenet_1x1").layers[::4]:
        x, w, b = layer_case("googlenet_1x1", L, 0, 2)
        ref, scale = oracle_ref(w, x, b, L.stride, L.pad, True)
        out, _ = run_gpu(w, x, b, L.stride, L.pad, True)
        check(out, ref, scale, b)


@pytest.mark.parametrize("wl,name", [("alexnet", "conv2"), ("alexnet", "conv3"), ("resnet50", "res5a_branch2b"),
                                     ("resnet50", "res2a_branch2b")])
def test_full_batch_sampled(wl, name):
    # BASELINE full size (N=128), in the launch configuration bench.py times;
    # sampled outputs checked one by one against the oracle.
    L = [l for l in workloads.workload(wl).layers if l.name == name][0]
    x, w, b = layer_case(wl, L, 0, 128)
    out, _ = run_gpu(w, x, b, L.stride, L.pad, True)
    rng = np.random.default_rng(5)
    npts = 4000
    coords = np.stack([rng.integers(0, 128, npts), rng.integers(0, L.M, npts), rng.integers(0, L.E, npts),
                       rng.integers(0, L.F, npts)], 1)
    corners = np.array([[n, m, h, ww] for n in (0, 127) for m in (0, L.M - 1) for h in (0, L.E - 1)
                        for ww in (0, L.F - 1)])
    coords = np.concatenate([coords, corners])
    rp, ci, v = oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad)
    ref, scale = oracle.sconv_points(x, rp, ci, v, L.M, L.K, L.stride, L.pad, coords, bias=b, relu=True)
    got = out[coords[:, 0], coords[:, 1], coords[:, 2], coords[:, 3]].astype(np.float64)
    assert np.all(np.abs(got - ref) <= TOL * (scale + np.abs(b[coords[:, 1]])))
    assert np.all(np.isfinite(out))


@pytest.mark.parametrize("wl,name", [("alexnet", "conv2"), ("alexnet", "conv3"), ("resnet50_v15", "res4a_branch2b"),
                                     ("googlenet_1x1", "inception_4e/1x1")])
def test_full_batch_autotuned_sampled(wl, name):
    # exactly the launch configuration bench.py times: N=128, the variant and
    # tiling escoin_csr_autotune picks on these buffers; sampled outputs vs oracle
    L = [l for l in workloads.workload(wl).layers if l.name == name][0]
    x, w, b = layer_case(wl, L, 0, 128)
    csr = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad).to_device(0)
    dx, db = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    out = torch.empty((128, L.M, L.E, L.F), device="cuda")
    csr.autotune(128, dx, out, db, True, 2, torch.cuda.current_stream().cuda_stream)
    out = escoin.forward(csr, dx, bias=db, relu=True)
    torch.cuda.synchronize()
    got_all = out.cpu().numpy()
    rng = np.random.default_rng(9)
    npts = 3000
    coords = np.stack([rng.integers(0, 128, npts), rng.integers(0, L.M, npts), rng.integers(0, L.E, npts),
                       rng.integers(0, L.F, npts)], 1)
    rp, ci, v = oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad)
    ref, scale = oracle.sconv_points(x, rp, ci, v, L.M, L.K, L.stride, L.pad, coords, bias=b, relu=True)
    got = got_all[coords[:, 0], coords[:, 1], coords[:, 2], coords[:, 3]].astype(np.float64)
    assert np.all(np.abs(got - ref) <= TOL * (scale + np.abs(b[coords[:, 1]]))), escoin.kernels()[csr.kernel()][1]
    assert np.all(np.isfinite(got_all))


# ------------------------------------------------------------------ ABI paths
def test_wrap_device_and_hostio_match():
    L = workloads.TINY
    x = inputs.activations("tiny", "tiny", 0, 3, L.C, L.H, L.W)
    w = inputs.layer_weights("tiny", L, 800)
    b = inputs.bias("tiny", "tiny", L.M)
    ref_out, csr = run_gpu(w, x, b, 1, 1, True)
    rp, ci, v = csr.host_arrays()
    d = [torch.from_numpy(a).cuda() for a in (rp, ci, v)]
    wrapped = escoin.Csr.wrap_device(d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), len(v), L.M, L.C, L.H, L.W,
                                     L.K, 1, 1, 0)
    out2, _ = run_gpu(w, x, b, 1, 1, True, csr=wrapped)
    assert out2.tobytes() == ref_out.tobytes()
    # host-buffer end-to-end entry point
    hx = torch.from_numpy(x).pin_memory()
    hout = torch.empty((3, L.M, L.E, L.F), dtype=torch.float32).pin_memory()
    dx = torch.empty_like(hx, device="cuda")
    dout = torch.empty_like(hout, device="cuda")
    db = torch.from_numpy(b).cuda()
    s = torch.cuda.current_stream().cuda_stream
    escoin.sconv_forward_hostio(3, L.C, L.H, L.W, L.M, L.K, 1, 1, csr, hx, hout, dx, dout, db, True, s)
    torch.cuda.synchronize()
    assert hout.numpy().tobytes() == ref_out.tobytes()


def test_fault_injection_detected():
    # a corrupted stretched colidx must fail verification
    L = workloads.TINY
    x = inputs.activations("tiny", "tiny", 0, 1, L.C, L.H, L.W)
    w = inputs.layer_weights("tiny", L, 800)
    rp, ci, v = oracle.csr_stretch(w, L.H, L.W, 1, 1)
    ref, scale = oracle.sconv(x, rp, ci, v, L.M, L.K, 1, 1)
    bad = ci.copy()
    bad[77] += 1
    d = [torch.from_numpy(a).cuda() for a in (rp, bad, v)]
    csr = escoin.Csr.wrap_device(d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), len(v), L.M, L.C, L.H, L.W,
                                 L.K, 1, 1, 0)
    out, _ = run_gpu(w, x, None, 1, 1, False, csr=csr)
    err = np.abs(out - ref) / np.maximum(scale, 1e-30)
    assert np.max(err) > TOL


def test_wrap_device_rejects_bad_csr():
    rp = torch.tensor([0, 2, 1], dtype=torch.int32, device="cuda")   # decreasing rowptr
    ci = torch.tensor([0, 1], dtype=torch.int32, device="cuda")
    v = torch.ones(2, dtype=torch.float32, device="cuda")
    with pytest.raises(escoin.EscoinError) as e:
        escoin.Csr.wrap_device(rp.data_ptr(), ci.data_ptr(), v.data_ptr(), 2, 2, 1, 4, 4, 3, 1, 1, 0)
    assert e.value.status == escoin.ERR_CSR_MISMATCH


def test_autotune_keeps_bits():
    L = workloads.alexnet_full()[3]  # conv4, grouped
    x, w, b = layer_case("alexnet", L, 0, 4)
    ref_out, csr = run_gpu(w, x, b, 1, 1, True)
    dx = torch.from_numpy(x).cuda()
    db = torch.from_numpy(b).cuda()
    out = torch.empty((4, L.M, L.E, L.F), device="cuda")
    kid, ms = csr.autotune(4, dx, out, db, True, 2, torch.cuda.current_stream().cuda_stream)
    assert 0 <= kid < len(escoin.kernels()) and ms > 0 and csr.kernel() == kid
    out2, _ = run_gpu(w, x, b, 1, 1, True, csr=csr)
    assert out2.tobytes() == ref_out.tobytes()


def test_bench_two_ranks_same_device():
    # the batch-shard driver end to end with 2 ranks (gloo over CUDA tensors, both
    # on cuda:0): CSR broadcast from rank 0, wrap_device on rank 1, strong scaling of the
    # global batch, max-over-ranks
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(root, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "1", "--workload", "tiny", "--batch", "6", "--no-baselines", "--no-cpu",
           "--dist-backend", "gloo", "--same-device"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 6 and d["config"]["batch_per_gpu"] == 3
    assert d["scaling"] == "strong" and d["value"] > 0


def test_two_ranks_shard_parity():
    # every rank checks ITS shard of the global batch against the oracle (same global image
    # indices) and bitwise against the full-batch forward sliced to its range
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29534", os.path.join(root, "tests", "mp_shard_check.py"),
           "--workload", "alexnet", "--layers", "conv3,conv4", "--batch", "10"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("[")]
    res = json.loads(lines[-1])
    assert [x["range"] for x in res] == [[0, 5], [5, 10]]
    for x in res:
        assert len(x["layers"]) == 2
        for l in x["layers"]:
            assert l["oracle_ok"] and l["slice_bitwise"], (x["rank"], l)


@pytest.mark.parametrize("seed", range(6))
def test_stretch_device_bit_exact(seed):
    # NEXT-4: the device stretch equals the host stretch bit for bit (and the oracle's)
    rng = np.random.default_rng(seed)
    K = int(rng.choice([1, 3, 5]))
    M, C, H, W, pad = int(rng.integers(1, 300)), int(rng.integers(1, 40)), 13, 11, K // 2
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) < 0.8] = 0.0
    w[rng.random(w.shape) < 0.05] = -0.0
    w.reshape(-1)[:3] = np.float32(1e-42)  # denormals are nonzero
    d = escoin.Csr.stretch_device(torch.from_numpy(w).cuda(), M, C, H, W, K, 1, pad, 0)
    h = escoin.Csr.stretch(w, H, W, 1, pad)
    for a, b in zip(d.host_arrays(), h.host_arrays()):
        assert a.tobytes() == b.tobytes()
    orp, oci, ov = oracle.csr_stretch(w, H, W, 1, pad)
    assert d.host_arrays()[1].tobytes() == oci.tobytes()
    x = rng.random((2, C, H, W)).astype(np.float32)
    o1, _ = run_gpu(w, x, None, 1, pad, False, csr=d)
    o2, _ = run_gpu(w, x, None, 1, pad, False, csr=h.to_device(0))
    assert o1.tobytes() == o2.tobytes()


def test_stretch_device_config_layer():
    L = workloads.alexnet_full()[3]
    w = inputs.layer_weights("alexnet", L, 800)
    d = escoin.Csr.stretch_device(torch.from_numpy(w).cuda(), L.M, L.C, L.H, L.W, L.K, 1, 1, 0)
    rp, ci, v = oracle.csr_stretch(w, L.H, L.W, 1, 1)
    a = d.host_arrays()
    assert a[0].tobytes() == rp.tobytes() and a[1].tobytes() == ci.tobytes() and a[2].tobytes() == v.tobytes()
