"""GPU parity of the pattern-specialised kernel (escoin_csr_jit, jit_sconv.cpp).

Same tolerance as tests/test_sconv_gpu.py (reading R#11) against the fp64
oracle, plus bitwise identity with the paper-mapping kernel (variant 0): the
specialised kernel performs the same fp32 FMAs in the same ascending
(c, kh, kw) order from 0.0f (R#10), so it must produce the same bits.
"""
import numpy as np
import pytest

import oracle
from paper_1802_10280_b200 import escoin, inputs, workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


def oracle_ref(w, x, bias, stride, pad, relu):
    M, C, K, _ = w.shape
    rp, ci, v = oracle.csr_stretch(w, x.shape[2], x.shape[3], stride, pad)
    return oracle.sconv(x, rp, ci, v, M, K, stride, pad, bias=bias, relu=relu)


def check(out, ref, scale, bias):
    b = 0.0 if bias is None else np.abs(bias.astype(np.float64))[None, :, None, None]
    err = np.abs(out.astype(np.float64) - ref)
    bound = TOL * (scale + b)
    assert not (err > bound).any(), "max err ratio %.3g" % np.max(err / np.maximum(bound, 1e-300))


def fwd(csr, x, b, relu):
    dx = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    db = None if b is None else torch.from_numpy(b).cuda()
    out = escoin.forward(csr, dx, bias=db, relu=relu)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def jit_and_paper(w, x, b, pad, relu, n_hint=0, **tun):
    N, C, H, W = x.shape
    csr = escoin.Csr.stretch(w, H, W, 1, pad).to_device(0)
    csr.jit(n_hint=n_hint or N, **tun)
    assert csr.kernel() == escoin.KERNEL_JIT
    out = fwd(csr, x, b, relu)
    csr.set_kernel(0)
    paper = fwd(csr, x, b, relu)
    return out, paper, csr


@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("with_bias", [False, True])
def test_tiny(relu, with_bias):
    L = workloads.TINY
    x = inputs.activations("tiny", "tiny", 0, 1, L.C, L.H, L.W)
    w = inputs.layer_weights("tiny", L, 800)
    b = inputs.bias("tiny", "tiny", L.M) if with_bias else None
    ref, scale = oracle_ref(w, x, b, L.stride, L.pad, relu)
    out, paper, _ = jit_and_paper(w, x, b, L.pad, relu)
    check(out, ref, scale, b)
    assert out.tobytes() == paper.tobytes()


GRID = [  # N, C, H, W, M, K, pad, density — stride 1, "same" padding
    (2, 5, 14, 14, 9, 3, 1, 0.3), (3, 16, 13, 13, 40, 3, 1, 0.2), (1, 7, 27, 27, 33, 5, 2, 0.2),
    (2, 3, 9, 17, 5, 5, 2, 0.5), (4, 20, 7, 7, 17, 3, 1, 0.2), (2, 9, 28, 28, 12, 3, 1, 0.2),
    (1, 12, 56, 56, 8, 3, 1, 0.15), (3, 11, 10, 12, 13, 1, 0, 0.3), (5, 2, 5, 6, 3, 3, 1, 1.0),
    (2, 33, 14, 14, 131, 3, 1, 0.1), (1, 1, 4, 4, 1, 3, 1, 1.0), (7, 9, 6, 9, 70, 3, 1, 0.25),
    (3, 37, 7, 7, 26, 1, 0, 0.2), (9, 13, 13, 13, 65, 3, 1, 0.2),
]
TUNINGS = [dict(), dict(Q=16, P=2, CC=3, NS=2), dict(Q=32, P=3, CC=5, NS=4, warps=4, minb=3),
           dict(Q=8, P=1, CC=1, NS=2, warps=2, minb=1), dict(NS=4, mbarrier=1),
           dict(Q=16, CC=3, NS=3, warps=4, mbarrier=1, prefetch=-1), dict(Q=8, CC=1, NS=5, warps=2, mbarrier=1),
           # FFMA2: slot pairs (P even, the default), scalar P = 2, horizontal pixel pairs (hp)
           dict(Q=8, P=2, pair=-1), dict(Q=16, P=4, CC=3, warps=4), dict(Q=16, P=2, CC=3, NS=2, hp=1),
           dict(Q=8, P=4, warps=4, hp=2), dict(Q=16, P=2, NS=4, mbarrier=1, hp=1),
           # prefetch warp (one extra warp one chunk ahead; no copies, no stores)
           dict(Q=16, warps=4, pw=1), dict(Q=8, P=2, CC=3, NS=2, warps=2, pw=1), dict(Q=16, CC=1, NS=4, pw=1)]


@pytest.mark.parametrize("tun", range(len(TUNINGS)))
@pytest.mark.parametrize("case", GRID)
def test_parity_grid(case, tun):
    N, C, H, W, M, K, p, d = case
    rng = np.random.default_rng(abs(hash(case)) % 2**32)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= d] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, 1, p, True)
    out, paper, _ = jit_and_paper(w, x, b, p, True, **TUNINGS[tun])
    check(out, ref, scale, b)
    assert out.tobytes() == paper.tobytes()


def test_batch_other_than_hint_and_empty_rows():
    rng = np.random.default_rng(3)
    N, C, H, M = 11, 10, 13, 30
    x = rng.random((N, C, H, H)).astype(np.float32)
    w = rng.standard_normal((M, C, 3, 3)).astype(np.float32)
    w[rng.random(w.shape) >= 0.2] = 0.0
    w[[0, 7, 29]] = 0.0  # empty rows: output = bias
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    csr = escoin.Csr.stretch(w, H, H, 1, 1).to_device(0)
    csr.jit(n_hint=128, Q=16)
    ref, scale = oracle_ref(w, x, b, 1, 1, False)
    for n0, n1 in [(0, 11), (3, 4), (2, 9)]:
        out = fwd(csr, x[n0:n1], b, False)
        check(out, ref[n0:n1], scale[n0:n1], b)


def test_exact_integer_regime():
    rng = np.random.default_rng(11)
    N, C, H, M = 3, 12, 14, 24
    x = rng.integers(0, 4, (N, C, H, H)).astype(np.float32)
    w = rng.integers(-3, 4, (M, C, 3, 3)).astype(np.float32)
    b = rng.integers(-3, 4, M).astype(np.float32)
    ref, _ = oracle_ref(w, x, b, 1, 1, True)
    out, _, _ = jit_and_paper(w, x, b, 1, True)
    assert np.array_equal(out.astype(np.float64), ref)


STRIDE_PAD = [  # N, C, H, W, M, K, stride, pad — window origins oh*S, ow*S in the stacked layout
    (3, 6, 15, 11, 13, 3, 2, 1), (2, 5, 9, 9, 7, 3, 1, 0), (2, 4, 8, 10, 9, 3, 1, 2), (4, 8, 16, 16, 12, 1, 2, 0),
    (2, 3, 11, 11, 5, 5, 2, 2), (3, 7, 13, 12, 6, 3, 3, 1), (5, 6, 14, 14, 40, 3, 2, 1), (2, 3, 7, 9, 4, 5, 1, 0),
]


@pytest.mark.parametrize("tun", [dict(), dict(Q=8, CC=3, NS=2, warps=4, minb=2)])
@pytest.mark.parametrize("case", STRIDE_PAD)
def test_stride_and_padding(case, tun):
    N, C, H, W, M, K, st, p = case
    rng = np.random.default_rng(abs(hash(case)) % 2**32)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= 0.3] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, st, p, True)
    csr = escoin.Csr.stretch(w, H, W, st, p).to_device(0)
    csr.jit(n_hint=N, **tun)
    assert csr.kernel() == escoin.KERNEL_JIT
    out = fwd(csr, x, b, True)
    check(out, ref, scale, b)
    csr.set_kernel(0)
    assert out.tobytes() == fwd(csr, x, b, True).tobytes()


def test_unsupported_shapes_rejected():
    w = np.ones((4, 3, 13, 13), np.float32)  # K > 11: no specialised form
    csr = escoin.Csr.stretch(w, 19, 19, 2, 1).to_device(0)
    with pytest.raises(escoin.EscoinError) as e:
        csr.jit()
    assert e.value.status == escoin.ERR_UNSUPPORTED
    assert csr.kernel() != escoin.KERNEL_JIT  # the previous kernel stays selected


@pytest.mark.parametrize("wl,name", [("alexnet", "conv3"), ("alexnet", "conv2"), ("resnet50", "res2a_branch2b"),
                                     ("googlenet", "inception_4a/5x5")])
def test_full_batch_sampled(wl, name):
    # BASELINE full size (N=128) with the default plan bench.py uses; sampled outputs vs oracle,
    # and bitwise identity with the autotuned interpreter kernel on the whole tensor.
    W = workloads.workload(wl)
    L = [l for l in W.layers if l.name == name][0]
    x = inputs.activations(W.net, L.name, 0, 128, L.C, L.H, L.W)
    w = inputs.layer_weights(W.net, L, W.sparsity_permille)
    b = inputs.bias(W.net, L.name, L.M)
    csr = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad).to_device(0)
    auto = fwd(csr, x, b, True)
    csr.jit(n_hint=128)
    out = fwd(csr, x, b, True)
    assert out.tobytes() == auto.tobytes()
    rng = np.random.default_rng(5)
    npts = 3000
    coords = np.stack([rng.integers(0, 128, npts), rng.integers(0, L.M, npts), rng.integers(0, L.E, npts),
                       rng.integers(0, L.F, npts)], 1)
    rp, ci, v = oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad)
    ref, scale = oracle.sconv_points(x, rp, ci, v, L.M, L.K, L.stride, L.pad, coords, bias=b, relu=True)
    got = out[coords[:, 0], coords[:, 1], coords[:, 2], coords[:, 3]].astype(np.float64)
    assert np.all(np.abs(got - ref) <= TOL * (scale + np.abs(b[coords[:, 1]])))


def test_autotune_considers_jit():
    L = workloads.TINY
    x = inputs.activations("tiny", "tiny", 0, 4, L.C, L.H, L.W)
    w = inputs.layer_weights("tiny", L, 800)
    csr = escoin.Csr.stretch(w, L.H, L.W, 1, 1).to_device(0)
    ref = fwd(csr, x, None, True)
    csr.jit(n_hint=4)
    csr.jit(n_hint=4, Q=8, warps=4)  # a second specialised kernel on the same handle
    csr.jit(n_hint=4, Q=16, CC=2, prefetch=-1)
    dx = torch.from_numpy(x).cuda()
    out = torch.empty((4, L.M, L.E, L.F), device="cuda")
    kid, ms = csr.autotune(4, dx, out, None, True, 2, torch.cuda.current_stream().cuda_stream)
    assert ms > 0 and csr.kernel() == kid
    assert fwd(csr, x, None, True).tobytes() == ref.tobytes()
    info = csr.jit_info()
    assert info["regs"] > 0 and info["code_bytes"] > 0 and info["Q"] > 0


@pytest.mark.parametrize("tun", [dict(), dict(Q=8, CC=3, NS=2, warps=4, minb=2), dict(Q=16, CC=5, NS=4),
                                 dict(Q=16, CC=2, NS=4, mbarrier=1)])
def test_grouped_block_diagonal_and_empty_groups(tun):
    # block-diagonal expansion of a g=3 grouped layer (R#18): every m-group touches a channel
    # sub-range only (the kernel skips the other chunks); one whole group of rows is empty
    rng = np.random.default_rng(21)
    N, C, H, M, g = 3, 24, 9, 48, 3
    x = rng.random((N, C, H, H)).astype(np.float32)
    w = np.zeros((M, C, 3, 3), np.float32)
    for k in range(g):
        blk = rng.standard_normal((M // g, C // g, 3, 3)).astype(np.float32)
        blk[rng.random(blk.shape) >= 0.3] = 0.0
        w[k * M // g:(k + 1) * M // g, k * C // g:(k + 1) * C // g] = blk
    w[16:32] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, 1, 1, True)
    out, paper, _ = jit_and_paper(w, x, b, 1, True, **tun)
    check(out, ref, scale, b)
    assert out.tobytes() == paper.tobytes()


# ------------------------------------------------------------------ units, graphs, cache, flushed autotune
def _layer_case(seed, N=6, C=24, H=13, M=96, K=3, pad=1, d=0.25):
    rng = np.random.default_rng(seed)
    x = rng.random((N, C, H, H)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= d] = 0.0
    w[20:24] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    return x, w, b


@pytest.mark.parametrize("units", [1, 2, 3, 6])
def test_units_parity_bitwise(units):
    # the m-groups split into separately compiled units launched concurrently on forked streams:
    # same bits as the paper-mapping kernel, within tolerance of the oracle
    x, w, b = _layer_case(100 + units)
    ref, scale = oracle_ref(w, x, b, 1, 1, True)
    out, paper, csr = jit_and_paper(w, x, b, 1, True, Q=16, units=units)
    assert csr.jit_info()["units"] == units
    check(out, ref, scale, b)
    assert out.tobytes() == paper.tobytes()


def test_multi_unit_forward_captures_into_a_graph():
    x, w, b = _layer_case(7, N=9)
    csr = escoin.Csr.stretch(w, 13, 13, 1, 1).to_device(0)
    csr.jit(n_hint=9, Q=16, units=4)
    dx = torch.from_numpy(x).cuda()
    db = torch.from_numpy(b).cuda()
    eager = escoin.forward(csr, dx, bias=db, relu=True)
    out = torch.zeros_like(eager)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        escoin.forward(csr, dx, bias=db, relu=True, out=out)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
    out.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)


def test_cubin_cache_roundtrip(tmp_path, monkeypatch):
    x, w, b = _layer_case(9)
    monkeypatch.setenv("ESCOIN_JIT_CACHE", str(tmp_path))
    c1 = escoin.Csr.stretch(w, 13, 13, 1, 1).to_device(0)
    c1.jit(n_hint=6, Q=16, units=3)
    st1 = c1.jit_stats()
    assert st1["units"] == 3 and st1["cache_hits"] == 0
    assert len(list(tmp_path.glob("*.cubin"))) == 4  # 3 units + the entry kernel (all relocatable objects)
    c2 = escoin.Csr.stretch(w, 13, 13, 1, 1).to_device(0)
    c2.jit(n_hint=6, Q=16, units=3)
    assert c2.jit_stats()["cache_hits"] == 3
    assert fwd(c1, x, b, True).tobytes() == fwd(c2, x, b, True).tobytes()
    w2 = w.copy()
    w2[0, 0, 0, 0] = 0.5  # one weight differs: a different kernel, no stale hit
    c3 = escoin.Csr.stretch(w2, 13, 13, 1, 1).to_device(0)
    c3.jit(n_hint=6, Q=16, units=3)
    assert c3.jit_stats()["cache_hits"] < 3
    ref, scale = oracle_ref(w2, x, b, 1, 1, True)
    check(fwd(c3, x, b, True), ref, scale, b)


def test_autotune_ex_flushed_jit_only_and_label():
    x, w, b = _layer_case(13, N=8)
    csr = escoin.Csr.stretch(w, 13, 13, 1, 1).to_device(0)
    ref = fwd(csr, x, b, True)
    csr.jit(n_hint=8, Q=16, units=2)
    csr.jit(n_hint=8, Q=32, warps=8, minb=2)
    dx = torch.from_numpy(x).cuda()
    db = torch.from_numpy(b).cuda()
    out = torch.empty((8, 96, 13, 13), device="cuda")
    flush = torch.empty(64 * 1024 * 1024 // 4, device="cuda")
    kid, ms = csr.autotune_ex(8, dx, out, db, True, 3, torch.cuda.current_stream().cuda_stream, flush=flush,
                              flags=escoin.TUNE_JIT)
    assert kid == escoin.KERNEL_JIT and ms > 0
    lab = csr.label()
    assert lab.startswith("jit_q") and "_u" in lab and "_ns" in lab and "_mb" in lab
    assert fwd(csr, x, b, True).tobytes() == ref.tobytes()
    kid, _ = csr.autotune_ex(8, dx, out, db, True, 2, torch.cuda.current_stream().cuda_stream,
                             flags=escoin.TUNE_VARIANTS)
    assert kid != escoin.KERNEL_JIT
    assert not csr.label().startswith("jit_")
    assert fwd(csr, x, b, True).tobytes() == ref.tobytes()


VEC_CASES = [  # N, C, H, W, M, K, stride, pad — rows of W % 4 == 0 / W % 2 == 0 / odd W
    (3, 10, 16, 16, 24, 3, 1, 1), (2, 7, 12, 20, 18, 5, 1, 2), (4, 9, 14, 14, 33, 3, 1, 1), (2, 5, 10, 6, 9, 3, 2, 1),
    (3, 6, 13, 13, 12, 3, 1, 1), (2, 12, 8, 8, 20, 1, 1, 0), (2, 4, 28, 28, 10, 3, 2, 0), (1, 3, 9, 8, 5, 3, 1, 3),
]


@pytest.mark.parametrize("case", VEC_CASES)
def test_vector_staging_bitwise(case):
    # 16/8-byte cp.async staging (per-CTA shifted, aligned buffer) vs 4-byte staging: same bits
    N, C, H, W, M, K, st, p = case
    rng = np.random.default_rng(abs(hash(case)) % 2**32)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= 0.3] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, st, p, True)
    outs = []
    for vec in (0, 1, 2):
        csr = escoin.Csr.stretch(w, H, W, st, p).to_device(0)
        csr.jit(n_hint=N, Q=8, warps=4, minb=2, vec=vec)
        outs.append(fwd(csr, x, b, True))
        if vec == 0:
            want = 4 if W % 4 == 0 else 2 if W % 2 == 0 else 1
            assert "_v%d" % want in csr.label()
    check(outs[0], ref, scale, b)
    assert outs[0].tobytes() == outs[1].tobytes() == outs[2].tobytes()


@pytest.mark.parametrize("case", [(2, 3, 35, 35, 16, 11, 4, 0), (3, 4, 31, 29, 10, 11, 4, 2), (2, 5, 19, 19, 9, 9, 2, 4),
                                  (1, 3, 227, 227, 24, 11, 4, 0)])
def test_large_filters_row_wise(case):
    # K up to 11 (AlexNet conv1, 11x11 / stride 4): taps loaded and consumed filter row by row
    N, C, H, W, M, K, st, p = case
    rng = np.random.default_rng(K * 100 + H)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= 0.2] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, st, p, True)
    csr = escoin.Csr.stretch(w, H, W, st, p).to_device(0)
    csr.jit(n_hint=N)
    assert csr.kernel() == escoin.KERNEL_JIT
    out = fwd(csr, x, b, True)
    check(out, ref, scale, b)
    csr.set_kernel(0)
    assert out.tobytes() == fwd(csr, x, b, True).tobytes()


@pytest.mark.parametrize("reorder", [1, 0])
def test_row_reordering_for_skewed_rows_bitwise(reorder):
    # skewed per-row sparsity (Beta(1, b) row densities): output channels regrouped so every group of
    # Q rows holds about the same nonzeros (load balance) — same bits, epilogue scatters
    from paper_1802_10280_b200.workloads import Layer
    L = Layer("skew", 48, 14, 14, 100, 3, 1, 1)
    w = inputs.layer_weights_skewed("skewtest", L, 800)
    rng = np.random.default_rng(4)
    x = rng.random((3, L.C, L.H, L.W)).astype(np.float32)
    b = (rng.random(L.M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, 1, 1, True)
    c0 = escoin.Csr.stretch(w, L.H, L.W, 1, 1).to_device(0)
    c0.jit(n_hint=3, Q=16, warps=8, reorder=-1)
    assert not c0.label().endswith("_ro")
    c1 = escoin.Csr.stretch(w, L.H, L.W, 1, 1).to_device(0)
    c1.jit(n_hint=3, Q=16, warps=8, reorder=reorder)
    assert c1.label().endswith("_ro")  # skewed enough that auto (0) regroups too
    o0, o1 = fwd(c0, x, b, True), fwd(c1, x, b, False)
    o1r = fwd(c1, x, b, True)
    check(o1r, ref, scale, b)
    assert o0.tobytes() == o1r.tobytes()
    ref_lin, scale_lin = oracle_ref(w, x, b, 1, 1, False)
    check(o1, ref_lin, scale_lin, b)


PERM_CASES = [  # N, C, H, W, M, K, stride, pad, tunables
    (3, 12, 13, 13, 40, 3, 1, 1, dict(Q=16, warps=4)), (5, 9, 7, 7, 33, 3, 1, 1, dict(Q=8, warps=8, P=2)),
    (2, 7, 14, 14, 24, 5, 1, 2, dict(Q=8, warps=4, minb=2)), (4, 6, 27, 27, 20, 5, 1, 2, dict(Q=16, warps=8)),
    (2, 8, 15, 11, 17, 3, 2, 1, dict(Q=8, warps=4)), (3, 10, 13, 13, 48, 3, 1, 1, dict(Q=16, warps=4, units=3)),
]


@pytest.mark.parametrize("relu", [True, False])
@pytest.mark.parametrize("case", PERM_CASES)
def test_lane_pixel_deal_bitwise(case, relu):
    # perm=1: lanes take the tile's pixels dealt by shared-memory bank; accumulators transposed through
    # shared memory before the (coalesced) stores — same bits as every other kernel, ragged tails included
    N, C, H, W, M, K, st, p, tun = case
    rng = np.random.default_rng(abs(hash(case[:8])) % 2**32)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= 0.25] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, st, p, relu)
    csr = escoin.Csr.stretch(w, H, W, st, p).to_device(0)
    csr.jit(n_hint=N, perm=1, reorder=-1, **tun)
    assert "_dl" in csr.label()
    out = fwd(csr, x, b, relu)
    check(out, ref, scale, b)
    csr.set_kernel(0)
    assert out.tobytes() == fwd(csr, x, b, relu).tobytes()
    for n0, n1 in [(1, N), (0, 1)]:  # other batch sizes (other tile phases / tails)
        csr2 = escoin.Csr.stretch(w, H, W, st, p).to_device(0)
        csr2.jit(n_hint=N, perm=1, reorder=-1, **tun)
        assert fwd(csr2, x[n0:n1], b, relu).tobytes() == out[n0:n1].tobytes()


SPLIT_CASES = [  # N, C, H, W, M, K, stride, pad, tunables
    (3, 12, 13, 13, 40, 3, 1, 1, dict(Q=16, warps=8, split=2)), (5, 9, 7, 7, 33, 3, 1, 1, dict(Q=8, warps=6, split=3)),
    (2, 7, 14, 14, 24, 5, 1, 2, dict(Q=8, warps=4, split=2, P=2)), (4, 6, 28, 28, 20, 3, 1, 1, dict(Q=16, warps=8, split=4)),
    (2, 8, 15, 11, 17, 3, 2, 1, dict(Q=8, warps=4, split=2)), (3, 10, 13, 13, 48, 3, 1, 1, dict(Q=16, warps=4, split=2,
                                                                                             units=3)),
]


@pytest.mark.parametrize("case", SPLIT_CASES)
def test_split_subtiles_bitwise(case):
    # split > 1: independent sub-tiles (own ring, own named barrier) inside one CTA — same bits
    N, C, H, W, M, K, st, p, tun = case
    rng = np.random.default_rng(abs(hash(case[:8])) % 2**32 + 1)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= 0.25] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, st, p, True)
    csr = escoin.Csr.stretch(w, H, W, st, p).to_device(0)
    csr.jit(n_hint=N, **tun)
    assert "_s%d" % tun["split"] in csr.label()
    out = fwd(csr, x, b, True)
    check(out, ref, scale, b)
    csr.set_kernel(0)
    assert out.tobytes() == fwd(csr, x, b, True).tobytes()


HP_CASES = [  # N, C, H, W, M, K, pad, tunables — horizontal pixel pairs: odd/even F, pad 0/1/2, K 1/3/5
    (3, 12, 13, 13, 40, 3, 1, dict(Q=16, P=2, warps=4, hp=1)), (2, 9, 14, 14, 24, 3, 1, dict(Q=8, P=2, warps=4, hp=1)),
    (2, 9, 14, 14, 24, 3, 1, dict(Q=8, P=2, warps=4, hp=2)), (2, 6, 56, 56, 16, 3, 1, dict(Q=16, P=2, warps=8, hp=1)),
    (2, 7, 7, 7, 33, 3, 1, dict(Q=8, P=4, warps=2, hp=1)), (3, 5, 11, 9, 12, 5, 2, dict(Q=8, P=2, warps=4, hp=1)),
    (2, 4, 12, 12, 10, 5, 2, dict(Q=4, P=2, warps=4, hp=1, CC=2, NS=4)), (4, 10, 6, 10, 9, 1, 0, dict(Q=8, P=2, hp=1)),
    (2, 8, 9, 8, 21, 3, 0, dict(Q=8, P=2, warps=2, hp=1)), (3, 12, 13, 13, 48, 3, 1, dict(Q=16, P=2, warps=4, hp=1,
                                                                                        units=3)),
    (2, 8, 14, 14, 24, 3, 1, dict(Q=8, P=2, warps=8, hp=1, split=2)),
    (5, 16, 7, 7, 64, 3, 1, dict(Q=32, P=2, warps=4, hp=1, reorder=1)),
]


@pytest.mark.parametrize("relu", [True, False])
@pytest.mark.parametrize("case", HP_CASES)
def test_horizontal_pairs_bitwise(case, relu):
    # hp: lanes hold pixel pairs (ow, ow+1) of one output row, taps from ld.shared.v2, FFMA2 — same
    # bits as the paper-mapping kernel, tolerance vs the oracle; phantom pixels (ow = -1 or F) never stored
    N, C, H, W, M, K, p, tun = case
    rng = np.random.default_rng(abs(hash(case[:7])) % 2**32 + 7)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= 0.25] = 0.0
    w[1] = 0.0  # an empty row
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, 1, p, relu)
    csr = escoin.Csr.stretch(w, H, W, 1, p).to_device(0)
    csr.jit(n_hint=N, **tun)
    lab = csr.label()
    assert "x2h" in lab, lab
    sentinel = torch.full((N, M, H + 2 * p - K + 1, W + 2 * p - K + 1), float("nan"), device="cuda")
    dx = torch.from_numpy(x).cuda()
    db = torch.from_numpy(b).cuda()
    escoin.sconv_forward(N, C, H, W, M, K, 1, p, csr, dx, sentinel, db, relu, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    out = sentinel.cpu().numpy()
    assert not np.isnan(out).any()  # every output written
    check(out, ref, scale, b)
    csr.set_kernel(0)
    assert out.tobytes() == fwd(csr, x, b, relu).tobytes()


KS_CASES = [  # N, C, H, W, M, K, stride, pad, tunables — split channels (few CTAs: small planes, few channels)
    (3, 40, 7, 7, 24, 3, 1, 1, dict(Q=8, CC=4, NS=3, ks=3)), (2, 64, 7, 7, 16, 5, 1, 2, dict(Q=16, CC=4, NS=4, ks=4)),
    (4, 96, 7, 7, 12, 1, 1, 0, dict(Q=12, CC=8, NS=3, ks=2)), (2, 30, 9, 11, 33, 3, 2, 1, dict(Q=16, CC=2, ks=5)),
    (3, 20, 13, 13, 40, 3, 1, 1, dict(Q=16, CC=4, NS=2, ks=4, units=2)), (2, 9, 6, 6, 5, 3, 1, 1, dict(Q=8, CC=1, ks=16)),
]


@pytest.mark.parametrize("relu", [True, False])
@pytest.mark.parametrize("case", KS_CASES)
def test_split_channels_tolerance_and_determinism(case, relu):
    # ks > 1: partial sums over channel ranges + fixed-order reduce: within R#11 of the oracle, identical
    # bits across runs and batch slices (not bitwise equal to the one-range kernels — a different order)
    N, C, H, W, M, K, st, p, tun = case
    rng = np.random.default_rng(abs(hash(case[:8])) % 2**32 + 11)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= 0.25] = 0.0
    w[2] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    ref, scale = oracle_ref(w, x, b, st, p, relu)
    csr = escoin.Csr.stretch(w, H, W, st, p).to_device(0)
    csr.jit(n_hint=N, **tun)
    assert "_k%d" % tun["ks"] in csr.label()
    out = fwd(csr, x, b, relu)
    check(out, ref, scale, b)
    assert fwd(csr, x, b, relu).tobytes() == out.tobytes()
    assert fwd(csr, x[1:], b, relu).tobytes() == out[1:].tobytes()
