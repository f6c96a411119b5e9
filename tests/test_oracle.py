"""Pins for the CPU oracle (oracle/) — checked against things other than itself.

Each test names what fixes the expected value: a SPEC worked example
(tests/golden/spec_examples.json, cited per entry), the brute-force 7-loop
Alg.1, torch conv2d in float64 (an independent library routine),
numpy matmul, closed forms, or invariants stated by the paper.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from paper_1802_10280_b200 import inputs, workloads

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rand_case(rng, N, C, H, W, M, K, density=0.3):
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= density] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    return x, w, b


# ------------------------------------------------------------------ golden values
@pytest.mark.parametrize("ex", GOLD["output_dims"])
def test_output_dims_golden(ex):
    assert oracle.output_dim(ex["H"], ex["K"], ex["stride"], ex["pad"]) == ex["E"]


def test_output_dims_invalid():
    assert oracle.output_dim(2, 3, 1, 0) == -1
    assert oracle.output_dim(5, 3, 0, 0) == -1


@pytest.mark.parametrize("ex", GOLD["layout_f"])
def test_layout_f_golden(ex):
    assert oracle.layout_f(ex["c"], ex["y"], ex["x"], ex["Hin"], ex["Win"]) == ex["f"]


def test_layout_f_additive_exhaustive():
    # f(c, y+r, x+s) = f(c, y, x) + f(0, r, s), all in-bounds points, dims <= 8
    for Hin, Win in [(3, 5), (8, 8), (6, 4)]:
        for c in range(3):
            for y, x, r, s in itertools.product(range(Hin), range(Win), range(Hin), range(Win)):
                if y + r < Hin and x + s < Win:
                    assert oracle.layout_f(c, y + r, x + s, Hin, Win) == \
                        oracle.layout_f(c, y, x, Hin, Win) + oracle.layout_f(0, r, s, Hin, Win)


@pytest.mark.parametrize("ex", GOLD["stretch_index"])
def test_stretch_golden(ex):
    K = ex["K"]
    w = np.zeros((1, ex["C"], K, K), np.float32)
    w.reshape(-1)[ex["kernel_index"]] = 1.5
    rowptr, colidx, value = oracle.csr_stretch(w, ex["H"], ex["W"], 1, ex["pad"])
    assert list(rowptr) == [0, 1] and list(colidx) == [ex["colidx"]] and value[0] == np.float32(1.5)


def test_csr_identity_and_zero():
    # identity viewed as m=3, CRS=3 (C=3, K=1)
    w = np.eye(3, dtype=np.float32).reshape(3, 3, 1, 1)
    rowptr, colidx, value = oracle.csr_stretch(w, 1, 1, 1, 0)  # Hp=Wp=1 -> colidx = c
    assert list(rowptr) == [0, 1, 2, 3] and list(colidx) == [0, 1, 2] and list(value) == [1, 1, 1]
    # all-zero 2x1x2x2
    rowptr, colidx, value = oracle.csr_stretch(np.zeros((2, 1, 2, 2), np.float32), 3, 3, 1, 0)
    assert list(rowptr) == [0, 0, 0] and colidx.size == 0


def test_conv_ones_golden():
    # 6x6 ones conv 3x3 ones -> 4x4 of 9.0
    x = np.ones((1, 1, 6, 6), np.float32)
    w = np.ones((1, 1, 3, 3), np.float32)
    rp, ci, v = oracle.csr_stretch(w, 6, 6, 1, 0)
    out, _ = oracle.sconv(x, rp, ci, v, 1, 3, 1, 0)
    assert out.shape == (1, 1, 4, 4) and np.all(out == 9.0)
    assert np.all(oracle.conv_dense(x, w, 1, 0) == 9.0)


def test_conv_scalar_golden():
    # n=m=c=1, 1x1 weight 2 -> 2*I
    rng = np.random.default_rng(0)
    x = rng.random((1, 1, 5, 7)).astype(np.float32)
    w = np.full((1, 1, 1, 1), 2.0, np.float32)
    rp, ci, v = oracle.csr_stretch(w, 5, 7, 1, 0)
    out, _ = oracle.sconv(x, rp, ci, v, 1, 1, 1, 0)
    assert np.array_equal(out, 2.0 * x.astype(np.float64))


@pytest.mark.parametrize("ex", GOLD["prune"])
def test_prune_golden(ex):
    w = np.array(ex["w"], np.float32)
    assert list(inputs.prune_by_magnitude(w, ex["sparsity_permille"])) == ex["out"]


@pytest.mark.parametrize("ex", GOLD["footprint"])
def test_footprint_golden(ex):
    # P:324-325 footprint model (2*nnz + M + 1) * 4 bytes, measured on the oracle's arrays
    M, nnz = ex["rows"], ex["nnz"]
    rng = np.random.default_rng(nnz)
    w = np.zeros((M, 1, 1, 100 if nnz else 1), np.float32).reshape(M, -1)
    flat = w.reshape(-1)
    flat[rng.choice(flat.size, nnz, replace=False)] = 1.0
    rp, ci, v = oracle.csr_stretch(w.reshape(M, -1, 1, 1), 1, 1, 1, 0)
    assert 4 * (rp.size + ci.size + v.size) == ex["bytes"]


@pytest.mark.parametrize("ex", GOLD["sparsity"])
def test_sparsity_golden(ex):
    # sparsity = zero cells / all cells of the weight matrix
    rows, cols, nnz = ex["rows"], ex["kernel_cols"], ex["nnz"]
    w = np.zeros((rows, cols), np.float32)
    w.reshape(-1)[:nnz] = 1.0
    rp, ci, v = oracle.csr_stretch(w.reshape(rows, cols, 1, 1), 1, 1, 1, 0)
    assert abs((1.0 - v.size / (rows * cols)) - ex["sparsity"]) < 1e-12


def test_footprint_below_40pct_when_sparse():
    # sparsity > 0.8 and M << nnz -> CSR < 40% of dense
    L = workloads.sweep_layer()
    w = inputs.layer_weights("alexnet", L, 810)
    rp, ci, v = oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad)
    assert 4 * (rp.size + ci.size + v.size) < 0.4 * 4 * w.size


# ------------------------------------------------------------------ stretch invariants
@pytest.mark.parametrize("seed", range(12))
def test_stretch_invariants_and_roundtrip(seed):
    rng = np.random.default_rng(100 + seed)
    M, C, K = rng.integers(1, 9), rng.integers(1, 7), int(rng.choice([1, 3, 5]))
    pad = int(rng.integers(0, 3))
    H = int(rng.integers(max(1, K - 2 * pad), 12))
    W = int(rng.integers(max(1, K - 2 * pad), 12))
    stride = int(rng.integers(1, 3))
    _, w, _ = rand_case(rng, 1, C, H, W, M, K, density=float(rng.choice([0.0, 0.2, 0.7, 1.0])))
    rp, ci, v = oracle.csr_stretch(w, H, W, stride, pad)
    Hp, Wp = H + 2 * pad, W + 2 * pad
    assert rp[0] == 0 and rp[-1] == v.size == np.count_nonzero(w) and np.all(np.diff(rp) >= 0)
    # decode (c, kh, kw) from the stretched offset; rebuild the dense tensor bitwise
    rebuilt = np.zeros_like(w)
    for m in range(M):
        row = ci[rp[m]:rp[m + 1]]
        assert np.all(np.diff(row) > 0)  # strictly increasing == ascending (c, kh, kw)
        for j in range(rp[m], rp[m + 1]):
            c, rem = divmod(int(ci[j]), Hp * Wp)
            kh, kw = divmod(rem, Wp)
            assert c < C and kh < K and kw < K
            rebuilt[m, c, kh, kw] = v[j]
    assert rebuilt.tobytes() == w.tobytes() or np.array_equal(rebuilt, w)
    assert np.array_equal(rebuilt.view(np.uint32)[w != 0], w.view(np.uint32)[w != 0])


def test_stretch_drops_signed_zero():
    w = np.array([0.0, -0.0, 1e-40, -2.0], np.float32).reshape(1, 4, 1, 1)
    rp, ci, v = oracle.csr_stretch(w, 2, 2, 1, 0)
    assert list(ci) == [2 * 4, 3 * 4] and v[0] == np.float32(1e-40)


# ------------------------------------------------------------------ Alg.2 vs Alg.1 brute force
SHAPES = [  # N, C, H, W, M, K, stride, pad
    (2, 3, 6, 6, 4, 3, 1, 0), (1, 2, 7, 5, 3, 3, 2, 1), (2, 4, 9, 8, 2, 5, 1, 2),
    (1, 3, 8, 11, 5, 1, 1, 0), (1, 2, 10, 7, 3, 3, 3, 2), (3, 1, 5, 5, 2, 5, 2, 2),
    (1, 5, 4, 4, 6, 3, 1, 1), (2, 2, 13, 13, 3, 3, 1, 1),
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("relu", [False, True])
def test_alg2_equals_alg1_bitwise(shape, relu):
    N, C, H, W, M, K, s, p = shape
    rng = np.random.default_rng(hash(shape) % 2**32)
    x, w, b = rand_case(rng, N, C, H, W, M, K, density=0.4)
    rp, ci, v = oracle.csr_stretch(w, H, W, s, p)
    out2, scale = oracle.sconv(x, rp, ci, v, M, K, s, p, bias=b, relu=relu)
    out1 = oracle.conv_dense(x, w, s, p, bias=b, relu=relu)
    # fp32 x fp32 products are exact in fp64 and nonzero terms are summed in the
    # same ascending (c, kh, kw) order; zero-weight terms add +-0 -> bitwise equal.
    assert np.array_equal(out2, out1)
    # scale bounds the pre-bias sum
    pre, _ = oracle.sconv(x, rp, ci, v, M, K, s, p)
    assert np.all(np.abs(pre) <= scale)


SCALE_SHAPES = [  # N, C, H, W, M, K, stride, pad — strides 1-3, pads 0-2
    (2, 3, 6, 6, 4, 3, 1, 0), (1, 2, 7, 5, 3, 3, 2, 1), (2, 4, 9, 8, 2, 5, 1, 2), (1, 3, 8, 11, 5, 1, 1, 0),
    (1, 2, 10, 7, 3, 3, 3, 2), (3, 1, 5, 5, 2, 5, 2, 2), (2, 5, 11, 9, 4, 3, 3, 0), (1, 4, 12, 12, 3, 5, 2, 1),
]


@pytest.mark.parametrize("shape", SCALE_SHAPES)
def test_scale_equals_abs_conv(shape):
    # scale = sum |w * x| over the stored nonzeros of row m (R#11, R#21) is the denominator of every
    # parity tolerance.  Pinned independently of the oracle: torch conv2d in float64 of |x| (zero
    # padded) with |w| computes sum_{c,kh,kw} |w| |x~| — the same set of terms (zero weights add 0,
    # taps in the padding add 0).  Signed x, so a scale that dropped the |.| on x would fail.
    # Every term is an exact fp64 product of two fp32 numbers; the sums differ only in order, so
    # they agree to a few ulps of the sum.
    torch = pytest.importorskip("torch")
    N, C, H, W, M, K, s, p = shape
    rng = np.random.default_rng(sum(shape) * 7919)
    x = (rng.random((N, C, H, W)) * 2 - 1).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= 0.4] = 0.0
    rp, ci, v = oracle.csr_stretch(w, H, W, s, p)
    _, scale = oracle.sconv(x, rp, ci, v, M, K, s, p, bias=None, relu=False)
    ind = torch.nn.functional.conv2d(torch.from_numpy(np.abs(x).astype(np.float64)),
                                     torch.from_numpy(np.abs(w).astype(np.float64)), stride=s, padding=p).numpy()
    assert scale.shape == ind.shape
    assert np.allclose(scale, ind, rtol=1e-13, atol=0.0)
    # and a bias does not enter scale (the tolerance adds |bias| separately)
    _, scale_b = oracle.sconv(x, rp, ci, v, M, K, s, p, bias=np.full(M, 5.0, np.float32), relu=True)
    assert np.array_equal(scale_b, scale)


@pytest.mark.parametrize("shape", SHAPES[:5])
def test_points_equal_full(shape):
    N, C, H, W, M, K, s, p = shape
    rng = np.random.default_rng(7)
    x, w, b = rand_case(rng, N, C, H, W, M, K)
    rp, ci, v = oracle.csr_stretch(w, H, W, s, p)
    out, scale = oracle.sconv(x, rp, ci, v, M, K, s, p, bias=b, relu=True)
    coords = np.array(list(itertools.product(range(N), range(M), range(out.shape[2]), range(out.shape[3]))))
    pts, psc = oracle.sconv_points(x, rp, ci, v, M, K, s, p, coords, bias=b, relu=True)
    assert np.array_equal(pts, out.reshape(-1)) and np.array_equal(psc, scale.reshape(-1))


# ------------------------------------------------------------------ special cases / invariants
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("shape", SHAPES)
def test_density_one_equals_torch_conv2d(shape):
    # north_star: density 1.0 equals dense conv (independent library routine, float64)
    N, C, H, W, M, K, s, p = shape
    rng = np.random.default_rng(11)
    x, w, b = rand_case(rng, N, C, H, W, M, K, density=1.0)
    rp, ci, v = oracle.csr_stretch(w, H, W, s, p)
    out, scale = oracle.sconv(x, rp, ci, v, M, K, s, p, bias=b)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x).double(), torch.from_numpy(w).double(),
                                     torch.from_numpy(b).double(), stride=s, padding=p).numpy()
    assert np.all(np.abs(out - ref) <= 1e-13 * (scale + np.abs(b)[None, :, None, None]) + 1e-300)


def test_pruned_layer_equals_torch_conv2d():
    L = workloads.TINY
    x = inputs.activations("tiny", "tiny", 0, 2, L.C, L.H, L.W)
    w = inputs.layer_weights("tiny", L, 800)
    b = inputs.bias("tiny", "tiny", L.M)
    rp, ci, v = oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad)
    assert v.size == 922  # 4608 - floor(0.8*4608) = 922
    out, scale = oracle.sconv(x, rp, ci, v, L.M, L.K, L.stride, L.pad, bias=b, relu=True)
    ref = torch.relu(torch.nn.functional.conv2d(torch.from_numpy(x).double(), torch.from_numpy(w).double(),
                                                torch.from_numpy(b).double(), padding=L.pad)).numpy()
    assert np.all(np.abs(out - ref) <= 1e-13 * (scale + 0.1))


def test_all_zero_weights_give_bias():
    rng = np.random.default_rng(3)
    x, _, b = rand_case(rng, 2, 3, 7, 7, 5, 3)
    w = np.zeros((5, 3, 3, 3), np.float32)
    rp, ci, v = oracle.csr_stretch(w, 7, 7, 1, 1)
    out, _ = oracle.sconv(x, rp, ci, v, 5, 3, 1, 1, bias=b)
    assert np.array_equal(out, np.broadcast_to(b.astype(np.float64)[None, :, None, None], out.shape))
    outr, _ = oracle.sconv(x, rp, ci, v, 5, 3, 1, 1, bias=b, relu=True)
    assert np.array_equal(outr, np.maximum(out, 0.0))


def test_1x1_equals_sparse_matmul():
    # north_star: a 1x1 kernel (s=1, p=0) is sparse W[M x C] times X[n][C x HW]
    rng = np.random.default_rng(5)
    x, w, _ = rand_case(rng, 3, 17, 6, 9, 11, 1, density=0.25)
    rp, ci, v = oracle.csr_stretch(w, 6, 9, 1, 0)
    out, scale = oracle.sconv(x, rp, ci, v, 11, 1, 1, 0)
    ref = np.einsum("mc,ncp->nmp", w.reshape(11, 17).astype(np.float64),
                    x.reshape(3, 17, 54).astype(np.float64)).reshape(out.shape)
    assert np.all(np.abs(out - ref) <= 1e-13 * scale + 1e-300)


def test_linear_in_weights_and_inputs():
    rng = np.random.default_rng(9)
    N, C, H, W, M, K, s, p = 2, 3, 8, 8, 4, 3, 1, 1
    x1, w1, _ = rand_case(rng, N, C, H, W, M, K, 0.3)
    x2, w2, _ = rand_case(rng, N, C, H, W, M, K, 0.3)

    def conv(x, w):
        rp, ci, v = oracle.csr_stretch(w, H, W, s, p)
        return oracle.sconv(x, rp, ci, v, M, K, s, p)

    a, b = np.float32(0.5), np.float32(-2.0)   # exact scalings keep fp32 weights exact
    o1, s1 = conv(x1, w1)
    o2, s2 = conv(x1, w2)
    o12, _ = conv(x1, (a * w1 + b * w2).astype(np.float32))
    tol = 1e-12 * (np.abs(a) * s1 + np.abs(b) * s2) + 1e-300
    # a*w1 + b*w2 is rounded to fp32 once; bound that rounding by 2^-24 relative
    tol = tol + 2.0 ** -23 * (np.abs(a) * s1 + np.abs(b) * s2)
    assert np.all(np.abs(o12 - (a * o1 + b * o2)) <= tol)
    i1, t1 = conv(x1, w1)
    i2, t2 = conv(x2, w1)
    i12, _ = conv((x1 + x2).astype(np.float32), w1)
    assert np.all(np.abs(i12 - (i1 + i2)) <= 2.0 ** -23 * (t1 + t2) + 1e-300)


def test_per_nonzero_decomposition_fig5():
    # P:483-489 (Fig.5): a 3x3 filter with two nonzeros ("2" and "3") over a 6x6
    # input equals the sum of the two nonzeros times their shifted 4x4 sub-matrices.
    rng = np.random.default_rng(2)
    x = rng.random((1, 1, 6, 6)).astype(np.float32)
    w = np.zeros((1, 1, 3, 3), np.float32)
    w[0, 0, 0, 1] = 2.0
    w[0, 0, 2, 2] = 3.0
    rp, ci, v = oracle.csr_stretch(w, 6, 6, 1, 0)
    out, _ = oracle.sconv(x, rp, ci, v, 1, 3, 1, 0)
    xd = x[0, 0].astype(np.float64)
    expect = 2.0 * xd[0:4, 1:5] + 3.0 * xd[2:6, 2:6]
    assert np.array_equal(out[0, 0], expect)


def test_pad_input_properties():
    x = np.array([[[[5.0]]]], np.float32)
    xp = oracle.pad_input(x, 1)
    assert xp.shape == (1, 1, 3, 3) and xp[0, 0, 1, 1] == 5.0 and xp.sum() == 5.0
    rng = np.random.default_rng(4)
    x = rng.random((2, 3, 5, 4)).astype(np.float32)
    for p in range(3):
        xp = oracle.pad_input(x, p)
        assert np.array_equal(xp[:, :, p:p + 5, p:p + 4], x.astype(np.float64))
        assert abs(xp.sum() - x.astype(np.float64).sum()) < 1e-9


def test_fault_injection_changes_output():
    # a corrupted stretched colidx must be detectable
    L = workloads.TINY
    x = inputs.activations("tiny", "tiny", 0, 1, L.C, L.H, L.W)
    w = inputs.layer_weights("tiny", L, 800)
    rp, ci, v = oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad)
    out, scale = oracle.sconv(x, rp, ci, v, L.M, L.K, 1, 1)
    bad = ci.copy()
    bad[100] += 1
    out2, _ = oracle.sconv(x, rp, bad, v, L.M, L.K, 1, 1)
    assert np.max(np.abs(out2 - out) / (scale + 1e-30)) > 1e-5


# ------------------------------------------------------------------ pruning + generator
def test_prune_contract():
    w = inputs.weights("t", "l", 8, 4, 3)
    for s in [0, 200, 800, 999]:
        pw = inputs.prune_by_magnitude(w, s)
        zeros = (s * w.size) // 1000
        assert np.count_nonzero(pw == 0) == zeros
        kept = np.abs(pw[pw != 0])
        if kept.size and zeros:
            assert kept.min() >= np.abs(w.reshape(-1)[np.argsort(np.abs(w.reshape(-1)), kind="stable")[zeros - 1]])
    ties = np.array([1.0, -1.0, 1.0, 2.0], np.float32)
    assert list(inputs.prune_by_magnitude(ties, 500)) == [0.0, 0.0, 1.0, 2.0]
    assert np.array_equal(inputs.prune_by_magnitude(inputs.prune_by_magnitude(w, 800), 800),
                          inputs.prune_by_magnitude(w, 800))


def test_generator_shard_invariance_and_ranges():
    a = inputs.activations("n", "l", 0, 8, 3, 5, 5)
    b = inputs.activations("n", "l", 4, 4, 3, 5, 5)
    assert np.array_equal(a[4:], b)
    assert a.dtype == np.float32 and a.min() >= 0.0 and a.max() < 1.0
    assert not np.array_equal(a[0], a[1])
    z = inputs.normal(inputs.key("x"), 200000)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    bb = inputs.bias("n", "l", 1000)
    assert bb.min() >= -0.1 and bb.max() < 0.1
    ex = inputs.activations("n", "l", 0, 2, 2, 3, 3, exact=True)
    assert set(np.unique(ex)) <= {0.0, 1.0, 2.0, 3.0}
    we = inputs.weights("n", "l", 4, 2, 3, exact=True)
    assert set(np.unique(we)) <= set(float(i) for i in range(-3, 4))


def test_expand_groups_block_diagonal():
    wg = inputs.weights("n", "l", 6, 2, 3)
    w = inputs.expand_groups(wg, 2)
    assert w.shape == (6, 4, 3, 3)
    assert np.all(w[:3, 2:] == 0) and np.all(w[3:, :2] == 0)
    assert np.array_equal(w[:3, :2], wg[:3]) and np.array_equal(w[3:, 2:], wg[3:])


# ------------------------------------------------------------------ Table 3
@pytest.mark.parametrize("ex", GOLD["table3"])
def test_table3_reproduced(ex):
    full = {"alexnet": workloads.alexnet_full, "googlenet": workloads.googlenet_full,
            "resnet50": workloads.resnet50_full}[ex["net"]]()
    convs = workloads.conv_layers(full)
    assert len(convs) == ex["conv_layers"]
    assert sum(l.sparse for l in convs) == ex["sparse_layers"]
    weights = sum(l.weights for l in full) / 1e6
    assert abs(weights - ex["weights_M"]) / ex["weights_M"] < 0.02
    macs = sum(l.macs for l in full) / 1e6
    if ex["net"] != "googlenet":  # reading R#17: GoogLeNet's 1.43G is not reproduced
        assert abs(macs - ex["macs_M"]) / ex["macs_M"] < 0.015
    if ex["net"] == "alexnet":
        assert round(macs) == 724 and round(weights) == 61


def test_resnet50_v15_macs():
    # v1.5 moves the stride to the 3x3: 4.09G MACs (SURVEY reading R#16), same weights
    full = workloads.resnet50_full(v15=True)
    assert abs(sum(l.macs for l in full) / 1e9 - 4.09) < 0.02
    assert sum(l.weights for l in full) == sum(l.weights for l in workloads.resnet50_full())
    sparse = [l for l in full if l.sparse]
    assert len(sparse) == 16 and sum(l.stride == 2 for l in sparse) == 3


def test_skewed_generator_contract():
    # SURVEY §8(d) skewed variant: per-row densities Beta(1, b) with the requested mean, each row pruned
    # to round(d_m * T_row) by magnitude; deterministic (counter-based keys)
    L = workloads.workload("resnet50").layers[10]
    w = inputs.layer_weights_skewed("resnet50", L, 800)
    w2 = inputs.layer_weights_skewed("resnet50", L, 800)
    assert w.tobytes() == w2.tobytes()
    d = inputs.skewed_row_density("resnet50", L.name, L.M, 0.2)
    T = L.C * L.K * L.K
    per_row = np.count_nonzero(w.reshape(L.M, -1), axis=1)
    assert np.array_equal(per_row, np.round(d * T).astype(int))
    assert abs(per_row.sum() / w.size - 0.2) < 0.03          # mean density ~ 0.2
    assert per_row.max() > 2.5 * per_row.mean()               # skewed: a heavy tail
    # surviving entries are the largest |w| of their row
    dense = inputs.weights("resnet50", L.name, L.M, L.C, L.K)
    for m in [0, 7, 100]:
        kept = np.abs(dense[m].reshape(-1))[w[m].reshape(-1) != 0]
        dropped = np.abs(dense[m].reshape(-1))[w[m].reshape(-1) == 0]
        if kept.size and dropped.size:
            assert kept.min() >= dropped.max()
