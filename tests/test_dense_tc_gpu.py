"""The dense tcgen05 implicit-GEMM comparison point (escoin_bench_dense_tc_forward).

NOT the method (it multiplies every weight, zeros included): north_star keeps
it "only as a measured comparison point".  Checked against the same fp64
oracle as the sparse path, element by element:
  * nsplit = 3 (3xTF32): the method's own tolerance 1e-5 * (sum|w*x| + |bias|);
  * nsplit = 1 (TF32): both operands rounded to 10-bit mantissas, each product
    off by <= 2^-10 relative -> tolerance 2e-3 * (sum|w*x| + |bias|).
"""
import numpy as np
import pytest

import oracle
from paper_1802_10280_b200 import escoin

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = [  # N, C, H, W, M, K, stride, pad, density
    (2, 16, 14, 14, 32, 3, 1, 1, 0.2),     # the tiny config shape (x2 images)
    (3, 7, 13, 11, 130, 5, 1, 2, 0.3),     # ragged M (> one 128-row tile), ragged pixels, K=5
    (2, 40, 9, 9, 20, 3, 2, 1, 0.5),       # stride 2, Kd = 360 (ragged k-chunks)
    (1, 5, 6, 6, 3, 1, 1, 0, 1.0),         # 1x1, tiny
    (4, 64, 28, 28, 64, 3, 1, 1, 0.2),     # several pixel tiles
    (2, 3, 31, 31, 10, 11, 4, 2, 0.5),     # K*K > 64: the explicit-bounds gather path (conv1-like)
]


@pytest.mark.parametrize("nsplit,tol", [(3, 1e-5), (1, 2e-3)])
@pytest.mark.parametrize("case", CASES)
def test_dense_tc_matches_oracle(case, nsplit, tol):
    N, C, H, W, M, K, s, p, d = case
    rng = np.random.default_rng(11)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= d] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    rp, ci, v = oracle.csr_stretch(w, H, W, s, p)
    ref, scale = oracle.sconv(x, rp, ci, v, M, K, s, p, bias=b, relu=True)
    out = escoin.bench_dense_tc_forward(torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda(),
                                        torch.from_numpy(b).cuda(), s, p, True, nsplit)
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.float64)
    bound = tol * (scale + np.abs(b.astype(np.float64))[None, :, None, None])
    err = np.abs(got - ref)
    assert np.all(err <= bound), "max err ratio %.3g" % np.max(err / np.maximum(bound, 1e-300))


@pytest.mark.parametrize("case", CASES[:5])
def test_dense_engine_on_a_handle(case):
    # ESCOIN_KERNEL_DENSE_TC: the handle's CSR densified on the device (inverse stretch) and run
    # through the 3xTF32 tcgen05 kernel behind escoin_sconv_forward — method tolerance vs oracle
    N, C, H, W, M, K, s, p, d = case
    rng = np.random.default_rng(23)
    x = rng.random((N, C, H, W)).astype(np.float32)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= d] = 0.0
    b = (rng.random(M) * 0.2 - 0.1).astype(np.float32)
    rp, ci, v = oracle.csr_stretch(w, H, W, s, p)
    ref, scale = oracle.sconv(x, rp, ci, v, M, K, s, p, bias=b, relu=True)
    csr = escoin.Csr.stretch(w, H, W, s, p).to_device(0)
    csr.set_kernel(escoin.KERNEL_DENSE_TC)
    assert csr.label() == "dense_tcgen05_3xtf32"
    out = escoin.forward(csr, torch.from_numpy(x).cuda(), bias=torch.from_numpy(b).cuda(), relu=True)
    direct = escoin.bench_dense_tc_forward(torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda(),
                                           torch.from_numpy(b).cuda(), s, p, True, 3)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert got.tobytes() == direct.cpu().numpy().tobytes()  # densify == the original dense weights
    bound = 1e-5 * (scale + np.abs(b.astype(np.float64))[None, :, None, None])
    assert np.all(np.abs(got.astype(np.float64) - ref) <= bound)


def test_select_engine_on_handles():
    rng = np.random.default_rng(5)
    N, C, H, M, K = 2, 16, 12, 32, 3
    x = torch.from_numpy(rng.random((N, C, H, H)).astype(np.float32)).cuda()
    for d, want in [(0.9, escoin.ENGINE_DENSE_TC), (0.2, escoin.ENGINE_SPARSE)]:
        w = rng.standard_normal((M, C, K, K)).astype(np.float32)
        w[rng.random(w.shape) >= d] = 0.0
        csr = escoin.Csr.stretch(w, H, H, 1, 1).to_device(0)
        sparse_out = escoin.forward(csr, x, relu=True)
        assert csr.select_engine() == want
        assert (csr.kernel() == escoin.KERNEL_DENSE_TC) == (want == escoin.ENGINE_DENSE_TC)
        out = escoin.forward(csr, x, relu=True)
        torch.cuda.synchronize()
        if want == escoin.ENGINE_SPARSE:
            assert torch.equal(out, sparse_out)
        else:
            assert torch.allclose(out, sparse_out, rtol=1e-4, atol=1e-4)
            assert csr.select_engine(threshold=0.0) == escoin.ENGINE_SPARSE  # override: back to sparse
            assert csr.kernel() != escoin.KERNEL_DENSE_TC
