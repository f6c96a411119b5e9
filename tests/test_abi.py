"""CPU-side checks of the C-ABI library: it loads, exports every symbol of
include/escoin.h, and its host-side stretch is bit-exact against the
oracle's independent stretch (no GPU compute calls here)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_1802_10280_b200 import escoin, inputs, workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "escoin.h")).read()
    return sorted(set(re.findall(r"^(?:int|void|double|const char\*)\s+(escoin_[a-z_0-9]+)\(", src, re.M)))


def test_header_symbols_exported():
    L = escoin.lib()
    syms = header_symbols()
    assert set(syms) == set(escoin.EXPORTS)
    for s in syms:
        assert hasattr(L, s), s
    assert "sm_100a" in escoin.version()


def test_library_has_no_oracle_dependency():
    # the product library must not link or embed the oracle
    data = open(escoin.LIB_PATH, "rb").read()
    assert b"oracle_" not in data


def test_kernel_table():
    ks = escoin.kernels()
    assert ks[0][1] == "paper_mapping" and ks[0][2] == 0
    assert any(k[2] == 3 and k[3] == 1 for k in ks)
    assert any(k[2] == 5 and k[3] == 1 for k in ks)


@pytest.mark.parametrize("seed", range(20))
def test_stretch_bit_exact_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    K = int(rng.choice([1, 3, 5]))
    pad = int(rng.integers(0, 3))
    H, W = int(rng.integers(max(1, K - 2 * pad), 15)), int(rng.integers(max(1, K - 2 * pad), 15))
    M, C, stride = int(rng.integers(1, 12)), int(rng.integers(1, 9)), int(rng.integers(1, 3))
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) < rng.random()] = 0.0
    if seed % 5 == 0:
        w[rng.random(w.shape) < 0.5] = -0.0
    csr = escoin.Csr.stretch(w, H, W, stride, pad)
    rp, ci, v = csr.host_arrays()
    orp, oci, ov = oracle.csr_stretch(w, H, W, stride, pad)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    assert v.view(np.uint32).tobytes() == ov.view(np.uint32).tobytes()
    info = csr.info()
    assert info == dict(M=M, C=C, H=H, W=W, K=K, stride=stride, pad=pad, nnz=int(ov.size))


@pytest.mark.parametrize("wl", ["tiny", "alexnet", "resnet50"])
def test_stretch_bit_exact_config_layers(wl):
    W = workloads.workload(wl)
    for L in W.layers[:4]:
        w = inputs.layer_weights(W.net, L, W.sparsity_permille)
        csr = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad)
        rp, ci, v = csr.host_arrays()
        orp, oci, ov = oracle.csr_stretch(w, L.H, L.W, L.stride, L.pad)
        assert np.array_equal(rp, orp) and np.array_equal(ci, oci) and np.array_equal(v, ov)


def test_stretch_errors():
    w = np.ones((2, 2, 3, 3), np.float32)
    with pytest.raises(escoin.EscoinError) as e:
        escoin.Csr.stretch(w, 1, 1, 1, 0)          # E < 1
    assert e.value.status == escoin.ERR_SHAPE
    with pytest.raises(escoin.EscoinError) as e:
        escoin.Csr.stretch(w, 5, 5, 0, 0)          # stride < 1
    assert e.value.status == escoin.ERR_SHAPE
    L = escoin.lib()
    h = ctypes.c_void_p()
    assert L.escoin_csr_stretch(None, 2, 2, 5, 5, 3, 1, 0, ctypes.byref(h)) == escoin.ERR_NULL
    assert L.escoin_sconv_forward(1, 2, 5, 5, 2, 3, 1, 0, None, None, None, None, 0, None) == escoin.ERR_NULL
    csr = escoin.Csr.stretch(w, 5, 5, 1, 0)
    # shape mismatch is detected before any device work
    assert L.escoin_sconv_forward(1, 3, 5, 5, 2, 3, 1, 0, csr.handle, None, None, None, 0, None) == \
        escoin.ERR_CSR_MISMATCH
    # forward on a handle with no device copy
    assert L.escoin_sconv_forward(1, 2, 5, 5, 2, 3, 1, 0, csr.handle, 1, 1, None, 0, None) == \
        escoin.ERR_NOT_ON_DEVICE
    # N == 0 is a no-op
    assert L.escoin_sconv_forward(0, 2, 5, 5, 2, 3, 1, 0, csr.handle, None, None, None, 0, None) == escoin.OK
    L.escoin_csr_free(None)  # NULL-safe
    assert escoin.lib().escoin_status_string(-6) == b"unsupported kernel variant / shape"


def test_select_engine_rule(monkeypatch):
    # SPEC select_engine: SPARSE iff sparsity >= threshold (ties -> SPARSE), else DENSE_TC
    monkeypatch.delenv("ESCOIN_SPARSE_THRESHOLD", raising=False)
    t = escoin.sparse_threshold()
    assert 0.0 < t < 1.0
    M, C, K = 64, 32, 3
    T = M * C * K * K
    assert escoin.select_engine(M, C, K, int(0.1 * T)) == escoin.ENGINE_SPARSE      # sparsity 0.9
    assert escoin.select_engine(M, C, K, T) == escoin.ENGINE_DENSE_TC               # sparsity 0.0
    assert escoin.select_engine(M, C, K, 0) == escoin.ENGINE_SPARSE                 # all zero
    nnz_at = T - 0.6 * T                                                            # sparsity exactly 0.6
    assert escoin.select_engine(M, C, K, int(nnz_at), 0.6) == escoin.ENGINE_SPARSE
    assert escoin.select_engine(M, C, K, int(nnz_at) + 1, 0.6) == escoin.ENGINE_DENSE_TC
    monkeypatch.setenv("ESCOIN_SPARSE_THRESHOLD", "0.95")                          # process-wide override
    assert escoin.sparse_threshold() == 0.95
    assert escoin.select_engine(M, C, K, int(0.1 * T)) == escoin.ENGINE_DENSE_TC
    assert escoin.select_engine(M, C, K, int(0.1 * T), 0.5) == escoin.ENGINE_SPARSE  # per-call override wins
    with pytest.raises(escoin.EscoinError):
        escoin.select_engine(0, C, K, 1)
