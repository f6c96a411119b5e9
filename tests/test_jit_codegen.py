"""Host-side checks of the pattern-specialised kernel's code generator (no GPU needed).

escoin_csr_jit compiles one `fma.rn.f32 acc, x, <weight immediate>, acc` per nonzero and
pixel.  These tests read the generated PTX (internal export escoin_internal_jit_ptx) and
check, independently of any device, that every accumulator receives exactly its CSR row —
the stretched CSR values bit for bit, at the taps its colidx encodes, in ascending
(c, kh, kw) order (reading R#10) — and that the text compiles for sm_100a in-process.
"""
import ctypes
import re

import numpy as np
import pytest

from paper_1802_10280_b200 import escoin, inputs, workloads


def _lib():
    L = escoin.lib()
    L.escoin_internal_jit_ptx.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                          ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
    L.escoin_internal_ptx_compile.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64)]
    return L


def gen_ptx(csr, n_hint=16, **tun):
    # reorder defaults to -1 here (identity grouping: accumulator (g, q) is row g*Q + q)
    keys = ["Q", "P", "CC", "NS", "warps", "minb", "prefetch", "mbarrier", "units", "vec", "reorder", "sws",
            "perm", "split", "pair", "hp", "pw", "ks"]
    tun.setdefault("reorder", -1)
    arr = (ctypes.c_int * 18)(*[tun.get(k, 0) for k in keys])
    L, n = _lib(), ctypes.c_int64()
    assert L.escoin_internal_jit_ptx(csr.handle, n_hint, arr, 18, None, 0, ctypes.byref(n)) == 0
    buf = ctypes.create_string_buffer(n.value + 1)
    assert L.escoin_internal_jit_ptx(csr.handle, n_hint, arr, 18, buf, n.value + 1, ctypes.byref(n)) == 0
    return buf.value.decode()


FMA = re.compile(r"fma\.rn\.f32 %a(\d+), %x(\d+), 0f([0-9A-F]{8}), %a(\d+);")
# FFMA2 slot pairs: {w, w} as a 64-bit immediate, pair registers %A (accumulators) and %X (taps)
FMA2 = re.compile(r"mov\.b64 %W, 0x([0-9A-F]{8})([0-9A-F]{8}); fma\.rn\.f32x2 %A(\d+), %X(\d+), %W, %A(\d+);")
PACK = re.compile(r"mov\.b64 %X(\d+), \{%x(\d+), %x(\d+)\};")
UNPACK = re.compile(r"mov\.b64 \{%a(\d+), %a(\d+)\}, %A(\d+);")
BLOCK = re.compile(r"^B(\d+)_(\d+):")


def fma_stream(ptx):
    """[(group, acc, xreg, bits)] in program order of the chunk blocks; an FFMA2 on pair registers
    counts as its two halves (acc 2A / 2A+1 at taps 2X / 2X+1), after checking that every pair is
    built from (and unpacked into) exactly those scalar registers."""
    g, out = None, []
    for line in ptx.splitlines():
        m = BLOCK.match(line)
        if m:
            g = int(m.group(1))
            continue
        m = FMA.search(line)
        if m:
            assert m.group(1) == m.group(4), line  # accumulates in place
            out.append((g, int(m.group(1)), int(m.group(2)), int(m.group(3), 16)))
            continue
        m = FMA2.search(line)
        if m:
            assert m.group(1) == m.group(2), line  # the same weight in both halves
            assert m.group(3) == m.group(5), line
            a, x, bits = int(m.group(3)), int(m.group(4)), int(m.group(1), 16)
            out.append((g, 2 * a, 2 * x, bits))
            out.append((g, 2 * a + 1, 2 * x + 1, bits))
            continue
        m = PACK.search(line)
        if m:
            assert (int(m.group(2)), int(m.group(3))) == (2 * int(m.group(1)), 2 * int(m.group(1)) + 1), line
            continue
        m = UNPACK.search(line)
        if m:
            assert (int(m.group(1)), int(m.group(2))) == (2 * int(m.group(3)), 2 * int(m.group(3)) + 1), line
    return out


def check_rows(csr, ptx, Q, P, stream=None, order=None):
    info = csr.info()
    M, K, H, W, pad = info["M"], info["K"], info["H"], info["W"], info["pad"]
    Hp, Wp = H + 2 * pad, W + 2 * pad
    rowptr, colidx, value = csr.host_arrays()
    stream = fma_stream(ptx) if stream is None else stream
    assert len(stream) == info["nnz"] * P  # one FFMA per nonzero and pixel, nothing else
    per_acc = {}
    for g, a, x, bits in stream:
        per_acc.setdefault((g, a), []).append((x, bits))
    slot_of = {m: divmod(m, Q) for m in range(M)} if order is None else {m: gq for gq, m in order.items()}
    for m in range(M):
        g, q = slot_of[m]
        r0, r1 = rowptr[m], rowptr[m + 1]
        bits = value[r0:r1].view(np.uint32).tolist()
        rem = colidx[r0:r1] % (Hp * Wp)
        taps = ((rem // Wp) * K + rem % Wp).tolist()
        for j in range(P):
            got = per_acc.get((g, q * P + j), [])
            assert [b for _, b in got] == bits, "row %d pixel %d: weights or order differ" % (m, j)
            assert [x for x, _ in got] == [t * P + j for t in taps], "row %d pixel %d: taps differ" % (m, j)


def resolved_q(ptx):
    return int(re.search(r"\.reg \.f32 %a<(\d+)>;", ptx).group(1))


def test_balanced_group_rows():
    # Q = 48 over M = 256 rows: 6 groups of ceil(256 / 6) = 43 rows instead of 5 x 48 + 16
    rng = np.random.default_rng(3)
    w = rng.standard_normal((256, 4, 3, 3)).astype(np.float32)
    w[rng.random(w.shape) >= 0.2] = 0.0
    csr = escoin.Csr.stretch(w, 6, 6, 1, 1)
    ptx = gen_ptx(csr, Q=48)
    assert resolved_q(ptx) == 43 and ".u32 mgr[12]" in ptx
    check_rows(csr, ptx, 43, 1)


CASES = [  # C, H, W, M, K, pad, density, tunables
    (16, 14, 14, 32, 3, 1, 0.2, dict()),
    (7, 9, 11, 33, 3, 1, 0.3, dict(Q=8, P=2, CC=3)),
    (6, 8, 8, 20, 5, 2, 0.25, dict(Q=16, CC=4, NS=4, mbarrier=1)),
    (12, 6, 7, 19, 1, 0, 0.4, dict(Q=4, P=3, warps=4, prefetch=-1)),
    (9, 10, 10, 21, 3, 1, 0.25, dict(Q=8, P=2, pair=-1)),            # scalar FFMAs at P = 2
    (10, 7, 9, 17, 3, 1, 0.3, dict(Q=8, P=4, CC=4, warps=4)),       # two FFMA2 pairs per lane
    (5, 12, 12, 12, 5, 2, 0.3, dict(Q=4, P=2, CC=2, mbarrier=1)),   # FFMA2 in the mbarrier pipeline
]
STRIDED = [  # C, H, W, M, K, stride, pad
    (6, 15, 11, 13, 3, 2, 1), (5, 9, 9, 7, 3, 1, 0), (3, 11, 11, 5, 5, 2, 2), (7, 13, 12, 6, 3, 3, 1),
]


@pytest.mark.parametrize("case", STRIDED)
def test_strided_and_padded_fma_stream(case):
    C, H, W, M, K, st, pad = case
    rng = np.random.default_rng(C * 100 + H)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= 0.3] = 0.0
    csr = escoin.Csr.stretch(w, H, W, st, pad)
    ptx = gen_ptx(csr, Q=8)
    check_rows(csr, ptx, resolved_q(ptx), 1)  # Q 8 -> ceil(M / groups) rows per group (balanced)


@pytest.mark.parametrize("case", CASES)
def test_generated_fma_stream_is_the_csr(case):
    C, H, W, M, K, pad, d, tun = case
    rng = np.random.default_rng(C * 1000 + M)
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= d] = 0.0
    w[min(3, M - 1)] = 0.0  # an empty row
    csr = escoin.Csr.stretch(w, H, W, 1, pad)
    ptx = gen_ptx(csr, **tun)
    P = tun.get("P", 1) or 1
    Q = resolved_q(ptx) // P
    check_rows(csr, ptx, Q, P)


def test_config_layer_and_grouped_blocks():
    # AlexNet conv4 (g = 2, block-diagonal expansion): every group only runs its channel half
    L = [l for l in workloads.workload("alexnet").layers if l.name == "conv4"][0]
    w = inputs.layer_weights("alexnet", L, 800)
    csr = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad)
    ptx = gen_ptx(csr, n_hint=128, Q=32, warps=32, minb=1)
    check_rows(csr, ptx, 32, 1)


def test_generated_ptx_compiles_for_sm100a():
    L = workloads.TINY
    w = inputs.layer_weights("tiny", L, 800)
    csr = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad)
    for tun in [dict(), dict(mbarrier=1, NS=4), dict(Q=8, P=2, prefetch=-1), dict(Q=8, P=2), dict(Q=4, P=4, pair=1),
                dict(Q=8, pw=1), dict(Q=8, CC=4, ks=3), dict(Q=8, P=2, hp=1)]:
        n = ctypes.c_int64()
        assert _lib().escoin_internal_ptx_compile(gen_ptx(csr, n_hint=1, **tun).encode(), ctypes.byref(n)) == 0
        assert n.value > 0


def test_unsupported_shapes_have_no_specialised_form():
    w = np.ones((4, 3, 13, 13), np.float32)  # K > 11
    csr = escoin.Csr.stretch(w, 19, 19, 2, 1)
    n = ctypes.c_int64()
    arr = (ctypes.c_int * 8)()
    assert _lib().escoin_internal_jit_ptx(csr.handle, 4, arr, 8, None, 0, ctypes.byref(n)) == escoin.ERR_UNSUPPORTED


def unit_split(csr, n_hint=16, **tun):
    keys = ["Q", "P", "CC", "NS", "warps", "minb", "prefetch", "mbarrier", "units", "vec", "reorder"]
    tun.setdefault("reorder", -1)
    arr = (ctypes.c_int * 11)(*[tun.get(k, 0) for k in keys])
    L = _lib()
    L.escoin_internal_jit_units.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                            ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                            ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                            ctypes.c_int, ctypes.c_int]
    rng = (ctypes.c_int * 64)()
    cnt = ctypes.c_int()
    assert L.escoin_internal_jit_units(csr.handle, n_hint, arr, 11, rng, 64, ctypes.byref(cnt), None, 0, None,
                                       0, 0) == 0
    ranges = [(rng[2 * u], rng[2 * u + 1]) for u in range(cnt.value)]
    ptxs = []
    for lo, hi in ranges:
        n = ctypes.c_int64()
        assert L.escoin_internal_jit_units(csr.handle, n_hint, arr, 11, None, 0, ctypes.byref(cnt), None, 0,
                                           ctypes.byref(n), lo, hi) == 0
        buf = ctypes.create_string_buffer(n.value + 1)
        assert L.escoin_internal_jit_units(csr.handle, n_hint, arr, 11, None, 0, ctypes.byref(cnt), buf,
                                           n.value + 1, ctypes.byref(n), lo, hi) == 0
        ptxs.append(buf.value.decode())
    return ranges, ptxs


@pytest.mark.parametrize("units", [1, 2, 3, 5])
def test_units_partition_groups_and_union_is_the_csr(units):
    # escoin_csr_jit splits the m-groups into separately compiled units (compiled in parallel,
    # launched concurrently): the ranges must tile [0, groups) and the union of the units'
    # FFMA streams (local group + the unit's first group) must still be exactly the CSR
    rng = np.random.default_rng(77 + units)
    M, C, H, K = 70, 9, 11, 3
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    w[rng.random(w.shape) >= 0.3] = 0.0
    w[8:16] = 0.0  # an empty group
    csr = escoin.Csr.stretch(w, H, H, 1, 1)
    ranges, ptxs = unit_split(csr, Q=8, units=units)
    ngroups = -(-M // 8)
    assert ranges[0][0] == 0 and ranges[-1][1] == ngroups and len(ranges) == min(units, ngroups)
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:])) and all(lo < hi for lo, hi in ranges)
    stream = []
    for (lo, hi), ptx in zip(ranges, ptxs):
        assert ".global .align 8 .u32 mgr[%d]" % (2 * (hi - lo)) in ptx
        stream += [(g + lo, a, x, b) for g, a, x, b in fma_stream(ptx)]
    check_rows(csr, None, 8, 1, stream=stream)


def _default_units(wl, name):
    L = [l for l in workloads.workload(wl).layers if l.name == name][0]
    w = inputs.layer_weights(wl, L, 800)
    csr = escoin.Csr.stretch(w, L.H, L.W, L.stride, L.pad)
    unit_split(csr, n_hint=128, Q=32, warps=32, minb=1)  # sets argtypes
    keys = (ctypes.c_int * 9)(32, 1, 0, 0, 32, 1, 0, 0, 0)
    rng = (ctypes.c_int * 64)()
    cnt = ctypes.c_int()
    assert _lib().escoin_internal_jit_units(csr.handle, 128, keys, 9, rng, 64, ctypes.byref(cnt), None, 0, None,
                                            0, 0) == 0
    rowptr = csr.host_arrays()[0]
    return [int(rowptr[min(L.M, rng[2 * u + 1] * 32)] - rowptr[rng[2 * u] * 32]) for u in range(cnt.value)]


def test_default_unit_split():
    # one unit up to 500k nonzeros / 1536 chunk blocks (a linked unit runs 2-12% slower), contiguous
    # ranges of about equal work above that: ResNet-50 v1 res5 (472k nonzeros, 1024 blocks) is one
    # kernel; v1.5 res5a (stride 2: 4-channel chunks, 2048 blocks) splits
    assert len(_default_units("resnet50", "res5a_branch2b")) == 1
    nnz = _default_units("resnet50_v15", "res5a_branch2b")
    assert len(nnz) >= 2 and max(nnz) < 1.25 * (sum(nnz) / len(nnz))


@pytest.mark.parametrize("units", [1, 3])
def test_multi_unit_compile_and_link_on_host(units):
    # several units: each compiled relocatable (its own host thread), linked with the entry kernel
    # into ONE cubin by nvJitLink — all on the host, no device needed
    L_ = _lib()
    L_.escoin_internal_jit_cubin.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64),
                                             ctypes.c_char_p, ctypes.c_int64]
    rng = np.random.default_rng(5)
    w = rng.standard_normal((40, 8, 3, 3)).astype(np.float32)
    w[rng.random(w.shape) >= 0.3] = 0.0
    csr = escoin.Csr.stretch(w, 10, 10, 1, 1)
    arr = (ctypes.c_int * 9)(8, 1, 0, 0, 4, 2, 0, 0, units)
    u, nb = ctypes.c_int(), ctypes.c_int64()
    log = ctypes.create_string_buffer(4096)
    rc = L_.escoin_internal_jit_cubin(csr.handle, 4, arr, 9, ctypes.byref(u), ctypes.byref(nb), log, 4096)
    assert rc == 0, log.value.decode()
    assert u.value == units and nb.value > 0


def test_reordered_groups_fma_stream_and_epilogue():
    # reorder=1: output channels regrouped (LPT by nonzeros); the per-group epilogue stores accumulator
    # (g, q) at channel m (offset 4*m*E*F): decode that map from the PTX, then every channel's FFMA
    # stream must still be exactly its CSR row, and every channel must be stored exactly once
    rng = np.random.default_rng(9)
    M, C, H, K, Q = 40, 6, 9, 3, 8
    w = rng.standard_normal((M, C, K, K)).astype(np.float32)
    dens = rng.beta(1.0, 4.0, M)
    w[rng.random(w.shape) >= dens[:, None, None, None]] = 0.0
    csr = escoin.Csr.stretch(w, H, H, 1, 1)
    ptx = gen_ptx(csr, Q=Q, reorder=1)
    order, g = {}, None
    for line in ptx.splitlines():
        m = re.match(r"^EG(\d+):", line)
        if m:
            g, acc = int(m.group(1)), None
            continue
        m = re.search(r"add\.rn\.f32 %v1, %a(\d+), %v0;", line)
        if m and g is not None:
            acc = int(m.group(1))
            continue
        m = re.search(r"st\.global\.f32 \[%rd\d+\+(\d+)\], %v1;", line)
        if m and g is not None and acc is not None:
            order.setdefault((g, acc), int(m.group(1)) // (4 * H * H))
    assert sorted(order.values()) == list(range(M))
    assert order != {divmod(m, Q): m for m in range(M)}  # actually regrouped
    check_rows(csr, ptx, Q, 1, order=order)
    # groups hold about equal nonzeros after regrouping
    rowptr = csr.host_arrays()[0]
    loads = [sum(int(rowptr[m + 1] - rowptr[m]) for (gg, _), m in order.items() if gg == gi) for gi in range(M // Q)]
    assert max(loads) <= 1.1 * (sum(loads) / len(loads))
