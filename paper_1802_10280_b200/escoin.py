"""Thin ctypes binding of libescoin.so (include/escoin.h) — marshalling only.

Every step of the method runs inside the library: the stretch on the host
in C++, the convolution in the sm_100a kernels.  This module converts Python
objects to pointers and status codes to exceptions.  There is no fallback:
if the library is missing or a call fails, an EscoinError is raised.

torch is used by callers only for device memory and streams; the functions
here accept raw integer pointers, and ``forward()`` accepts torch tensors for
convenience (their ``data_ptr()`` is passed through).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ESCOIN_LIB", os.path.join(_HERE, "libescoin.so"))

OK = 0
ERR_NULL, ERR_SHAPE, ERR_CSR_MISMATCH, ERR_NOT_ON_DEVICE = -1, -2, -3, -4
ERR_OVERFLOW, ERR_UNSUPPORTED, ERR_ALLOC, ERR_CUDA = -5, -6, -7, -8
KERNEL_AUTO = -1
KERNEL_JIT = 1000  # the handle's pattern-specialised kernel (escoin_csr_jit)

# Every symbol include/escoin.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "escoin_csr_stretch", "escoin_csr_info", "escoin_csr_host_arrays", "escoin_csr_to_device",
    "escoin_csr_wrap_device", "escoin_csr_free", "escoin_sconv_forward", "escoin_sconv_forward_hostio",
    "escoin_kernel_count", "escoin_kernel_info", "escoin_csr_set_kernel", "escoin_csr_get_kernel",
    "escoin_status_string", "escoin_version", "escoin_csr_autotune", "escoin_csr_stretch_device",
    "escoin_bench_dense_tc_forward", "escoin_csr_jit", "escoin_csr_jit_info", "escoin_csr_autotune_ex",
    "escoin_csr_kernel_label", "escoin_csr_jit_stats", "escoin_sparse_threshold", "escoin_select_engine",
    "escoin_csr_select_engine",
]
TUNE_VARIANTS, TUNE_JIT = 1, 2
ENGINE_SPARSE, ENGINE_DENSE_TC = 0, 1
KERNEL_DENSE_TC = 2000


class EscoinError(RuntimeError):
    def __init__(self, fn, status):
        self.status = status
        msg = _lib.escoin_status_string(status).decode() if _lib is not None else str(status)
        super().__init__("%s failed: %s (%d)" % (fn, msg, status))


_lock = threading.Lock()
_lib = None


def lib():
    """Load libescoin.so (fails loudly if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    "libescoin.so not found at %s — run __graft_entry__.build() / "
                    "python paper_1802_10280_b200/build.py" % LIB_PATH)
            L = ctypes.CDLL(LIB_PATH)
            ci, cl, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
            pp = ctypes.POINTER(ctypes.c_void_p)
            ip = ctypes.POINTER(ctypes.c_int)
            L.escoin_csr_stretch.argtypes = [vp, ci, ci, ci, ci, ci, ci, ci, pp]
            L.escoin_csr_stretch_device.argtypes = [vp, ci, ci, ci, ci, ci, ci, ci, ci, vp, pp]
            L.escoin_csr_info.argtypes = [vp, ip, ip, ip, ip, ip, ip, ip, ctypes.POINTER(cl)]
            L.escoin_csr_host_arrays.argtypes = [vp, pp, pp, pp]
            L.escoin_csr_to_device.argtypes = [vp, ci, vp]
            L.escoin_csr_wrap_device.argtypes = [vp, vp, vp, cl, ci, ci, ci, ci, ci, ci, ci, ci, vp, pp]
            L.escoin_csr_free.argtypes = [vp]
            L.escoin_csr_free.restype = None
            L.escoin_sconv_forward.argtypes = [ci] * 8 + [vp, vp, vp, vp, ci, vp]
            L.escoin_sconv_forward_hostio.argtypes = [ci] * 8 + [vp, vp, vp, vp, vp, vp, ci, vp]
            L.escoin_kernel_count.argtypes = []
            L.escoin_kernel_info.argtypes = [ci, ctypes.POINTER(ctypes.c_char_p), ip, ip]
            L.escoin_csr_set_kernel.argtypes = [vp, ci]
            L.escoin_csr_get_kernel.argtypes = [vp, ip]
            L.escoin_csr_autotune.argtypes = [vp, ci, vp, vp, vp, ci, ci, vp, ip, ctypes.POINTER(ctypes.c_float)]
            L.escoin_bench_dense_tc_forward.argtypes = [ci] * 8 + [vp, vp, vp, vp, ci, ci, vp]
            L.escoin_csr_jit.argtypes = [vp, ci, ip, ci]
            L.escoin_csr_jit_info.argtypes = [vp, ip, ip, ip, ctypes.POINTER(cl)]
            L.escoin_csr_autotune_ex.argtypes = [vp, ci, vp, vp, vp, ci, ci, vp, vp, cl, ci, ip,
                                                 ctypes.POINTER(ctypes.c_float)]
            L.escoin_csr_kernel_label.argtypes = [vp, ctypes.c_char_p, ci]
            L.escoin_csr_jit_stats.argtypes = [vp, ip, ip, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(cl)]
            L.escoin_sparse_threshold.argtypes = []
            L.escoin_sparse_threshold.restype = ctypes.c_double
            L.escoin_select_engine.argtypes = [ci, ci, ci, cl, ctypes.c_double]
            L.escoin_csr_select_engine.argtypes = [vp, ctypes.c_double, ip]
            L.escoin_status_string.argtypes = [ci]
            L.escoin_status_string.restype = ctypes.c_char_p
            L.escoin_version.restype = ctypes.c_char_p
            for name in EXPORTS:
                if name not in ("escoin_csr_free", "escoin_status_string", "escoin_version",
                                "escoin_sparse_threshold"):
                    getattr(L, name).restype = ci
            _lib = L
    return _lib


def _check(fn, status):
    if status != OK:
        raise EscoinError(fn, status)


def version() -> str:
    return lib().escoin_version().decode()


def kernels():
    """[(id, name, K, stride)] of the compiled sconv variants (K = stride = 0: any)."""
    L = lib()
    out = []
    for i in range(L.escoin_kernel_count()):
        name, K, S = ctypes.c_char_p(), ctypes.c_int(), ctypes.c_int()
        _check("escoin_kernel_info", L.escoin_kernel_info(i, ctypes.byref(name), ctypes.byref(K), ctypes.byref(S)))
        out.append((i, name.value.decode(), K.value, S.value))
    return out


def sparse_threshold() -> float:
    """The active sparse/dense threshold (ESCOIN_SPARSE_THRESHOLD or the library default)."""
    return float(lib().escoin_sparse_threshold())


def select_engine(M, C, K, nnz, threshold=-1.0) -> int:
    """escoin_select_engine: ENGINE_SPARSE if sparsity >= threshold (default: the active one)."""
    r = lib().escoin_select_engine(M, C, K, nnz, threshold)
    if r < 0:
        raise EscoinError("escoin_select_engine", r)
    return r


def kernel_name(kernel_id: int) -> str:
    """Name of a kernel id as returned by Csr.kernel() (variants, or "jit" for KERNEL_JIT)."""
    if kernel_id == KERNEL_JIT:
        return "jit"
    if kernel_id == KERNEL_DENSE_TC:
        return "dense_tc"
    return kernels()[kernel_id][1]


class Csr:
    """Owning wrapper of an escoin_csr* handle (one pruned, stretched layer)."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)

    @classmethod
    def stretch(cls, w: np.ndarray, H: int, W: int, stride: int, pad: int) -> "Csr":
        """escoin_csr_stretch on dense pruned weights [M][C][K][K] (host fp32)."""
        w = np.ascontiguousarray(w, dtype=np.float32)
        M, C, K, K2 = w.shape
        assert K == K2, "square filters only"
        h = ctypes.c_void_p()
        _check("escoin_csr_stretch", lib().escoin_csr_stretch(w.ctypes.data, M, C, H, W, K, stride, pad,
                                                              ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def stretch_device(cls, d_w, M, C, H, W, K, stride, pad, device=0, stream=0) -> "Csr":
        """escoin_csr_stretch_device on dense pruned weights already on the GPU (pointer or torch tensor)."""
        h = ctypes.c_void_p()
        _check("escoin_csr_stretch_device", lib().escoin_csr_stretch_device(
            _ptr(d_w), M, C, H, W, K, stride, pad, device, stream, ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def wrap_device(cls, d_rowptr: int, d_colidx: int, d_value: int, nnz: int, M, C, H, W, K, stride, pad,
                    device: int, stream: int = 0) -> "Csr":
        h = ctypes.c_void_p()
        _check("escoin_csr_wrap_device", lib().escoin_csr_wrap_device(
            d_rowptr, d_colidx, d_value, nnz, M, C, H, W, K, stride, pad, device, stream, ctypes.byref(h)))
        return cls(h.value)

    @property
    def handle(self) -> int:
        return self._h.value

    def info(self):
        v = [ctypes.c_int() for _ in range(7)]
        nnz = ctypes.c_int64()
        _check("escoin_csr_info", lib().escoin_csr_info(self._h, *[ctypes.byref(x) for x in v], ctypes.byref(nnz)))
        M, C, H, W, K, S, P = (x.value for x in v)
        return dict(M=M, C=C, H=H, W=W, K=K, stride=S, pad=P, nnz=nnz.value)

    def host_arrays(self):
        """Copies of (rowptr int32[M+1], colidx int32[nnz], value fp32[nnz])."""
        info = self.info()
        r, c, v = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _check("escoin_csr_host_arrays", lib().escoin_csr_host_arrays(self._h, ctypes.byref(r), ctypes.byref(c),
                                                                      ctypes.byref(v)))
        M, nnz = info["M"], info["nnz"]
        rowptr = np.ctypeslib.as_array(ctypes.cast(r, ctypes.POINTER(ctypes.c_int32)), (M + 1,)).copy()
        if nnz == 0:
            return rowptr, np.zeros(0, np.int32), np.zeros(0, np.float32)
        colidx = np.ctypeslib.as_array(ctypes.cast(c, ctypes.POINTER(ctypes.c_int32)), (nnz,)).copy()
        value = np.ctypeslib.as_array(ctypes.cast(v, ctypes.POINTER(ctypes.c_float)), (nnz,)).copy()
        return rowptr, colidx, value

    def to_device(self, device: int = 0, stream: int = 0) -> "Csr":
        _check("escoin_csr_to_device", lib().escoin_csr_to_device(self._h, device, stream))
        return self

    def set_kernel(self, kernel_id: int) -> "Csr":
        _check("escoin_csr_set_kernel", lib().escoin_csr_set_kernel(self._h, kernel_id))
        return self

    def kernel(self) -> int:
        k = ctypes.c_int()
        _check("escoin_csr_get_kernel", lib().escoin_csr_get_kernel(self._h, ctypes.byref(k)))
        return k.value

    def autotune(self, N, inp, out, bias=None, relu=False, reps=3, stream=0):
        """escoin_csr_autotune: time every applicable variant on these buffers, keep the fastest."""
        bid, bms = ctypes.c_int(), ctypes.c_float()
        _check("escoin_csr_autotune", lib().escoin_csr_autotune(self._h, N, _ptr(inp), _ptr(out), _ptr(bias),
                                                                1 if relu else 0, reps, stream, ctypes.byref(bid),
                                                                ctypes.byref(bms)))
        return bid.value, bms.value

    def autotune_ex(self, N, inp, out, bias=None, relu=False, reps=3, stream=0, flush=None,
                    flags=TUNE_VARIANTS | TUNE_JIT):
        """escoin_csr_autotune_ex: as autotune, timing each rep alone after an L2 flush (memset of `flush`,
        a device tensor or None), median of reps; flags choose the candidate sets."""
        bid, bms = ctypes.c_int(), ctypes.c_float()
        nbytes = 0 if flush is None else flush.numel() * flush.element_size()
        _check("escoin_csr_autotune_ex", lib().escoin_csr_autotune_ex(
            self._h, N, _ptr(inp), _ptr(out), _ptr(bias), 1 if relu else 0, reps, stream, _ptr(flush), nbytes, flags,
            ctypes.byref(bid), ctypes.byref(bms)))
        return bid.value, bms.value

    def select_engine(self, threshold=-1.0) -> int:
        """escoin_csr_select_engine: apply the sparse/dense rule to this handle (on its device)."""
        e = ctypes.c_int()
        _check("escoin_csr_select_engine", lib().escoin_csr_select_engine(self._h, threshold, ctypes.byref(e)))
        return e.value

    def label(self) -> str:
        """escoin_csr_kernel_label: the current kernel with every tunable."""
        buf = ctypes.create_string_buffer(256)
        _check("escoin_csr_kernel_label", lib().escoin_csr_kernel_label(self._h, buf, 256))
        return buf.value.decode()

    def jit(self, n_hint=128, Q=0, P=0, CC=0, NS=0, warps=0, minb=0, prefetch=0, mbarrier=0, units=0,
            vec=0, reorder=0, sws=0, perm=0, split=0, pair=0, hp=0, pw=0, ks=0) -> "Csr":
        """escoin_csr_jit: compile this layer's pattern-specialised kernel and select it."""
        tun = (ctypes.c_int * 18)(Q, P, CC, NS, warps, minb, prefetch, mbarrier, units, vec, reorder, sws, perm,
                                  split, pair, hp, pw, ks)
        _check("escoin_csr_jit", lib().escoin_csr_jit(self._h, n_hint, tun, 18))
        return self

    def jit_info(self):
        """dict(Q, P, CC, NS, warps, minb, units, regs, code_bytes) of the specialised kernel."""
        tun = (ctypes.c_int * 6)()
        units, regs, code = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        _check("escoin_csr_jit_info", lib().escoin_csr_jit_info(self._h, tun, ctypes.byref(units),
                                                                ctypes.byref(regs), ctypes.byref(code)))
        d = dict(zip(["Q", "P", "CC", "NS", "warps", "minb"], list(tun)))
        d.update(units=units.value, regs=regs.value, code_bytes=code.value)
        return d

    def jit_stats(self):
        """dict(units, cache_hits, compile_s, ptx_bytes) of the selected specialised kernel's build."""
        u, hits, sec, ptx = ctypes.c_int(), ctypes.c_int(), ctypes.c_double(), ctypes.c_int64()
        _check("escoin_csr_jit_stats", lib().escoin_csr_jit_stats(self._h, ctypes.byref(u), ctypes.byref(hits),
                                                                  ctypes.byref(sec), ctypes.byref(ptx)))
        return dict(units=u.value, cache_hits=hits.value, compile_s=sec.value, ptx_bytes=ptx.value)

    def free(self):
        if self._h.value:
            lib().escoin_csr_free(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def sconv_forward(N, C, H, W, M, K, stride, pad, csr: Csr, inp, out, bias=None, relu=False, stream=0):
    """escoin_sconv_forward.  inp/out/bias: device pointers (int) or torch CUDA tensors."""
    _check("escoin_sconv_forward", lib().escoin_sconv_forward(
        N, C, H, W, M, K, stride, pad, csr.handle, _ptr(inp), _ptr(out), _ptr(bias), 1 if relu else 0, stream))


def sconv_forward_hostio(N, C, H, W, M, K, stride, pad, csr: Csr, h_in, h_out, d_in, d_out, bias=None,
                         relu=False, stream=0):
    """escoin_sconv_forward_hostio: host in/out (pinned for async), device scratch d_in/d_out."""
    _check("escoin_sconv_forward_hostio", lib().escoin_sconv_forward_hostio(
        N, C, H, W, M, K, stride, pad, csr.handle, _ptr(h_in), _ptr(h_out), _ptr(d_in), _ptr(d_out), _ptr(bias),
        1 if relu else 0, stream))


def bench_dense_tc_forward(w, x, bias=None, stride=1, pad=0, relu=False, nsplit=3, out=None, stream=None):
    """escoin_bench_dense_tc_forward — the dense tcgen05 comparison point (NOT the method).
    w: torch CUDA fp32 [M][C][K][K] dense pruned weights; x: [N][C][H][W]."""
    import torch
    M, C, K, _ = w.shape
    N, _, H, W = x.shape
    E, F = out_dims(H, W, K, stride, pad)
    if out is None:
        out = torch.empty((N, M, E, F), dtype=torch.float32, device=x.device)
    s = (stream if stream is not None else torch.cuda.current_stream(x.device)).cuda_stream
    _check("escoin_bench_dense_tc_forward", lib().escoin_bench_dense_tc_forward(
        N, C, H, W, M, K, stride, pad, _ptr(w), _ptr(x), _ptr(out), _ptr(bias), 1 if relu else 0, nsplit, s))
    return out


def out_dims(H, W, K, stride, pad):
    return (H + 2 * pad - K) // stride + 1, (W + 2 * pad - K) // stride + 1


def forward(csr: Csr, x, bias=None, relu=False, out=None, stream=None):
    """Convenience: x torch CUDA tensor [N][C][H][W] fp32 -> out [N][M][E][F]."""
    import torch
    info = csr.info()
    N, C, H, W = x.shape
    E, F = out_dims(H, W, info["K"], info["stride"], info["pad"])
    if out is None:
        out = torch.empty((N, info["M"], E, F), dtype=torch.float32, device=x.device)
    s = (stream if stream is not None else torch.cuda.current_stream(x.device)).cuda_stream
    sconv_forward(N, C, H, W, info["M"], info["K"], info["stride"], info["pad"], csr, x, out, bias, relu, s)
    return out
