"""CPU oracle for the Escoin direct sparse convolution (arXiv 1802.10280).

TEST INFRASTRUCTURE ONLY: importable by tests/, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``).  The product
package ``paper_1802_10280_b200`` never imports this module, and this module
imports nothing from the product package.

Everything here is a thin ctypes marshalling layer over ``escoin_oracle.c``
(plain C, fp64 accumulation, OpenMP over disjoint (n, m) pairs).  See the C
file for the paper passages each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "escoin_oracle.c")
_LIB = os.path.join(_HERE, "libescoin_oracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-fno-fast-math", "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
            f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
            f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
            i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
            ci, cl, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
            L.oracle_output_dim.argtypes = [ci, ci, ci, ci]
            L.oracle_output_dim.restype = ci
            L.oracle_layout_f.argtypes = [cl, cl, cl, cl, cl]
            L.oracle_layout_f.restype = cl
            L.oracle_num_threads.restype = ci
            L.oracle_set_threads.argtypes = [ci]
            L.oracle_set_threads.restype = None
            L.oracle_csr_stretch.argtypes = [f32p, ci, ci, ci, ci, ci, ci, ci, i32p, i32p, f32p, cl,
                                             ctypes.POINTER(cl)]
            L.oracle_csr_stretch.restype = ci
            L.oracle_pad_input.argtypes = [f32p, ci, ci, ci, ci, ci, f64p]
            L.oracle_sconv.argtypes = [ci] * 8 + [i32p, i32p, f32p, f32p, vp, ci, f64p, vp]
            L.oracle_sconv.restype = ci
            L.oracle_sconv_points.argtypes = [ci] * 8 + [i32p, i32p, f32p, f32p, vp, ci, i64p, cl, f64p, vp]
            L.oracle_sconv_points.restype = ci
            L.oracle_conv_dense.argtypes = [ci] * 8 + [f32p, f32p, vp, ci, f64p]
            L.oracle_conv_dense.restype = ci
            _lib = L
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return None if a is None else a.ctypes.data


def output_dim(H: int, K: int, stride: int, pad: int) -> int:
    return int(lib().oracle_output_dim(H, K, stride, pad))


def layout_f(c: int, y: int, x: int, Hin: int, Win: int) -> int:
    return int(lib().oracle_layout_f(c, y, x, Hin, Win))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's loops (timing only; results do not depend on it)."""
    lib().oracle_set_threads(int(n))


def csr_stretch(w: np.ndarray, H: int, W: int, stride: int, pad: int):
    """O-1: dense pruned weights [M][C][K][K] -> stretched (rowptr, colidx, value)."""
    w = _f32(w)
    M, C, K, K2 = w.shape
    assert K == K2
    cap = int(np.count_nonzero(w))
    rowptr = np.zeros(M + 1, np.int32)
    colidx = np.zeros(max(cap, 1), np.int32)
    value = np.zeros(max(cap, 1), np.float32)
    nnz = ctypes.c_int64(0)
    rc = lib().oracle_csr_stretch(w, M, C, H, W, K, stride, pad, rowptr, colidx, value, cap, ctypes.byref(nnz))
    if rc != 0:
        raise ValueError("oracle_csr_stretch failed (%d)" % rc)
    n = nnz.value
    return rowptr, colidx[:n].copy(), value[:n].copy()


def pad_input(x: np.ndarray, pad: int) -> np.ndarray:
    x = _f32(x)
    N, C, H, W = x.shape
    out = np.empty((N, C, H + 2 * pad, W + 2 * pad), np.float64)
    lib().oracle_pad_input(x, N, C, H, W, pad, out)
    return out


def sconv(x, rowptr, colidx, value, M, K, stride, pad, bias=None, relu=False, want_scale=True):
    """O-2: Alg.2 in fp64.  Returns (out, scale), both float64 [N][M][E][F]."""
    x = _f32(x)
    N, C, H, W = x.shape
    E, F = output_dim(H, K, stride, pad), output_dim(W, K, stride, pad)
    out = np.empty((N, M, E, F), np.float64)
    scale = np.empty((N, M, E, F), np.float64) if want_scale else None
    b = None if bias is None else _f32(bias)
    rc = lib().oracle_sconv(N, C, H, W, M, K, stride, pad,
                            np.ascontiguousarray(rowptr, np.int32), np.ascontiguousarray(colidx, np.int32),
                            _f32(value), x, _ptr(b), int(bool(relu)), out, _ptr(scale))
    if rc != 0:
        raise ValueError("oracle_sconv failed (%d)" % rc)
    return out, scale


def sconv_points(x, rowptr, colidx, value, M, K, stride, pad, coords, bias=None, relu=False):
    """O-2 at explicit output coordinates; coords int64 [npts][4] = (n, m, h, w)."""
    x = _f32(x)
    N, C, H, W = x.shape
    coords = np.ascontiguousarray(coords, np.int64).reshape(-1, 4)
    out = np.empty(coords.shape[0], np.float64)
    scale = np.empty(coords.shape[0], np.float64)
    b = None if bias is None else _f32(bias)
    rc = lib().oracle_sconv_points(N, C, H, W, M, K, stride, pad,
                                   np.ascontiguousarray(rowptr, np.int32), np.ascontiguousarray(colidx, np.int32),
                                   _f32(value), x, _ptr(b), int(bool(relu)), coords, coords.shape[0], out,
                                   _ptr(scale))
    if rc != 0:
        raise ValueError("oracle_sconv_points failed (%d)" % rc)
    return out, scale


def conv_dense(x, w, stride, pad, bias=None, relu=False):
    """O-3: Alg.1 7-loop brute force on the dense pruned weights (tiny shapes only)."""
    x, w = _f32(x), _f32(w)
    N, C, H, W = x.shape
    M, C2, K, _ = w.shape
    assert C2 == C
    E, F = output_dim(H, K, stride, pad), output_dim(W, K, stride, pad)
    out = np.empty((N, M, E, F), np.float64)
    b = None if bias is None else _f32(bias)
    rc = lib().oracle_conv_dense(N, C, H, W, M, K, stride, pad, w, x, _ptr(b), int(bool(relu)), out)
    if rc != 0:
        raise ValueError("oracle_conv_dense failed (%d)" % rc)
    return out
