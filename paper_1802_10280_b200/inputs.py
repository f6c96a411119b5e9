"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no CSR, no stretching, no
convolution).  It only draws numbers: activations, He-initialised weights,
biases, and the magnitude pruning that turns dense random weights into the
"pruned model" the paper takes as given (P:290-297, P:576-579 — the paper
uses externally pruned SkimCaffe models; we substitute deterministic
magnitude pruning, SURVEY §8(c) reading R#13).

Generator: counter-based splitmix64.  Element i
of a stream with 64-bit key k is ``mix(k + GAMMA*(i+1))`` — the i-th output
of a splitmix64 seeded with k.  Keys are derived by folding string/int parts
(seed, net, layer, tensor kind, GLOBAL image index) through the same mixer,
so image n's activations are identical whatever the batch size or the shard
it lands in.

Value distributions:
  activations  U[0,1)                       fp32 = (u >> 40) * 2^-24 (exact)
  weights      N(0, 2/(C/g*K*K)) (He)       Box-Muller in fp64 -> fp32
  bias         U[-0.1, 0.1)                 fp32
  exact regime weights/bias integers in [-3,3], activations integers in [0,3]
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
DEFAULT_SEED = 42


def _mix(z):
    """splitmix64 finaliser on uint64 scalars/arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(z, dtype=np.uint64)
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def _fnv1a(s: str) -> np.uint64:
    h = 0xCBF29CE484222325
    for b in s.encode("utf-8"):
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return np.uint64(h)


def key(*parts) -> np.uint64:
    """Fold parts (str or int) into a 64-bit stream key."""
    k = _mix(np.uint64(DEFAULT_SEED))
    for p in parts:
        v = _fnv1a(p) if isinstance(p, str) else np.uint64(int(p) & 0xFFFFFFFFFFFFFFFF)
        with np.errstate(over="ignore"):
            k = _mix(k ^ v ^ GAMMA)
    return np.uint64(k)


def stream_u64(k, count: int, keys_axis=None) -> np.ndarray:
    """u64 stream(s).  k scalar -> shape [count]; k array [B] -> shape [B, count]."""
    i = np.arange(1, count + 1, dtype=np.uint64)
    k = np.asarray(k, dtype=np.uint64)
    with np.errstate(over="ignore"):
        if k.ndim == 0:
            return _mix(k + GAMMA * i)
        return _mix(k[:, None] + GAMMA * i[None, :])


def u01(u: np.ndarray) -> np.ndarray:
    """uniform fp32 in [0,1): top 24 bits, exactly representable."""
    return ((u >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)).astype(np.float32)


def normal(k, count: int) -> np.ndarray:
    """Standard normals via Box-Muller (fp64) from two sub-streams of k."""
    a = stream_u64(key(int(k), "bm-r"), count)
    b = stream_u64(key(int(k), "bm-t"), count)
    r1 = ((a >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)  # (0, 1]
    t = (b >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)           # [0, 1)
    return np.sqrt(-2.0 * np.log(r1)) * np.cos(2.0 * np.pi * t)


# ---------------------------------------------------------------- tensors
def activations(net: str, layer: str, n0: int, n: int, C: int, H: int, W: int,
                kind: str = "x", exact: bool = False) -> np.ndarray:
    """Images [n0, n0+n) of a layer's input, fp32 NCHW; keyed by GLOBAL image index."""
    keys = np.array([key(net, layer, kind, g) for g in range(n0, n0 + n)], dtype=np.uint64)
    u = stream_u64(keys, C * H * W) if n > 0 else np.zeros((0, C * H * W), np.uint64)
    if exact:
        x = np.floor(u01(u).astype(np.float64) * 4.0).astype(np.float32)
    else:
        x = u01(u)
    return x.reshape(n, C, H, W)


def weights(net: str, layer: str, M: int, Cg: int, K: int, exact: bool = False) -> np.ndarray:
    """Dense (unpruned) grouped weights [M][C/g][K][K] fp32, He normal (or small ints)."""
    T = M * Cg * K * K
    k = key(net, layer, "w")
    if exact:
        w = np.floor(u01(stream_u64(k, T)).astype(np.float64) * 7.0) - 3.0
        return w.astype(np.float32).reshape(M, Cg, K, K)
    std = np.sqrt(2.0 / (Cg * K * K))
    return (normal(k, T) * std).astype(np.float32).reshape(M, Cg, K, K)


def bias(net: str, layer: str, M: int, exact: bool = False) -> np.ndarray:
    u = u01(stream_u64(key(net, layer, "b"), M))
    if exact:
        return (np.floor(u.astype(np.float64) * 7.0) - 3.0).astype(np.float32)
    return (u.astype(np.float64) * 0.2 - 0.1).astype(np.float32)


def prune_by_magnitude(w: np.ndarray, sparsity_permille: int) -> np.ndarray:
    """Zero the floor(s*T) smallest-|w| entries (reading R#13).

    s is given in per-mille so the zero count is exact integer arithmetic.
    Ties at the cut: lower flat index pruned first (stable sort on |w|).
    """
    assert 0 <= sparsity_permille <= 1000
    flat = np.array(w, dtype=np.float32, copy=True).reshape(-1)
    zeros = (int(sparsity_permille) * flat.size) // 1000
    order = np.argsort(np.abs(flat), kind="stable")
    flat[order[:zeros]] = 0.0
    return flat.reshape(w.shape)


def expand_groups(wg: np.ndarray, groups: int) -> np.ndarray:
    """Grouped weights [M][C/g][K][K] -> block-diagonal dense [M][C][K][K] (reading R#18)."""
    M, Cg, K, _ = wg.shape
    if groups == 1:
        return np.ascontiguousarray(wg)
    out = np.zeros((M, Cg * groups, K, K), np.float32)
    Mg = M // groups
    for g in range(groups):
        out[g * Mg:(g + 1) * Mg, g * Cg:(g + 1) * Cg] = wg[g * Mg:(g + 1) * Mg]
    return out


def layer_weights(net: str, layer, sparsity_permille: int, exact: bool = False) -> np.ndarray:
    """Pruned, group-expanded dense weights [M][C][K][K] for a workloads.Layer."""
    wg = weights(net, layer.name, layer.M, layer.C // layer.groups, layer.K, exact=exact)
    return expand_groups(prune_by_magnitude(wg, sparsity_permille), layer.groups)


def skewed_row_density(net: str, layer: str, M: int, mean_density: float) -> np.ndarray:
    """Per-output-channel densities d_m ~ Beta(1, b) with mean 1/(1+b) = mean_density (SURVEY §8(d),
    the optional "skewed" variant for load balance): inverse CDF d = 1 - (1-u)^(1/b), so most rows
    are sparser than the mean and a few are much denser."""
    assert 0.0 < mean_density < 1.0
    b = 1.0 / mean_density - 1.0
    u = u01(stream_u64(key(net, layer, "skew"), M)).astype(np.float64)
    return 1.0 - np.power(1.0 - u, 1.0 / b)


def prune_rows_by_magnitude(w: np.ndarray, density: np.ndarray) -> np.ndarray:
    """Row m keeps its round(d_m * T_row) largest-|w| entries (ties: lower index pruned first)."""
    out = np.array(w, dtype=np.float32, copy=True).reshape(w.shape[0], -1)
    T = out.shape[1]
    for m in range(out.shape[0]):
        zeros = T - int(round(float(density[m]) * T))
        order = np.argsort(np.abs(out[m]), kind="stable")
        out[m, order[:zeros]] = 0.0
    return out.reshape(w.shape)


def layer_weights_skewed(net: str, layer, sparsity_permille: int) -> np.ndarray:
    """As layer_weights, but with per-row densities drawn from Beta(1, b) (mean 1 - sparsity)."""
    wg = weights(net, layer.name, layer.M, layer.C // layer.groups, layer.K)
    d = skewed_row_density(net, layer.name, layer.M, 1.0 - sparsity_permille / 1000.0)
    return expand_groups(prune_rows_by_magnitude(wg, d), layer.groups)
