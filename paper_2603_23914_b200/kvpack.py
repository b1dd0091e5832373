"""kvpack-compatible Python surface over the B200 C-ABI.

Mirrors the reference module's functions for this path (bindings/module.cpp:
129-238, re-exported by python/kvpack/__init__.py:8-34): same names, argument
meaning, defaults, return types and exception classes (the reference's
parameter/shape/data errors surface as ValueError, module.cpp:117-127).
Arrays are copied, never aliased (module.cpp:6, 29-47).  The factorisation,
the importance EMA and the tier assignment run on the GPU through
libkvp_b200.so; compression_ratio and partial_decompress_flops are the
reference's closed-form integer/f64 accounting and stay on the host.
quantize_roundtrip (the 4-bit groupwise store's round trip) runs on the GPU,
bit-identical to the reference.

Not mirrored (outside this path): run_simulation (the INI-driven
harness).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _capi as capi

__version__ = "0.1.0"

__all__ = [
    "__version__",
    "quantize_roundtrip",
    "assign_groups",
    "compression_ratio",
    "ema_update",
    "explained_variance_ratio",
    "partial_decompress_flops",
    "rank_for_variance",
    "singular_values",
    "truncated_svd",
]


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("kvpack (B200): a CUDA device is required; there is no CPU fallback")
    return torch


def _matrix(a, name="a"):
    m = np.asarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise ValueError(f"{name} must be 2-D")
    return np.ascontiguousarray(m)


def truncated_svd(a, rank, method="exact", seed=0, oversampling=8, power_iterations=2):
    """Rank-R factorisation (linalg.hpp:29-30): left T x R with the singular
    values folded in, right R x W with orthonormal rows.  `method` is "exact"
    or "randomized" (linalg.cpp:68-105: k = min(R + oversampling, min(T, W)),
    `power_iterations` re-orthonormalised power iterations, Philox sketch)."""
    m = _matrix(a)
    rows, cols = m.shape
    if rows == 0 or cols == 0:
        raise ValueError("truncated_svd: matrix must be non-empty")
    rank = int(rank)
    if rank < 1 or rank > min(rows, cols):
        raise ValueError("truncated_svd: rank must be in [1, min(rows, cols)]")
    if not np.all(np.isfinite(m)):
        raise ValueError("truncated_svd: matrix contains non-finite values")
    if method not in ("exact", "randomized"):
        raise ValueError(f"truncated_svd: unknown method '{method}'")
    if not np.any(m):  # linalg.cpp:51-58: zero left against coordinate rows
        right = np.zeros((rank, cols))
        right[np.arange(rank), np.arange(rank)] = 1.0
        return np.zeros((rows, rank)), right
    torch = _torch()
    dev = torch.as_tensor(m, dtype=torch.float32, device="cuda").contiguous()
    left = torch.empty((rows, rank), dtype=torch.float32, device="cuda")
    right = torch.empty((rank, cols), dtype=torch.float32, device="cuda")
    capi.call("kvp_truncated_svd", dev.data_ptr(), 1, rows, cols, rank, 0 if method == "exact" else 1, int(seed),
              int(oversampling), int(power_iterations), left.data_ptr(), right.data_ptr(), None, None)
    torch.cuda.synchronize()
    return left.cpu().numpy().astype(np.float64), right.cpu().numpy().astype(np.float64)


def singular_values(a):
    """All singular values, descending (linalg.cpp:119-128)."""
    m = _matrix(a)
    rows, cols = m.shape
    if rows == 0 or cols == 0:
        raise ValueError("singular_values: matrix must be non-empty")
    if not np.any(m):
        return np.zeros(min(rows, cols))
    torch = _torch()
    r = min(rows, cols)
    dev = torch.as_tensor(m, dtype=torch.float32, device="cuda").contiguous()
    left = torch.empty((rows, r), dtype=torch.float32, device="cuda")
    right = torch.empty((r, cols), dtype=torch.float32, device="cuda")
    sv = torch.empty((r,), dtype=torch.float32, device="cuda")
    capi.call("kvp_truncated_svd", dev.data_ptr(), 1, rows, cols, r, 0, 0, 0, 2, left.data_ptr(), right.data_ptr(),
              sv.data_ptr(), None)
    torch.cuda.synchronize()
    return sv.cpu().numpy().astype(np.float64)


def explained_variance_ratio(a, rank):
    """Fraction of the squared Frobenius mass in the top `rank` directions (linalg.cpp:130-142)."""
    m = _matrix(a)
    rank = int(rank)
    if rank > min(m.shape):
        raise ValueError("explained_variance_ratio: rank exceeds min(rows, cols)")
    s = singular_values(m)
    total = head = 0.0
    for i, v in enumerate(s):
        total += v * v
        if i < rank:
            head += v * v
    return 1.0 if total == 0.0 else head / total  # zero matrix: any rank explains everything


def rank_for_variance(a, target, max_rank):
    """Smallest rank reaching the explained-variance target, clamped to
    max_rank; returns (rank, achieved) (linalg.cpp:144-165)."""
    m = _matrix(a)
    target = float(target)
    if not (target > 0.0) or target > 1.0:
        raise ValueError("rank_for_variance: target must be in (0, 1]")
    max_rank = int(max_rank)
    if max_rank < 1:
        raise ValueError("rank_for_variance: max_rank must be >= 1")
    hard_cap = min(max_rank, min(m.shape))
    s = singular_values(m)
    total = 0.0
    for v in s:
        total += v * v
    if total == 0.0:
        return 1, 1.0
    head, rank, achieved = 0.0, 0, 0.0
    for r in range(1, hard_cap + 1):
        head += s[r - 1] * s[r - 1]
        rank, achieved = r, head / total
        if achieved >= target:
            break
    return rank, achieved  # target unreachable within max_rank: clamp, report achieved


def compression_ratio(tokens, width, rank):
    """Scalar-count ratio T*W / (T*R + R*W); rank 0 reports 1 (cache.cpp:221-229)."""
    tokens, width, rank = int(tokens), int(width), int(rank)
    if tokens == 0 or width == 0:
        raise ValueError("compression_ratio: token count and width must be positive")
    dense = float(tokens) * float(width)
    if rank == 0:
        return 1.0  # uncompressed storage
    return dense / (float(tokens) * float(rank) + float(rank) * float(width))


def partial_decompress_flops(tokens, width, ratios, ranks):
    """Closed-form tiered decompression cost llround(2*T*W*sum_f r_f R_f) and
    the reduction 1 - weighted/R_0 against the first tier's rank
    (importance.cpp:119-133); returns (flops, reduction)."""
    tokens, width = int(tokens), int(width)
    ratios = [float(r) for r in ratios]
    ranks = [int(r) for r in ranks]
    if not ratios or len(ratios) != len(ranks):
        raise ValueError("flops_partial_decompress: ratios and ranks must align")
    weighted = 0.0
    for r, k in zip(ratios, ranks):
        weighted += r * float(k)
    x = 2.0 * float(tokens) * float(width) * weighted
    flops = int(math.floor(x + 0.5))  # std::llround (non-negative)
    reduction = 0.0 if ranks[0] == 0 else 1.0 - weighted / float(ranks[0])
    return flops, reduction


def ema_update(scores, attn, alpha=0.25):
    """One EMA step: alpha^Tq * scores + (1 - alpha^Tq) * column means of the
    Tq x n head-averaged attention rows (importance.cpp:33-65), on the GPU."""
    s = np.asarray(scores, dtype=np.float64)
    if s.ndim != 1:
        raise ValueError("scores must be 1-D")
    rows = _matrix(attn, "attn")
    if rows.shape[1] != s.shape[0]:
        raise ValueError("ema_update: attention width must match the score count")
    torch = _torch()
    ds = torch.as_tensor(s, device="cuda").contiguous()
    da = torch.as_tensor(rows, device="cuda").contiguous()
    capi.call("kvp_update_importance", 1, int(s.shape[0]), ds.data_ptr(), int(rows.shape[0]), da.data_ptr(),
              float(alpha), 1, None)
    torch.cuda.synchronize()
    return ds.cpu().numpy()


def assign_groups(scores, ratios, ranks):
    """Token indices per tier by descending score, ties by position
    (importance.cpp:67-117); one ascending index list per tier, on the GPU."""
    s = np.asarray(scores, dtype=np.float64)
    if s.ndim != 1:
        raise ValueError("scores must be 1-D")
    ratios = np.asarray([float(r) for r in ratios], dtype=np.float64)
    ranks = np.asarray([int(r) for r in ranks], dtype=np.int32)
    if len(ratios) != len(ranks) or len(ratios) == 0:
        raise ValueError("assign_groups: ratios and ranks must be non-empty and of equal length")
    n = int(s.shape[0])
    if n == 0:
        return [[] for _ in ratios]
    torch = _torch()
    ds = torch.as_tensor(s, device="cuda").contiguous()
    tier = torch.empty((n,), dtype=torch.uint8, device="cuda")
    capi.call("kvp_assign_tiers", 1, n, ds.data_ptr(), n, len(ratios), ratios.ctypes.data_as(C.c_void_p),
              ranks.ctypes.data_as(C.c_void_p), ranks.ctypes.data_as(C.c_void_p), tier.data_ptr(), None, None, None)
    torch.cuda.synchronize()
    t = tier.cpu().numpy()
    return [np.flatnonzero(t == f).tolist() for f in range(len(ratios))]


def quantize_roundtrip(a, group_size=64):
    """4-bit groupwise quantize + dequantize (module.cpp:223-230, quantize.cpp:10-54):
    per column, groups of ``group_size`` rows share a min and a scale (max - min) / 15;
    per-element error <= (group max - group min) / 30.  Bit-identical to the reference."""
    m = _matrix(a)
    group_size = int(group_size)
    if group_size < 1:
        raise ValueError("quantize_4bit: group_size must be >= 1")
    if not np.all(np.isfinite(m)):
        raise ValueError("quantize_4bit: matrix contains non-finite values")
    rows, cols = m.shape
    if rows == 0 or cols == 0:
        return m.copy()
    torch = _torch()
    dev = torch.as_tensor(m, dtype=torch.float64, device="cuda").contiguous()
    out = torch.empty_like(dev)
    capi.call("kvp_quantize_roundtrip", dev.data_ptr(), rows, cols, group_size, out.data_ptr(), None)
    torch.cuda.synchronize()
    return out.cpu().numpy()
