"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes driver for ``oracle/_ref/libkvpack_ref.so`` — the reference's own C++
sources (``/root/reference/proj/src/*.cpp``, compiled unmodified by
``oracle/Makefile``) plus the Eigen-free linalg restatement
(``oracle/linalg_lapack.cpp``).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
module; the product package never does.

All matrices cross as float64 numpy arrays (the reference's pybind11 module
does the same, bindings/module.cpp:29-47); ``dtype`` selects the engine
precision T of the reference templates: "f64" -> double, "f32" -> float.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_ref" / "libkvpack_ref.so"

_lib = None


class RefError(RuntimeError):
    """Raised with the reference's exception text; ``code`` mirrors kvp_status."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class PlanEntry(C.Structure):
    _fields_ = [
        ("segment", C.c_int32),
        ("block", C.c_int32),
        ("row", C.c_uint32),
        ("rank_k", C.c_uint32),
        ("rank_v", C.c_uint32),
        ("pad", C.c_uint32),
        ("position", C.c_uint64),
    ]


class StepReport(C.Structure):
    _fields_ = [
        ("step", C.c_uint64),
        ("bytes_before", C.c_uint64),
        ("bytes_after", C.c_uint64),
        ("importance_bytes", C.c_uint64),
        ("decompress_flops", C.c_uint64),
        ("decompress_flops_full", C.c_uint64),
        ("flops_reduction", C.c_double),
        ("compression_event", C.c_int32),
        ("n_warnings", C.c_int32),
    ]


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(
                f"{LIB_PATH} missing: run `make -C oracle` (needs /root/reference)")
        _lib = C.CDLL(str(LIB_PATH))
        _lib.kvref_last_error.restype = C.c_char_p
        _lib.kvref_cache_new.restype = C.c_void_p
        _lib.kvref_cache_new.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t]
        _lib.kvref_cache_free.argtypes = [C.c_void_p]
        _lib.kvref_save_cache.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
        _lib.kvref_load_cache.argtypes = [C.c_int, C.c_char_p, C.POINTER(C.c_void_p)]
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, lib().kvref_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ini(decode_ini: str | None) -> bytes:
    return (decode_ini or "").encode()


class RefCache:
    """A reference ``LayerCache<T>`` (cache.hpp:120-146) owned by the oracle lib."""

    def __init__(self, heads, kv_heads, head_dim, dtype="f64", layer=0):
        self.H, self.Hkv, self.D = heads, kv_heads, head_dim
        self.W = kv_heads * head_dim
        self.HD = heads * head_dim
        self.dtype = dtype
        self._h = lib().kvref_cache_new(1 if dtype == "f32" else 0, heads, kv_heads, head_dim, layer)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().kvref_cache_free(C.c_void_p(self._h))
            self._h = None

    def save(self, path: str, width: int = 8):
        """save_cache (snapshot.cpp:251-307)."""
        _check(lib().kvref_save_cache(C.c_void_p(self._h), path.encode(), width))

    @classmethod
    def load(cls, path: str, heads, kv_heads, head_dim, dtype="f64"):
        """load_cache (snapshot.cpp:309-371)."""
        h = C.c_void_p()
        _check(lib().kvref_load_cache(1 if dtype == "f32" else 0, path.encode(), C.byref(h)))
        obj = cls.__new__(cls)
        obj.H, obj.Hkv, obj.D = heads, kv_heads, head_dim
        obj.W, obj.HD, obj.dtype = kv_heads * head_dim, heads * head_dim, dtype
        obj._h = h.value
        return obj

    def append(self, modality: int, k, v):
        k, v = _f64(k), _f64(v)
        _check(lib().kvref_append(C.c_void_p(self._h), modality, C.c_size_t(k.shape[0]), _dp(k), _dp(v)))

    def compress_now(self, decode_ini=None):
        _check(lib().kvref_compress_now(C.c_void_p(self._h), _ini(decode_ini)))

    def factor_tail(self, modality, k_factors, v_factors):
        """Install (left, right) factors (or None = dense) as the segment's joint
        block in place of its tail (kvref_factor_tail)."""
        args = []
        for fac in (k_factors, v_factors):
            if fac is None:
                args += [C.c_size_t(0), None, None]
            else:
                left, right = _f64(fac[0]), _f64(fac[1])
                args += [C.c_size_t(left.shape[1]), _dp(left), _dp(right)]
                self._keep = getattr(self, "_keep", []) + [left, right]
        _check(lib().kvref_factor_tail(C.c_void_p(self._h), modality, *args))
        self._keep = []

    def decode_step(self, x, wq, wk, wv, wo, decode_ini=None):
        x = _f64(np.atleast_2d(x))
        out = np.zeros((x.shape[0], self.HD))
        rep = StepReport()
        ws = [_f64(w) for w in (wq, wk, wv, wo)]
        _check(lib().kvref_decode_step(C.c_void_p(self._h), _ini(decode_ini), C.c_size_t(x.shape[0]),
                                       _dp(x), *[_dp(w) for w in ws], _dp(out), C.byref(rep)))
        return out, rep

    def plan_size(self, decode_ini=None) -> int:
        n = C.c_size_t()
        _check(lib().kvref_plan_size(C.c_void_p(self._h), _ini(decode_ini), C.byref(n)))
        return n.value

    def attend(self, queries, qpos, decode_ini=None, fused=False, tile=64):
        q = _f64(np.atleast_2d(queries))
        tq = q.shape[0]
        qp = np.ascontiguousarray(qpos, dtype=np.uint64)
        n = self.plan_size(decode_ini)
        ctx = np.zeros((tq, self.HD))
        ha = np.zeros((tq, n))
        ents = (PlanEntry * n)()
        _check(lib().kvref_attend(C.c_void_p(self._h), _ini(decode_ini), C.c_size_t(tq), _dp(q), _u64p(qp),
                                  int(fused), C.c_size_t(tile), _dp(ctx), _dp(ha), ents))
        plan = np.array([(e.segment, e.block, e.row, e.rank_k, e.rank_v, e.position) for e in ents],
                        dtype=np.int64).reshape(n, 6)
        return ctx, ha, plan

    def importance(self):
        n = C.c_size_t()
        _check(lib().kvref_importance_size(C.c_void_p(self._h), C.byref(n)))
        pos = np.zeros(n.value, dtype=np.uint64)
        sc = np.zeros(n.value)
        _check(lib().kvref_importance_get(C.c_void_p(self._h), _u64p(pos), _dp(sc)))
        return pos, sc

    def set_importance(self, scores):
        s = _f64(scores)
        _check(lib().kvref_importance_set(C.c_void_p(self._h), _dp(s)))

    def segment_info(self, modality):
        nb, tl, nxt = C.c_size_t(), C.c_size_t(), C.c_uint64()
        _check(lib().kvref_segment_info(C.c_void_p(self._h), modality, C.byref(nb), C.byref(tl), C.byref(nxt)))
        return nb.value, tl.value, nxt.value

    def block(self, modality, block, kind):
        """Returns ("lowrank", left, right, positions) or ("dense", rows, None, positions)."""
        t, r, w = C.c_size_t(), C.c_size_t(), C.c_size_t()
        _check(lib().kvref_block_info(C.c_void_p(self._h), modality, C.c_size_t(block), kind,
                                      C.byref(t), C.byref(r), C.byref(w)))
        t, r, w = t.value, r.value, w.value
        pos = np.zeros(t, dtype=np.uint64)
        if r == 0:
            rows = np.zeros((t, w))
            _check(lib().kvref_block_get(C.c_void_p(self._h), modality, C.c_size_t(block), kind,
                                         _dp(rows), None, _u64p(pos)))
            return "dense", rows, None, pos
        left, right = np.zeros((t, r)), np.zeros((r, w))
        _check(lib().kvref_block_get(C.c_void_p(self._h), modality, C.c_size_t(block), kind,
                                     _dp(left), _dp(right), _u64p(pos)))
        return "lowrank", left, right, pos

    def tail(self, modality):
        _, tl, _ = self.segment_info(modality)
        k, v = np.zeros((tl, self.W)), np.zeros((tl, self.W))
        pos = np.zeros(tl, dtype=np.uint64)
        _check(lib().kvref_tail_get(C.c_void_p(self._h), modality, _dp(k), _dp(v), _u64p(pos)))
        return k, v, pos


def truncated_svd(a, rank, method="exact", seed=0, oversampling=8, power_iterations=2, dtype="f64"):
    a = _f64(a)
    m, n = a.shape
    left, right = np.zeros((m, rank)), np.zeros((rank, n))
    _check(lib().kvref_truncated_svd(1 if dtype == "f32" else 0, C.c_size_t(m), C.c_size_t(n), _dp(a),
                                     C.c_size_t(rank), int(method == "randomized"), C.c_uint64(seed),
                                     C.c_size_t(oversampling), C.c_size_t(power_iterations),
                                     _dp(left), _dp(right)))
    return left, right


def singular_values(a):
    a = _f64(a)
    out = np.zeros(min(a.shape))
    _check(lib().kvref_singular_values(C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]), _dp(a), _dp(out)))
    return out


def assign_groups(scores, ratios, ranks, positions=None):
    s = _f64(scores)
    n = s.shape[0]
    pos = np.arange(n, dtype=np.uint64) if positions is None else np.ascontiguousarray(positions, np.uint64)
    r = _f64(ratios)
    rk = np.ascontiguousarray(ranks, dtype=np.uint64)
    tier = np.zeros(n, dtype=np.uint32)
    _check(lib().kvref_assign_groups(C.c_size_t(n), _dp(s), _u64p(pos), C.c_size_t(len(r)), _dp(r),
                                     rk.ctypes.data_as(C.POINTER(C.c_size_t)),
                                     tier.ctypes.data_as(C.POINTER(C.c_uint32))))
    return tier


def update_importance(scores, attn, alpha=0.25):
    s = _f64(scores).copy()
    a = _f64(np.atleast_2d(attn))
    _check(lib().kvref_update_importance(C.c_size_t(s.shape[0]), _dp(s), C.c_size_t(a.shape[0]), _dp(a),
                                         C.c_double(alpha)))
    return s


def flops_partial_decompress(tokens, width, ratios, ranks):
    r = _f64(ratios)
    rk = np.ascontiguousarray(ranks, dtype=np.uint64)
    fl, red = C.c_uint64(), C.c_double()
    _check(lib().kvref_flops_partial_decompress(C.c_size_t(tokens), C.c_size_t(width), C.c_size_t(len(r)),
                                                _dp(r), rk.ctypes.data_as(C.POINTER(C.c_size_t)),
                                                C.byref(fl), C.byref(red)))
    return fl.value, red.value


def quantize_roundtrip(a, group_size=64):
    """dequantize(quantize_4bit(a, group_size)) (quantize.cpp:10-54), double."""
    a = _f64(a)
    out = np.zeros_like(a)
    _check(lib().kvref_quantize_roundtrip(C.c_size_t(a.shape[0]), C.c_size_t(a.shape[1]), _dp(a),
                                          C.c_size_t(group_size), _dp(out)))
    return out


def compression_ratio(tokens, width, rank):
    out = C.c_double()
    _check(lib().kvref_compression_ratio(C.c_size_t(tokens), C.c_size_t(width), C.c_size_t(rank), C.byref(out)))
    return out.value


def gaussian_matrix(rows, cols, seed, stream=0):
    out = np.zeros((rows, cols))
    _check(lib().kvref_gaussian_matrix(C.c_size_t(rows), C.c_size_t(cols), C.c_uint64(seed),
                                       C.c_uint64(stream), _dp(out)))
    return out


def latent_factor_matrix(tokens, heads, kv_heads, head_dim, true_rank, decay, shared, noise, seed, stream):
    out = np.zeros((tokens, kv_heads * head_dim))
    _check(lib().kvref_latent_factor_matrix(C.c_size_t(tokens), C.c_size_t(heads), C.c_size_t(kv_heads),
                                            C.c_size_t(head_dim), C.c_size_t(true_rank), C.c_double(decay),
                                            C.c_size_t(shared), C.c_double(noise), C.c_uint64(seed),
                                            C.c_uint64(stream), _dp(out)))
    return out


def reference_attention(heads, kv_heads, head_dim, x, k, v, wq, wk, wv, wo):
    x = _f64(np.atleast_2d(x))
    k, v = _f64(k), _f64(v)
    out = np.zeros((x.shape[0], heads * head_dim))
    ws = [_f64(w) for w in (wq, wk, wv, wo)]
    _check(lib().kvref_reference_attention(C.c_size_t(heads), C.c_size_t(kv_heads), C.c_size_t(head_dim),
                                           C.c_size_t(x.shape[0]), _dp(x), C.c_size_t(k.shape[0]), _dp(k),
                                           _dp(v), *[_dp(w) for w in ws], _dp(out)))
    return out


def run_simulation(ini_text: str, threads: int = 1) -> str:
    p = C.c_char_p()
    _check(lib().kvref_run_simulation(ini_text.encode(), int(threads), C.byref(p)))
    text = C.string_at(p).decode()
    lib().kvref_free(p)
    return text


def host_cores() -> int:
    return len(os.sched_getaffinity(0))
