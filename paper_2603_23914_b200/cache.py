"""The reference's cache + decoder API (cache.hpp:120-176, decoder.hpp:18-191,
compressor.hpp:14-56) over a device-resident LayerCache batch.

Same names, argument meanings and error behaviour as the reference:
``DecodeConfig`` / ``TierSpec`` / ``MatrixRanks`` / ``SvdOptions`` /
``RankScheme`` mirror decoder.hpp:31-75 and linalg.hpp:12-19;
``decode_step(h, cache, weights, cfg)`` and ``compress_now(cache, cfg)``
mirror decoder.hpp:166-191 and return the per-instance ``StepReport``s.  A
``LayerCacheBatch`` is ``batch`` LayerCaches of one layer that step together
(the reference harness's per-request caches, harness.cpp:239-360).  All compute
runs in libkvp_b200.so (csrc/cache.cu); parameter/shape/data errors raise
``ValueError`` like the reference's Python module (bindings/module.cpp:117-127).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi as capi

VISUAL, TEXTUAL = 0, 1
KEY, VALUE = 0, 1
_DT = {"f32": capi.KVP_F32, "f64": capi.KVP_F64, "bf16": capi.KVP_BF16}


@dataclass
class TierSpec:
    """Attention-aware tiering (decoder.hpp:28-36)."""
    ratios: list
    key_fractions: list
    value_fractions: list


@dataclass
class MatrixRanks:
    """Per-matrix compression ranks, 0 = dense (decoder.hpp:40-51)."""
    key_visual: int = 64
    value_visual: int = 64
    key_textual: int = 0
    value_textual: int = 0


@dataclass
class SvdOptions:
    """linalg.hpp:12-19."""
    method: str = "exact"
    oversampling: int = 8
    power_iterations: int = 2
    seed: int = 0


@dataclass
class RankScheme:
    """compressor.hpp:14-30: fixed / linear_schedule / variance_target."""
    kind: str = "fixed"
    fixed_rank: int = 64
    first_layer_rank: int = 16
    last_layer_rank: int = 128
    num_layers: int = 32
    variance_target: float = 0.95
    max_rank: int = 256


@dataclass
class DecodeConfig:
    """decoder.hpp:53-75 (the eviction / quantization variants are not on the device)."""
    compression_period: int | None = 512
    ranks: MatrixRanks = field(default_factory=MatrixRanks)
    rank_scheme: RankScheme | None = None
    tiering: TierSpec | None = None
    alpha: float = 0.25
    svd: SvdOptions = field(default_factory=SvdOptions)
    recompress: str = "joint"
    bytes_per_scalar: int = 2

    @classmethod
    def from_ini(cls, text: str) -> "DecodeConfig":
        """The [decode], [decode.ranks], [decode.rank_scheme] and [decode.tiering]
        sections of a reference INI config (config.cpp:96-184)."""
        cfg = cls()
        section = ""
        for raw in text.splitlines():
            line = raw.split("#", 1)[0].split(";", 1)[0].strip()
            if not line:
                continue
            if line.startswith("["):
                section = line.strip("[]").strip()
                if section == "decode.rank_scheme" and cfg.rank_scheme is None:
                    cfg.rank_scheme = RankScheme()
                if section == "decode.tiering" and cfg.tiering is None:
                    cfg.tiering = TierSpec([], [], [])
                continue
            key, _, value = (x.strip() for x in line.partition("="))
            if section == "decode":
                if key == "compression_period":
                    cfg.compression_period = None if value in ("none", "inf") else int(value)
                elif key == "alpha":
                    cfg.alpha = float(value)
                elif key == "svd_method":
                    cfg.svd.method = value
                elif key == "svd_seed":
                    cfg.svd.seed = int(value)
                elif key == "svd_oversampling":
                    cfg.svd.oversampling = int(value)
                elif key == "svd_power_iterations":
                    cfg.svd.power_iterations = int(value)
                elif key == "recompress":
                    cfg.recompress = value
                elif key == "bytes_per_scalar":
                    cfg.bytes_per_scalar = int(value)
                elif key in ("eviction", "quantization") and value == "true":
                    raise ValueError(f"decode.{key}: the hybrid variants are not part of the device path")
            elif section == "decode.ranks":
                setattr(cfg.ranks, key, int(value))
            elif section == "decode.rank_scheme":
                s = cfg.rank_scheme
                if key == "kind":
                    s.kind = value
                elif key == "variance_target":
                    s.variance_target = float(value)
                else:
                    setattr(s, key, int(value))
            elif section == "decode.tiering":
                vals = [float(x) for x in value.split(",")]
                if key == "ratios":
                    cfg.tiering.ratios = vals
                elif key == "key_rank_fractions":
                    cfg.tiering.key_fractions = vals
                elif key == "value_rank_fractions":
                    cfg.tiering.value_fractions = vals
        return cfg

    def to_c(self):
        c = capi.DecodeConfigC()
        c.compression_period = -1 if self.compression_period is None else int(self.compression_period)
        if self.compression_period is not None and self.compression_period < 1:
            raise ValueError("DecodeConfig: compression_period must be >= 1")
        r = self.ranks
        c.rank_key_visual, c.rank_value_visual = r.key_visual, r.value_visual
        c.rank_key_textual, c.rank_value_textual = r.key_textual, r.value_textual
        s = self.rank_scheme
        kinds = {"fixed": 0, "linear_schedule": 1, "variance_target": 2}
        if s is None:
            c.rank_scheme = -1
        else:
            if s.kind not in kinds:
                raise ValueError(f"RankScheme: unknown kind '{s.kind}'")
            c.rank_scheme = kinds[s.kind]
            c.scheme_fixed_rank, c.scheme_first_layer_rank = s.fixed_rank, s.first_layer_rank
            c.scheme_last_layer_rank, c.scheme_num_layers = s.last_layer_rank, s.num_layers
            c.scheme_variance_target, c.scheme_max_rank = s.variance_target, s.max_rank
        keep = []
        if self.tiering is not None:
            t = self.tiering
            arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (t.ratios, t.key_fractions, t.value_fractions)]
            if len({a.size for a in arrs}) != 1 or arrs[0].size == 0:
                raise ValueError("TierSpec: one rank fraction per group required")
            keep += arrs
            c.n_tiers = arrs[0].size
            c.tier_ratios, c.tier_key_fractions, c.tier_value_fractions = (
                a.ctypes.data_as(C.POINTER(C.c_double)) for a in arrs)
        c.alpha = self.alpha
        if self.svd.method not in ("exact", "randomized"):
            raise ValueError(f"SvdOptions: unknown method '{self.svd.method}'")
        c.svd_method = 1 if self.svd.method == "randomized" else 0
        c.svd_seed, c.svd_oversampling, c.svd_power_iterations = (self.svd.seed, self.svd.oversampling,
                                                                  self.svd.power_iterations)
        if self.recompress not in ("joint", "separate_epochs"):
            raise ValueError(f"DecodeConfig: unknown recompress mode '{self.recompress}'")
        c.recompress = 0 if self.recompress == "joint" else 1
        c.bytes_per_scalar = self.bytes_per_scalar
        c._keep = keep
        return c


@dataclass
class StepReport:
    """decoder.hpp:145-160 (integer accounting fields)."""
    step: int = 0
    bytes_before: int = 0
    bytes_after: int = 0
    importance_bytes: int = 0
    decompress_flops: int = 0
    decompress_flops_full: int = 0
    flops_reduction: float = 0.0
    compression_event: bool = False
    n_warnings: int = 0

    @classmethod
    def from_c(cls, r):
        return cls(r.step, r.bytes_before, r.bytes_after, r.importance_bytes, r.decompress_flops,
                   r.decompress_flops_full, r.flops_reduction, bool(r.compression_event), r.n_warnings)


def _torch():
    import torch
    return torch


class AttentionWeights:
    """decoder.hpp:18-26, uploaded once to the device in the cache's storage dtype."""

    def __init__(self, w_q, w_k, w_v, w_o, dtype="f64"):
        torch = _torch()
        tdt = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16}[dtype]
        self.dtype = dtype
        self.t = [torch.as_tensor(np.ascontiguousarray(w, dtype=np.float64)).to("cuda", tdt).contiguous()
                  for w in (w_q, w_k, w_v, w_o)]
        self.c = capi.WeightsC(*[x.data_ptr() for x in self.t])


class LayerCacheBatch:
    """`batch` device LayerCaches of one layer (cache.hpp:120-146)."""

    def __init__(self, heads, kv_heads, head_dim, batch=1, dtype="f64", layer_index=0):
        self.H, self.Hkv, self.D, self.batch, self.dtype = heads, kv_heads, head_dim, batch, dtype
        self.layer_index = layer_index
        self.W, self.HD = kv_heads * head_dim, heads * head_dim
        self._h = C.c_void_p()
        cfg = capi.CacheConfigC(heads, kv_heads, head_dim, _DT[dtype], batch, layer_index)
        capi.call("kvp_cache_create", C.byref(cfg), C.byref(self._h))

    def close(self):
        if self._h:
            capi.call("kvp_cache_destroy", self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _rows(self, x, cols):
        a = np.ascontiguousarray(x, dtype=np.float64)
        if a.ndim == 2:
            a = a[None]
        if a.shape[0] != self.batch or a.shape[2] != cols:
            raise ValueError("append_tokens: rows must be cache_width wide, one block per instance")
        return a

    def append_tokens(self, modality, k_rows, v_rows):
        k, v = self._rows(k_rows, self.W), self._rows(v_rows, self.W)
        if k.shape != v.shape:
            raise ValueError("append_tokens: K and V row counts disagree")
        capi.call("kvp_cache_append", self._h, modality, k.shape[1], k.ctypes.data, v.ctypes.data)

    def factor_tail(self, modality, k_factors, v_factors):
        """Install host factors (left, right) — or None for a dense kind — as a block
        made of the segment's current tail (uploading a host LayerCache image)."""
        args, keep = [], []
        for fac in (k_factors, v_factors):
            if fac is None:
                args += [0, None, None]
            else:
                l, r = (np.ascontiguousarray(x, dtype=np.float64) for x in fac)
                if l.ndim == 2:
                    l, r = l[None], r[None]
                keep += [l, r]
                args += [l.shape[2], l.ctypes.data, r.ctypes.data]
        capi.call("kvp_cache_factor_tail", self._h, modality, *args)

    def shape(self):
        ts, nx, st = C.c_int32(), C.c_uint64(), C.c_uint64()
        nb, tl = (C.c_int32 * 2)(), (C.c_int32 * 2)()
        capi.call("kvp_cache_shape", self._h, C.byref(ts), C.byref(nx), C.byref(st), nb, tl)
        return dict(table_size=ts.value, next_position=nx.value, steps_taken=st.value, n_blocks=list(nb),
                    tail_len=list(tl))

    def importance(self):
        n = self.shape()["table_size"]
        pos = np.zeros(n, dtype=np.uint64)
        sc = np.zeros((self.batch, n))
        capi.call("kvp_cache_get_importance", self._h, pos.ctypes.data, sc.ctypes.data)
        return pos, sc

    def set_importance(self, scores):
        s = np.ascontiguousarray(np.broadcast_to(scores, (self.batch, self.shape()["table_size"])), dtype=np.float64)
        capi.call("kvp_cache_set_importance", self._h, s.ctypes.data)

    def block(self, instance, modality, block, kind):
        t, r = C.c_int32(), C.c_int32()
        capi.call("kvp_cache_block_info", self._h, instance, modality, block, kind, C.byref(t), C.byref(r))
        t, r = t.value, r.value
        pos = np.zeros(t, dtype=np.uint64)
        if r == 0:
            rows = np.zeros((t, self.W))
            capi.call("kvp_cache_block_get", self._h, instance, modality, block, kind, rows.ctypes.data, None,
                      pos.ctypes.data)
            return "dense", rows, None, pos
        left, right = np.zeros((t, r)), np.zeros((r, self.W))
        capi.call("kvp_cache_block_get", self._h, instance, modality, block, kind, left.ctypes.data,
                  right.ctypes.data, pos.ctypes.data)
        return "lowrank", left, right, pos

    def tail(self, instance, modality):
        n = self.shape()["tail_len"][modality]
        k, v = np.zeros((n, self.W)), np.zeros((n, self.W))
        pos = np.zeros(n, dtype=np.uint64)
        capi.call("kvp_cache_tail_get", self._h, instance, modality, k.ctypes.data, v.ctypes.data, pos.ctypes.data)
        return k, v, pos

    def memory_bytes(self, instance=0, bytes_per_scalar=2):
        out = capi.CacheBytesC()
        capi.call("kvp_cache_memory_bytes", self._h, instance, bytes_per_scalar, C.byref(out))
        return dict(visual=out.visual_bytes, textual=out.textual_bytes, cache_bytes=out.cache_bytes,
                    importance_bytes=out.importance_bytes)

    @classmethod
    def from_state(cls, states, dtype="f64"):
        """Upload reference LayerCache images (oracle.cases.export_state dicts, one per
        instance, identical structure): blocks in append order, tails, importance."""
        st0 = states[0]
        c = cls(int(st0["H"]), int(st0["Hkv"]), int(st0["D"]), batch=len(states), dtype=dtype)
        W = c.W
        # rebuild by position order: each block / tail is a run of consecutive positions
        runs = []
        for s in (0, 1):
            for b in range(int(st0[f"s{s}_nblocks"])):
                runs.append((int(st0[f"s{s}b{b}_positions"][0]), s, b))
            if st0[f"s{s}_tail_positions"].size:
                runs.append((int(st0[f"s{s}_tail_positions"][0]), s, -1))
        for _, s, b in sorted(runs):
            if b < 0:
                c.append_tokens(s, np.stack([x[f"s{s}_tail_k"] for x in states]),
                                np.stack([x[f"s{s}_tail_v"] for x in states]))
                continue
            n = st0[f"s{s}b{b}_positions"].size
            facs, rows = [], []
            for kn in ("k", "v"):
                if f"s{s}b{b}_{kn}_left" in st0:
                    facs.append((np.stack([x[f"s{s}b{b}_{kn}_left"] for x in states]),
                                 np.stack([x[f"s{s}b{b}_{kn}_right"] for x in states])))
                    rows.append(np.zeros((len(states), n, W)))
                else:  # a dense kind keeps the appended rows
                    facs.append(None)
                    rows.append(np.stack([x[f"s{s}b{b}_{kn}_rows"] for x in states]))
            c.append_tokens(s, rows[0], rows[1])
            c.factor_tail(s, facs[0], facs[1])
        c.set_importance(np.stack([x["imp_scores"] for x in states]))
        return c


def _reports(arr):
    return [StepReport.from_c(r) for r in arr]


def compress_now(cache: LayerCacheBatch, cfg: DecodeConfig):
    """decoder.hpp:184-186: re-factorise every compressible segment with a tail."""
    reps = (capi.StepReportC * cache.batch)()
    cc = cfg.to_c()
    capi.call("kvp_compress_now", cache._h, C.byref(cc), reps, None)
    return _reports(reps)


def decode_step(h, cache: LayerCacheBatch, weights: AttentionWeights, cfg: DecodeConfig, modality=TEXTUAL):
    """decoder.hpp:166-169 for every instance: h [batch][tq][HD] (numpy or a CUDA
    tensor); returns (output [batch][tq][HD] as a CUDA tensor, [StepReport])."""
    torch = _torch()
    adt = torch.float64 if cache.dtype == "f64" else torch.float32
    x = h if isinstance(h, torch.Tensor) else torch.as_tensor(np.asarray(h))
    if x.dim() == 2:
        x = x[None]
    x = x.to("cuda", adt).contiguous()
    if x.shape[0] != cache.batch or x.shape[2] != cache.HD:
        raise ValueError("decode_step: activations must be model_width wide, one block per instance")
    out = torch.empty_like(x)
    reps = (capi.StepReportC * cache.batch)()
    cc = cfg.to_c()
    capi.call("kvp_decode_step", cache._h, C.c_void_p(x.data_ptr()), x.shape[1], modality, C.byref(weights.c),
              C.byref(cc), C.c_void_p(out.data_ptr()), reps, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    return out, _reports(reps)


def segment_full_matrix(cache: LayerCacheBatch, modality, kind):
    """decoder.hpp:188-191: [blocks at full stored rank; tail] per instance."""
    torch = _torch()
    sh = cache.shape()
    n = sum(cache.block(0, modality, b, kind)[3].size for b in range(sh["n_blocks"][modality])) + \
        sh["tail_len"][modality]
    out = torch.empty((cache.batch, n, cache.W), dtype=torch.float64, device="cuda")
    capi.call("kvp_segment_full_matrix", cache._h, modality, kind, C.c_void_p(out.data_ptr()),
              C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return out.cpu().numpy()
