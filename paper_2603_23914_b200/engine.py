"""Python handle on the device decode engine (include/kvp_b200.h kvp_engine_*).

The engine is the batched serving form of the reference's harness loop
(harness.cpp:239-360): per layer a projection GEMM, tail append, the fused
compressed-cache attention (qdots -> cluster core -> vsum) with the fused
importance EMA, and the output GEMM — captured once as a CUDA graph.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import _capi as capi


@dataclass
class ProfileSpec:
    true_rank: int
    shared_subspace: int
    spectrum_decay: float
    noise_floor: float


@dataclass
class EngineSpec:
    heads: int
    kv_heads: int
    head_dim: int
    layers: int
    batch: int
    visual_tokens: int
    textual_tokens: int
    decode_steps: int
    rank_k: int
    rank_v: int
    alpha: float = 0.25
    seed: int = 0
    visual: ProfileSpec = None
    textual: ProfileSpec = field(default_factory=lambda: ProfileSpec(48, 4, 0.98, 1e-2))
    svd_method: str = "randomized"
    svd_seed: int = 0
    svd_oversampling: int = 8
    svd_power_iterations: int = 2
    factor_init: str = "compaction"  # or "placeholder"
    cluster: int = 0
    tier_ratio: float = 0.0           # two-tier values: first-group ratio (0 = untiered)
    tier_value_fraction: float = 1.0  # value-rank fraction of the second group
    instance_offset: int = 0          # global index of instance 0 (Philox streams of the sharded batch)

    def to_c(self) -> capi.EngineConfig:
        vis = self.visual or ProfileSpec(2 * self.rank_k, self.rank_k, 0.98, 1e-2)
        c = capi.EngineConfig()
        for k in ("heads", "kv_heads", "head_dim", "layers", "batch", "visual_tokens", "textual_tokens",
                  "decode_steps", "rank_k", "rank_v", "alpha", "seed", "svd_seed", "svd_oversampling",
                  "svd_power_iterations", "cluster", "tier_ratio", "tier_value_fraction", "instance_offset"):
            setattr(c, k, getattr(self, k))
        c.visual = capi.Profile(vis.true_rank, vis.shared_subspace, vis.spectrum_decay, vis.noise_floor)
        t = self.textual
        c.textual = capi.Profile(t.true_rank, t.shared_subspace, t.spectrum_decay, t.noise_floor)
        c.svd_method = 1 if self.svd_method == "randomized" else 0
        c.factor_init = 1 if self.factor_init == "placeholder" else 0
        return c


class Engine:
    def __init__(self, spec: EngineSpec):
        self.spec = spec
        self._h = C.c_void_p()
        self._cfg = spec.to_c()
        capi.call("kvp_engine_create", C.byref(self._cfg), C.byref(self._h))

    def close(self):
        if self._h:
            capi.call("kvp_engine_destroy", self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prefill(self):
        capi.call("kvp_engine_prefill", self._h)

    def step(self, x_dev_ptr: int, y_dev_ptr: int, stream: int = 0):
        capi.call("kvp_engine_step", self._h, C.c_void_p(x_dev_ptr), C.c_void_p(y_dev_ptr), C.c_void_p(stream))

    def step_host(self, x_host_ptr: int, y_host_ptr: int):
        capi.call("kvp_engine_step_host", self._h, C.c_void_p(x_host_ptr), C.c_void_p(y_host_ptr))

    def reset_steps(self):
        capi.call("kvp_engine_reset_steps", self._h)

    def info(self) -> capi.EngineInfo:
        i = capi.EngineInfo()
        capi.call("kvp_engine_get_info", self._h, C.byref(i))
        return i

    def time_attention(self, iters: int = 3):
        ms, by = C.c_double(), C.c_double()
        capi.call("kvp_engine_time_attention", self._h, iters, C.byref(ms), C.byref(by))
        return ms.value, by.value

    def layer(self, l: int) -> capi.LayerView:
        v = capi.LayerView()
        capi.call("kvp_engine_layer_state", self._h, l, C.byref(v))
        return v
