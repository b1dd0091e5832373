"""ctypes binding of the C-ABI in include/kvp_b200.h (libkvp_b200.so).

The product path: every call lands in hand-written sm_100a kernels.  There is
no CPU fallback — if the shared library is missing the import fails loudly.
Status codes become the exception types the reference's Python module raises
(bindings/module.cpp:117-127): io -> OSError, parameter/shape/data -> ValueError.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libkvp_b200.so"

KVP_OK, KVP_ERR_PARAMETER, KVP_ERR_SHAPE, KVP_ERR_DATA, KVP_ERR_IO, KVP_ERR_CUDA = range(6)
KVP_F32, KVP_F64, KVP_BF16 = 0, 1, 2
KVP_DENSE, KVP_LOWRANK = 0, 1


class KvpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class KvpParameterError(KvpError, ValueError):
    pass


class KvpShapeError(KvpParameterError):
    pass


class KvpDataError(KvpError, ValueError):
    pass


class KvpIOError(KvpError, OSError):
    pass


class KvpCudaError(KvpError):
    pass


_ERRORS = {KVP_ERR_PARAMETER: KvpParameterError, KVP_ERR_SHAPE: KvpShapeError, KVP_ERR_DATA: KvpDataError,
           KVP_ERR_IO: KvpIOError, KVP_ERR_CUDA: KvpCudaError}


class Store(C.Structure):
    _fields_ = [("form", C.c_int32), ("rank", C.c_int32), ("a", C.c_void_p), ("b", C.c_void_p),
                ("lda", C.c_int64), ("ldb", C.c_int64)]


class PlanEntry(C.Structure):
    _fields_ = [("k_store", C.c_int32), ("v_store", C.c_int32), ("row", C.c_uint32), ("rank_k", C.c_uint32),
                ("rank_v", C.c_uint32), ("table_index", C.c_int32), ("position", C.c_uint64)]


class AttendDesc(C.Structure):
    _fields_ = [("heads", C.c_int32), ("kv_heads", C.c_int32), ("head_dim", C.c_int32), ("dtype", C.c_int32),
                ("n_stores", C.c_int32), ("n_entries", C.c_int32), ("tq", C.c_int32), ("table_size", C.c_int32),
                ("stores", C.POINTER(Store)), ("entries", C.POINTER(PlanEntry)), ("queries", C.c_void_p),
                ("query_positions", C.c_void_p), ("context", C.c_void_p), ("head_avg", C.c_void_p),
                ("head_avg_table", C.c_void_p)]


class FusedDesc(C.Structure):
    _fields_ = [("heads", C.c_int32), ("kv_heads", C.c_int32), ("head_dim", C.c_int32), ("batch", C.c_int32),
                ("n_comp", C.c_int32), ("rank_k", C.c_int32), ("rank_v", C.c_int32), ("tier2_value_rank", C.c_int32),
                ("tail_cap", C.c_int32), ("n_tail", C.c_int32), ("n_tail_dev", C.c_void_p),
                ("cluster", C.c_int32), ("context_bf16", C.c_int32),
                ("left_k", C.c_void_p), ("right_k", C.c_void_p), ("left_v", C.c_void_p), ("right_v", C.c_void_p),
                ("tail_k", C.c_void_p), ("tail_v", C.c_void_p), ("queries", C.c_void_p),
                ("importance", C.c_void_p), ("imp_stride", C.c_int64), ("alpha", C.c_double),
                ("head_avg", C.c_void_p), ("context", C.c_void_p), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("value_tier", C.c_void_p)]


class Profile(C.Structure):
    _fields_ = [("true_rank", C.c_int32), ("shared_subspace", C.c_int32), ("spectrum_decay", C.c_double),
                ("noise_floor", C.c_double)]


class EngineConfig(C.Structure):
    _fields_ = [("heads", C.c_int32), ("kv_heads", C.c_int32), ("head_dim", C.c_int32), ("layers", C.c_int32),
                ("batch", C.c_int32), ("visual_tokens", C.c_int32), ("textual_tokens", C.c_int32),
                ("decode_steps", C.c_int32), ("rank_k", C.c_int32), ("rank_v", C.c_int32), ("alpha", C.c_double),
                ("seed", C.c_uint64), ("visual", Profile), ("textual", Profile), ("svd_method", C.c_int32),
                ("svd_seed", C.c_uint64), ("svd_oversampling", C.c_int32), ("svd_power_iterations", C.c_int32),
                ("factor_init", C.c_int32), ("cluster", C.c_int32), ("tier_ratio", C.c_double),
                ("tier_value_fraction", C.c_double), ("instance_offset", C.c_int32)]


class EngineInfo(C.Structure):
    _fields_ = [("cluster", C.c_int32), ("rank_k", C.c_int32), ("rank_v", C.c_int32), ("ld_left", C.c_int32),
                ("tail_cap", C.c_int32), ("steps_taken", C.c_int32), ("compaction_ms", C.c_double),
                ("launches_per_step", C.c_uint64), ("weight_bytes_per_step", C.c_uint64),
                ("factor_bytes_per_step", C.c_uint64), ("tail_row_bytes", C.c_uint64),
                ("importance_bytes_per_token", C.c_uint64)]


class LayerView(C.Structure):
    _fields_ = [("left_k", C.c_void_p), ("left_v", C.c_void_p), ("right_k", C.c_void_p), ("right_v", C.c_void_p),
                ("tail_k", C.c_void_p), ("tail_v", C.c_void_p), ("importance", C.c_void_p), ("w_qkv", C.c_void_p),
                ("w_o", C.c_void_p), ("n_tail", C.c_int32)]


# name -> (restype, argtypes); every symbol include/kvp_b200.h declares.
class CacheConfigC(C.Structure):
    _fields_ = [("heads", C.c_int32), ("kv_heads", C.c_int32), ("head_dim", C.c_int32), ("dtype", C.c_int32),
                ("batch", C.c_int32), ("layer_index", C.c_int32)]


class DecodeConfigC(C.Structure):
    _fields_ = [("compression_period", C.c_int64), ("rank_key_visual", C.c_int32), ("rank_value_visual", C.c_int32),
                ("rank_key_textual", C.c_int32), ("rank_value_textual", C.c_int32), ("rank_scheme", C.c_int32),
                ("scheme_fixed_rank", C.c_int32), ("scheme_first_layer_rank", C.c_int32),
                ("scheme_last_layer_rank", C.c_int32), ("scheme_num_layers", C.c_int32),
                ("scheme_variance_target", C.c_double), ("scheme_max_rank", C.c_int32), ("n_tiers", C.c_int32),
                ("tier_ratios", C.POINTER(C.c_double)), ("tier_key_fractions", C.POINTER(C.c_double)),
                ("tier_value_fractions", C.POINTER(C.c_double)), ("alpha", C.c_double), ("svd_method", C.c_int32),
                ("svd_seed", C.c_uint64), ("svd_oversampling", C.c_int32), ("svd_power_iterations", C.c_int32),
                ("recompress", C.c_int32), ("bytes_per_scalar", C.c_int32)]


class StepReportC(C.Structure):
    _fields_ = [("step", C.c_uint64), ("bytes_before", C.c_uint64), ("bytes_after", C.c_uint64),
                ("importance_bytes", C.c_uint64), ("decompress_flops", C.c_uint64),
                ("decompress_flops_full", C.c_uint64), ("flops_reduction", C.c_double),
                ("compression_event", C.c_int32), ("n_warnings", C.c_int32)]


class WeightsC(C.Structure):
    _fields_ = [("w_q", C.c_void_p), ("w_k", C.c_void_p), ("w_v", C.c_void_p), ("w_o", C.c_void_p)]


class CacheBytesC(C.Structure):
    _fields_ = [("visual_scalars", C.c_uint64), ("textual_scalars", C.c_uint64), ("visual_bytes", C.c_uint64),
                ("textual_bytes", C.c_uint64), ("cache_bytes", C.c_uint64), ("importance_bytes", C.c_uint64)]


_P = C.c_void_p
SIGNATURES = {
    "kvp_cache_create": (C.c_int, [C.POINTER(CacheConfigC), C.POINTER(C.c_void_p)]),
    "kvp_cache_destroy": (C.c_int, [_P]),
    "kvp_cache_append": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P]),
    "kvp_cache_factor_tail": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, C.c_int32, _P, _P]),
    "kvp_cache_set_importance": (C.c_int, [_P, _P]),
    "kvp_cache_get_importance": (C.c_int, [_P, _P, _P]),
    "kvp_cache_shape": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "kvp_cache_set_counters": (C.c_int, [_P, C.c_uint64, C.c_uint64]),
    "kvp_quantize_roundtrip": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, _P, _P]),
    "kvp_cache_block_info": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, _P]),
    "kvp_cache_block_get": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P]),
    "kvp_cache_tail_get": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _P]),
    "kvp_cache_memory_bytes": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(CacheBytesC)]),
    "kvp_segment_full_matrix": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P]),
    "kvp_compress_now": (C.c_int, [_P, C.POINTER(DecodeConfigC), _P, _P]),
    "kvp_decode_step": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.POINTER(WeightsC), C.POINTER(DecodeConfigC), _P,
                                  _P, _P]),
    "kvp_abi_version": (C.c_int, []),
    "kvp_last_error_message": (C.c_char_p, []),
    "kvp_launch_count": (C.c_uint64, []),
    "kvp_attend_plan": (C.c_int, [C.POINTER(AttendDesc), C.c_void_p]),
    "kvp_update_importance": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_double,
                                        C.c_int32, C.c_void_p]),
    "kvp_assign_tiers": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "kvp_update_importance_host": (C.c_int, [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_double]),
    "kvp_assign_groups_host": (C.c_int, [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "kvp_packed_left_bytes": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int32]),
    "kvp_pack_left": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "kvp_packed_weight_bytes": (C.c_size_t, [C.c_int32, C.c_int32]),
    "kvp_pack_weight": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "kvp_matmul_packed_workspace": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int32]),
    "kvp_matmul_packed": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                    C.c_int32, C.c_void_p, C.c_void_p]),
    "kvp_truncated_svd": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64,
                                    C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "kvp_gaussian_matrix": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, C.c_int32, C.c_void_p,
                                      C.c_void_p]),
    "kvp_decode_fused": (C.c_int, [C.POINTER(FusedDesc), C.c_void_p]),
    "kvp_decode_fused_workspace": (C.c_size_t, [C.POINTER(FusedDesc)]),
    "kvp_engine_create": (C.c_int, [C.POINTER(EngineConfig), C.POINTER(C.c_void_p)]),
    "kvp_engine_destroy": (C.c_int, [C.c_void_p]),
    "kvp_engine_prefill": (C.c_int, [C.c_void_p]),
    "kvp_engine_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "kvp_engine_step_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "kvp_engine_reset_steps": (C.c_int, [C.c_void_p]),
    "kvp_engine_get_info": (C.c_int, [C.c_void_p, C.POINTER(EngineInfo)]),
    "kvp_engine_layer_state": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(LayerView)]),
    "kvp_engine_time_attention": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing — build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (no CPU fallback exists)")
        l = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def check(rc: int):
    if rc != KVP_OK:
        msg = lib().kvp_last_error_message().decode()
        raise _ERRORS.get(rc, KvpError)(rc, msg)


def call(name, *args):
    check(getattr(lib(), name)(*args))


def launch_count() -> int:
    return int(lib().kvp_launch_count())
