"""ctypes binding of libplora.so (C ABI: include/plora.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2512_20210_b200/csrc``).  There is no fallback: if the
library is missing every entry point fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, LogicError, ParseError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
# PLORA_LIB: diagnostics only (A/B builds of the same ABI, scripts/); default in-tree
LIB_PATH = os.environ.get("PLORA_LIB", os.path.join(_HERE, "libplora.so"))

PLORA_OK = 0
PLORA_E_VALIDATION = -1
PLORA_E_LOGIC = -2
PLORA_E_CONFIG = -3
PLORA_E_PARSE = -4
PLORA_E_CUDA = -5
PLORA_E_NOMEM = -6

PLORA_MAX_PROJ = 8
PLORA_BF16 = 0
PLORA_F32 = 1
PLORA_COPY_CE = 0
PLORA_COPY_SM = 1
PLORA_COPY_AUTO = 2
PLORA_ADMIT_LOADING = 0
PLORA_ADMIT_READY = 1
PLORA_ADMIT_FAILED = 2
PLORA_NOT_RESIDENT = 0
PLORA_STAGING = 1
PLORA_RESIDENT = 2


class CudaError(RuntimeError):
    """A CUDA runtime failure inside libplora."""


class plora_frag_report(C.Structure):
    _fields_ = [("external_frag", C.c_double), ("internal_frag", C.c_double),
                ("utilization", C.c_double)]


class plora_reloc(C.Structure):
    _fields_ = [("adapter", C.c_uint32), ("logical", C.c_uint32), ("src", C.c_uint32),
                ("dst", C.c_uint32)]


class plora_policy(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("theta", "alpha", "beta", "gamma", "tau_ms",
                                          "freq_half_life_ms", "staging_fraction")]


class plora_dynamics(C.Structure):
    _fields_ = [("status", C.c_int32), ("busy", C.c_uint32), ("last_access_ms", C.c_double),
                ("decayed_count", C.c_double), ("decay_stamp_ms", C.c_double),
                ("prediction", C.c_double), ("transfer_active", C.c_int32),
                ("reserved", C.c_int32)]


class plora_synthetic_profile(C.Structure):
    _fields_ = [("num_adapters", C.c_uint32), ("base_rate", C.c_double),
                ("diurnal_amplitude", C.c_double), ("period_s", C.c_double),
                ("hot_set_size", C.c_uint32), ("hot_rotation_s", C.c_double),
                ("hot_share", C.c_double), ("rotation_jitter", C.c_double),
                ("burstiness_cv", C.c_double), ("input_median", C.c_double),
                ("input_sigma", C.c_double), ("output_median", C.c_double),
                ("output_sigma", C.c_double), ("max_tokens", C.c_uint32)]


class plora_model(C.Structure):
    _fields_ = [("n_layers", C.c_uint32), ("n_proj", C.c_uint32),
                ("d_in", C.c_uint32 * PLORA_MAX_PROJ), ("d_out", C.c_uint32 * PLORA_MAX_PROJ),
                ("dtype", C.c_uint32)]


class plora_engine_config(C.Structure):
    _fields_ = [("policy", plora_policy), ("copy_mode", C.c_int32), ("prefetch", C.c_int32),
                ("compaction", C.c_int32), ("reserved", C.c_int32), ("chunk_bytes", C.c_uint64),
                ("prefetch_inflight_bytes", C.c_uint64)]


class plora_engine_stats(C.Structure):
    _fields_ = ([(n, C.c_uint64) for n in (
        "arrivals", "hits", "demand_loads", "prefetch_issued", "promotions", "evictions",
        "admission_failures", "upgrades", "compactions", "relocations", "prediction_rounds",
        "transfers_completed", "bytes_h2d")]
        + [("transfer_ms", C.c_double), ("demand_transfer_ms", C.c_double),
           ("predictor_ms", C.c_double)]
        + [(n, C.c_uint64) for n in ("in_flight", "staged", "resident")]
        + [("copy_mode", C.c_int32), ("reserved", C.c_int32)]
        + [("acc_sum", C.c_double)]
        + [(n, C.c_uint64) for n in ("acc_intervals", "acc_tp", "acc_fp", "acc_fn")])


class plora_decision(C.Structure):
    _fields_ = [("t_ms", C.c_double), ("score", C.c_double), ("adapter", C.c_uint32),
                ("action", C.c_uint32), ("detail", C.c_uint64)]


class plora_lstm_config(C.Structure):
    _fields_ = [("window", C.c_uint32), ("hidden", C.c_uint32), ("layers", C.c_uint32),
                ("embedding_dim", C.c_uint32), ("num_adapters", C.c_uint32),
                ("learning_rate", C.c_double), ("adam_beta1", C.c_double),
                ("adam_beta2", C.c_double), ("adam_eps", C.c_double)]


class plora_predictor_config(C.Structure):
    _fields_ = [("model", plora_lstm_config), ("interval_ms", C.c_double),
                ("train_every", C.c_uint32), ("batch_size", C.c_uint32),
                ("replay_capacity", C.c_uint32)]


class plora_predictor_stats_t(C.Structure):
    _fields_ = [("observed", C.c_uint64), ("train_steps", C.c_uint64), ("known", C.c_uint64),
                ("buffered", C.c_uint64), ("current_interval", C.c_int64),
                ("last_loss", C.c_double)]


_u32, _u64, _i32, _i64, _int, _dbl, _vp = (C.c_uint32, C.c_uint64, C.c_int32, C.c_int64,
                                           C.c_int, C.c_double, C.c_void_p)
_P = C.POINTER

# name -> (restype, argtypes)
_SIGS = {
    "plora_last_error": (C.c_char_p, []),
    "plora_version": (C.c_char_p, []),
    "plora_kernel_launch_count": (_u64, []),
    "plora_lora_dims_validate": (_int, [_u32, _u32, _u32, _u32, _u32]),
    "plora_param_count": (_int, [_u32, _u32, _u32, _u32, _u32, _P(_u64)]),
    "plora_size_table_create": (_int, [_u32, _u64, _int, _P(_vp)]),
    "plora_size_table_destroy": (None, [_vp]),
    "plora_size_table_set": (_int, [_vp, _u32, _u64]),
    "plora_size_table_bytes_for": (_int, [_vp, _u32, _P(_u64)]),
    "plora_load_catalog_json": (_i64, [C.c_char_p, _vp, _u32, _u32, _u32, _u32, _P(_u32),
                                        _P(_u64), C.c_char_p, _u64, _u64]),
    "plora_generate_catalog": (_int, [_u32, _P(_u32), _P(_dbl), _u64, _u64, _vp, _u32, _u32,
                                      _u32, _u32, _P(_u32), _P(_u64)]),
    "plora_pool_create": (_int, [_u64, _u32, _P(_vp)]),
    "plora_pool_destroy": (None, [_vp]),
    "plora_pool_pages_needed": (_u32, [_vp, _u64]),
    "plora_pool_alloc": (_int, [_vp, _u32, _u64]),
    "plora_pool_free": (_int, [_vp, _u32]),
    "plora_pool_translate": (_int, [_vp, _u32, _u32, _P(_u32)]),
    "plora_pool_table": (_int, [_vp, _u32, _P(_P(_u32)), _P(_u32), _P(_u64)]),
    "plora_pool_has": (_int, [_vp, _u32]),
    "plora_pool_compact": (_int, [_vp, _P(_u64)]),
    "plora_pool_last_relocations": (_int, [_vp, _P(_P(plora_reloc)), _P(_u64)]),
    "plora_pool_report": (None, [_vp, _P(plora_frag_report)]),
    "plora_pool_free_pages": (_u32, [_vp]),
    "plora_pool_total_pages": (_u32, [_vp]),
    "plora_pool_page_bytes": (_u64, [_vp]),
    "plora_pool_used_bytes": (_u64, [_vp]),
    "plora_pool_allocated_bytes": (_u64, [_vp]),
    "plora_pool_total_bytes": (_u64, [_vp]),
    "plora_pool_resident": (_u64, [_vp, _P(_u32), _u64]),
    "plora_pool_check_invariants": (_int, [_vp]),
    "plora_pool_dump": (_int, [_vp, C.c_char_p, _u64, _P(_u64)]),
    "plora_policy_default": (None, [_P(plora_policy)]),
    "plora_policy_validate": (_int, [_P(plora_policy)]),
    "plora_dynamics_init": (None, [_P(plora_dynamics)]),
    "plora_record_access": (None, [_P(plora_dynamics), _dbl, _dbl]),
    "plora_decayed_at": (_dbl, [_P(plora_dynamics), _dbl, _dbl]),
    "plora_recency_score": (_dbl, [_dbl, _dbl, _dbl]),
    "plora_eviction_score": (_dbl, [_P(plora_dynamics), _P(plora_policy), _dbl, _dbl]),
    "plora_scored_residents": (_u64, [_P(plora_dynamics), _u64, _P(plora_policy), _dbl,
                                      _P(_dbl), _P(_u32)]),
    "plora_select_prefetch": (_u64, [_P(_dbl), _u64, _P(plora_dynamics), _u64,
                                     _P(plora_policy), _P(_u64), _u64, _u64, _P(_u32)]),
    "plora_plan_evictions": (_int, [_u64, _u64, _P(_u32), _u64, _P(_u64), _u64, _P(_u32),
                                    _P(_u64)]),
    "plora_synthetic_profile_default": (None, [_P(plora_synthetic_profile)]),
    "plora_generate_synthetic": (_i64, [_P(plora_synthetic_profile), _dbl, _u64, _P(_dbl),
                                        _P(_u32), _P(_u32), _P(_u32), _u64]),
    "plora_model_adapter_bytes": (_u64, [_P(plora_model), _u32]),
    "plora_model_block_offset": (_u64, [_P(plora_model), _u32, _u32, _u32]),
    "plora_store_create": (_int, [_vp, _int, _P(plora_model), _u32, _P(_vp)]),
    "plora_store_destroy": (None, [_vp]),
    "plora_store_arena": (_vp, [_vp]),
    "plora_store_register": (_int, [_vp, _u32, _u32]),
    "plora_store_rank": (_int, [_vp, _u32, _P(_u32)]),
    "plora_store_write_pages": (_int, [_vp, _u32, _vp, _u64, _int, _vp]),
    "plora_store_read_pages": (_int, [_vp, _u32, _vp, _u64, _vp]),
    "plora_store_publish": (_int, [_vp, _u32, _vp]),
    "plora_store_retire": (_int, [_vp, _u32, _vp]),
    "plora_store_is_published": (_int, [_vp, _u32]),
    "plora_store_apply_relocations": (_int, [_vp, _P(plora_reloc), _u64, _vp]),
    "plora_hoststore_create": (_int, [_P(_u64), _P(_u32), _u32, _u64, _P(_vp)]),
    "plora_hoststore_open": (_int, [C.c_char_p, _P(_vp)]),
    "plora_hoststore_save": (_int, [_vp, C.c_char_p]),
    "plora_hoststore_destroy": (None, [_vp]),
    "plora_hoststore_count": (_u32, [_vp]),
    "plora_hoststore_entry": (_int, [_vp, _u32, _P(_vp), _P(_u64), _P(_u32)]),
    "plora_hoststore_bytes": (_int, [_vp, _P(_u64)]),
    "plora_plan_create": (_int, [_vp, _P(_i32), _u32, _vp, _P(_vp)]),
    "plora_plan_update": (_int, [_vp, _P(_i32), _u32, _vp]),
    "plora_plan_destroy": (None, [_vp]),
    "plora_plan_num_segments": (_u32, [_vp]),
    "plora_bgmv": (_int, [_vp, _u32, _u32, _vp, _u64, _vp, _u64, C.c_float, _vp]),
    "plora_bgmv_layer": (_int, [_vp, _u32, _vp, _u64, _P(_vp), _P(_u64), C.c_float, _vp]),
    "plora_bgmv_layers": (_int, [_vp, _u32, _u32, _vp, _u64, _u64, _P(_vp), _P(_u64), _P(_u64),
                                 C.c_float, _vp]),
    "plora_sgmv": (_int, [_vp, _u32, _u32, _vp, _u64, _vp, _u64, C.c_float, _vp]),
    "plora_sgmv_layer": (_int, [_vp, _u32, _vp, _u64, _P(_vp), _P(_u64), C.c_float, _vp]),
    "plora_sgmv_fused": (_int, [_vp, _u32, _u32, _vp, _u64, _vp, _u64, _vp, _u64, C.c_float, _vp]),
    "plora_sgmv_fused_layer": (_int, [_vp, _u32, _vp, _u64, _P(_vp), _P(_u64), _P(_vp), _P(_u64),
                                      C.c_float, _vp]),
    "plora_engine_config_default": (None, [_P(plora_engine_config)]),
    "plora_engine_create": (_int, [_vp, _P(plora_engine_config), _P(_vp)]),
    "plora_engine_destroy": (None, [_vp]),
    "plora_engine_set_source": (_int, [_vp, _u32, _vp, _u64]),
    "plora_engine_attach_predictor": (_int, [_vp, _vp, _int]),
    "plora_engine_flush_predictor": (_int, [_vp]),
    "plora_engine_on_arrival": (_int, [_vp, _u32, _dbl, _vp]),
    "plora_engine_round": (_int, [_vp, _dbl, _vp]),
    "plora_engine_set_predictions": (_int, [_vp, _P(_dbl), _u64]),
    "plora_engine_acquire": (_int, [_vp, _u32, _dbl, _vp]),
    "plora_engine_wait_ready": (_int, [_vp, _u32, _vp]),
    "plora_engine_release": (_int, [_vp, _u32]),
    "plora_engine_boundary": (_int, [_vp, _dbl, _vp]),
    "plora_engine_sync": (_int, [_vp]),
    "plora_engine_on_arrivals": (_i64, [_vp, _P(_u32), _u64, _dbl, _vp]),
    "plora_engine_admit": (_int, [_vp, _P(_u32), _u64, _dbl, _vp, _int, _P(_i32)]),
    "plora_engine_release_many": (_int, [_vp, _P(_u32), _u64]),
    "plora_engine_status": (_int, [_vp, _u32, _P(plora_dynamics)]),
    "plora_engine_decisions": (_u64, [_vp, _u64, _P(plora_decision), _u64]),
    "plora_engine_set_decision_log": (_int, [_vp, C.c_int]),
    "plora_engine_set_accuracy_interval": (_int, [_vp, C.c_double, C.c_double]),
    "plora_engine_get_stats": (None, [_vp, _P(plora_engine_stats)]),
    "plora_engine_streams": (_int, [_vp, _P(_vp), _P(_vp)]),
    "plora_lstm_config_default": (None, [_P(plora_lstm_config)]),
    "plora_predictor_config_default": (None, [_P(plora_predictor_config)]),
    "plora_cross_entropy": (_int, [_P(_dbl), _P(_dbl), _u64, _P(_dbl)]),
    "plora_lstm_create": (_int, [_P(plora_lstm_config), _u64, _P(_vp)]),
    "plora_lstm_destroy": (None, [_vp]),
    "plora_lstm_param_count": (_u64, [_vp]),
    "plora_lstm_parameters": (_P(_dbl), [_vp]),
    "plora_lstm_get_config": (None, [_vp, _P(plora_lstm_config)]),
    "plora_lstm_forward": (_int, [_vp, _P(_u32), _P(_dbl), _u64, _P(_dbl)]),
    "plora_lstm_loss": (_int, [_vp, _P(_u32), _P(_dbl), _P(_dbl), _u64, _P(_dbl)]),
    "plora_lstm_gradient": (_int, [_vp, _P(_u32), _P(_dbl), _P(_dbl), _u64, _P(_dbl)]),
    "plora_lstm_train_step": (_int, [_vp, _P(_u32), _P(_dbl), _P(_dbl), _u64, _P(_dbl)]),
    "plora_lstm_save": (_int, [_vp, C.c_char_p]),
    "plora_lstm_load": (_int, [C.c_char_p, _P(_vp)]),
    "plora_predictor_create": (_int, [_P(plora_predictor_config), _u64, _P(_vp)]),
    "plora_predictor_destroy": (None, [_vp]),
    "plora_predictor_model": (_vp, [_vp]),
    "plora_predictor_observe": (_int, [_vp, _u32, _dbl]),
    "plora_predictor_roll_to": (_int, [_vp, _dbl]),
    "plora_predictor_train_step": (_int, [_vp, _P(_dbl)]),
    "plora_predictor_set_device": (_int, [_vp, C.c_int]),
    "plora_predictor_predict_all": (_i64, [_vp, _dbl, _P(_u32), _P(_dbl), _u64]),
    "plora_predictor_window": (_int, [_vp, _u32, _P(_dbl)]),
    "plora_predictor_known": (_int, [_vp, _u32]),
    "plora_predictor_stats": (None, [_vp, _P(plora_predictor_stats_t)]),
    "plora_predictor_buffer_at": (_int, [_vp, _u64, _P(_u32), _P(_dbl), _P(_dbl)]),
    "plora_tp_shard_rows": (_u32, [_vp, _u32]),
    "plora_bgmv_tp_shrink": (_int, [_vp, _u32, _u32, _u32, _u32, _vp, _u64, _vp, _vp]),
    "plora_bgmv_tp_expand": (_int, [_vp, _u32, _u32, _u32, _u32, _vp, _vp, _u64, C.c_float, _vp]),
    "plora_bgmv_tp_shrink_push": (_int, [_vp, _u32, _u32, _u32, _u32, _vp, _u64, _vp, _vp, _vp]),
    "plora_bgmv_tp_expand_wait": (_int, [_vp, _u32, _u32, _u32, _u32, _vp, _vp, _vp, _u64,
                                         C.c_float, _vp]),
    "plora_debug_set_trace": (_int, [_vp, _u64]),
    "plora_debug_set_bgmv_impl": (_int, [C.c_int]),
    "plora_debug_set_bgmv_flags": (_int, [_u32]),
    "plora_debug_set_stream_prefetch": (_int, [_u32]),
    "plora_debug_set_route_tokens": (_int, [_u32]),
    "plora_debug_plan_routed": (_int, [C.c_void_p, C.POINTER(_u32)]),
    "plora_debug_set_stream_ctas": (_int, [_u32]),
    "plora_debug_set_hybrid_share": (_int, [C.c_double]),
    "plora_debug_plan_hybrid": (_int, [_vp, _P(C.c_double)]),
    "plora_debug_set_hybrid_per_layer": (_int, [C.c_int]),
    "plora_debug_plan_geom": (_int, [_vp, _u32, _P(_u32)]),
    "plora_debug_set_sgmv_flags": (_int, [_u32]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib() -> C.CDLL:
    """The loaded libplora.so (loads on first use; raises if it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (no CPU fallback exists)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    return lib().plora_last_error().decode("utf-8", "replace")


def check(rc: int) -> int:
    """Map a plora status code onto the reference's exception types."""
    if rc >= 0:
        return rc
    msg = last_error()
    if rc == PLORA_E_VALIDATION:
        raise ValidationError(msg)
    if rc == PLORA_E_CONFIG:
        raise ConfigError(msg)
    if rc == PLORA_E_PARSE:
        raise ParseError(msg)
    if rc == PLORA_E_CUDA:
        raise CudaError(msg)
    if rc == PLORA_E_NOMEM:
        raise MemoryError(msg)
    raise LogicError(msg)


def u32_array(values):
    arr = (C.c_uint32 * max(len(values), 1))()
    for i, v in enumerate(values):
        arr[i] = v
    return arr


def u64_array(values):
    arr = (C.c_uint64 * max(len(values), 1))()
    for i, v in enumerate(values):
        arr[i] = v
    return arr


def f64_array(values):
    arr = (C.c_double * max(len(values), 1))()
    for i, v in enumerate(values):
        arr[i] = v
    return arr


def i32_array(values):
    arr = (C.c_int32 * max(len(values), 1))()
    for i, v in enumerate(values):
        arr[i] = v
    return arr
