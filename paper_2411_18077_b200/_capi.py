"""ctypes binding of the C ABI in include/minikv_b200.h.

Loads the in-tree ``libminikv_b200.so`` (built by ``make -C paper_2411_18077_b200``
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing, or the device is not sm_100, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MKV_LIB_PATH") or os.path.join(HERE, "libminikv_b200.so")  # override: A/B builds
HEADER = os.path.join(os.path.dirname(HERE), "include", "minikv_b200.h")

MKV_OK = 0
MKV_ERR_INVALID_ARGUMENT = 1
MKV_ERR_DOMAIN = 2
MKV_ERR_RUNTIME = 3
MKV_ERR_OUT_OF_RANGE = 4
MKV_ERR_CUDA = 5
MKV_ERR_UNSUPPORTED = 6


class MkvError(Exception):
    """Base class; subclasses mirror the reference's exception types."""

    status = -1


class InvalidArgument(MkvError, ValueError):      # std::invalid_argument
    status = MKV_ERR_INVALID_ARGUMENT


class DomainError(MkvError, ArithmeticError):     # std::domain_error
    status = MKV_ERR_DOMAIN


class RuntimeFailure(MkvError, RuntimeError):     # std::runtime_error
    status = MKV_ERR_RUNTIME


class OutOfRange(MkvError, IndexError):           # std::out_of_range
    status = MKV_ERR_OUT_OF_RANGE


class CudaError(MkvError, RuntimeError):
    status = MKV_ERR_CUDA


class Unsupported(MkvError, RuntimeError):
    status = MKV_ERR_UNSUPPORTED


_BY_STATUS = {c.status: c for c in (InvalidArgument, DomainError, RuntimeFailure, OutOfRange,
                                    CudaError, Unsupported)}

i64 = C.c_int64
i32 = C.c_int
vp = C.c_void_p


class PrefillArgs(C.Structure):
    _fields_ = [("q", vp), ("q_sb", i64), ("q_sh", i64), ("q_st", i64),
                ("k", vp), ("k_sb", i64), ("k_sh", i64), ("k_st", i64),
                ("v", vp), ("v_sb", i64), ("v_sh", i64), ("v_st", i64),
                ("out", vp), ("o_sb", i64), ("o_sh", i64), ("o_st", i64),
                ("lse", vp), ("a_cumul", vp),
                ("batch", i32), ("n_q_heads", i32), ("n_kv_heads", i32), ("len_q", i32),
                ("len_k", i32), ("head_dim", i32), ("scale", C.c_float), ("causal", i32)]


class AttnF32Args(C.Structure):
    _fields_ = [("q", vp), ("ld_q", i64), ("k", vp), ("ld_k", i64), ("v", vp), ("ld_v", i64),
                ("out", vp), ("ld_o", i64), ("lse", vp), ("a_cumul", vp),
                ("len_q", i32), ("len_k", i32), ("d", i32), ("dv", i32), ("scale", C.c_float), ("causal", i32)]


class SelectArgs(C.Structure):
    _fields_ = [("a_cumul", vp), ("a_stride", i64), ("n_units", i32), ("length", i32),
                ("hh_count", C.POINTER(C.c_int32)), ("rw_count", i32), ("kept", vp),
                ("kept_stride", i64), ("n_kept", vp)]


class CacheConfig(C.Structure):
    _fields_ = [("n_units", i32), ("head_dim", i32), ("n_r", i32), ("group_size", i32),
                ("prefill_capacity", C.POINTER(C.c_int32)), ("max_decode_tokens", i32),
                ("keep_fp32_params", i32)]


class CachePrefillArgs(C.Structure):
    _fields_ = [("unit_begin", i32), ("n_units", i32),
                ("k", vp), ("k_su", i64), ("k_st", i64),
                ("v", vp), ("v_su", i64), ("v_st", i64),
                ("kept", vp), ("kept_stride", i64), ("n_kept_host", C.POINTER(C.c_int32))]


class PrefillSelectArgs(C.Structure):
    _fields_ = [("unit_begin", i32), ("n_units", i32), ("length", i32),
                ("a_cumul", vp), ("a_stride", i64), ("hh_count", C.POINTER(C.c_int32)),
                ("rw_count", i32),
                ("k", vp), ("k_su", i64), ("k_st", i64),
                ("v", vp), ("v_su", i64), ("v_st", i64)]


class H2OArgs(C.Structure):
    _fields_ = [("prompt_k", vp), ("ld_k", i64), ("prompt_scores", vp), ("qs", vp), ("ks", vp),
                ("l_prompt", i32), ("d", i32), ("steps", i32), ("hh_budget", i64), ("rw_budget", i64),
                ("scale", C.c_float), ("kept", vp), ("kept_stride", i64), ("kept_count", vp)]


class DecodeArgs(C.Structure):
    _fields_ = [("unit_begin", i32), ("n_units", i32), ("group", i32),
                ("q", vp), ("k_new", vp), ("v_new", vp), ("out", vp), ("scale", C.c_float)]


class DecodeStepsArgs(C.Structure):
    _fields_ = [("unit_begin", i32), ("n_units", i32), ("group", i32), ("n_steps", i32),
                ("q", vp), ("q_step", C.c_int64), ("k_new", vp), ("v_new", vp), ("kv_step", C.c_int64),
                ("out", vp), ("out_step", C.c_int64), ("scale", C.c_float)]


# every symbol the header declares (checked by tests/test_capi_symbols.py)
EXPORTS = [
    "mkv_last_error", "mkv_abi_version", "mkv_device_check",
    "mkv_prefill_attn", "mkv_select", "mkv_allocate_pyramid", "mkv_allocate_uniform",
    "mkv_allocate_variance", "mkv_score_variance",
    "mkv_cache_create", "mkv_cache_destroy", "mkv_cache_bytes", "mkv_cache_unit_info",
    "mkv_cache_prefill", "mkv_cache_prefill_select", "mkv_decode_step", "mkv_cache_append",
    "mkv_decode_step_layers", "mkv_decode_steps", "mkv_debug_decode_trace", "mkv_debug_launch_count", "mkv_decode_pages_only", "mkv_cache_export_sizes", "mkv_cache_export_reference",
    "mkv_cache_export_residual", "mkv_cache_check", "mkv_cache_save_mkvc", "mkv_cache_load_mkvc",
    "mkv_synth_fp16", "mkv_synth_fp16_rows", "mkv_synth_uniform_f32", "mkv_h2o_dynamic_baseline",
    "mkv_attention_f32", "mkv_decode_attention_f32", "mkv_quantize_block_f32", "mkv_dequantize_f32"]

_lib = None


def lib():
    """The loaded C ABI (raises if the in-tree library was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build with `make -C paper_2411_18077_b200` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.mkv_last_error.restype = C.c_char_p
    L.mkv_prefill_attn.argtypes = [C.POINTER(PrefillArgs), vp]
    L.mkv_select.argtypes = [C.POINTER(SelectArgs), vp]
    L.mkv_allocate_pyramid.argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, i32, C.POINTER(C.c_int64)]
    L.mkv_allocate_uniform.argtypes = [C.c_size_t, C.c_size_t, C.POINTER(C.c_int64)]
    L.mkv_allocate_variance.argtypes = [vp, C.c_size_t, C.c_size_t, i32, C.POINTER(C.c_int64), C.POINTER(C.c_int)]
    L.mkv_score_variance.argtypes = [vp, i64, i32, i32, vp, vp]
    if hasattr(L, "mkv_h2o_dynamic_baseline"):
        L.mkv_h2o_dynamic_baseline.argtypes = [C.POINTER(H2OArgs), vp]
    L.mkv_cache_create.argtypes = [C.POINTER(CacheConfig), C.POINTER(vp)]
    L.mkv_cache_destroy.argtypes = [vp]
    L.mkv_cache_bytes.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    L.mkv_cache_unit_info.argtypes = [vp, i32] + [C.POINTER(C.c_int64)] * 4
    L.mkv_cache_prefill.argtypes = [vp, C.POINTER(CachePrefillArgs), vp]
    L.mkv_cache_prefill_select.argtypes = [vp, C.POINTER(PrefillSelectArgs), vp]
    L.mkv_decode_step.argtypes = [vp, C.POINTER(DecodeArgs), vp]
    L.mkv_decode_pages_only.argtypes = [vp, C.POINTER(DecodeArgs), vp]
    L.mkv_decode_step_layers.argtypes = [vp, i32, C.POINTER(DecodeArgs), vp]
    L.mkv_decode_steps.argtypes = [vp, C.POINTER(DecodeStepsArgs), vp]
    L.mkv_cache_append.argtypes = [vp, i32, i32, vp, vp, vp]
    L.mkv_cache_export_sizes.argtypes = [vp, i32, i32] + [C.POINTER(C.c_int64)] * 3
    L.mkv_cache_export_reference.argtypes = [vp, i32, i32, vp, vp, vp]
    L.mkv_cache_export_residual.argtypes = [vp, i32, vp, vp]
    L.mkv_cache_check.argtypes = [vp]
    L.mkv_cache_save_mkvc.argtypes = [vp, i32, C.c_char_p]
    L.mkv_cache_load_mkvc.argtypes = [vp, i32, C.c_char_p]
    if hasattr(L, "mkv_debug_decode_trace"):  # diagnostics entry (absent in older A/B builds)
        L.mkv_debug_decode_trace.argtypes = [vp, vp, i32]
    if hasattr(L, "mkv_debug_launch_count"):
        L.mkv_debug_launch_count.argtypes = []
        L.mkv_debug_launch_count.restype = C.c_uint64
    L.mkv_synth_fp16.argtypes = [vp, i64, C.c_uint64, C.c_uint64, vp]
    L.mkv_synth_fp16_rows.argtypes = [vp, i64, i64, i64, C.c_uint64, C.c_uint64, C.c_uint64, vp]
    L.mkv_synth_uniform_f32.argtypes = [vp, i64, i64, i64, C.c_uint64, C.c_uint64, C.c_uint64, vp]
    L.mkv_attention_f32.argtypes = [C.POINTER(AttnF32Args), vp]
    L.mkv_decode_attention_f32.argtypes = [vp, vp, i64, vp, i64, i32, i32, i32, C.c_float, vp, vp, vp]
    L.mkv_quantize_block_f32.argtypes = [vp, i64, vp, i32, i32, i32, i32, i64, C.c_uint32, vp, vp, vp]
    L.mkv_dequantize_f32.argtypes = [vp, vp, C.POINTER(C.c_int64), i32, i32, i32, i32, vp, i64, vp]
    _lib = L
    return L


def check(status: int, what: str = ""):
    if status != MKV_OK:
        msg = lib().mkv_last_error().decode(errors="replace")
        raise _BY_STATUS.get(status, MkvError)(f"{what}: {msg}" if what else msg)
