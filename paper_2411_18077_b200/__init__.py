"""B200-native MiniKV attention hot path (arXiv 2411.18077).

Four sm_100a CUDA kernels behind the C ABI ``include/minikv_b200.h``:
K1 two-pass selective flash-attention prefill (X_O, LSE, A_cumul),
K2 rectified top-k / pyramid token selection, K3 2-bit quantize + pack,
K4 fused unpack-and-multiply 2-bit decode attention.  ``ops`` mirrors the
reference C++ operator interface (namespace minikv) on torch device tensors.
"""
from ._capi import (CudaError, DomainError, InvalidArgument, MkvError, OutOfRange,  # noqa: F401
                    RuntimeFailure, Unsupported)
from .ops import (AttentionResult, H2OBaselineTrace, KVCache, PersistenceReport, VarianceMode,  # noqa: F401
                  allocate_pyramid, allocate_uniform, allocate_variance, default_scale, h2o_dynamic_baseline,
                  layer_score_variance, persistence_analysis, select_token_counts,
                  select_tokens, selective_flash_attn, synth_fp16, synth_uniform,
                  selective_flash_attn_f32, decode_attention, quantize_block, dequantize)

__all__ = [
    "AttentionResult", "KVCache", "VarianceMode", "allocate_pyramid", "allocate_uniform", "allocate_variance",
    "layer_score_variance", "default_scale", "H2OBaselineTrace", "PersistenceReport", "h2o_dynamic_baseline",
    "persistence_analysis",
    "select_token_counts", "select_tokens", "selective_flash_attn", "synth_fp16", "synth_uniform",
    "MkvError", "InvalidArgument", "DomainError", "RuntimeFailure", "OutOfRange", "CudaError",
    "Unsupported", "selective_flash_attn_f32", "decode_attention", "quantize_block", "dequantize",
]
