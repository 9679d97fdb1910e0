"""Shared helpers for the GPU parity tests (oracle = oracle/ C restatement)."""
from __future__ import annotations

import numpy as np

import oracle

SEED = 2024


def synth_np(seed, stream, shape):
    """Host copy of the synthetic fp16 generator (bit-identical to the device)."""
    n = int(np.prod(shape))
    return oracle.port().synth_fp16(seed, stream, n).reshape(shape)


def f32(x_fp16):
    return np.asarray(x_fp16, dtype=np.float16).astype(np.float32)


def oracle_select(a, hh, rw):
    return oracle.port().select_token_counts(a, hh, rw)[0]


def max_abs(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)))) if np.size(a) else 0.0
