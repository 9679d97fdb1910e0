"""The C ABI library loads and exports every symbol include/minikv_b200.h
declares; host-only entry points work without a GPU; compute entry points
fail loudly (never silently fall back) when no sm_100 device is present.  CPU only.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest
import torch

import oracle
from paper_2411_18077_b200 import _capi

HEADER = _capi.HEADER


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mkv_[a-z0-9_]+)\s*\(", txt)))


def test_header_matches_binding_list():
    assert declared_symbols() == sorted(_capi.EXPORTS)


def test_library_exports_every_declared_symbol():
    assert os.path.exists(_capi.LIB_PATH), "build the library first (__graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (mkv_[a-z0-9_]+)$", out, flags=re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    L = _capi.lib()
    for s in declared_symbols():
        assert hasattr(L, s)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_host_helpers_match_oracle_without_gpu():
    from paper_2411_18077_b200 import allocate_pyramid, allocate_uniform
    P = oracle.port()
    for x, layers, depth, bh in [(3276, 32, 7, True), (70, 8, 7, False), (26214, 32, 7, True), (5, 1, 3, True),
                                 (0, 4, 7, True), (12345, 17, 2, False)]:
        assert allocate_pyramid(x, layers, depth, bh) == list(P.allocate_pyramid(x, layers, depth, bh))
    assert allocate_uniform(33, 32) == list(P.allocate_uniform(33, 32))
    with pytest.raises(_capi.InvalidArgument):
        allocate_pyramid(10, 0)
    with pytest.raises(_capi.InvalidArgument):
        allocate_pyramid(10, 4, 0)


def test_variance_allocation_matches_oracle_without_gpu():  # selection.cpp:85-128 (host, bit-exact)
    from paper_2411_18077_b200 import VarianceMode, allocate_variance
    P = oracle.port()
    rng = np.random.default_rng(11)
    for t in range(200):
        layers, total = int(rng.integers(1, 33)), int(rng.integers(0, 300000))
        v = (rng.random(layers) * 5).astype(np.float32)
        if t % 5 == 0:
            v[:] = 0.0
        for mode in (VarianceMode.Prop, VarianceMode.Inv):
            hh, fb = allocate_variance(v, total, mode)
            exp, efb = P.allocate_variance(v, total, inverse=mode == VarianceMode.Inv)
            assert hh == list(exp) and fb == efb
    with pytest.raises(_capi.InvalidArgument):
        allocate_variance([], 5)
    with pytest.raises(_capi.InvalidArgument):
        allocate_variance([1.0, -0.5], 5)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_compute_calls_fail_loudly_without_device():
    L = _capi.lib()
    caps = (C.c_int32 * 1)(16)
    cfg = _capi.CacheConfig(1, 128, 128, 16, caps, 0, 0)
    h = C.c_void_p()
    st = L.mkv_cache_create(C.byref(cfg), C.byref(h))
    assert st in (_capi.MKV_ERR_UNSUPPORTED, _capi.MKV_ERR_CUDA)
    assert L.mkv_last_error()
    with pytest.raises(_capi.MkvError):
        _capi.check(L.mkv_synth_fp16(C.c_void_p(16), 4, 1, 1, None), "synth")


def test_argument_errors_map_to_reference_exceptions():
    L = _capi.lib()
    caps = (C.c_int32 * 1)(16)
    h = C.c_void_p()
    cfg = _capi.CacheConfig(1, 128, 24, 16, caps, 0, 0)   # n_r % group_size != 0
    with pytest.raises(_capi.InvalidArgument):
        _capi.check(L.mkv_cache_create(C.byref(cfg), C.byref(h)))
    cfg = _capi.CacheConfig(1, 0, 128, 16, caps, 0, 0)    # d == 0
    with pytest.raises(_capi.InvalidArgument):
        _capi.check(L.mkv_cache_create(C.byref(cfg), C.byref(h)))
    a = _capi.PrefillArgs()
    a.len_q, a.len_k, a.causal, a.head_dim = 8, 4, 1, 128     # causal requires lq <= lk
    with pytest.raises(_capi.InvalidArgument):
        _capi.check(L.mkv_prefill_attn(C.byref(a), None))
    a.len_q = 0
    with pytest.raises(_capi.InvalidArgument):
        _capi.check(L.mkv_prefill_attn(C.byref(a), None))
