"""MKVC snapshots (snapshot.cpp:71-198) of device caches.

* save: a device cache (fp32 params kept) written as MKVC is byte-identical to the
  reference's save_cache of the reference cache built from the same fp16 inputs
  (oracle/_ref = the unmodified reference sources) -- through a prefill block with a
  partial page, two n_r flushes and a residual;
* load: the reference's file loaded into a fresh device unit exports the same streams
  and then decodes bit-identically to the device cache it came from;
* errors keep the reference's classes (bad magic / truncation -> std::runtime_error).
"""
import os

import numpy as np
import pytest
import torch

import oracle
from tests.gpu_util import f32

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def mkv():
    import paper_2411_18077_b200 as m
    return m


def _build(mkv, rng, L=700, hh=70, rw=61, steps=280, n_r=128):
    d = 128
    k = rng.standard_normal((L, d)).astype(np.float16)
    v = rng.standard_normal((L, d)).astype(np.float16)
    a = rng.random(L).astype(np.float32)
    dev = mkv.KVCache(2, hh + rw, max_decode_tokens=steps + 2 * n_r, n_r=n_r, keep_fp32_params=True)
    dev.prefill(torch.from_numpy(k)[None].cuda(), torch.from_numpy(v)[None].cuda(), torch.from_numpy(a)[None].cuda(),
                hh, rw)
    ref = oracle.ref().cache_prefill(f32(k), f32(v), a, hh, rw, n_r=n_r)
    for _ in range(steps):
        tk = rng.standard_normal((1, d)).astype(np.float16)
        tv = rng.standard_normal((1, d)).astype(np.float16)
        dev.append(torch.from_numpy(tk).cuda(), torch.from_numpy(tv).cuda())
        ref.append(f32(tk[0]), f32(tv[0]))
    dev.check()
    return dev, ref


def test_save_matches_reference_bytes(mkv, tmp_path):
    dev, ref = _build(mkv, np.random.default_rng(1))
    p_dev, p_ref = str(tmp_path / "dev.mkvc"), str(tmp_path / "ref.mkvc")
    dev.save_mkvc(0, p_dev)
    ref.save(p_ref)
    a, b = open(p_dev, "rb").read(), open(p_ref, "rb").read()
    assert a[:4] == b"MKVC" and len(a) == len(b)
    assert a == b


def test_load_reference_snapshot_then_decode(mkv, tmp_path):
    rng = np.random.default_rng(2)
    dev, ref = _build(mkv, rng, steps=150)
    path = str(tmp_path / "ref.mkvc")
    ref.save(path)
    dev.load_mkvc(1, path)  # unit 1 (empty so far) <- the reference's cache
    i0, i1 = dev.unit_info(0), dev.unit_info(1)
    assert i0 == i1
    for which in (0, 1):
        w0, p0, b0 = dev.export_reference(0, which)
        w1, p1, b1 = dev.export_reference(1, which)
        rw_, rp_, rb_ = ref.export(which)
        assert np.array_equal(w1, rw_) and np.array_equal(p1.reshape(-1), rp_.reshape(-1)) and list(b1) == list(rb_)
        assert np.array_equal(w0, w1) and np.array_equal(p0, p1)
    r0, v0 = dev.export_residual(0)
    r1, v1 = dev.export_residual(1)
    assert np.array_equal(r0, r1) and np.array_equal(v0, v1)
    d = 128
    for _ in range(140):  # both units decode identically, through another flush
        q = torch.from_numpy(rng.standard_normal((1, 4, d)).astype(np.float16)).cuda()
        tk = torch.from_numpy(rng.standard_normal((1, d)).astype(np.float16)).cuda()
        tv = torch.from_numpy(rng.standard_normal((1, d)).astype(np.float16)).cuda()
        o0 = dev.decode_step(q, tk, tv, 0.088, unit_begin=0)
        o1 = dev.decode_step(q, tk, tv, 0.088, unit_begin=1)
        assert torch.equal(o0, o1)


def test_snapshot_errors(mkv, tmp_path):
    dev = mkv.KVCache(1, 32, max_decode_tokens=16)
    bad = tmp_path / "bad.mkvc"
    bad.write_bytes(b"XXXX" + b"\0" * 60)
    with pytest.raises(mkv.RuntimeFailure):
        dev.load_mkvc(0, str(bad))
    rng = np.random.default_rng(3)
    src, ref = _build(mkv, rng, L=100, hh=10, rw=10, steps=3)
    good = str(tmp_path / "good.mkvc")
    ref.save(good)
    data = open(good, "rb").read()
    (tmp_path / "trunc.mkvc").write_bytes(data[: len(data) // 2])
    with pytest.raises(mkv.RuntimeFailure):
        dev.load_mkvc(0, str(tmp_path / "trunc.mkvc"))
    other = mkv.KVCache(1, 32, max_decode_tokens=16, n_r=64)  # n_r differs from the snapshot
    with pytest.raises(mkv.InvalidArgument):
        other.load_mkvc(0, good)
    with pytest.raises(mkv.RuntimeFailure):
        dev.load_mkvc(0, str(tmp_path / "missing.mkvc"))
