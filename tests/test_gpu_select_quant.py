"""K2 (selection) and K3 (quantize + pack) on the B200 vs the oracle: bit-exact.

Selection: select_token_counts (selection.cpp:10-33), ties to the lower index.
Quantizer: prefill -> append_block PerChannel K / PerToken V
(quantizer.cpp:102-136), compared through the reference-format export.
"""
import numpy as np
import pytest
import torch

import oracle
from tests.gpu_util import SEED, f32, oracle_select

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mkv():
    import paper_2411_18077_b200 as m
    return m


def _ties(rng, n, levels):
    return (rng.integers(0, levels, n).astype(np.float32) * np.float32(0.125))


@pytest.mark.parametrize("L,hh,rw,kind", [
    (256, 64, 64, "uniform"), (1000, 100, 100, "ties"), (4096, 409, 409, "uniform"),
    (777, 0, 50, "uniform"), (777, 50, 0, "ties"), (100, 95, 10, "uniform"),  # clamped
    (300, 300, 0, "ties"), (1, 1, 0, "uniform"), (65536, 6553, 6553, "ties"),
    (5000, 2500, 100, "allequal"), (32768, 6084, 3276, "uniform"),
])
def test_select_matches_oracle(mkv, L, hh, rw, kind):
    rng = np.random.default_rng(L * 7 + hh)
    if kind == "uniform":
        a = rng.random(L).astype(np.float32)
    elif kind == "ties":
        a = _ties(rng, L, 7)
    else:
        a = np.ones(L, np.float32)
    a[rng.integers(0, L, max(1, L // 50))] = 0.0
    a[rng.integers(0, L, max(1, L // 97))] = -0.0
    ta = torch.from_numpy(a).cuda()
    kept, nk = mkv.select_token_counts(ta, hh, rw)
    got = kept.cpu().numpy().astype(np.int64)
    exp = oracle_select(a, hh, rw)
    assert nk == len(exp)
    np.testing.assert_array_equal(got, exp)


def test_select_batched_units(mkv):
    rng = np.random.default_rng(5)
    n, L = 37, 3000
    a = _ties(rng, n * L, 40).reshape(n, L)
    hh = [int(x) for x in rng.integers(0, 1500, n)]
    kept, nks = mkv.select_token_counts(torch.from_numpy(a).cuda(), hh, 200)
    kept = kept.cpu().numpy()
    for u in range(n):
        exp = oracle_select(a[u], hh[u], 200)
        np.testing.assert_array_equal(kept[u, :nks[u]], exp)


def _prefill_case(mkv, L, hh, rw, n_units, fp32_params, dist_scale=1.0):
    rng = np.random.default_rng(L + hh + rw)
    d = 128
    k = (rng.standard_normal((n_units, L, d)) * dist_scale).astype(np.float16)
    v = (rng.standard_normal((n_units, L, d)) * dist_scale).astype(np.float16)
    a = rng.random((n_units, L)).astype(np.float32)
    cap = min(hh + rw, L)
    cache = mkv.KVCache(n_units, cap, max_decode_tokens=256, keep_fp32_params=fp32_params)
    cache.prefill(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(a).cuda(), hh, rw)
    cache.check()
    return cache, k, v, a


@pytest.mark.parametrize("L,hh,rw", [(300, 40, 30), (1000, 100, 100), (64, 16, 16), (37, 5, 3),
                                     (4096, 409, 409), (20, 100, 0)])
@pytest.mark.parametrize("fp32_params", [True, False])
def test_prefill_pack_bit_exact(mkv, L, hh, rw, fp32_params):
    n_units = 3
    cache, k, v, a = _prefill_case(mkv, L, hh, rw, n_units, fp32_params)
    P = oracle.port()
    for u in range(n_units):
        oc = P.cache()
        oc.prefill(f32(k[u]), f32(v[u]), a[u], hh, rw)
        for which in (0, 1):
            w_ref, p_ref, br_ref = oc.export(which)
            w, p, br = cache.export_reference(u, which)
            np.testing.assert_array_equal(br, br_ref)
            np.testing.assert_array_equal(w, w_ref)  # codes: bit-exact
            if fp32_params:
                np.testing.assert_array_equal(p, p_ref)
            else:
                np.testing.assert_array_equal(p, p_ref.astype(np.float16).astype(np.float32))


def test_flush_blocks_bit_exact(mkv):
    """decode_append flushes a full n_r block into 2-bit pages (cache_engine.cpp:79-90)."""
    L, hh, rw, n_units, d = 500, 60, 45, 2, 128
    cache, k, v, a = _prefill_case(mkv, L, hh, rw, n_units, True)
    P = oracle.port()
    ocs = []
    for u in range(n_units):
        oc = P.cache()
        oc.prefill(f32(k[u]), f32(v[u]), a[u], hh, rw)
        ocs.append(oc)
    rng = np.random.default_rng(9)
    for step in range(300):
        tk = rng.standard_normal((n_units, d)).astype(np.float16)
        tv = rng.standard_normal((n_units, d)).astype(np.float16)
        cache.append(torch.from_numpy(tk).cuda(), torch.from_numpy(tv).cuda())
        for u in range(n_units):
            ocs[u].append(f32(tk[u]), f32(tv[u]))
    cache.check()
    for u in range(n_units):
        info = cache.unit_info(u)
        assert info["tokens_quantized"] == ocs[u].tokens_quantized == hh + rw + 256
        assert info["tokens_residual"] == ocs[u].tokens_residual == 300 - 256
        for which in (0, 1):
            w_ref, p_ref, br_ref = ocs[u].export(which)
            w, p, br = cache.export_reference(u, which)
            np.testing.assert_array_equal(br, br_ref)
            np.testing.assert_array_equal(w, w_ref)
            np.testing.assert_array_equal(p, p_ref)
        rk, rv = cache.export_residual(u)
        ork, orv = ocs[u].residual()
        np.testing.assert_array_equal(rk.astype(np.float32), ork)
        np.testing.assert_array_equal(rv.astype(np.float32), orv)


def test_nonfinite_input_is_domain_error(mkv):
    L, d = 64, 128
    k = np.zeros((1, L, d), np.float16)
    v = np.zeros((1, L, d), np.float16)
    k[0, 3, 7] = np.float16(np.inf)
    a = np.ones((1, L), np.float32)
    cache = mkv.KVCache(1, L, 0)
    cache.prefill(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(a).cuda(), L, 0)
    with pytest.raises(mkv.DomainError):
        cache.check()


def test_prefill_errors(mkv):
    cache = mkv.KVCache(1, 64, 0)
    k = torch.zeros((1, 64, 128), dtype=torch.float16, device="cuda")
    a = torch.ones((1, 64), dtype=torch.float32, device="cuda")
    with pytest.raises(mkv.RuntimeFailure):   # zero kept tokens (cache_engine.cpp:66-68)
        cache.prefill(k, k, a, 0, 0)
    with pytest.raises(mkv.InvalidArgument):  # make_cache: n_r not a multiple of group_size
        mkv.KVCache(1, 64, 0, n_r=24)
    with pytest.raises(mkv.RuntimeFailure):   # decode_step on an empty cache
        q = torch.zeros((1, 1, 128), dtype=torch.float16, device="cuda")
        cache.decode_step(q, None, None, 0.1)


def test_synth_matches_oracle(mkv):
    t = mkv.synth_fp16((4, 1000), SEED, 12345, 7).cpu().numpy()
    for r in range(4):
        exp = oracle.port().synth_fp16(SEED, 12345 + 7 * r, 1000)
        np.testing.assert_array_equal(t[r].view(np.uint16), exp.view(np.uint16))
    u = mkv.synth_uniform((2, 500), SEED, 99, 1).cpu().numpy()
    for r in range(2):
        np.testing.assert_array_equal(u[r], oracle.port().synth_uniform(SEED, 99 + r, 500))


@pytest.mark.parametrize("kind", ["half_points", "tiny_range", "huge_range", "constant_rows", "near_thresholds",
                                  "signed_zero", "subnormal"])
def test_quantizer_rounding_edges_bit_exact(mkv, kind):
    """Quotients on/near the .5 rounding points, tiny and huge group ranges, constant groups:
    codes and params must equal the reference's exact fp32 arithmetic (quantizer.cpp:28-53)."""
    rng = np.random.default_rng(77)
    L, d = 160, 128
    if kind == "half_points":   # values on a 0.5 grid: many quotients exactly k + 0.5
        k = (rng.integers(0, 7, (1, L, d)) * 0.5).astype(np.float16)
    elif kind == "tiny_range":
        k = (1000.0 + rng.integers(0, 4, (1, L, d)) * 0.5).astype(np.float16)
    elif kind == "huge_range":
        k = (rng.standard_normal((1, L, d)) * 3000.0).astype(np.float16)
    elif kind == "near_thresholds":  # values at (j + 0.5) / 3 of the range, nudged by +-1, 2 fp16 ulps
        base = rng.standard_normal((1, L, d)).astype(np.float16)
        span = np.abs(rng.standard_normal((1, 1, d))).astype(np.float16) + np.float16(0.25)
        frac = rng.choice(np.array([0.0, 0.5 / 3, 1.5 / 3, 2.5 / 3, 1.0], np.float32), (1, L, d))
        k = (base * 0 + (span * frac)).astype(np.float16)
        k[:, ::16] = np.float16(0.0)   # every 16-token group holds its minimum ...
        k[:, 1::16] = span             # ... and its maximum
        nudge = rng.integers(-2, 3, (1, L, d)).astype(np.int16)
        bits = k.view(np.int16) + nudge * (rng.random((1, L, d)) < 0.5)
        bits[:, ::16] = k.view(np.int16)[:, ::16]
        bits[:, 1::16] = k.view(np.int16)[:, 1::16]
        k = bits.astype(np.int16).view(np.float16)
        k[~np.isfinite(k)] = np.float16(0.0)
    elif kind == "signed_zero":  # +0 / -0 as group minima / maxima: the first one wins (std::min/max)
        k = rng.choice(np.array([-0.0, 0.0, 0.0, -0.0, 0.5, -0.5, 1.0], np.float16), (1, L, d))
        k[:, ::5] = np.where(rng.random((1, (L + 4) // 5, d)) < 0.5, np.float16(-0.0), np.float16(0.0))
    elif kind == "subnormal":  # fp16 subnormals and zeros: the smallest scales
        k = (rng.integers(-3, 4, (1, L, d)) * 2.0 ** -24).astype(np.float16)
    else:
        k = np.repeat(rng.standard_normal((1, L, 1)).astype(np.float16), d, axis=2)
    v = k[:, ::-1].copy()
    a = rng.random((1, L)).astype(np.float32)
    cache = mkv.KVCache(1, L, 0, keep_fp32_params=True)
    cache.prefill(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(a).cuda(), L, 0)
    cache.check()
    oc = oracle.port().cache()
    oc.prefill(f32(k[0]), f32(v[0]), a[0], L, 0)
    for which in (0, 1):
        w, p, br = cache.export_reference(0, which)
        w_ref, p_ref, br_ref = oc.export(which)
        np.testing.assert_array_equal(w, w_ref)
        np.testing.assert_array_equal(p, p_ref)


@pytest.mark.parametrize("cluster", ["0", "2", "8", "16"])
@pytest.mark.parametrize("L,hh,rw,kind", [
    (131072, 13107, 13107, "ties"), (131072, 65536, 0, "uniform"), (65536, 100, 3000, "allequal"),
    (40000, 19999, 1, "ties"),
])
def test_select_cluster_path_matches_oracle(mkv, monkeypatch, cluster, L, hh, rw, kind):
    """Few long units (configs[3]: 8 x 128K) take the thread-block-cluster radix select;
    every cluster size gives the single-CTA kernel's (= the reference's) indices."""
    monkeypatch.setenv("MKV_SELECT_CLUSTER", cluster)
    rng = np.random.default_rng(L + hh + int(cluster))
    n = 3
    if kind == "uniform":
        a = rng.random((n, L)).astype(np.float32)
    elif kind == "ties":
        a = _ties(rng, n * L, 5).reshape(n, L)
    else:
        a = np.ones((n, L), np.float32)
    a[:, rng.integers(0, L, L // 50)] = -0.0
    kept, nks = mkv.select_token_counts(torch.from_numpy(a).cuda(), hh, rw)
    kept = kept.cpu().numpy()
    for u in range(n):
        np.testing.assert_array_equal(kept[u, :nks[u]], oracle_select(a[u], hh, rw))



def test_layer_score_variance_device(mkv):
    """layer_score_variance (selection.cpp:130-146) on the device, batched over rows.
    Known answers are exact; random rows agree with the oracle to 1e-6 relative (the
    device sums in a fixed tree order instead of index order, both in fp64)."""
    P = oracle.port()
    assert float(mkv.layer_score_variance(torch.tensor([5.0, 5.0, 5.0]).cuda())) == 0.0
    assert float(mkv.layer_score_variance(torch.tensor([0.0, 2.0]).cuda())) == 1.0
    rng = np.random.default_rng(12)
    for L in (1, 7, 1000, 32768, 131072):
        a = (rng.random((5, L)) ** 3).astype(np.float32)
        got = mkv.layer_score_variance(torch.from_numpy(a).cuda()).cpu().numpy()
        for u in range(5):
            exp = P.layer_score_variance(a[u])
            assert abs(got[u] - exp) <= 1e-6 * max(abs(exp), 1e-30), (L, u, got[u], exp)
