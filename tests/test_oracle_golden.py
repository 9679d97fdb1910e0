"""Pin the C restatement (oracle/minikv_oracle.c) -- CPU only.

1. Known-answer cases transcribed from the reference's own unit tests
   (proj/tests/test_{attention,quantizer,selection,cache_engine}.cpp).
2. tests/golden/minikv_golden.npz, produced by running the reference itself
   (tests/golden/make_golden.py -> oracle/_ref), compared BIT-EXACTLY.
"""
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "minikv_golden.npz")


@pytest.fixture(scope="module")
def P():
    return oracle.port()


@pytest.fixture(scope="module")
def G():
    return np.load(GOLDEN)


# ---- known answers from the reference test suites ----

def test_single_token_acumul_is_one(P):  # test_attention.cpp:24-33
    rng = np.random.default_rng(1)
    q, k, v = (rng.standard_normal((1, 4)).astype(np.float32) for _ in range(3))
    r = P.selective_flash_attn(q, k, v, 0.5, True, 4, 4)
    assert r.a_cumul[0] == np.float32(1.0)


def test_causal_column_sums_total_rows(P):  # test_attention.cpp:35-45
    x = np.random.default_rng(2).standard_normal((8, 16)).astype(np.float32)
    r = P.selective_flash_attn(x, x, x, 0.25, True, 4, 4)
    assert np.all(r.a_cumul >= 0)
    assert abs(float(np.sum(r.a_cumul, dtype=np.float64)) - 8.0) < 1e-5


def test_aux_memory_linear(P):  # test_attention.cpp:96-108
    prev = 0
    for l in (128, 256, 512, 1024):
        x = np.random.default_rng(l).standard_normal((l, 16)).astype(np.float32)
        r = P.selective_flash_attn(x, x, x, 0.25, True, 32, 32)
        assert r.aux_elements <= 8 * (2 * l) + 32 * 32 + 64
        if prev:
            assert r.aux_elements / prev <= 2.2
        prev = r.aux_elements


def test_decode_attention_trivial(P):  # test_attention.cpp:169-190
    out, attn = P.decode_attention(np.array([1, 2], np.float32), np.array([[2, 4]], np.float32),
                                   np.array([[5, 6]], np.float32), 1.0)
    assert attn[0] == 1.0 and out[0] == 5.0 and out[1] == 6.0
    out, attn = P.decode_attention(np.array([1, 2], np.float32), np.array([[1, 0], [1, 0]], np.float32),
                                   np.array([[1, 0], [0, 1]], np.float32), 1.0)
    assert abs(attn[0] - 0.5) < 1e-6 and abs(out[0] - 0.5) < 1e-6
    with pytest.raises(ValueError):
        P.decode_attention(np.zeros(2, np.float32), np.zeros((0, 2), np.float32), np.zeros((0, 2), np.float32), 1.0)


def test_quantize_known_groups(P):  # test_quantizer.cpp:26-64
    codes, sc, zp = P.quantize_group(np.array([5, 5, 5, 5], np.float32))
    assert sc == 0.0 and zp == 5.0 and np.all(codes == 0)
    codes, sc, zp = P.quantize_group(np.array([0, 1, 2, 3], np.float32))
    assert sc == 1.0 and zp == 0.0 and list(codes) == [0, 1, 2, 3]
    with pytest.raises(ArithmeticError):
        P.quantize_group(np.array([1.0, np.nan, 2.0], np.float32))


def test_pack_known_words(P):  # test_quantizer.cpp:86-104
    assert list(P.pack_codes(np.full(16, 3, np.uint8))) == [0xFFFFFFFF]
    one = np.zeros(16, np.uint8)
    one[0] = 1
    assert list(P.pack_codes(one)) == [1]


def test_short_final_group_param_count(P):  # test_quantizer.cpp:189-202
    m = np.random.default_rng(27).standard_normal((20, 4)).astype(np.float32)
    _, params = P.quantize_block(m, 0)
    assert params.shape[0] == 4 * 2


def test_transpose_duality(P):  # test_quantizer.cpp:158-174
    rng = np.random.default_rng(25)
    for _ in range(20):
        rows, cols = (int(x) for x in rng.integers(1, 41, 2))
        m = (rng.standard_normal((rows, cols)) * 3).astype(np.float32)
        ca, pa = P.quantize_block(m, 1)
        cb, pb = P.quantize_block(np.ascontiguousarray(m.T), 0)
        assert np.array_equal(pa, pb) and np.array_equal(P.pack_codes(ca), P.pack_codes(cb))


def test_selection_known(P):  # test_selection.cpp:13-54
    kept, cl = P.select_token_counts(np.array([4, 3, 2, 1], np.float32), 1, 1)
    assert list(kept) == [0, 3] and not cl
    kept, cl = P.select_token_counts(np.array([1, 2, 3], np.float32), 5, 5)
    assert list(kept) == [0, 1, 2] and cl
    kept, _ = P.select_token_counts(np.ones(6, np.float32), 2, 1)
    assert list(kept) == [0, 1, 5]


def test_pyramid_known(P):  # test_selection.cpp:113-137
    assert list(P.allocate_pyramid(100, 8, 1)) == [100] * 8
    p = P.allocate_pyramid(70, 8, 7)
    assert p[0] == 130 and p[-1] == 10 and 556 <= p.sum() <= 564
    t = P.allocate_pyramid(70, 8, 7, bottom_heavy=False)
    assert t[0] == 10 and t[-1] == 130
    assert list(P.allocate_uniform(33, 32)) == [2] + [1] * 31


def test_variance_allocation_known(P):  # test_selection.cpp:151-179
    for inv in (False, True):
        hh, fb = P.allocate_variance([1, 1, 1, 1], 40, inverse=inv)
        assert list(hh) == [10] * 4 and not fb
    assert list(P.allocate_variance([3, 1], 40)[0]) == [30, 10]
    hh, fb = P.allocate_variance([0, 0, 0], 30)
    assert fb and list(hh) == [10] * 3
    rng = np.random.default_rng(36)
    for _ in range(100):
        layers, total = int(rng.integers(1, 25)), int(rng.integers(0, 3000))
        v = (rng.random(layers) * 4).astype(np.float32)
        for inv in (False, True):
            assert int(P.allocate_variance(v, total, inverse=inv)[0].sum()) == total
    with pytest.raises(ValueError):
        P.allocate_variance([], 10)
    with pytest.raises(ValueError):
        P.allocate_variance([1.0, -1.0], 10)


def test_population_variance_known(P):  # test_selection.cpp:180-196
    assert P.layer_score_variance([5, 5, 5]) == 0.0
    assert P.layer_score_variance([0, 2]) == 1.0
    a = np.random.default_rng(37).standard_normal(64).astype(np.float32)
    assert abs(P.layer_score_variance(a) - float(np.var(a.astype(np.float64)))) < 1e-6


def test_cache_flush_counts(P):  # test_cache_engine.cpp:116-128
    rng = np.random.default_rng(45)
    c = P.cache(d=16, n_r=128)
    c.prefill(rng.standard_normal((16, 16)), rng.standard_normal((16, 16)), np.ones(16), 16, 0)
    for _ in range(1000):
        c.append(rng.standard_normal(16), rng.standard_normal(16))
        assert c.tokens_residual < 128
    _, _, br = c.export(0)
    assert len(br) - 1 == 7 and c.tokens_residual == 104 and c.tokens_quantized + c.tokens_residual == 1016


def test_cache_errors(P):  # test_cache_engine.cpp:36-41,74-78
    with pytest.raises(ValueError):
        P.cache(d=16, n_r=24)
    c = P.cache(d=16, n_r=128)
    with pytest.raises(RuntimeError):
        c.prefill(np.zeros((4, 16)), np.zeros((4, 16)), np.ones(4), 0, 0)
    with pytest.raises(RuntimeError):
        c.decode_step(np.zeros(16), np.zeros(16), np.zeros(16), 1.0)


# ---- golden fixtures produced by the reference itself ----

def test_golden_attention(P, G):
    i = 0
    while f"att{i}_shape" in G:
        lq, lk, d, causal, bm, bn = (int(x) for x in G[f"att{i}_shape"])
        r = P.selective_flash_attn(G[f"att{i}_q"], G[f"att{i}_k"], G[f"att{i}_v"], 1.0 / np.sqrt(d),
                                   bool(causal), bm, bn)
        np.testing.assert_array_equal(r.output, G[f"att{i}_out"])
        np.testing.assert_array_equal(r.lse, G[f"att{i}_lse"])
        np.testing.assert_array_equal(r.a_cumul, G[f"att{i}_acumul"])
        i += 1
    assert i >= 7
    o, a = P.decode_attention(G["dec_q"], G["dec_k"], G["dec_v"], 1.0 / np.sqrt(8))
    np.testing.assert_array_equal(o, G["dec_out"])
    np.testing.assert_array_equal(a, G["dec_attn"])


def test_golden_quantizer(P, G):
    i = 0
    while f"qm{i}_m" in G:
        m = G[f"qm{i}_m"]
        for axis in (0, 1):
            codes, params = P.quantize_block(m, axis)
            np.testing.assert_array_equal(P.pack_codes(codes), G[f"qm{i}_ax{axis}_words"])
            np.testing.assert_array_equal(params, G[f"qm{i}_ax{axis}_params"])
            deq = P.dequantize_block(codes, params, m.shape[0], m.shape[1], axis)
            np.testing.assert_array_equal(deq, G[f"qm{i}_ax{axis}_deq"])
        i += 1
    assert i >= 5


def test_golden_selection(P, G):
    i = 0
    while f"sel{i}_a" in G:
        hh, rw = (int(x) for x in G[f"sel{i}_args"])
        kept, cl = P.select_token_counts(G[f"sel{i}_a"], hh, rw)
        np.testing.assert_array_equal(kept, G[f"sel{i}_kept"])
        assert cl == bool(G[f"sel{i}_clamped"][0])
        i += 1
    j = 0
    while f"pyr{j}_args" in G:
        x, layers, depth, bh = (int(v) for v in G[f"pyr{j}_args"])
        np.testing.assert_array_equal(P.allocate_pyramid(x, layers, depth, bool(bh)), G[f"pyr{j}_out"])
        j += 1
    assert i >= 5 and j >= 6


def test_golden_cache_engine(P, G):
    hh, rw = (int(x) for x in G["cache_args"])
    c = P.cache(d=128, n_r=128)
    c.prefill(G["cache_k"], G["cache_v"], G["cache_a"], hh, rw)
    tq, tk, tv = G["cache_tq"], G["cache_tk"], G["cache_tv"]
    for s in range(tq.shape[0]):
        out = c.decode_step(tq[s], tk[s], tv[s], 1.0 / np.sqrt(128))
        np.testing.assert_array_equal(out, G["cache_out"][s])
    for which in (0, 1):
        w, p, br = c.export(which)
        np.testing.assert_array_equal(w, G[f"cache_ex{which}_words"])
        np.testing.assert_array_equal(p, G[f"cache_ex{which}_params"])
        np.testing.assert_array_equal(br, G[f"cache_ex{which}_blocks"])


def test_synth_generator_stats(P):
    x = P.synth_fp16(2024, 5, 200000).astype(np.float64)
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1.0) < 0.01
