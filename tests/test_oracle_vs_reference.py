"""The C restatement vs the reference itself (oracle/_ref, compiled from the
unmodified sources): bit-identical on fresh seeded inputs.  CPU only; skipped
where the reference .so could not be built (the golden fixtures then pin it).
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def PR():
    return oracle.port(), oracle.ref()


def test_attention_random_shapes(PR):  # mirrors acceptance.cpp:103-142 (210 random cases)
    P, R = PR
    rng = np.random.default_rng(7)
    for _ in range(60):
        d = int(rng.choice([8, 16, 64, 128]))
        lk = int(rng.integers(1, 200))
        lq = int(rng.integers(1, lk + 1))
        causal = bool(rng.integers(0, 2))
        bm, bn = int(rng.integers(1, 97)), int(rng.integers(1, 97))
        q = rng.standard_normal((lq, d)).astype(np.float32)
        k = rng.standard_normal((lk, d)).astype(np.float32)
        v = rng.standard_normal((lk, d)).astype(np.float32)
        a = P.selective_flash_attn(q, k, v, 1 / np.sqrt(d), causal, bm, bn)
        b = R.selective_flash_attn(q, k, v, 1 / np.sqrt(d), causal, bm, bn)
        assert np.array_equal(a.output, b.output) and np.array_equal(a.lse, b.lse)
        assert np.array_equal(a.a_cumul, b.a_cumul) and a.aux_elements == b.aux_elements


def test_quantizer_random(PR):
    P, R = PR
    rng = np.random.default_rng(8)
    for _ in range(100):
        rows, cols = int(rng.integers(1, 140)), int(rng.integers(1, 140))
        m = (rng.standard_normal((rows, cols)) * rng.uniform(0.01, 100)).astype(np.float32)
        if rng.random() < 0.2:
            m = np.round(m)  # many exact-tie / constant groups
        for axis in (0, 1):
            codes, params = P.quantize_block(m, axis)
            w, p = R.quantize_matrix(m, axis)
            assert np.array_equal(P.pack_codes(codes), w) and np.array_equal(params, p)


def test_selection_random(PR):
    P, R = PR
    rng = np.random.default_rng(9)
    for _ in range(200):
        L = int(rng.integers(1, 3000))
        a = rng.random(L).astype(np.float32)
        if rng.random() < 0.5:
            a = np.floor(a * 6).astype(np.float32)
        hh, rw = int(rng.integers(0, L + 5)), int(rng.integers(0, L // 2 + 2))
        assert np.array_equal(P.select_token_counts(a, hh, rw)[0], R.select_token_counts(a, hh, rw)[0])


def test_pyramid_random(PR):
    P, R = PR
    rng = np.random.default_rng(10)
    for _ in range(300):
        x, layers, depth = int(rng.integers(0, 60000)), int(rng.integers(1, 80)), int(rng.integers(1, 12))
        bh = bool(rng.integers(0, 2))
        assert np.array_equal(P.allocate_pyramid(x, layers, depth, bh), R.allocate_pyramid(x, layers, depth, bh))


def test_cache_decode_random(PR):
    P, R = PR
    rng = np.random.default_rng(11)
    for trial in range(4):
        L, d = int(rng.integers(20, 400)), int(rng.choice([16, 64, 128]))
        n_r = int(rng.choice([16, 32, 128]))
        hh, rw = int(rng.integers(0, L)), int(rng.integers(1, L // 2 + 2))
        k = rng.standard_normal((L, d)).astype(np.float32)
        v = rng.standard_normal((L, d)).astype(np.float32)
        a = rng.random(L).astype(np.float32)
        pc = P.cache(d=d, n_r=n_r)
        pc.prefill(k, v, a, hh, rw)
        rc = R.cache_prefill(k, v, a, hh, rw, n_r=n_r)
        for s in range(int(rng.integers(1, 2 * n_r + 10))):
            tq, tk, tv = (rng.standard_normal(d).astype(np.float32) for _ in range(3))
            assert np.array_equal(pc.decode_step(tq, tk, tv, 0.1), rc.decode_step(tq, tk, tv, 0.1))
        for which in (0, 1):
            for x, y in zip(pc.export(which), rc.export(which)):
                assert np.array_equal(x, y)


def test_variance_allocation_random(PR):  # selection.cpp:85-146, bit-identical allocations
    P, R = PR
    rng = np.random.default_rng(9)
    for t in range(300):
        layers, total = int(rng.integers(1, 40)), int(rng.integers(0, 100000))
        v = (rng.random(layers) * (10.0 ** rng.integers(-6, 4))).astype(np.float32)
        if t % 7 == 0:
            v[rng.integers(0, layers)] = 0.0
        if t % 11 == 0:
            v[:] = v[0]  # equal shares -> fraction ties resolved to the lower layer
        for inv in (False, True):
            a, fa = P.allocate_variance(v, total, inverse=inv)
            b, fb = R.allocate_variance(v, total, inverse=inv)
            assert np.array_equal(a, b) and fa == fb
    for _ in range(50):
        a = (rng.random(int(rng.integers(1, 5000))) * 3).astype(np.float32)
        assert P.layer_score_variance(a) == R.layer_score_variance(a)


def test_h2o_dynamic_baseline_random(PR):  # harness.cpp:83-150: identical kept sets at every step
    P, R = PR
    rng = np.random.default_rng(41)
    for _ in range(40):
        l = int(rng.integers(1, 300))
        d = int(rng.choice([2, 8, 16, 64, 128]))
        steps = int(rng.integers(0, 60))
        hh, rw = int(rng.integers(0, 200)), int(rng.integers(0, 50))
        hh = max(hh, 1 - rw)
        pk = rng.standard_normal((l, d)).astype(np.float32)
        sc = rng.random(l).astype(np.float32)
        qs = rng.standard_normal((steps, d)).astype(np.float32)
        ks = rng.standard_normal((steps, d)).astype(np.float32)
        assert P.h2o_dynamic_baseline(pk, sc, qs, ks, hh, rw, 1 / np.sqrt(d)) == \
            R.h2o_dynamic_baseline(pk, sc, qs, ks, hh, rw, 1 / np.sqrt(d))
