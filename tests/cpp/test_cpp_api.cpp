// test_cpp_api.cpp -- the C++ host API (include/minikv_b200.hpp) against the oracle
// (oracle/minikv_oracle.c, the C restatement pinned to the reference), written like
// the reference's own unit tests (proj/tests/test_{selection,attention,cache_engine}.cpp):
// known answers first, then seeded random cases.  Needs an sm_100 GPU; run by
// tests/test_gpu_cpp_api.py.  Exit status = number of failed checks.
#include <cmath>
#include <cstdio>
#include <functional>
#include <numeric>
#include <random>
#include <stdexcept>
#include <vector>

#include "minikv_b200.hpp"
extern "C" {
#include "minikv_oracle.h"
}

namespace mk = minikv_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                             \
    do {                                                                        \
        ++g_checks;                                                             \
        if (!(cond)) {                                                          \
            ++g_fail;                                                           \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);         \
        }                                                                       \
    } while (0)
template <typename E>
static bool throws(const std::function<void()>& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static std::vector<float> fp16_values(std::mt19937& rng, size_t n) {  // device-representable inputs
    std::normal_distribution<float> nd(0.0f, 1.0f);
    std::vector<float> v(n);
    for (auto& x : v) x = mko_round_fp16(nd(rng));
    return v;
}

static void test_selection() {  // test_selection.cpp:13-54, 113-196
    auto s = mk::select_token_counts({4, 3, 2, 1}, 1, 1);
    CHECK((s.kept == std::vector<size_t>{0, 3}) && !s.clamped);
    CHECK((s.hh == std::vector<size_t>{0}) && (s.rw == std::vector<size_t>{3}));
    s = mk::select_token_counts({1, 2, 3}, 5, 5);
    CHECK(s.clamped && (s.kept == std::vector<size_t>{0, 1, 2}));
    s = mk::select_token_counts(std::vector<float>(6, 1.0f), 2, 1);  // all equal: lowest indices
    CHECK((s.hh == std::vector<size_t>{0, 1}) && (s.rw == std::vector<size_t>{5}));
    s = mk::select_tokens({4, 3, 2, 1}, mk::CacheBudget{0.25, 0.25}, 4);
    CHECK((s.kept == std::vector<size_t>{0, 3}));
    CHECK(throws<std::invalid_argument>([] { mk::select_tokens({1, 2}, mk::CacheBudget{0.1, 0.1}, 3); }));
    std::mt19937 rng(1);
    for (int t = 0; t < 20; ++t) {
        const size_t l = 1 + rng() % 5000, hh = rng() % (l + 10), rw = rng() % (l / 2 + 1);
        std::vector<float> a(l);
        for (auto& x : a) x = (float)(rng() % 23) * 0.125f;  // heavy ties
        s = mk::select_token_counts(a, hh, rw);
        std::vector<int64_t> kept(l + 1);
        size_t nk = 0;
        int clamped = 0;
        mko_select_token_counts(a.data(), l, hh, rw, kept.data(), &nk, nullptr, nullptr, nullptr, nullptr, &clamped);
        bool same = nk == s.kept.size() && clamped == (int)s.clamped;
        for (size_t i = 0; same && i < nk; ++i) same = (size_t)kept[i] == s.kept[i];
        CHECK(same);
    }
    auto p = mk::allocate_pyramid(70, 8, 7);
    CHECK(p.per_layer_hh.front() == 130 && p.per_layer_hh.back() == 10);
    CHECK((mk::allocate_pyramid(100, 8, 1).per_layer_hh == std::vector<size_t>(8, 100)));
    CHECK((mk::allocate_variance({1, 1, 1, 1}, 40, mk::VarianceMode::Inv).per_layer_hh == std::vector<size_t>(4, 10)));
    CHECK((mk::allocate_variance({3, 1}, 40, mk::VarianceMode::Prop).per_layer_hh == std::vector<size_t>{30, 10}));
    auto z = mk::allocate_variance({0, 0, 0}, 30, mk::VarianceMode::Prop);
    CHECK(z.uniform_fallback && (z.per_layer_hh == std::vector<size_t>(3, 10)));
    CHECK(throws<std::invalid_argument>([] { mk::allocate_variance({1, -1}, 10, mk::VarianceMode::Prop); }));
    CHECK(mk::layer_score_variance({5, 5, 5}) == 0.0f);
    CHECK(mk::layer_score_variance({0, 2}) == 1.0f);
    CHECK(throws<std::invalid_argument>([] { mk::layer_score_variance({}); }));
}

static void test_attention() {  // test_attention.cpp:24-45, 110-135 at the device tolerances
    std::mt19937 rng(2);
    const size_t d = 128;
    {  // l = 1: the only key gets all the attention
        mk::Matrix q(1, d), k(1, d), v(1, d);
        q.data = fp16_values(rng, d); k.data = fp16_values(rng, d); v.data = fp16_values(rng, d);
        auto r = mk::selective_flash_attn(q, k, v, mk::default_scale(d), true);
        CHECK(std::fabs(r.a_cumul[0] - 1.0f) < 1e-5f);
        bool same = true;
        for (size_t c = 0; c < d; ++c) same &= std::fabs(r.output.at(0, c) - v.at(0, c)) < 1e-3f;
        CHECK(same);
    }
    for (auto [lq, lk, causal] : {std::tuple<size_t, size_t, bool>{300, 300, true}, {100, 400, true},
                                  {257, 190, false}}) {
        mk::Matrix q(lq, d), k(lk, d), v(lk, d);
        q.data = fp16_values(rng, lq * d); k.data = fp16_values(rng, lk * d); v.data = fp16_values(rng, lk * d);
        const float sc = mk::default_scale(d);
        auto r = mk::selective_flash_attn(q, k, v, sc, causal);
        std::vector<float> out(lq * d), lse(lq), ac(lk);
        size_t aux = 0;
        mko_selective_flash_attn(q.data.data(), k.data.data(), v.data.data(), lq, lk, d, d, sc, causal, 64, 64,
                                 out.data(), lse.data(), ac.data(), &aux);
        float eo = 0, el = 0;
        bool acok = true;
        double sum = 0;
        for (size_t i = 0; i < lq * d; ++i) eo = std::fmax(eo, std::fabs(out[i] - r.output.data[i]));
        for (size_t i = 0; i < lq; ++i) el = std::fmax(el, std::fabs(lse[i] - r.lse[i]));
        for (size_t j = 0; j < lk; ++j) {
            acok &= std::fabs(ac[j] - r.a_cumul[j]) <= 1e-3f + 2e-3f * std::fabs(ac[j]);
            sum += r.a_cumul[j];
        }
        CHECK(eo <= 5e-3f);
        CHECK(el <= 1e-3f);
        CHECK(acok);
        CHECK(std::fabs(sum - (double)lq) <= 1e-3 * lq);  // columns sum to the number of query rows
        CHECK(r.aux_elements <= 2 * (lq + lk));            // linear auxiliary memory
    }
    CHECK(throws<std::invalid_argument>([] {
        mk::Matrix q(8, 128), k(4, 128), v(4, 128);
        mk::selective_flash_attn(q, k, v, 0.1f, true);  // causal needs l_query <= l_key
    }));
}

static bool same_tensor(const mk::QuantizedTensor& t, const mko_cache* oc, int which) {
    const size_t nw = (mko_cache_total_codes(oc, which) + 15) / 16, np = mko_cache_n_params(oc, which);
    std::vector<uint32_t> w(nw + 1);
    std::vector<float> p(2 * np + 2);
    std::vector<int64_t> br(mko_cache_n_blocks(oc) + 1);
    mko_cache_export(oc, which, w.data(), p.data(), br.data());
    if (t.packed_words.size() != nw || t.params.size() != np || t.block_rows.size() != mko_cache_n_blocks(oc))
        return false;
    for (size_t i = 0; i < nw; ++i)
        if (w[i] != t.packed_words[i]) return false;
    for (size_t g = 0; g < np; ++g)
        if (!(p[2 * g] == t.params[g].scale && p[2 * g + 1] == t.params[g].zero_point)) return false;
    for (size_t b = 0; b < t.block_rows.size(); ++b)
        if ((size_t)br[b] != t.block_rows[b]) return false;
    return true;
}

static void test_cache() {  // test_cache_engine.cpp:64-128, 154-218 at the device tolerances
    std::mt19937 rng(3);
    const size_t d = 128, l = 500, hh = 60, rw = 40, n_r = 128;
    mk::Matrix k(l, d), v(l, d);
    k.data = fp16_values(rng, l * d);
    v.data = fp16_values(rng, l * d);
    std::vector<float> a(l);
    for (auto& x : a) x = (float)(rng() % 1000) / 997.0f;
    auto [cache, rep] = mk::prefill(k, v, a, hh, rw, n_r);
    mko_cache* oc = nullptr;
    mko_cache_create(d, n_r, 16, &oc);
    mko_cache_prefill(oc, k.data.data(), v.data.data(), a.data(), l, hh, rw);
    CHECK(rep.kept.kept.size() == hh + rw && rep.bytes_before == 4ull * l * d);
    CHECK(cache.tokens_quantized() == hh + rw && cache.tokens_residual() == 0);
    CHECK(same_tensor(cache.q_key(), oc, 0));    // codes, params and block rows bit-exact
    CHECK(same_tensor(cache.q_value(), oc, 1));
    CHECK(rep.bytes_after == mk::measured_bytes(cache));
    const float sc = mk::default_scale(d);
    float worst = 0.0f;
    for (int s = 0; s < 300; ++s) {  // through two n_r flushes
        auto q = fp16_values(rng, d), tk = fp16_values(rng, d), tv = fp16_values(rng, d);
        auto out = mk::decode_step(cache, q, tk, tv, sc);
        std::vector<float> exp(d);
        mko_cache_decode_step(oc, q.data(), tk.data(), tv.data(), sc, 1, exp.data());
        for (size_t c = 0; c < d; ++c) worst = std::fmax(worst, std::fabs(out[c] - exp[c]));
    }
    CHECK(worst <= 5e-3f);
    CHECK(cache.tokens_quantized() == mko_cache_tokens_quantized(oc));
    CHECK(cache.tokens_residual() == mko_cache_tokens_residual(oc));
    CHECK(same_tensor(cache.q_key(), oc, 0) && same_tensor(cache.q_value(), oc, 1));
    {  // stored_keys = dequantize_matrix(q_key), and the residual rows round-trip exactly
        auto sk = mk::stored_keys(cache);
        CHECK(sk.rows == cache.tokens_quantized() && sk.cols == d);
        auto rk = cache.r_key();
        std::vector<float> ork(mko_cache_tokens_residual(oc) * d), orv(ork.size());
        mko_cache_residual(oc, ork.data(), orv.data());
        CHECK(rk.data == ork);
    }
    mko_cache_destroy(oc);
    {  // 1000 appends from an empty cache: 7 flushed blocks, 104 residual rows
        auto c = mk::make_cache(d, n_r);
        auto t = fp16_values(rng, d);
        for (int i = 0; i < 1000; ++i) mk::decode_append(c, t, t);
        CHECK(c.tokens_quantized() == 7 * 128 && c.tokens_residual() == 104);
        CHECK(c.q_key().block_rows.size() == 7);
    }
    CHECK(throws<std::invalid_argument>([] { mk::make_cache(128, 24, 16); }));  // n_r % group != 0
    CHECK(throws<std::runtime_error>([&] { mk::prefill(k, v, a, 0, 0, n_r); }));  // zero kept
    CHECK(throws<std::invalid_argument>([&] { mk::decode_append(cache, std::vector<float>(3), std::vector<float>(3)); }));
    CHECK(throws<std::domain_error>([&] {
        mk::Matrix kn = k;
        kn.at(l - 1, 5) = NAN;  // a kept (RW) token is non-finite: quantize_group throws
        mk::prefill(kn, v, a, hh, rw, n_r);
    }));
}

int main() {
    test_selection();
    test_attention();
    test_cache();
    std::printf("%s: %d checks, %d failed\n", g_fail ? "FAILED" : "OK", g_checks, g_fail);
    return g_fail;
}
