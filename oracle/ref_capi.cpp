// ref_capi.cpp -- TEST / BASELINE INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper around the UNMODIFIED MiniKV reference library,
// compiled from its own sources under /root/reference/proj/core/src by
// oracle/Makefile into oracle/_ref/libminikv_ref.so.  The reference namespace
// is renamed with -Dminikv=minikv_ref so this .so can sit beside the product
// library in one process.  Nothing here re-implements reference logic: every
// entry point forwards to the reference symbol named in its comment.  Used by
//   * tests/ to pin the C restatement (oracle/minikv_oracle.c) bit-for-bit,
//   * tests/golden/make_golden.py to write golden fixtures,
//   * bench.py --impl reference / cpu_baseline to time the reference CPU path
//     on the GPU box's host cores (std::thread pool over independent units,
//     legal per SPEC.md:144,401 -- distinct caches are independent).
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "minikv/attention.hpp"
#include "minikv/cache_engine.hpp"
#include "minikv/harness.hpp"
#include "minikv/snapshot.hpp"
#include "minikv/quantizer.hpp"
#include "minikv/selection.hpp"
#include "minikv_oracle.h"

using namespace minikv;  // expands to minikv_ref

namespace {

int status_of(const std::exception_ptr& e) {
    try {
        std::rethrow_exception(e);
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::domain_error&) {
        return 2;
    } catch (const std::out_of_range&) {
        return 4;
    } catch (const std::runtime_error&) {
        return 3;
    } catch (...) {
        return 5;
    }
}

#define GUARD(...)                                   \
    try {                                            \
        __VA_ARGS__;                                 \
    } catch (...) {                                  \
        return status_of(std::current_exception());  \
    }                                                \
    return 0;

Matrix mat(const float* p, std::size_t r, std::size_t c) {
    Matrix m(r, c);
    if (r * c) std::memcpy(m.data.data(), p, sizeof(float) * r * c);
    return m;
}

}  // namespace

extern "C" {

// attention.cpp:29-117
int mkr_selective_flash_attn(const float* q, const float* k, const float* v, size_t lq, size_t lk,
                             size_t d, size_t dv, float scale, int causal, size_t bm, size_t bn,
                             float* out, float* lse, float* a_cumul, size_t* aux) {
    GUARD({
        AttentionResult r = selective_flash_attn(mat(q, lq, d), mat(k, lk, d), mat(v, lk, dv),
                                                 scale, causal != 0, TileConfig{bm, bn});
        std::memcpy(out, r.output.data.data(), sizeof(float) * lq * dv);
        std::memcpy(lse, r.lse.data(), sizeof(float) * lq);
        std::memcpy(a_cumul, r.a_cumul.data(), sizeof(float) * lk);
        if (aux) *aux = r.aux_elements;
    })
}

// attention.cpp:119-143
int mkr_decode_attention(const float* q, const float* keys, const float* values, size_t n,
                         size_t d, size_t dv, float scale, float* out, float* attn) {
    GUARD({
        auto [o, a] = decode_attention(Vector(q, q + d), mat(keys, n, d), mat(values, n, dv), scale);
        std::memcpy(out, o.data(), sizeof(float) * dv);
        std::memcpy(attn, a.data(), sizeof(float) * n);
    })
}

// quantizer.cpp:28-53
int mkr_quantize_group(const float* values, size_t n, uint8_t* codes, float* scale, float* zero) {
    GUARD({
        auto [c, p] = quantize_group(std::span<const float>(values, n));
        std::memcpy(codes, c.data(), c.size());
        *scale = p.scale;
        *zero = p.zero_point;
    })
}

// quantizer.cpp:67-77
int mkr_pack_codes(const uint8_t* codes, size_t n, uint32_t* words) {
    GUARD({
        auto w = pack_codes(std::span<const std::uint8_t>(codes, n));
        std::memcpy(words, w.data(), sizeof(uint32_t) * w.size());
    })
}

// quantize_matrix / append_block (quantizer.cpp:102-151): packed stream + params.
int mkr_quantize_matrix(const float* m, size_t rows, size_t cols, int axis, size_t gs,
                        uint32_t* words, size_t* n_words, float* params, size_t* n_groups) {
    GUARD({
        QuantizedTensor t = quantize_matrix(mat(m, rows, cols),
                                            axis == 0 ? GroupAxis::PerChannel : GroupAxis::PerToken,
                                            gs);
        std::memcpy(words, t.packed_words.data(), sizeof(uint32_t) * t.packed_words.size());
        *n_words = t.packed_words.size();
        for (std::size_t i = 0; i < t.params.size(); ++i) {
            params[2 * i] = t.params[i].scale;
            params[2 * i + 1] = t.params[i].zero_point;
        }
        *n_groups = t.params.size();
    })
}

// dequantize_matrix (quantizer.cpp:153-195) of quantize_matrix(m).
int mkr_quant_dequant_matrix(const float* m, size_t rows, size_t cols, int axis, size_t gs,
                             float* out) {
    GUARD({
        QuantizedTensor t = quantize_matrix(mat(m, rows, cols),
                                            axis == 0 ? GroupAxis::PerChannel : GroupAxis::PerToken,
                                            gs);
        Matrix back = dequantize_matrix(t);
        std::memcpy(out, back.data.data(), sizeof(float) * rows * cols);
    })
}

// selection.cpp:10-33
int mkr_select_token_counts(const float* a, size_t l, size_t hh, size_t rw, int64_t* kept,
                            size_t* n_kept, int* clamped) {
    GUARD({
        SelectionResult s = select_token_counts(Vector(a, a + l), hh, rw);
        for (std::size_t i = 0; i < s.kept.size(); ++i) kept[i] = static_cast<int64_t>(s.kept[i]);
        *n_kept = s.kept.size();
        *clamped = s.clamped ? 1 : 0;
    })
}

// selection.cpp:61-83
int mkr_allocate_pyramid(size_t x, size_t layers, size_t depth, int bottom_heavy, int64_t* out) {
    GUARD({
        LayerAllocation a = allocate_pyramid(
            x, layers, depth,
            bottom_heavy ? PyramidOrientation::BottomHeavy : PyramidOrientation::TopHeavy);
        for (std::size_t i = 0; i < layers; ++i) out[i] = static_cast<int64_t>(a.per_layer_hh[i]);
    })
}

// selection.cpp:48-59
int mkr_allocate_uniform(size_t total, size_t layers, int64_t* out) {
    GUARD({
        LayerAllocation a = allocate_uniform(total, layers);
        for (std::size_t i = 0; i < layers; ++i) out[i] = static_cast<int64_t>(a.per_layer_hh[i]);
    })
}

// selection.cpp:85-128
int mkr_allocate_variance(const float* variance, size_t layers, size_t total, int inverse, int64_t* out,
                          int* uniform_fallback) {
    GUARD({
        LayerAllocation a = allocate_variance(Vector(variance, variance + layers), total,
                                              inverse ? VarianceMode::Inv : VarianceMode::Prop);
        for (std::size_t i = 0; i < layers; ++i) out[i] = static_cast<int64_t>(a.per_layer_hh[i]);
        *uniform_fallback = a.uniform_fallback ? 1 : 0;
    })
}

// selection.cpp:130-146
int mkr_layer_score_variance(const float* a, size_t n, float* out) {
    GUARD({ *out = layer_score_variance(Vector(a, a + n)); })
}

// harness.cpp:108-150
int mkr_h2o_dynamic_baseline(const float* pk, size_t l, size_t d, const float* scores, const float* qs,
                             const float* ks, size_t steps, size_t hh, size_t rw, float scale, int32_t* kept,
                             size_t stride, int32_t* counts) {
    GUARD({
        std::vector<Vector> q, k;
        for (size_t s = 0; s < steps; ++s) {
            q.emplace_back(qs + s * d, qs + (s + 1) * d);
            k.emplace_back(ks + s * d, ks + (s + 1) * d);
        }
        const H2OBaselineTrace t = h2o_dynamic_baseline(mat(pk, l, d), Vector(scores, scores + l), q, k, hh, rw, scale);
        for (size_t s = 0; s < t.kept_per_step.size(); ++s) {
            counts[s] = static_cast<int32_t>(t.kept_per_step[s].size());
            for (size_t i = 0; i < t.kept_per_step[s].size(); ++i)
                kept[s * stride + i] = static_cast<int32_t>(t.kept_per_step[s][i]);
        }
    })
}

// ---- cache engine: an opaque KVCacheLayer handle ----

struct mkr_cache {
    KVCacheLayer layer;
};

// cache_engine.cpp:56-77
int mkr_cache_prefill(const float* k, const float* v, const float* a, size_t l, size_t d,
                      size_t hh, size_t rw, size_t n_r, size_t gs, mkr_cache** out) {
    GUARD({
        auto [cache, rep] = prefill(mat(k, l, d), mat(v, l, d), Vector(a, a + l), hh, rw, n_r, gs);
        *out = new mkr_cache{std::move(cache)};
    })
}

void mkr_cache_destroy(mkr_cache* c) { delete c; }

// cache_engine.cpp:79-90
int mkr_cache_append(mkr_cache* c, const float* tk, const float* tv) {
    GUARD({ decode_append(c->layer, Vector(tk, tk + c->layer.d), Vector(tv, tv + c->layer.d)); })
}

// cache_engine.cpp:100-138
int mkr_cache_decode_step(mkr_cache* c, const float* tq, const float* tk, const float* tv,
                          float scale, float* out) {
    GUARD({
        const std::size_t d = c->layer.d;
        Vector o = decode_step(c->layer, Vector(tq, tq + d), Vector(tk, tk + d), Vector(tv, tv + d),
                               scale);
        std::memcpy(out, o.data(), sizeof(float) * d);
    })
}

// snapshot.cpp:71-198
int mkr_cache_save(const mkr_cache* c, const char* path) { GUARD({ save_cache(c->layer, std::string(path)); }) }
int mkr_cache_load(const char* path, mkr_cache** out) {
    GUARD({ *out = new mkr_cache{load_cache(std::string(path))}; })
}

size_t mkr_cache_tokens_quantized(const mkr_cache* c) { return c->layer.tokens_quantized; }
size_t mkr_cache_tokens_residual(const mkr_cache* c) { return c->layer.tokens_residual(); }

// QuantizedTensor fields of the cache (which 0 = q_key, 1 = q_value).
size_t mkr_cache_n_words(const mkr_cache* c, int which) {
    return (which ? c->layer.q_value : c->layer.q_key).packed_words.size();
}
size_t mkr_cache_n_params(const mkr_cache* c, int which) {
    return (which ? c->layer.q_value : c->layer.q_key).params.size();
}
size_t mkr_cache_n_blocks(const mkr_cache* c) { return c->layer.q_key.block_rows.size(); }
int mkr_cache_export(const mkr_cache* c, int which, uint32_t* words, float* params,
                     int64_t* block_rows) {
    const QuantizedTensor& t = which ? c->layer.q_value : c->layer.q_key;
    std::memcpy(words, t.packed_words.data(), sizeof(uint32_t) * t.packed_words.size());
    for (std::size_t i = 0; i < t.params.size(); ++i) {
        params[2 * i] = t.params[i].scale;
        params[2 * i + 1] = t.params[i].zero_point;
    }
    for (std::size_t i = 0; i < t.block_rows.size(); ++i) block_rows[i] = static_cast<int64_t>(t.block_rows[i]);
    return 0;
}

// ---- timing drivers for the CPU baseline (bench.py) ----
// Each unit is an independent (seq, layer, kv-head) cache.  GQA decode of one
// unit = decode_append once, stored_keys/stored_values once (the reference's
// full dequantize), then decode_attention per q-head over [stored ; residual]
// (bit-identical to decode_step for G = 1).

struct mkr_decode_set {
    std::vector<KVCacheLayer> units;
    std::size_t d = 0, g = 1;
};

namespace {
// Synthetic inputs shared bit-for-bit with the GPU run (oracle/minikv_oracle.h).
void synth_floats(uint64_t seed, uint64_t stream, std::size_t n, float* out) {
    std::vector<uint16_t> h(n);
    mko_synth_fp16(seed, stream, n, h.data());
    for (std::size_t i = 0; i < n; ++i) out[i] = mko_half_bits_to_float(h[i]);
}
void synth_uniform(uint64_t seed, uint64_t stream, std::size_t n, float* out) {
    for (std::size_t i = 0; i < n; ++i)
        out[i] = static_cast<float>(mko_synth_mix(seed, stream, i) >> 40) * (1.0f / 16777216.0f);
}
}  // namespace

// Build n_units caches: unit u (global id unit_ids[u]) keeps hh[u] + rw of l tokens.
// K/V = synthetic fp16 N(0,1) (streams MKV_STREAM(2|3, id, 0)), a_cumul = synthetic
// uniform [0,1) (stream MKV_STREAM(7, id, 0)).
int mkr_decode_set_create(size_t n_units, size_t l, size_t d, size_t g, const int64_t* hh,
                          size_t rw, size_t n_r, size_t gs, uint64_t seed, const uint64_t* unit_ids,
                          int threads, mkr_decode_set** out) {
    GUARD({
        auto* s = new mkr_decode_set;
        s->d = d;
        s->g = g;
        s->units.resize(n_units);
        std::atomic<std::size_t> next{0};
        std::atomic<int> err{0};
        auto worker = [&]() {
            for (std::size_t u; (u = next.fetch_add(1)) < n_units;) {
                try {
                    Matrix km(l, d), vm(l, d);
                    Vector a(l);
                    synth_floats(seed, (2ull << 48) | (unit_ids[u] << 16), l * d, km.data.data());
                    synth_floats(seed, (3ull << 48) | (unit_ids[u] << 16), l * d, vm.data.data());
                    synth_uniform(seed, (7ull << 48) | (unit_ids[u] << 16), l, a.data());
                    auto [cache, rep] = prefill(km, vm, a, static_cast<std::size_t>(hh[u]), rw, n_r, gs);
                    s->units[u] = std::move(cache);
                } catch (...) {
                    err = status_of(std::current_exception());
                }
            }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < (threads > 0 ? threads : 1); ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
        if (err) {
            delete s;
            return err.load();
        }
        *out = s;
    })
}

void mkr_decode_set_destroy(mkr_decode_set* s) { delete s; }

// decode_append (cache_engine.cpp:79-90) of one token per unit: k/v[u][d].
int mkr_decode_set_append(mkr_decode_set* s, const float* k, const float* v, int threads) {
    GUARD({
        const std::size_t n = s->units.size(), d = s->d;
        std::atomic<std::size_t> next{0};
        std::atomic<int> err{0};
        auto worker = [&]() {
            for (std::size_t u; (u = next.fetch_add(1)) < n;) {
                try {
                    decode_append(s->units[u], Vector(k + u * d, k + (u + 1) * d), Vector(v + u * d, v + (u + 1) * d));
                } catch (...) {
                    err = status_of(std::current_exception());
                }
            }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < (threads > 0 ? threads : 1); ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
        if (err) return err.load();
    })
}

// One decode step for every unit: q[u][g][d], k/v[u][d] inputs, out[u][g][d].
// Returns wall seconds in *secs.
int mkr_decode_set_step(mkr_decode_set* s, const float* q, const float* k, const float* v,
                        float scale, float* out, int threads, double* secs) {
    GUARD({
        const std::size_t n = s->units.size(), d = s->d, g = s->g;
        std::atomic<std::size_t> next{0};
        std::atomic<int> err{0};
        auto t0 = std::chrono::steady_clock::now();
        auto worker = [&]() {
            for (std::size_t u; (u = next.fetch_add(1)) < n;) {
                try {
                    KVCacheLayer& c = s->units[u];
                    decode_append(c, Vector(k + u * d, k + (u + 1) * d), Vector(v + u * d, v + (u + 1) * d));
                    Matrix keys = stored_keys(c), vals = stored_values(c);
                    keys.data.insert(keys.data.end(), c.r_key.data.begin(), c.r_key.data.end());
                    keys.rows += c.r_key.rows;
                    vals.data.insert(vals.data.end(), c.r_value.data.begin(), c.r_value.data.end());
                    vals.rows += c.r_value.rows;
                    keys.cols = d;
                    vals.cols = d;
                    for (std::size_t h = 0; h < g; ++h) {
                        const float* qh = q + (u * g + h) * d;
                        auto [o, a] = decode_attention(Vector(qh, qh + d), keys, vals, scale);
                        std::memcpy(out + (u * g + h) * d, o.data(), sizeof(float) * d);
                    }
                } catch (...) {
                    err = status_of(std::current_exception());
                }
            }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < (threads > 0 ? threads : 1); ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
        *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (err) return err.load();
    })
}

// selective_flash_attn (tiles 64x64, attention.hpp:12-15) over n_heads independent
// causal heads of length l on a thread pool.  Head h uses synthetic Q stream
// MKV_STREAM(1, h, 0) and K/V streams MKV_STREAM(2|3, h / g, 0).  Wall seconds in
// *secs; *a_cumul_sum = sum of every head's a_cumul (= n_heads * l, a checksum).
int mkr_prefill_heads(size_t n_heads, size_t g, size_t l, size_t d, uint64_t seed, int threads,
                      double* secs, double* a_cumul_sum) {
    GUARD({
        std::atomic<std::size_t> next{0};
        std::atomic<int> err{0};
        std::vector<double> sums(n_heads, 0.0);
        std::vector<Matrix> qs(n_heads), ks(n_heads), vs(n_heads);
        for (std::size_t h = 0; h < n_heads; ++h) {  // inputs generated outside the timed region
            qs[h] = Matrix(l, d); ks[h] = Matrix(l, d); vs[h] = Matrix(l, d);
            synth_floats(seed, (1ull << 48) | (static_cast<uint64_t>(h) << 16), l * d, qs[h].data.data());
            synth_floats(seed, (2ull << 48) | (static_cast<uint64_t>(h / g) << 16), l * d, ks[h].data.data());
            synth_floats(seed, (3ull << 48) | (static_cast<uint64_t>(h / g) << 16), l * d, vs[h].data.data());
        }
        auto worker = [&]() {
            for (std::size_t h; (h = next.fetch_add(1)) < n_heads;) {
                try {
                    AttentionResult r = selective_flash_attn(
                        qs[h], ks[h], vs[h], 1.0f / std::sqrt(static_cast<float>(d)), true, TileConfig{64, 64});
                    double s = 0.0;
                    for (float x : r.a_cumul) s += x;
                    sums[h] = s;
                } catch (...) {
                    err = status_of(std::current_exception());
                }
            }
        };
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < (threads > 0 ? threads : 1); ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
        *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (a_cumul_sum) {
            double tot = 0.0;
            for (double s : sums) tot += s;
            *a_cumul_sum = tot;
        }
        if (err) return err.load();
    })
}

// The whole single-layer chain the reference CLI runs (minikv_cli.cpp:180-201), per kv-head
// unit h of n_kv (G = g q-heads each), every unit independent on a thread pool:
//   selective_flash_attn (tiles 64x64) per q-head -> a_cumul (GQA: fp32 sum over the unit's
//   q-heads in head order) -> prefill(k, v, a_cumul, hh, rw, n_r, gs) -> `steps` decode
//   iterations: g == 1 -> decode_step (cache_engine.cpp:100-138) itself; g > 1 ->
//   decode_append once + decode_attention per q-head over [stored ; residual].
// Inputs: Q stream (1, hq), K/V (2|3, h), decode q (4, h, s+1) [g*d], k/v (5|6, h, s+1) [d].
// Outputs (any may be null): out[steps][n_kv*g][d], kept[n_kv][kept_stride] + n_kept[n_kv],
// x_o[n_kv*g][l][d].  secs[0..3] = wall seconds of the whole pool, and per-phase thread-time
// sums: attention, prefill (select + gather + quantize), decode.
int mkr_pipeline_run(size_t n_kv, size_t g, size_t l, size_t d, size_t hh, size_t rw, size_t n_r, size_t gs,
                     size_t steps, uint64_t seed, int threads, float* out, int64_t* kept, size_t kept_stride,
                     int64_t* n_kept, float* x_o, double* secs) {
    GUARD({
        std::atomic<std::size_t> next{0};
        std::atomic<int> err{0};
        std::vector<double> t_attn(n_kv, 0.0), t_pre(n_kv, 0.0), t_dec(n_kv, 0.0);
        const float scale = 1.0f / std::sqrt(static_cast<float>(d));
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto dt = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
        auto worker = [&]() {
            for (std::size_t h; (h = next.fetch_add(1)) < n_kv;) {
                try {
                    Matrix km(l, d), vm(l, d);
                    synth_floats(seed, (2ull << 48) | (static_cast<uint64_t>(h) << 16), l * d, km.data.data());
                    synth_floats(seed, (3ull << 48) | (static_cast<uint64_t>(h) << 16), l * d, vm.data.data());
                    Vector acc(l, 0.0f);
                    auto t0 = now();
                    double attn_s = 0.0;
                    for (std::size_t j = 0; j < g; ++j) {
                        const std::size_t hq = h * g + j;
                        Matrix qm(l, d);
                        synth_floats(seed, (1ull << 48) | (static_cast<uint64_t>(hq) << 16), l * d, qm.data.data());
                        auto ta = now();
                        AttentionResult r = selective_flash_attn(qm, km, vm, scale, true, TileConfig{64, 64});
                        attn_s += dt(ta, now());
                        for (std::size_t c = 0; c < l; ++c) acc[c] += r.a_cumul[c];
                        if (x_o) std::memcpy(x_o + hq * l * d, r.output.data.data(), sizeof(float) * l * d);
                    }
                    (void)t0;
                    t_attn[h] = attn_s;
                    auto tp = now();
                    auto [cache, rep] = prefill(km, vm, acc, hh, rw, n_r, gs);
                    t_pre[h] = dt(tp, now());
                    if (kept) {
                        for (std::size_t i = 0; i < rep.kept.kept.size() && i < kept_stride; ++i)
                            kept[h * kept_stride + i] = static_cast<int64_t>(rep.kept.kept[i]);
                    }
                    if (n_kept) n_kept[h] = static_cast<int64_t>(rep.kept.kept.size());
                    Vector tq(g * d), tk(d), tv(d);
                    double dec_s = 0.0;
                    for (std::size_t st = 0; st < steps; ++st) {
                        const uint64_t id = (static_cast<uint64_t>(h) << 16) | (st + 1);
                        synth_floats(seed, (4ull << 48) | id, g * d, tq.data());
                        synth_floats(seed, (5ull << 48) | id, d, tk.data());
                        synth_floats(seed, (6ull << 48) | id, d, tv.data());
                        auto td = now();
                        if (g == 1) {
                            Vector o = decode_step(cache, tq, tk, tv, scale);
                            dec_s += dt(td, now());
                            if (out) std::memcpy(out + (st * n_kv + h) * d, o.data(), sizeof(float) * d);
                        } else {
                            decode_append(cache, tk, tv);
                            Matrix keys = stored_keys(cache), vals = stored_values(cache);
                            keys.data.insert(keys.data.end(), cache.r_key.data.begin(), cache.r_key.data.end());
                            keys.rows += cache.r_key.rows;
                            vals.data.insert(vals.data.end(), cache.r_value.data.begin(), cache.r_value.data.end());
                            vals.rows += cache.r_value.rows;
                            keys.cols = vals.cols = d;
                            for (std::size_t j = 0; j < g; ++j) {
                                auto [o, a] = decode_attention(Vector(tq.begin() + j * d, tq.begin() + (j + 1) * d),
                                                               keys, vals, scale);
                                if (out) std::memcpy(out + ((st * n_kv + h) * g + j) * d, o.data(), sizeof(float) * d);
                            }
                            dec_s += dt(td, now());
                        }
                    }
                    t_dec[h] = dec_s;
                } catch (...) {
                    err = status_of(std::current_exception());
                }
            }
        };
        auto t0 = now();
        std::vector<std::thread> pool;
        for (int t = 0; t < (threads > 0 ? threads : 1); ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
        if (secs) {
            secs[0] = dt(t0, now());
            secs[1] = secs[2] = secs[3] = 0.0;
            for (std::size_t h = 0; h < n_kv; ++h) { secs[1] += t_attn[h]; secs[2] += t_pre[h]; secs[3] += t_dec[h]; }
        }
        if (err) return err.load();
    })
}

}  // extern "C"
