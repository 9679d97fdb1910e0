// minikv_reference_adapter.cpp -- what a maintainer links INTO the reference build to route
// its hot-path declarations (proj/core/include/minikv/*.hpp, unchanged) to the B200 library.
//
// Each definition below has exactly the reference's signature and forwards to the C++ host
// API of include/minikv_b200.hpp; the reference's own CPU definitions of these functions are
// dropped from its build when this file is linked (dropin/Makefile weakens them).  Routed:
//   attention.cpp:29-143     selective_flash_attn, decode_attention  (fp32 device kernels)
//   selection.cpp:10-146     select_token_counts / select_tokens (K2), allocate_*, variance
//   quantizer.cpp:28-151,153 quantize_group, quantize_matrix, append_block, dequantize_matrix
//   cache_engine.cpp:9-138   make_cache, prefill, decode_append, decode_step, stored_keys/values
// The reference's KVCacheLayer is a value type whose public fields the callers read and copy
// (tests, snapshot.cpp, pipeline.cpp), so its state stays in those host fields: each call
// moves them into minikv_b200::value::KVCacheLayer (no copy), runs selection / gather +
// quantize + pack / dequantize / attention on the device, and moves them back.  Left to the
// reference: bit-packing helpers (pack_codes, unpack_codes, push_code, code_at,
// dequantize_group), matrix helpers, accounting, snapshots, the pipeline driver.
#include <stdexcept>

#include "minikv/attention.hpp"
#include "minikv/cache_engine.hpp"
#include "minikv/quantizer.hpp"
#include "minikv/selection.hpp"
#include "minikv_b200.hpp"

namespace minikv {
namespace {
minikv_b200::Matrix to_b200(const Matrix& m) {
    minikv_b200::Matrix r;
    r.rows = m.rows;
    r.cols = m.cols;
    r.data = m.data;
    return r;
}
Matrix from_b200(minikv_b200::Matrix&& m) {
    Matrix r;
    r.rows = m.rows;
    r.cols = m.cols;
    r.data = std::move(m.data);
    return r;
}
// zero-copy moves between the two (field-identical) matrix / tensor types
void move_into(minikv_b200::Matrix& d, Matrix& s) {
    d.rows = s.rows;
    d.cols = s.cols;
    d.data = std::move(s.data);
}
void move_into(Matrix& d, minikv_b200::Matrix& s) {
    d.rows = s.rows;
    d.cols = s.cols;
    d.data = std::move(s.data);
}
minikv_b200::GroupAxis axis_b200(GroupAxis a) {
    return a == GroupAxis::PerChannel ? minikv_b200::GroupAxis::PerChannel : minikv_b200::GroupAxis::PerToken;
}
void move_into(minikv_b200::QuantizedTensor& d, QuantizedTensor& s) {
    d.axis = axis_b200(s.axis);
    d.group_size = s.group_size;
    d.logical_rows = s.logical_rows;
    d.logical_cols = s.logical_cols;
    d.packed_words = std::move(s.packed_words);
    d.params.resize(s.params.size());
    for (std::size_t g = 0; g < s.params.size(); ++g) d.params[g] = {s.params[g].scale, s.params[g].zero_point};
    s.params.clear();
    d.block_rows = std::move(s.block_rows);
    d.total_codes = s.total_codes;
}
void move_into(QuantizedTensor& d, minikv_b200::QuantizedTensor& s) {
    d.axis = s.axis == minikv_b200::GroupAxis::PerChannel ? GroupAxis::PerChannel : GroupAxis::PerToken;
    d.group_size = s.group_size;
    d.logical_rows = s.logical_rows;
    d.logical_cols = s.logical_cols;
    d.packed_words = std::move(s.packed_words);
    d.params.resize(s.params.size());
    for (std::size_t g = 0; g < s.params.size(); ++g) d.params[g] = {s.params[g].scale, s.params[g].zero_point};
    s.params.clear();
    d.block_rows = std::move(s.block_rows);
    d.total_codes = s.total_codes;
}
minikv_b200::QuantizedTensor copy_b200(const QuantizedTensor& t) {
    QuantizedTensor c = t;
    minikv_b200::QuantizedTensor r;
    move_into(r, c);
    return r;
}
using VCache = minikv_b200::value::KVCacheLayer;
minikv_b200::value::QuantMode mode_b200(QuantMode m) {
    return m == QuantMode::Identity ? minikv_b200::value::QuantMode::Identity : minikv_b200::value::QuantMode::TwoBit;
}
void move_into(VCache& d, KVCacheLayer& s) {
    d.d = s.d;
    d.n_r = s.n_r;
    d.group_size = s.group_size;
    d.mode = mode_b200(s.mode);
    move_into(d.q_key, s.q_key);
    move_into(d.q_value, s.q_value);
    move_into(d.fp_key, s.fp_key);
    move_into(d.fp_value, s.fp_value);
    move_into(d.r_key, s.r_key);
    move_into(d.r_value, s.r_value);
    d.tokens_quantized = s.tokens_quantized;
}
void move_into(KVCacheLayer& d, VCache& s) {
    d.d = s.d;
    d.n_r = s.n_r;
    d.group_size = s.group_size;
    d.mode = s.mode == minikv_b200::value::QuantMode::Identity ? QuantMode::Identity : QuantMode::TwoBit;
    move_into(d.q_key, s.q_key);
    move_into(d.q_value, s.q_value);
    move_into(d.fp_key, s.fp_key);
    move_into(d.fp_value, s.fp_value);
    move_into(d.r_key, s.r_key);
    move_into(d.r_value, s.r_value);
    d.tokens_quantized = s.tokens_quantized;
}
// Runs f on the cache's state moved into the B200 value type; the state is moved back whether
// f returns or throws (the reference validates before mutating, so a throwing call leaves the
// cache as it was).
template <typename F>
auto with_state(KVCacheLayer& cache, F&& f) {
    VCache v;
    move_into(v, cache);
    struct Back {
        KVCacheLayer& c;
        VCache& v;
        ~Back() { move_into(c, v); }
    } back{cache, v};
    return f(v);
}
SelectionResult from_b200(const minikv_b200::SelectionResult& s) {
    SelectionResult r;
    r.kept = s.kept;
    r.hh = s.hh;
    r.rw = s.rw;
    r.clamped = s.clamped;
    return r;
}
LayerAllocation from_b200(const minikv_b200::LayerAllocation& a) {
    LayerAllocation r;
    r.per_layer_hh = a.per_layer_hh;
    r.uniform_fallback = a.uniform_fallback;
    return r;
}
}  // namespace

// ---- attention.hpp:38-44 ----
AttentionResult selective_flash_attn(const Matrix& q, const Matrix& k, const Matrix& v, float scale, bool causal,
                                     TileConfig tiles) {
    auto r = minikv_b200::selective_flash_attn_f32(to_b200(q), to_b200(k), to_b200(v), scale, causal,
                                                   minikv_b200::TileConfig{tiles.block_m, tiles.block_n});
    AttentionResult out;
    out.output = from_b200(std::move(r.output));
    out.lse = std::move(r.lse);
    out.a_cumul = std::move(r.a_cumul);
    out.aux_elements = r.aux_elements;
    return out;
}

std::pair<Vector, Vector> decode_attention(const Vector& q_row, const Matrix& keys, const Matrix& values,
                                           float scale) {
    return minikv_b200::decode_attention(q_row, to_b200(keys), to_b200(values), scale);
}

// ---- selection.hpp:30-59 ----
SelectionResult select_token_counts(const Vector& a_cumul, std::size_t hh_count, std::size_t rw_count) {
    return from_b200(minikv_b200::select_token_counts(a_cumul, hh_count, rw_count));
}

SelectionResult select_tokens(const Vector& a_cumul, const CacheBudget& budget, std::size_t l_prompt) {
    return from_b200(
        minikv_b200::select_tokens(a_cumul, minikv_b200::CacheBudget{budget.alpha_hh, budget.alpha_rw}, l_prompt));
}

LayerAllocation allocate_uniform(std::size_t total_hh, std::size_t layers) {
    return from_b200(minikv_b200::allocate_uniform(total_hh, layers));
}

LayerAllocation allocate_pyramid(std::size_t mean_budget_x, std::size_t layers, std::size_t depth_d,
                                 PyramidOrientation orientation) {
    return from_b200(minikv_b200::allocate_pyramid(mean_budget_x, layers, depth_d,
                                                   orientation == PyramidOrientation::BottomHeavy
                                                       ? minikv_b200::PyramidOrientation::BottomHeavy
                                                       : minikv_b200::PyramidOrientation::TopHeavy));
}

LayerAllocation allocate_variance(const Vector& per_layer_variance, std::size_t total_hh, VarianceMode mode) {
    return from_b200(minikv_b200::allocate_variance(
        per_layer_variance, total_hh,
        mode == VarianceMode::Prop ? minikv_b200::VarianceMode::Prop : minikv_b200::VarianceMode::Inv));
}

float layer_score_variance(const Vector& a_cumul) { return minikv_b200::layer_score_variance(a_cumul); }

// ---- quantizer.hpp:44-68 ----
std::pair<std::vector<std::uint8_t>, GroupQuantParams> quantize_group(std::span<const float> values) {
    if (values.empty()) throw std::invalid_argument("quantize_group: empty group");
    // one group = a 1 x n PerToken block with group size n, quantized on the device
    minikv_b200::Matrix m(1, values.size());
    std::copy(values.begin(), values.end(), m.data.begin());
    const minikv_b200::QuantizedTensor t =
        minikv_b200::quantize_matrix(m, minikv_b200::GroupAxis::PerToken, values.size());
    std::vector<std::uint8_t> codes(values.size());
    for (std::size_t i = 0; i < values.size(); ++i) codes[i] = (t.packed_words[i / 16] >> (2 * (i % 16))) & 3u;
    return {std::move(codes), GroupQuantParams{t.params[0].scale, t.params[0].zero_point}};
}

QuantizedTensor quantize_matrix(const Matrix& m, GroupAxis axis, std::size_t group_size) {
    minikv_b200::QuantizedTensor t = minikv_b200::quantize_matrix(to_b200(m), axis_b200(axis), group_size);
    QuantizedTensor r;
    move_into(r, t);
    return r;
}

void append_block(QuantizedTensor& t, const Matrix& block) {
    minikv_b200::QuantizedTensor b;
    move_into(b, t);
    struct Back {
        QuantizedTensor& t;
        minikv_b200::QuantizedTensor& b;
        ~Back() { move_into(t, b); }
    } back{t, b};
    minikv_b200::append_block(b, to_b200(block));
}

Matrix dequantize_matrix(const QuantizedTensor& t) { return from_b200(minikv_b200::dequantize_matrix(copy_b200(t))); }

// ---- cache_engine.hpp:44-67 ----
KVCacheLayer make_cache(std::size_t d, std::size_t n_r, std::size_t group_size, QuantMode mode) {
    VCache v = minikv_b200::value::make_cache(d, n_r, group_size, mode_b200(mode));
    KVCacheLayer c;
    move_into(c, v);
    return c;
}

std::pair<KVCacheLayer, PrefillReport> prefill(const Matrix& k, const Matrix& v, const Vector& a_cumul,
                                               std::size_t hh_count, std::size_t rw_count, std::size_t n_r,
                                               std::size_t group_size, QuantMode mode) {
    auto [vc, rep] = minikv_b200::value::prefill(to_b200(k), to_b200(v), a_cumul, hh_count, rw_count, n_r, group_size,
                                                 mode_b200(mode));
    KVCacheLayer cache;
    move_into(cache, vc);
    PrefillReport report;
    report.kept = from_b200(rep.kept);
    report.bytes_before = rep.bytes_before;
    report.bytes_after = rep.bytes_after;
    report.a_cumul = std::move(rep.a_cumul);
    return {std::move(cache), std::move(report)};
}

void decode_append(KVCacheLayer& cache, const Vector& t_k, const Vector& t_v) {
    with_state(cache, [&](VCache& s) {
        minikv_b200::value::decode_append(s, t_k, t_v);
        return 0;
    });
}

Vector decode_step(KVCacheLayer& cache, const Vector& t_q, const Vector& t_k, const Vector& t_v, float scale) {
    return with_state(cache, [&](VCache& s) { return minikv_b200::value::decode_step(s, t_q, t_k, t_v, scale); });
}

Matrix stored_keys(const KVCacheLayer& cache) {
    if (cache.mode == QuantMode::Identity) return cache.fp_key;
    return dequantize_matrix(cache.q_key);
}

Matrix stored_values(const KVCacheLayer& cache) {
    if (cache.mode == QuantMode::Identity) return cache.fp_value;
    return dequantize_matrix(cache.q_value);
}

}  // namespace minikv
