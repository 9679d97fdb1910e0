// minikv_reference_adapter.cpp -- what a maintainer links INTO the reference build to route
// its hot-path declarations (proj/core/include/minikv/*.hpp, unchanged) to the B200 library.
//
// Each definition below has exactly the reference's signature and forwards to the C++
// host API of include/minikv_b200.hpp (types converted field by field).  The reference's
// own CPU definitions of these functions (attention.cpp:29, selection.cpp:10-146,
// cache_engine.cpp:56) are dropped from its build when this file is linked.  Decode
// (decode_step over a host KVCacheLayer) stays on the batched device-handle API
// (minikv_b200::KVCacheLayer / mkv_decode_step): the reference's value-type cache has no
// place for device state.  Built by dropin/Makefile against the reference headers as a
// signature check (compile only); see INTEGRATION.md.
#include "minikv/attention.hpp"
#include "minikv/cache_engine.hpp"
#include "minikv/selection.hpp"
#include "minikv_b200.hpp"

namespace minikv {
namespace {
minikv_b200::Matrix to_b200(const Matrix& m) {
    minikv_b200::Matrix r(m.rows, m.cols);
    r.data = m.data;
    return r;
}
Matrix from_b200(const minikv_b200::Matrix& m) {
    Matrix r(m.rows, m.cols);
    r.data = m.data;
    return r;
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
QuantizedTensor from_b200(const minikv_b200::QuantizedTensor& t) {
    QuantizedTensor r;
    r.axis = t.axis == minikv_b200::GroupAxis::PerChannel ? GroupAxis::PerChannel : GroupAxis::PerToken;
    r.group_size = t.group_size;
    r.logical_rows = t.logical_rows;
    r.logical_cols = t.logical_cols;
    r.packed_words = t.packed_words;
    r.params.resize(t.params.size());
    for (std::size_t g = 0; g < t.params.size(); ++g) r.params[g] = {t.params[g].scale, t.params[g].zero_point};
    r.block_rows = t.block_rows;
    r.total_codes = t.total_codes;
    return r;
}
}  // namespace

AttentionResult selective_flash_attn(const Matrix& q, const Matrix& k, const Matrix& v, float scale, bool causal,
                                     TileConfig tiles) {
    auto r = minikv_b200::selective_flash_attn(to_b200(q), to_b200(k), to_b200(v), scale, causal,
                                               minikv_b200::TileConfig{tiles.block_m, tiles.block_n});
    AttentionResult out;
    out.output = from_b200(r.output);
    out.lse = r.lse;
    out.a_cumul = r.a_cumul;
    out.aux_elements = r.aux_elements;
    return out;
}

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

// prefill on the device (K2 select + K3 quantize/pack), returned as the reference's
// host KVCacheLayer: q_key / q_value are the device pages exported bit-exactly.
std::pair<KVCacheLayer, PrefillReport> prefill(const Matrix& k, const Matrix& v, const Vector& a_cumul,
                                               std::size_t hh_count, std::size_t rw_count, std::size_t n_r,
                                               std::size_t group_size, QuantMode mode) {
    if (mode != QuantMode::TwoBit) throw std::invalid_argument("prefill: the device cache is 2-bit");
    auto [dc, rep] = minikv_b200::prefill(to_b200(k), to_b200(v), a_cumul, hh_count, rw_count, n_r, group_size);
    KVCacheLayer cache = make_cache(k.cols, n_r, group_size, mode);
    cache.q_key = from_b200(dc.q_key());
    cache.q_value = from_b200(dc.q_value());
    cache.tokens_quantized = dc.tokens_quantized();
    PrefillReport report;
    report.kept = from_b200(rep.kept);
    report.bytes_before = rep.bytes_before;
    report.bytes_after = rep.bytes_after;
    report.a_cumul = rep.a_cumul;
    return {std::move(cache), std::move(report)};
}

}  // namespace minikv
