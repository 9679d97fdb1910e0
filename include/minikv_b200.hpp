// minikv_b200.hpp -- C++ host API of the B200 MiniKV hot path.
//
// Mirrors the reference's public C++ operator interface (namespace minikv,
// proj/core/include/minikv/{matrix,attention,selection,quantizer,cache_engine}.hpp):
// the same function names, argument meaning, result fields and exception classes,
// implemented on the device through the C ABI of minikv_b200.h.  Values are host
// fp32 like the reference's; they are rounded ONCE to fp16 on upload (the device
// format), so codes and selected indices are bit-identical to the reference for
// fp16-representable inputs and attention outputs agree within the tolerances of
// DESIGN.md.  No CPU fallback: without an sm_100 device every compute call throws.
//
// The namespace is minikv_b200 so that this library links next to the reference
// (the parity tests do exactly that); INTEGRATION.md shows the one-line bodies a
// maintainer gives the reference's own declarations to route them here.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

namespace minikv_b200 {

using Vector = std::vector<float>;

// Dense row-major fp32 matrix (matrix.hpp:11-26).
struct Matrix {
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::vector<float> data;
    Matrix() = default;
    Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0f) {}
    float& at(std::size_t r, std::size_t c) { return data[r * cols + c]; }
    float at(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
    float* row(std::size_t r) { return data.data() + r * cols; }
    const float* row(std::size_t r) const { return data.data() + r * cols; }
    bool empty() const { return rows == 0 || cols == 0; }
};

// ---- attention.hpp:12-39 ----
struct TileConfig {  // accepted for signature parity; the device tiles are fixed (128 x 128)
    std::size_t block_m = 64;
    std::size_t block_n = 64;
};
struct AttentionResult {
    Matrix output;  // l_query x d
    Vector lse;     // natural-log LSE per query row
    Vector a_cumul; // per key: sum of attention weights over all query rows
    std::size_t aux_elements = 0;  // auxiliary fp32 elements beyond inputs/outputs (linear)
};
inline float default_scale(std::size_t d_head) {
    return 1.0f / static_cast<float>(std::sqrt(static_cast<double>(d_head)));
}
// K1: two-pass selective flash attention (attention.cpp:29-117).  d = 128.
AttentionResult selective_flash_attn(const Matrix& q, const Matrix& k, const Matrix& v, float scale, bool causal,
                                     TileConfig tiles = {});

// ---- selection.hpp:11-59 ----
struct CacheBudget {
    double alpha_hh = 0.0;
    double alpha_rw = 0.0;
};
struct LayerAllocation {
    std::vector<std::size_t> per_layer_hh;
    bool uniform_fallback = false;
};
struct SelectionResult {
    std::vector<std::size_t> kept;  // ascending: sort(hh) ++ rw
    std::vector<std::size_t> hh;
    std::vector<std::size_t> rw;
    bool clamped = false;
};
// K2 (selection.cpp:10-46)
SelectionResult select_token_counts(const Vector& a_cumul, std::size_t hh_count, std::size_t rw_count);
SelectionResult select_tokens(const Vector& a_cumul, const CacheBudget& budget, std::size_t l_prompt);
enum class PyramidOrientation { BottomHeavy, TopHeavy };
enum class VarianceMode { Prop, Inv };
LayerAllocation allocate_uniform(std::size_t total_hh, std::size_t layers);
LayerAllocation allocate_pyramid(std::size_t mean_budget_x, std::size_t layers, std::size_t depth_d = 7,
                                 PyramidOrientation orientation = PyramidOrientation::BottomHeavy);
LayerAllocation allocate_variance(const Vector& per_layer_variance, std::size_t total_hh, VarianceMode mode);
float layer_score_variance(const Vector& a_cumul);  // on the device (fp64 two-pass)

// ---- harness.hpp:33-52: the H2O comparison baseline (device) and persistence ----
struct H2OBaselineTrace {
    std::vector<std::vector<std::size_t>> kept_per_step;  // [0] = post-prefill set
};
H2OBaselineTrace h2o_dynamic_baseline(const Matrix& prompt_k, const Vector& prompt_scores,
                                      const std::vector<Vector>& decode_qs, const std::vector<Vector>& decode_ks,
                                      std::size_t hh_budget, std::size_t rw_budget, float scale);
struct PersistenceReport {
    Vector fractions;
    double final_fraction = 0.0;
};
PersistenceReport persistence_analysis(const H2OBaselineTrace& trace, const std::vector<std::size_t>& prefill_hh);

// ---- quantizer.hpp:15-42: the reference's QuantizedTensor stream format ----
enum class GroupAxis { PerChannel, PerToken };
struct GroupQuantParams {
    float scale = 0.0f;
    float zero_point = 0.0f;
};
inline constexpr std::size_t kDefaultGroupSize = 16;
struct QuantizedTensor {
    GroupAxis axis = GroupAxis::PerToken;
    std::size_t group_size = kDefaultGroupSize;
    std::size_t logical_rows = 0;
    std::size_t logical_cols = 0;
    std::vector<std::uint32_t> packed_words;
    std::vector<GroupQuantParams> params;
    std::vector<std::size_t> block_rows;
    std::size_t total_codes = 0;
};
// ---- exact-fp32 reference-format path (any head dim / group size; csrc/refmt.cu) ----
// quantize_matrix / append_block (quantizer.cpp:102-151): codes, packed words and params
// bit-identical to the reference (quantize_group's IEEE division and rounding on the device).
QuantizedTensor quantize_matrix(const Matrix& m, GroupAxis axis, std::size_t group_size = kDefaultGroupSize);
void append_block(QuantizedTensor& t, const Matrix& block);
// dequantize_matrix (quantizer.cpp:153-195) on the device: v = fl(fl(code * scale) + zero), no FMA
Matrix dequantize_matrix(const QuantizedTensor& t);
// selective_flash_attn on fp32 matrices, any d (attention.cpp:29-117): fp32 device kernels in the
// reference's dot-product and A_cumul accumulation order (the fp16 tensor-core K1 above is d = 128)
AttentionResult selective_flash_attn_f32(const Matrix& q, const Matrix& k, const Matrix& v, float scale, bool causal,
                                         TileConfig tiles = {});
// decode_attention (attention.cpp:119-143) on the device: (output row, attention row)
std::pair<Vector, Vector> decode_attention(const Vector& q_row, const Matrix& keys, const Matrix& values, float scale);

// ---- cache_engine.hpp:15-67: a device-resident KVCacheLayer ----
class KVCacheLayer {
public:
    std::size_t d = 0;
    std::size_t n_r = 128;
    std::size_t group_size = kDefaultGroupSize;
    std::size_t decode_reserve = 4096;  // decode tokens the device cache can grow by

    KVCacheLayer();
    ~KVCacheLayer();
    KVCacheLayer(KVCacheLayer&&) noexcept;
    KVCacheLayer& operator=(KVCacheLayer&&) noexcept;
    KVCacheLayer(const KVCacheLayer&) = delete;
    KVCacheLayer& operator=(const KVCacheLayer&) = delete;

    std::size_t tokens_quantized() const;
    std::size_t tokens_residual() const;
    std::size_t total_tokens() const { return tokens_quantized() + tokens_residual(); }
    // The reference's fields, exported from the device (bit-identical stream format).
    QuantizedTensor q_key() const;    // PerChannel
    QuantizedTensor q_value() const;  // PerToken
    Matrix r_key() const;             // residual rows (fp16 values widened)
    Matrix r_value() const;

    struct Impl;
    std::unique_ptr<Impl> impl;
};
struct PrefillReport {
    SelectionResult kept;
    std::uint64_t bytes_before = 0;  // fp16 K+V of the whole prompt
    std::uint64_t bytes_after = 0;   // measured cache bytes (accounting.cpp:101-114)
    Vector a_cumul;
};
KVCacheLayer make_cache(std::size_t d, std::size_t n_r, std::size_t group_size = kDefaultGroupSize);
// K2 + K3 (cache_engine.cpp:56-77)
std::pair<KVCacheLayer, PrefillReport> prefill(const Matrix& k, const Matrix& v, const Vector& a_cumul,
                                               std::size_t hh_count, std::size_t rw_count, std::size_t n_r,
                                               std::size_t group_size = kDefaultGroupSize);
void decode_append(KVCacheLayer& cache, const Vector& t_k, const Vector& t_v);  // cache_engine.cpp:79-90
// K4 (cache_engine.cpp:100-138)
Vector decode_step(KVCacheLayer& cache, const Vector& t_q, const Vector& t_k, const Vector& t_v, float scale);
Matrix stored_keys(const KVCacheLayer& cache);    // dequantize_matrix(q_key)
Matrix stored_values(const KVCacheLayer& cache);  // dequantize_matrix(q_value)
std::uint64_t measured_bytes(const KVCacheLayer& cache);

// ---- the reference's value-type KVCacheLayer (cache_engine.hpp:11-67), any d / group size ----
// The state lives in the reference's own host fields (so copies, snapshots and field reads behave
// exactly as the reference's); every computation -- selection (K2), gather + quantize + pack,
// dequantization and the decode attention -- runs on the device through the fp32
// reference-format kernels.  This is what the drop-in adapter (dropin/) routes the reference's
// make_cache / prefill / decode_append / decode_step / stored_* to.  The batched device-handle
// cache above (K3 pages, K4) is the throughput path for d = 128, group 16, fp16.
namespace value {
enum class QuantMode { TwoBit, Identity };
struct KVCacheLayer {
    std::size_t d = 0;
    std::size_t n_r = 128;
    std::size_t group_size = kDefaultGroupSize;
    QuantMode mode = QuantMode::TwoBit;
    QuantizedTensor q_key;    // PerChannel
    QuantizedTensor q_value;  // PerToken
    Matrix fp_key;            // identity-mode stores
    Matrix fp_value;
    Matrix r_key;             // residual, < n_r rows after any public operation
    Matrix r_value;
    std::size_t tokens_quantized = 0;
    std::size_t tokens_residual() const { return r_key.rows; }
    std::size_t total_tokens() const { return tokens_quantized + tokens_residual(); }
};
KVCacheLayer make_cache(std::size_t d, std::size_t n_r, std::size_t group_size = kDefaultGroupSize,
                        QuantMode mode = QuantMode::TwoBit);
std::pair<KVCacheLayer, PrefillReport> prefill(const Matrix& k, const Matrix& v, const Vector& a_cumul,
                                               std::size_t hh_count, std::size_t rw_count, std::size_t n_r,
                                               std::size_t group_size = kDefaultGroupSize,
                                               QuantMode mode = QuantMode::TwoBit);
void decode_append(KVCacheLayer& cache, const Vector& t_k, const Vector& t_v);
Vector decode_step(KVCacheLayer& cache, const Vector& t_q, const Vector& t_k, const Vector& t_v, float scale);
Matrix stored_keys(const KVCacheLayer& cache);
Matrix stored_values(const KVCacheLayer& cache);
std::uint64_t measured_bytes(const KVCacheLayer& cache);  // accounting.cpp:101-114
}  // namespace value

}  // namespace minikv_b200
