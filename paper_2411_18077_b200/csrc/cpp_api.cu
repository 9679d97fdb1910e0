// cpp_api.cu -- the C++ host API (include/minikv_b200.hpp) over the C ABI.
//
// Host code only: uploads the reference-shaped host values (fp32 rounded once to
// fp16, the device format), calls the C ABI on the default stream, synchronises and
// returns reference-shaped results.  Status codes become the reference's exception
// classes: invalid_argument, domain_error, runtime_error, out_of_range.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#include "minikv_b200.h"
#include "minikv_b200.hpp"

namespace minikv_b200 {

namespace {

void throw_status(int st, const char* where) {
    if (st == MKV_OK) return;
    const std::string m = std::string(where) + ": " + mkv_last_error();
    switch (st) {
        case MKV_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
        case MKV_ERR_DOMAIN: throw std::domain_error(m);
        case MKV_ERR_OUT_OF_RANGE: throw std::out_of_range(m);
        default: throw std::runtime_error(m);  // RUNTIME, CUDA, UNSUPPORTED
    }
}

void cuda_check(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
}

// RAII device buffer
struct Dev {
    void* p = nullptr;
    explicit Dev(size_t bytes) { cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc"); }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    Dev(Dev&& o) noexcept : p(o.p) { o.p = nullptr; }
    Dev& operator=(Dev&& o) noexcept {
        if (this != &o) {
            cudaFree(p);
            p = o.p;
            o.p = nullptr;
        }
        return *this;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

std::vector<__half> to_half(const float* x, size_t n) {
    std::vector<__half> h(n);
    for (size_t i = 0; i < n; ++i) h[i] = __float2half_rn(x[i]);
    return h;
}

Dev upload_half(const float* x, size_t n) {
    Dev d(n * sizeof(__half));
    const std::vector<__half> h = to_half(x, n);
    cuda_check(cudaMemcpy(d.p, h.data(), n * sizeof(__half), cudaMemcpyHostToDevice), "upload");
    return d;
}

Dev upload_f32(const float* x, size_t n) {
    Dev d(n * sizeof(float));
    cuda_check(cudaMemcpy(d.p, x, n * sizeof(float), cudaMemcpyHostToDevice), "upload");
    return d;
}

std::vector<float> download_half(const Dev& d, size_t n) {
    std::vector<__half> h(n);
    cuda_check(cudaMemcpy(h.data(), d.p, n * sizeof(__half), cudaMemcpyDeviceToHost), "download");
    std::vector<float> out(n);
    for (size_t i = 0; i < n; ++i) out[i] = __half2float(h[i]);
    return out;
}

constexpr int kD = 128;  // the device head dimension

}  // namespace

// ---------------------------------------------------------------------------
// attention (attention.cpp:29-117)
// ---------------------------------------------------------------------------
AttentionResult selective_flash_attn(const Matrix& q, const Matrix& k, const Matrix& v, float scale, bool causal,
                                     TileConfig) {
    if (q.cols != k.cols) throw std::invalid_argument("selective_flash_attn: q/k width mismatch");
    if (k.rows != v.rows) throw std::invalid_argument("selective_flash_attn: k/v length mismatch");
    if (q.rows == 0 || k.rows == 0) throw std::invalid_argument("selective_flash_attn: empty input");
    if (causal && q.rows > k.rows) throw std::invalid_argument("selective_flash_attn: causal requires l_query <= l_key");
    if (q.cols != kD || v.cols != kD) throw std::invalid_argument("selective_flash_attn: the device kernel is d = 128");
    const size_t lq = q.rows, lk = k.rows;
    Dev dq = upload_half(q.data.data(), lq * kD), dk = upload_half(k.data.data(), lk * kD),
        dv = upload_half(v.data.data(), lk * kD);
    Dev dout(lq * kD * sizeof(__half)), dlse(lq * sizeof(float)), dacc(lk * sizeof(float));
    mkv_prefill_args a{};
    a.q = dq.p; a.q_st = kD; a.q_sh = (int64_t)lq * kD; a.q_sb = a.q_sh;
    a.k = dk.p; a.k_st = kD; a.k_sh = (int64_t)lk * kD; a.k_sb = a.k_sh;
    a.v = dv.p; a.v_st = kD; a.v_sh = (int64_t)lk * kD; a.v_sb = a.v_sh;
    a.out = dout.p; a.o_st = kD; a.o_sh = (int64_t)lq * kD; a.o_sb = a.o_sh;
    a.lse = dlse.as<float>(); a.a_cumul = dacc.as<float>();
    a.batch = 1; a.n_q_heads = 1; a.n_kv_heads = 1;
    a.len_q = (int)lq; a.len_k = (int)lk; a.head_dim = kD;
    a.scale = scale; a.causal = causal ? 1 : 0;
    throw_status(mkv_prefill_attn(&a, nullptr), "selective_flash_attn");
    AttentionResult r;
    r.output = Matrix(lq, kD);
    r.output.data = download_half(dout, lq * kD);
    r.lse.resize(lq);
    r.a_cumul.resize(lk);
    cuda_check(cudaMemcpy(r.lse.data(), dlse.p, lq * sizeof(float), cudaMemcpyDeviceToHost), "download");
    cuda_check(cudaMemcpy(r.a_cumul.data(), dacc.p, lk * sizeof(float), cudaMemcpyDeviceToHost), "download");
    r.aux_elements = lq + lk;  // LSE + A_cumul: linear in the sequence (attention.hpp:21-23)
    return r;
}

// ---------------------------------------------------------------------------
// selection (selection.cpp)
// ---------------------------------------------------------------------------
SelectionResult select_token_counts(const Vector& a_cumul, size_t hh_count, size_t rw_count) {
    const size_t l = a_cumul.size();
    SelectionResult res;
    if (hh_count + rw_count >= l) {  // keep everything (selection.cpp:14-18)
        res.clamped = hh_count + rw_count > l;
        rw_count = std::min(rw_count, l);
        hh_count = l - rw_count;
    }
    for (size_t i = l - rw_count; i < l; ++i) res.rw.push_back(i);
    if (l == 0) return res;
    if (l > (size_t)INT32_MAX || hh_count > (size_t)INT32_MAX) throw std::invalid_argument("select: length too large");
    Dev da = upload_f32(a_cumul.data(), l);
    Dev dk(l * sizeof(int32_t));
    const int32_t hh = (int32_t)hh_count;
    mkv_select_args s{};
    s.a_cumul = da.as<float>(); s.a_stride = (int64_t)l; s.n_units = 1; s.length = (int)l;
    s.hh_count = &hh; s.rw_count = (int)rw_count; s.kept = dk.as<int32_t>(); s.kept_stride = (int64_t)l;
    throw_status(mkv_select(&s, nullptr), "select_token_counts");
    const size_t n_kept = std::min(hh_count + rw_count, l);
    std::vector<int32_t> kept(n_kept);
    cuda_check(cudaMemcpy(kept.data(), dk.p, n_kept * sizeof(int32_t), cudaMemcpyDeviceToHost), "download");
    res.kept.assign(kept.begin(), kept.end());
    res.hh.assign(res.kept.begin(), res.kept.begin() + (n_kept - rw_count));
    return res;
}

SelectionResult select_tokens(const Vector& a_cumul, const CacheBudget& budget, size_t l_prompt) {
    if (a_cumul.size() != l_prompt) throw std::invalid_argument("select_tokens: a_cumul length != l_prompt");
    if (budget.alpha_hh < 0 || budget.alpha_rw < 0) throw std::invalid_argument("select_tokens: negative budget");
    const auto hh = static_cast<size_t>(std::floor(budget.alpha_hh * static_cast<double>(l_prompt)));
    const auto rw = static_cast<size_t>(std::floor(budget.alpha_rw * static_cast<double>(l_prompt)));
    return select_token_counts(a_cumul, hh, rw);
}

static LayerAllocation from_i64(const std::vector<int64_t>& v, bool fallback) {
    LayerAllocation a;
    a.per_layer_hh.assign(v.begin(), v.end());
    a.uniform_fallback = fallback;
    return a;
}

LayerAllocation allocate_uniform(size_t total_hh, size_t layers) {
    if (layers < 1) throw std::invalid_argument("allocate_uniform: layers must be >= 1");
    std::vector<int64_t> out(layers);
    throw_status(mkv_allocate_uniform(total_hh, layers, out.data()), "allocate_uniform");
    return from_i64(out, false);
}

LayerAllocation allocate_pyramid(size_t x, size_t layers, size_t depth, PyramidOrientation o) {
    if (layers < 1) throw std::invalid_argument("allocate_pyramid: layers must be >= 1");
    std::vector<int64_t> out(layers);
    throw_status(mkv_allocate_pyramid(x, layers, depth, o == PyramidOrientation::BottomHeavy ? 1 : 0, out.data()),
                 "allocate_pyramid");
    return from_i64(out, false);
}

LayerAllocation allocate_variance(const Vector& var, size_t total_hh, VarianceMode mode) {
    std::vector<int64_t> out(std::max<size_t>(var.size(), 1));
    int fb = 0;
    throw_status(mkv_allocate_variance(var.data(), var.size(), total_hh, mode == VarianceMode::Inv ? 1 : 0,
                                       out.data(), &fb),
                 "allocate_variance");
    out.resize(var.size());
    return from_i64(out, fb != 0);
}

float layer_score_variance(const Vector& a_cumul) {
    if (a_cumul.empty()) throw std::invalid_argument("layer_score_variance: empty input");
    Dev da = upload_f32(a_cumul.data(), a_cumul.size());
    Dev dout(sizeof(float));
    throw_status(mkv_score_variance(da.as<float>(), (int64_t)a_cumul.size(), 1, (int)a_cumul.size(),
                                    dout.as<float>(), nullptr),
                 "layer_score_variance");
    float r = 0.0f;
    cuda_check(cudaMemcpy(&r, dout.p, sizeof(float), cudaMemcpyDeviceToHost), "download");
    return r;
}

// harness.cpp:108-150 on the device (mkv_h2o_dynamic_baseline)
H2OBaselineTrace h2o_dynamic_baseline(const Matrix& prompt_k, const Vector& prompt_scores,
                                      const std::vector<Vector>& decode_qs, const std::vector<Vector>& decode_ks,
                                      size_t hh_budget, size_t rw_budget, float scale) {
    if (prompt_k.rows != prompt_scores.size())
        throw std::invalid_argument("h2o_dynamic_baseline: prompt score length mismatch");
    if (decode_qs.size() != decode_ks.size())
        throw std::invalid_argument("h2o_dynamic_baseline: decode stream length mismatch");
    if (hh_budget + rw_budget < 1) throw std::invalid_argument("h2o_dynamic_baseline: budget must be >= 1");
    const size_t L = prompt_k.rows, steps = decode_qs.size();
    const size_t d = prompt_k.cols ? prompt_k.cols : (steps ? decode_ks[0].size() : 1);
    std::vector<float> qs(steps * d), ks(steps * d);
    for (size_t s = 0; s < steps; ++s) {
        if (decode_ks[s].size() != d) throw std::invalid_argument("append_row: width mismatch");
        if (decode_qs[s].size() != d) throw std::invalid_argument("h2o_dynamic_baseline: query width mismatch");
        std::copy(decode_qs[s].begin(), decode_qs[s].end(), qs.begin() + s * d);
        std::copy(decode_ks[s].begin(), decode_ks[s].end(), ks.begin() + s * d);
    }
    const size_t stride = std::max<size_t>(1, std::min(L + steps, hh_budget + rw_budget));
    Dev dk = upload_f32(prompt_k.data.data(), L * d), dsc = upload_f32(prompt_scores.data(), L);
    Dev dq = upload_f32(qs.data(), steps * d), dks = upload_f32(ks.data(), steps * d);
    Dev dkept((steps + 1) * stride * sizeof(int32_t)), dcnt((steps + 1) * sizeof(int32_t));
    mkv_h2o_args a{};
    a.prompt_k = dk.as<float>(); a.ld_k = (int64_t)d; a.prompt_scores = dsc.as<float>();
    a.qs = dq.as<float>(); a.ks = dks.as<float>();
    a.l_prompt = (int)L; a.d = (int)d; a.steps = (int)steps;
    a.hh_budget = (int64_t)hh_budget; a.rw_budget = (int64_t)rw_budget; a.scale = scale;
    a.kept = dkept.as<int32_t>(); a.kept_stride = (int64_t)stride; a.kept_count = dcnt.as<int32_t>();
    throw_status(mkv_h2o_dynamic_baseline(&a, nullptr), "h2o_dynamic_baseline");
    std::vector<int32_t> kept((steps + 1) * stride), cnt(steps + 1);
    cuda_check(cudaMemcpy(kept.data(), dkept.p, kept.size() * sizeof(int32_t), cudaMemcpyDeviceToHost), "download");
    cuda_check(cudaMemcpy(cnt.data(), dcnt.p, cnt.size() * sizeof(int32_t), cudaMemcpyDeviceToHost), "download");
    H2OBaselineTrace t;
    t.kept_per_step.resize(steps + 1);
    for (size_t s = 0; s <= steps; ++s)
        t.kept_per_step[s].assign(kept.begin() + s * stride, kept.begin() + s * stride + cnt[s]);
    return t;
}

// harness.cpp:152-169 (host arithmetic on the device-produced kept sets)
PersistenceReport persistence_analysis(const H2OBaselineTrace& trace, const std::vector<size_t>& prefill_hh) {
    if (prefill_hh.empty()) throw std::runtime_error("persistence_analysis: empty prefill heavy-hitter set");
    PersistenceReport r;
    for (const auto& kept : trace.kept_per_step) {
        size_t hit = 0;
        for (size_t idx : prefill_hh)
            if (std::binary_search(kept.begin(), kept.end(), idx)) ++hit;
        r.fractions.push_back(static_cast<float>(hit) / static_cast<float>(prefill_hh.size()));
    }
    r.final_fraction = r.fractions.back();
    return r;
}

// ---------------------------------------------------------------------------
// exact-fp32 reference-format path (refmt.cu through the C ABI)
// ---------------------------------------------------------------------------
namespace {

int axis_id(GroupAxis a) { return a == GroupAxis::PerChannel ? 0 : 1; }

int64_t group_count(GroupAxis axis, size_t rows, size_t cols, size_t gs) {
    return axis == GroupAxis::PerChannel ? (int64_t)cols * (int64_t)((rows + gs - 1) / gs)
                                         : (int64_t)rows * (int64_t)((cols + gs - 1) / gs);
}

// append_block (quantizer.cpp:102-136) of a block already on the device (rows gathered through
// d_idx when non-null): quantize + pack on the device, append words / params / block_rows.
void append_block_device(QuantizedTensor& t, const float* d_src, int64_t ld, const int32_t* d_idx, size_t rows,
                         size_t cols) {
    if (rows == 0 || cols == 0) throw std::invalid_argument("append_block: empty block");
    if (t.logical_cols == 0) t.logical_cols = cols;
    if (cols != t.logical_cols) throw std::invalid_argument("append_block: channel count mismatch");
    if (t.group_size < 1) throw std::invalid_argument("append_block: group_size must be >= 1");
    const int64_t n = (int64_t)rows * (int64_t)cols;
    const int64_t off = (int64_t)t.total_codes;
    const int64_t nw = (off + n + 15) / 16 - off / 16;
    const int64_t ng = group_count(t.axis, rows, cols, t.group_size);
    const uint32_t init = (off % 16) ? t.packed_words.at((size_t)(off / 16)) : 0u;
    Dev dw(nw * sizeof(uint32_t)), dp(ng * 2 * sizeof(float));
    throw_status(mkv_quantize_block_f32(d_src, ld, d_idx, (int)rows, (int)cols, (int)t.group_size, axis_id(t.axis),
                                        off, init, dw.as<uint32_t>(), dp.as<float>(), nullptr),
                 "append_block");
    std::vector<uint32_t> words(nw);
    std::vector<float> params(2 * ng);
    cuda_check(cudaMemcpy(words.data(), dw.p, nw * sizeof(uint32_t), cudaMemcpyDeviceToHost), "download");
    cuda_check(cudaMemcpy(params.data(), dp.p, 2 * ng * sizeof(float), cudaMemcpyDeviceToHost), "download");
    t.packed_words.resize((size_t)(off / 16));  // the partial last word is re-emitted by the device
    t.packed_words.insert(t.packed_words.end(), words.begin(), words.end());
    for (int64_t g = 0; g < ng; ++g) t.params.push_back(GroupQuantParams{params[2 * g], params[2 * g + 1]});
    t.block_rows.push_back(rows);
    t.logical_rows += rows;
    t.total_codes += (size_t)n;
}

// dequantize_matrix (quantizer.cpp:153-195) into a device buffer with row stride ld; returns rows
size_t dequantize_device(const QuantizedTensor& t, float* d_out, int64_t ld) {
    int64_t groups = 0, codes = 0;
    size_t rows = 0;
    for (size_t R : t.block_rows) {
        groups += group_count(t.axis, R, t.logical_cols, t.group_size);
        codes += (int64_t)R * (int64_t)t.logical_cols;
        rows += R;
    }
    if ((size_t)groups != t.params.size()) throw std::runtime_error("dequantize_matrix: corrupted group count");
    if ((size_t)codes > t.total_codes || t.packed_words.size() * 16 < (size_t)codes)
        throw std::out_of_range("QuantizedTensor: code index out of range");
    if (rows > t.logical_rows) throw std::runtime_error("dequantize_matrix: block rows exceed logical rows");
    if (t.block_rows.empty() || t.logical_cols == 0) return rows;
    Dev dw(t.packed_words.size() * sizeof(uint32_t)), dp(t.params.size() * 2 * sizeof(float));
    cuda_check(cudaMemcpy(dw.p, t.packed_words.data(), t.packed_words.size() * sizeof(uint32_t), cudaMemcpyHostToDevice),
               "upload");
    cuda_check(cudaMemcpy(dp.p, t.params.data(), t.params.size() * 2 * sizeof(float), cudaMemcpyHostToDevice), "upload");
    std::vector<int64_t> br(t.block_rows.begin(), t.block_rows.end());
    throw_status(mkv_dequantize_f32(dw.as<uint32_t>(), dp.as<float>(), br.data(), (int)br.size(), (int)t.logical_cols,
                                    (int)t.group_size, axis_id(t.axis), d_out, ld, nullptr),
                 "dequantize_matrix");
    return rows;
}

Matrix download_f32(const Dev& d, size_t rows, size_t cols) {
    Matrix m(rows, cols);
    if (rows * cols)
        cuda_check(cudaMemcpy(m.data.data(), d.p, rows * cols * sizeof(float), cudaMemcpyDeviceToHost), "download");
    return m;
}

}  // namespace

QuantizedTensor quantize_matrix(const Matrix& m, GroupAxis axis, size_t group_size) {
    if (m.empty()) throw std::invalid_argument("quantize_matrix: empty matrix");
    if (group_size < 1) throw std::invalid_argument("quantize_matrix: group_size must be >= 1");
    QuantizedTensor t;
    t.axis = axis;
    t.group_size = group_size;
    t.logical_cols = m.cols;
    append_block(t, m);
    return t;
}

void append_block(QuantizedTensor& t, const Matrix& block) {
    if (block.empty()) throw std::invalid_argument("append_block: empty block");
    Dev d = upload_f32(block.data.data(), block.rows * block.cols);
    append_block_device(t, d.as<float>(), (int64_t)block.cols, nullptr, block.rows, block.cols);
}

Matrix dequantize_matrix(const QuantizedTensor& t) {
    Matrix m(t.logical_rows, t.logical_cols);
    Dev d(std::max<size_t>(t.logical_rows * t.logical_cols, 1) * sizeof(float));
    // rows past the blocks (an inconsistent tensor) stay 0, as in the reference's Matrix
    cuda_check(cudaMemset(d.p, 0, std::max<size_t>(t.logical_rows * t.logical_cols, 1) * sizeof(float)), "memset");
    const size_t rows = dequantize_device(t, d.as<float>(), (int64_t)t.logical_cols);
    if (rows * t.logical_cols)
        cuda_check(cudaMemcpy(m.data.data(), d.p, rows * t.logical_cols * sizeof(float), cudaMemcpyDeviceToHost),
                   "download");
    return m;
}

AttentionResult selective_flash_attn_f32(const Matrix& q, const Matrix& k, const Matrix& v, float scale, bool causal,
                                         TileConfig tiles) {
    // check_shapes (attention.cpp:12-25) and the tile check (:32-34)
    if (q.rows == 0 || k.rows == 0) throw std::invalid_argument("attention: zero-length sequence");
    if (q.cols != k.cols) throw std::invalid_argument("attention: q/k head dimension mismatch");
    if (v.rows != k.rows) throw std::invalid_argument("attention: k/v token count mismatch");
    if (causal && q.rows > k.rows) throw std::invalid_argument("attention: causal requires l_query <= l_key");
    if (tiles.block_m < 1 || tiles.block_n < 1) throw std::invalid_argument("attention: tile sizes must be >= 1");
    const size_t lq = q.rows, lk = k.rows, d = q.cols, dv = v.cols;
    Dev dq = upload_f32(q.data.data(), lq * d), dk = upload_f32(k.data.data(), lk * d),
        dvv = upload_f32(v.data.data(), lk * dv);
    Dev dout(lq * dv * sizeof(float)), dlse(lq * sizeof(float)), dacc(lk * sizeof(float));
    mkv_attention_f32_args a{};
    a.q = dq.as<float>(); a.ld_q = (int64_t)d;
    a.k = dk.as<float>(); a.ld_k = (int64_t)d;
    a.v = dvv.as<float>(); a.ld_v = (int64_t)dv;
    a.out = dout.as<float>(); a.ld_o = (int64_t)dv;
    a.lse = dlse.as<float>(); a.a_cumul = dacc.as<float>();
    a.len_q = (int)lq; a.len_k = (int)lk; a.d = (int)d; a.dv = (int)dv;
    a.scale = scale; a.causal = causal ? 1 : 0;
    throw_status(mkv_attention_f32(&a, nullptr), "selective_flash_attn");
    AttentionResult r;
    r.output = download_f32(dout, lq, dv);
    r.lse.resize(lq);
    r.a_cumul.resize(lk);
    cuda_check(cudaMemcpy(r.lse.data(), dlse.p, lq * sizeof(float), cudaMemcpyDeviceToHost), "download");
    cuda_check(cudaMemcpy(r.a_cumul.data(), dacc.p, lk * sizeof(float), cudaMemcpyDeviceToHost), "download");
    // per-row running max / sum (registers of the row CTA) + one 128-key weight chunk: linear in l
    r.aux_elements = 2 * lq + 128;
    return r;
}

std::pair<Vector, Vector> decode_attention(const Vector& q_row, const Matrix& keys, const Matrix& values, float scale) {
    if (keys.rows == 0) throw std::invalid_argument("decode_attention: empty key set");
    if (q_row.size() != keys.cols) throw std::invalid_argument("decode_attention: query dimension mismatch");
    if (values.rows != keys.rows) throw std::invalid_argument("decode_attention: k/v token count mismatch");
    const size_t n = keys.rows, d = keys.cols, dv = values.cols;
    Dev dq = upload_f32(q_row.data(), d), dk = upload_f32(keys.data.data(), n * d),
        dvv = upload_f32(values.data.data(), n * dv);
    Dev dout(std::max<size_t>(dv, 1) * sizeof(float)), dattn(n * sizeof(float));
    Vector out(dv, 0.0f), attn(n);
    if (dv == 0) {  // the reference still computes the (unused) softmax row
        Matrix one(n, 1);
        Dev d1 = upload_f32(one.data.data(), n);
        throw_status(mkv_decode_attention_f32(dq.as<float>(), dk.as<float>(), (int64_t)d, d1.as<float>(), 1, (int)n,
                                              (int)d, 1, scale, dout.as<float>(), dattn.as<float>(), nullptr),
                     "decode_attention");
    } else {
        throw_status(mkv_decode_attention_f32(dq.as<float>(), dk.as<float>(), (int64_t)d, dvv.as<float>(), (int64_t)dv,
                                              (int)n, (int)d, (int)dv, scale, dout.as<float>(), dattn.as<float>(),
                                              nullptr),
                     "decode_attention");
        cuda_check(cudaMemcpy(out.data(), dout.p, dv * sizeof(float), cudaMemcpyDeviceToHost), "download");
    }
    cuda_check(cudaMemcpy(attn.data(), dattn.p, n * sizeof(float), cudaMemcpyDeviceToHost), "download");
    return {std::move(out), std::move(attn)};
}

// ---------------------------------------------------------------------------
// the value-type KVCacheLayer (cache_engine.cpp:9-138) on the reference-format kernels
// ---------------------------------------------------------------------------
namespace value {

KVCacheLayer make_cache(size_t d, size_t n_r, size_t group_size, QuantMode mode) {
    if (d == 0) throw std::invalid_argument("make_cache: d must be >= 1");
    if (group_size < 1 || n_r == 0 || n_r % group_size != 0)
        throw std::invalid_argument("make_cache: n_r must be a positive multiple of group_size");
    KVCacheLayer c;
    c.d = d;
    c.n_r = n_r;
    c.group_size = group_size;
    c.mode = mode;
    c.q_key.axis = GroupAxis::PerChannel;
    c.q_key.group_size = group_size;
    c.q_key.logical_cols = d;
    c.q_value.axis = GroupAxis::PerToken;
    c.q_value.group_size = group_size;
    c.q_value.logical_cols = d;
    c.r_key = Matrix(0, d);
    c.r_value = Matrix(0, d);
    return c;
}

namespace {

void append_rows(Matrix& dst, const Matrix& src) {
    if (dst.rows == 0) {
        dst = src;
        return;
    }
    dst.data.insert(dst.data.end(), src.data.begin(), src.data.end());
    dst.rows += src.rows;
}

// store_block (cache_engine.cpp:34-52) of rows already on the device (optionally gathered)
void store_block_device(KVCacheLayer& c, const float* dk, const float* dv, const int32_t* d_idx, size_t rows,
                        size_t cols) {
    append_block_device(c.q_key, dk, (int64_t)cols, d_idx, rows, cols);
    append_block_device(c.q_value, dv, (int64_t)cols, d_idx, rows, cols);
    c.tokens_quantized += rows;
}

void store_block(KVCacheLayer& c, const Matrix& kb, const Matrix& vb) {
    if (c.mode == QuantMode::Identity) {  // full-precision copies, no computation
        append_rows(c.fp_key, kb);
        append_rows(c.fp_value, vb);
        c.tokens_quantized += kb.rows;
        return;
    }
    if (kb.empty()) throw std::invalid_argument("append_block: empty block");
    Dev dk = upload_f32(kb.data.data(), kb.rows * kb.cols), dv = upload_f32(vb.data.data(), vb.rows * vb.cols);
    store_block_device(c, dk.as<float>(), dv.as<float>(), nullptr, kb.rows, kb.cols);
}

Matrix gather(const Matrix& m, const std::vector<size_t>& idx) {  // gather_rows (matrix.cpp:38-47)
    Matrix out(idx.size(), m.cols);
    for (size_t i = 0; i < idx.size(); ++i) {
        if (idx[i] >= m.rows) throw std::out_of_range("gather_rows: index out of range");
        std::copy_n(m.row(idx[i]), m.cols, out.row(i));
    }
    return out;
}

// the stored part (dequantized or identity) followed by the residual rows, on the device
size_t stack_device(const KVCacheLayer& c, bool values, Dev& out) {
    const QuantizedTensor& t = values ? c.q_value : c.q_key;
    const Matrix& fp = values ? c.fp_value : c.fp_key;
    const Matrix& res = values ? c.r_value : c.r_key;
    const size_t nq = c.mode == QuantMode::Identity ? fp.rows : t.logical_rows;
    const size_t n = nq + res.rows;
    out = Dev(std::max<size_t>(n * c.d, 1) * sizeof(float));
    cuda_check(cudaMemset(out.p, 0, std::max<size_t>(n * c.d, 1) * sizeof(float)), "memset");
    if (c.mode == QuantMode::Identity) {
        if (nq)
            cuda_check(cudaMemcpy(out.p, fp.data.data(), nq * c.d * sizeof(float), cudaMemcpyHostToDevice), "upload");
    } else if (nq) {
        dequantize_device(t, out.as<float>(), (int64_t)c.d);
    }
    if (res.rows)
        cuda_check(cudaMemcpy(out.as<float>() + nq * c.d, res.data.data(), res.rows * c.d * sizeof(float),
                              cudaMemcpyHostToDevice),
                   "upload");
    return n;
}

}  // namespace

std::uint64_t measured_bytes(const KVCacheLayer& c) {
    std::uint64_t bytes = 0;
    if (c.mode == QuantMode::Identity) {
        bytes += (std::uint64_t)c.fp_key.data.size() * 2 + (std::uint64_t)c.fp_value.data.size() * 2;
    } else {
        bytes += (std::uint64_t)c.q_key.packed_words.size() * 4 + (std::uint64_t)c.q_key.params.size() * 4;
        bytes += (std::uint64_t)c.q_value.packed_words.size() * 4 + (std::uint64_t)c.q_value.params.size() * 4;
    }
    bytes += (std::uint64_t)c.r_key.data.size() * 2 + (std::uint64_t)c.r_value.data.size() * 2;
    return bytes;
}

std::pair<KVCacheLayer, PrefillReport> prefill(const Matrix& k, const Matrix& v, const Vector& a_cumul,
                                               size_t hh_count, size_t rw_count, size_t n_r, size_t group_size,
                                               QuantMode mode) {
    if (k.rows != v.rows || k.rows != a_cumul.size()) throw std::invalid_argument("prefill: k/v/a_cumul length mismatch");
    if (k.cols != v.cols) throw std::invalid_argument("prefill: k/v width mismatch");
    if (hh_count + rw_count == 0) throw std::runtime_error("prefill: zero kept tokens");
    KVCacheLayer c = make_cache(k.cols, n_r, group_size, mode);
    PrefillReport report;
    report.kept = select_token_counts(a_cumul, hh_count, rw_count);  // K2 on the device
    report.a_cumul = a_cumul;
    report.bytes_before = (std::uint64_t)2 * k.rows * k.cols * 2;
    const std::vector<size_t>& kept = report.kept.kept;
    if (mode == QuantMode::Identity || kept.empty()) {
        store_block(c, gather(k, kept), gather(v, kept));
    } else {
        // gather_rows + append_block in one device pass: the quantizer reads the kept rows in place
        std::vector<int32_t> idx(kept.begin(), kept.end());
        Dev dk = upload_f32(k.data.data(), k.rows * k.cols), dv = upload_f32(v.data.data(), v.rows * v.cols);
        Dev di(idx.size() * sizeof(int32_t));
        cuda_check(cudaMemcpy(di.p, idx.data(), idx.size() * sizeof(int32_t), cudaMemcpyHostToDevice), "upload");
        store_block_device(c, dk.as<float>(), dv.as<float>(), di.as<int32_t>(), kept.size(), k.cols);
    }
    report.bytes_after = measured_bytes(c);
    return {std::move(c), std::move(report)};
}

void decode_append(KVCacheLayer& c, const Vector& t_k, const Vector& t_v) {
    if (t_k.size() != c.d || t_v.size() != c.d) throw std::invalid_argument("decode_append: token dimension mismatch");
    c.r_key.data.insert(c.r_key.data.end(), t_k.begin(), t_k.end());
    c.r_key.cols = c.d;
    ++c.r_key.rows;
    c.r_value.data.insert(c.r_value.data.end(), t_v.begin(), t_v.end());
    c.r_value.cols = c.d;
    ++c.r_value.rows;
    if (c.r_key.rows == c.n_r) {
        store_block(c, c.r_key, c.r_value);
        c.r_key = Matrix(0, c.d);
        c.r_value = Matrix(0, c.d);
    }
}

Vector decode_step(KVCacheLayer& c, const Vector& t_q, const Vector& t_k, const Vector& t_v, float scale) {
    if (c.total_tokens() == 0) throw std::runtime_error("decode_step: empty cache");
    if (t_q.size() != c.d) throw std::invalid_argument("decode_step: query dimension mismatch");
    decode_append(c, t_k, t_v);
    Dev keys(16), vals(16);
    const size_t n = stack_device(c, false, keys);
    stack_device(c, true, vals);
    Dev dq = upload_f32(t_q.data(), c.d), dout(c.d * sizeof(float)), dattn(n * sizeof(float));
    throw_status(mkv_decode_attention_f32(dq.as<float>(), keys.as<float>(), (int64_t)c.d, vals.as<float>(),
                                          (int64_t)c.d, (int)n, (int)c.d, (int)c.d, scale, dout.as<float>(),
                                          dattn.as<float>(), nullptr),
                 "decode_step");
    Vector out(c.d);
    cuda_check(cudaMemcpy(out.data(), dout.p, c.d * sizeof(float), cudaMemcpyDeviceToHost), "download");
    return out;
}

Matrix stored_keys(const KVCacheLayer& c) {
    return c.mode == QuantMode::Identity ? c.fp_key : dequantize_matrix(c.q_key);
}
Matrix stored_values(const KVCacheLayer& c) {
    return c.mode == QuantMode::Identity ? c.fp_value : dequantize_matrix(c.q_value);
}

}  // namespace value

// ---------------------------------------------------------------------------
// device KV cache (cache_engine.cpp)
// ---------------------------------------------------------------------------
struct KVCacheLayer::Impl {
    mkv_cache* h = nullptr;
    ~Impl() {
        if (h) mkv_cache_destroy(h);
    }
};

KVCacheLayer::KVCacheLayer() = default;
KVCacheLayer::~KVCacheLayer() = default;
KVCacheLayer::KVCacheLayer(KVCacheLayer&&) noexcept = default;
KVCacheLayer& KVCacheLayer::operator=(KVCacheLayer&&) noexcept = default;

static mkv_cache* handle(const KVCacheLayer& c) {
    if (!c.impl || !c.impl->h) throw std::runtime_error("KVCacheLayer: no device cache");
    return c.impl->h;
}

static void create_device_cache(KVCacheLayer& c, size_t prefill_capacity) {
    const int32_t cap = (int32_t)prefill_capacity;
    mkv_cache_config cfg{};
    cfg.n_units = 1;
    cfg.head_dim = (int)c.d;
    cfg.n_r = (int)c.n_r;
    cfg.group_size = (int)c.group_size;
    cfg.prefill_capacity = &cap;
    cfg.max_decode_tokens = (int)c.decode_reserve;
    cfg.keep_fp32_params = 1;  // exports carry the reference's fp32 (scale, zero) bit-exactly
    c.impl.reset(new KVCacheLayer::Impl());
    throw_status(mkv_cache_create(&cfg, &c.impl->h), "make_cache");
}

KVCacheLayer make_cache(size_t d, size_t n_r, size_t group_size) {
    if (d < 1) throw std::invalid_argument("make_cache: d must be >= 1");
    if (group_size < 1 || n_r == 0 || n_r % group_size != 0)
        throw std::invalid_argument("make_cache: n_r must be a positive multiple of group_size");
    KVCacheLayer c;
    c.d = d;
    c.n_r = n_r;
    c.group_size = group_size;
    create_device_cache(c, 0);
    return c;
}

size_t KVCacheLayer::tokens_quantized() const {
    int64_t tq = 0;
    throw_status(mkv_cache_unit_info(handle(*this), 0, &tq, nullptr, nullptr, nullptr), "tokens_quantized");
    return (size_t)tq;
}

size_t KVCacheLayer::tokens_residual() const {
    int64_t tr = 0;
    throw_status(mkv_cache_unit_info(handle(*this), 0, nullptr, &tr, nullptr, nullptr), "tokens_residual");
    return (size_t)tr;
}

static QuantizedTensor export_tensor(const KVCacheLayer& c, int which) {
    int64_t nw = 0, np = 0, nb = 0;
    throw_status(mkv_cache_export_sizes(handle(c), 0, which, &nw, &np, &nb), "export");
    QuantizedTensor t;
    t.axis = which == 0 ? GroupAxis::PerChannel : GroupAxis::PerToken;
    t.group_size = c.group_size;
    t.logical_rows = c.tokens_quantized();
    t.logical_cols = c.d;
    t.packed_words.resize(std::max<int64_t>(nw, 1));
    std::vector<float> params(std::max<int64_t>(2 * np, 2));
    std::vector<int64_t> br(std::max<int64_t>(nb, 1));
    throw_status(mkv_cache_export_reference(handle(c), 0, which, t.packed_words.data(), params.data(), br.data()),
                 "export");
    t.packed_words.resize(nw);
    t.params.resize(np);
    for (int64_t g = 0; g < np; ++g) t.params[g] = GroupQuantParams{params[2 * g], params[2 * g + 1]};
    t.block_rows.assign(br.begin(), br.begin() + nb);
    t.total_codes = t.logical_rows * t.logical_cols;
    return t;
}

QuantizedTensor KVCacheLayer::q_key() const { return export_tensor(*this, 0); }
QuantizedTensor KVCacheLayer::q_value() const { return export_tensor(*this, 1); }

static Matrix residual(const KVCacheLayer& c, bool value) {
    const size_t n = c.tokens_residual();
    std::vector<uint16_t> rk(std::max<size_t>(n, 1) * c.d), rv(std::max<size_t>(n, 1) * c.d);
    throw_status(mkv_cache_export_residual(handle(c), 0, rk.data(), rv.data()), "residual");
    Matrix m(n, c.d);
    const std::vector<uint16_t>& src = value ? rv : rk;
    for (size_t i = 0; i < n * c.d; ++i) {
        __half_raw r;
        r.x = src[i];
        m.data[i] = __half2float(__half(r));
    }
    return m;
}

Matrix KVCacheLayer::r_key() const { return residual(*this, false); }
Matrix KVCacheLayer::r_value() const { return residual(*this, true); }

std::uint64_t measured_bytes(const KVCacheLayer& c) {  // accounting.cpp:101-114
    std::uint64_t bytes = 0;
    for (int which = 0; which < 2; ++which) {
        int64_t nw = 0, np = 0;
        throw_status(mkv_cache_export_sizes(handle(c), 0, which, &nw, &np, nullptr), "measured_bytes");
        bytes += (std::uint64_t)nw * 4 + (std::uint64_t)np * 4;  // (scale, zero) counted as 2 x fp16
    }
    bytes += (std::uint64_t)c.tokens_residual() * c.d * 2 * 2;
    return bytes;
}

std::pair<KVCacheLayer, PrefillReport> prefill(const Matrix& k, const Matrix& v, const Vector& a_cumul,
                                               size_t hh_count, size_t rw_count, size_t n_r, size_t group_size) {
    if (k.rows != v.rows || k.rows != a_cumul.size()) throw std::invalid_argument("prefill: k/v/a_cumul length mismatch");
    if (k.cols != v.cols) throw std::invalid_argument("prefill: k/v width mismatch");
    if (hh_count + rw_count == 0) throw std::runtime_error("prefill: zero kept tokens");
    KVCacheLayer c;
    c.d = k.cols;
    c.n_r = n_r;
    c.group_size = group_size;
    if (group_size < 1 || n_r == 0 || n_r % group_size != 0)
        throw std::invalid_argument("make_cache: n_r must be a positive multiple of group_size");
    const size_t l = k.rows;
    const size_t n_kept = std::min(hh_count + rw_count, l);
    create_device_cache(c, n_kept);
    PrefillReport report;
    report.kept = select_token_counts(a_cumul, hh_count, rw_count);
    report.a_cumul = a_cumul;
    report.bytes_before = (std::uint64_t)2 * l * k.cols * 2;  // K + V at fp16
    if (l > 0) {
        Dev dk = upload_half(k.data.data(), l * c.d), dv = upload_half(v.data.data(), l * c.d);
        Dev da = upload_f32(a_cumul.data(), l);
        const int32_t hh = (int32_t)hh_count;
        mkv_prefill_select_args a{};
        a.unit_begin = 0; a.n_units = 1; a.length = (int)l;
        a.a_cumul = da.as<float>(); a.a_stride = (int64_t)l;
        a.hh_count = &hh; a.rw_count = (int)rw_count;
        a.k = dk.p; a.k_su = (int64_t)l * c.d; a.k_st = (int64_t)c.d;
        a.v = dv.p; a.v_su = (int64_t)l * c.d; a.v_st = (int64_t)c.d;
        throw_status(mkv_cache_prefill_select(handle(c), &a, nullptr), "prefill");
        throw_status(mkv_cache_check(handle(c)), "prefill");  // non-finite input -> domain_error
    }
    report.bytes_after = measured_bytes(c);
    return {std::move(c), std::move(report)};
}

void decode_append(KVCacheLayer& c, const Vector& t_k, const Vector& t_v) {
    if (t_k.size() != c.d || t_v.size() != c.d) throw std::invalid_argument("decode_append: token dimension mismatch");
    Dev dk = upload_half(t_k.data(), c.d), dv = upload_half(t_v.data(), c.d);
    throw_status(mkv_cache_append(handle(c), 0, 1, dk.p, dv.p, nullptr), "decode_append");
    throw_status(mkv_cache_check(handle(c)), "decode_append");
}

Vector decode_step(KVCacheLayer& c, const Vector& t_q, const Vector& t_k, const Vector& t_v, float scale) {
    if (t_q.size() != c.d || t_k.size() != c.d || t_v.size() != c.d)
        throw std::invalid_argument("decode_step: token dimension mismatch");
    Dev dq = upload_half(t_q.data(), c.d), dk = upload_half(t_k.data(), c.d), dv = upload_half(t_v.data(), c.d);
    Dev dout(c.d * sizeof(__half));
    mkv_decode_args a{};
    a.unit_begin = 0; a.n_units = 1; a.group = 1;
    a.q = dq.p; a.k_new = dk.p; a.v_new = dv.p; a.out = dout.p; a.scale = scale;
    throw_status(mkv_decode_step(handle(c), &a, nullptr), "decode_step");
    throw_status(mkv_cache_check(handle(c)), "decode_step");
    return download_half(dout, c.d);
}

Matrix stored_keys(const KVCacheLayer& c) { return dequantize_matrix(c.q_key()); }
Matrix stored_values(const KVCacheLayer& c) { return dequantize_matrix(c.q_value()); }

}  // namespace minikv_b200
