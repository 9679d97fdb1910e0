/*
 * minikv_oracle.c -- TEST INFRASTRUCTURE ONLY (see minikv_oracle.h).
 *
 * Plain-C restatement of the MiniKV reference hot path.  Citations are
 * relative to /root/reference/proj/core/src.  Build: see oracle/Makefile
 * (gcc -O2 -ffp-contract=off, no -march: no FMA contraction, like the
 * reference's Release build).
 */
#include "minikv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* numerics (matrix.cpp)                                              */
/* ------------------------------------------------------------------ */

/* matrix.cpp:60-66: sequential fp32 sum, no FMA. */
float mko_dot(const float* a, const float* b, size_t n) {
    float acc = 0.0f;
    for (size_t k = 0; k < n; ++k) {
        float p = a[k] * b[k];
        acc += p;
    }
    return acc;
}

/* std::max(a, b) == (a < b) ? b : a */
static inline float smax(float a, float b) { return (a < b) ? b : a; }
/* std::min(a, b) == (b < a) ? b : a */
static inline float smin(float a, float b) { return (b < a) ? b : a; }

/* matrix.cpp:83-99: max-subtract, exp, sum, divide. */
int mko_softmax_inplace(float* x, size_t n) {
    if (n == 0) return MKO_INVALID;
    float m = x[0];
    for (size_t i = 1; i < n; ++i) m = smax(m, x[i]);
    float sum = 0.0f;
    for (size_t i = 0; i < n; ++i) {
        x[i] = expf(x[i] - m);
        sum += x[i];
    }
    for (size_t i = 0; i < n; ++i) x[i] /= sum;
    return MKO_OK;
}

/* IEEE binary32 -> binary16, round to nearest even (handles subnormals, inf, nan). */
uint16_t mko_float_to_half_bits(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    uint32_t sign = (x >> 16) & 0x8000u;
    uint32_t exp = (x >> 23) & 0xFFu;
    uint32_t man = x & 0x7FFFFFu;
    if (exp == 0xFFu) return (uint16_t)(sign | 0x7C00u | (man ? 0x200u : 0u));
    int32_t e = (int32_t)exp - 127 + 15;
    if (e >= 31) return (uint16_t)(sign | 0x7C00u);
    if (e <= 0) {
        if (e < -10) return (uint16_t)sign;
        man |= 0x800000u;
        uint32_t shift = (uint32_t)(14 - e);
        uint32_t half_man = man >> shift;
        uint32_t rem = man & ((1u << shift) - 1u);
        uint32_t halfway = 1u << (shift - 1);
        if (rem > halfway || (rem == halfway && (half_man & 1u))) half_man++;
        return (uint16_t)(sign | half_man);
    }
    uint32_t half = sign | ((uint32_t)e << 10) | (man >> 13);
    uint32_t rem = man & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (half & 1u))) half++;
    return (uint16_t)half;
}

float mko_half_bits_to_float(uint16_t h) {
    uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    uint32_t exp = ((uint32_t)h >> 10) & 0x1Fu;
    uint32_t man = (uint32_t)h & 0x3FFu;
    uint32_t x;
    if (exp == 0) {
        if (man == 0) {
            x = sign;
        } else {
            int32_t e = -1;
            do { man <<= 1; ++e; } while (!(man & 0x400u));
            man &= 0x3FFu;
            x = sign | ((uint32_t)(127 - 15 - e) << 23) | (man << 13);
        }
    } else if (exp == 31) {
        x = sign | 0x7F800000u | (man << 13);
    } else {
        x = sign | ((exp - 15 + 127) << 23) | (man << 13);
    }
    float f;
    memcpy(&f, &x, 4);
    return f;
}

float mko_round_fp16(float x) { return mko_half_bits_to_float(mko_float_to_half_bits(x)); }

/* ------------------------------------------------------------------ */
/* attention (attention.cpp)                                          */
/* ------------------------------------------------------------------ */

/* attention.cpp:29-117 (check_shapes :12-25, tile clamp :39-40, offset :42). */
int mko_selective_flash_attn(const float* q, const float* k, const float* v, size_t lq, size_t lk,
                             size_t d, size_t dv, float scale, int causal, size_t block_m,
                             size_t block_n, float* out, float* lse, float* a_cumul,
                             size_t* aux_elements) {
    if (lq == 0 || lk == 0) return MKO_INVALID;
    if (causal && lq > lk) return MKO_INVALID;
    if (block_m < 1 || block_n < 1) return MKO_INVALID;
    const size_t bm = block_m < lq ? block_m : lq;
    const size_t bn = block_n < lk ? block_n : lk;
    const size_t offset = causal ? (lk - lq) : 0;

    memset(out, 0, sizeof(float) * lq * dv);
    for (size_t i = 0; i < lq; ++i) lse[i] = 0.0f;
    for (size_t j = 0; j < lk; ++j) a_cumul[j] = 0.0f;

    float* tile = (float*)malloc(sizeof(float) * bm * bn);
    float* run_max = (float*)malloc(sizeof(float) * lq);
    float* run_sum = (float*)malloc(sizeof(float) * lq);
    for (size_t i = 0; i < lq; ++i) {
        run_max[i] = -INFINITY;
        run_sum[i] = 0.0f;
    }
    if (aux_elements) *aux_elements = bm * bn + lq + lq;

    /* Pass 1 (:54-91): online softmax over key tiles. */
    for (size_t r0 = 0; r0 < lq; r0 += bm) {
        const size_t rend = (r0 + bm < lq) ? r0 + bm : lq;
        for (size_t c0 = 0; c0 < lk; c0 += bn) {
            const size_t cend = (c0 + bn < lk) ? c0 + bn : lk;
            for (size_t i = r0; i < rend; ++i) {
                size_t limit = cend;
                if (causal && offset + i + 1 < limit) limit = offset + i + 1;
                if (limit <= c0) continue;
                float* trow = tile + (i - r0) * bn;
                float tmax = -INFINITY;
                for (size_t j = c0; j < limit; ++j) {
                    const float s = scale * mko_dot(q + i * d, k + j * d, d);
                    trow[j - c0] = s;
                    tmax = smax(tmax, s);
                }
                const float new_max = smax(run_max[i], tmax);
                const float rescale = (run_sum[i] > 0.0f) ? expf(run_max[i] - new_max) : 0.0f;
                float* orow = out + i * dv;
                if (rescale != 1.0f) {
                    run_sum[i] *= rescale;
                    for (size_t c = 0; c < dv; ++c) orow[c] *= rescale;
                }
                for (size_t j = c0; j < limit; ++j) {
                    const float w = expf(trow[j - c0] - new_max);
                    run_sum[i] += w;
                    const float* vrow = v + j * dv;
                    for (size_t c = 0; c < dv; ++c) {
                        float p = w * vrow[c];
                        orow[c] += p;
                    }
                }
                run_max[i] = new_max;
            }
        }
    }
    /* :92-99 normalize and LSE (natural log). */
    for (size_t i = 0; i < lq; ++i) {
        const float inv = 1.0f / run_sum[i];
        float* orow = out + i * dv;
        for (size_t c = 0; c < dv; ++c) orow[c] *= inv;
        lse[i] = run_max[i] + logf(run_sum[i]);
    }
    /* Pass 2 (:101-115): column sums in fixed row order. */
    for (size_t c0 = 0; c0 < lk; c0 += bn) {
        const size_t cend = (c0 + bn < lk) ? c0 + bn : lk;
        for (size_t r0 = 0; r0 < lq; r0 += bm) {
            const size_t rend = (r0 + bm < lq) ? r0 + bm : lq;
            for (size_t i = r0; i < rend; ++i) {
                size_t limit = cend;
                if (causal && offset + i + 1 < limit) limit = offset + i + 1;
                for (size_t j = c0; j < limit; ++j) {
                    const float s = scale * mko_dot(q + i * d, k + j * d, d);
                    a_cumul[j] += expf(s - lse[i]);
                }
            }
        }
    }
    free(tile);
    free(run_max);
    free(run_sum);
    return MKO_OK;
}

/* attention.cpp:119-143 */
int mko_decode_attention(const float* q, const float* keys, const float* values, size_t n,
                         size_t d, size_t dv, float scale, float* out, float* attn) {
    if (n == 0) return MKO_INVALID;
    for (size_t j = 0; j < n; ++j) attn[j] = scale * mko_dot(q, keys + j * d, d);
    mko_softmax_inplace(attn, n);
    for (size_t c = 0; c < dv; ++c) out[c] = 0.0f;
    for (size_t j = 0; j < n; ++j) {
        const float* vrow = values + j * dv;
        for (size_t c = 0; c < dv; ++c) {
            float p = attn[j] * vrow[c];
            out[c] += p;
        }
    }
    return MKO_OK;
}

/* ------------------------------------------------------------------ */
/* quantizer (quantizer.cpp)                                          */
/* ------------------------------------------------------------------ */

/* quantizer.cpp:28-53: asymmetric min/max 2-bit, round half away from zero, clamp. */
int mko_quantize_group(const float* values, size_t n, uint8_t* codes, float* scale,
                       float* zero_point) {
    if (n == 0) return MKO_INVALID;
    float lo = values[0], hi = values[0];
    for (size_t i = 0; i < n; ++i) {
        const float v = values[i];
        if (!isfinite(v)) return MKO_DOMAIN;
        lo = smin(lo, v);
        hi = smax(hi, v);
    }
    const float zp = lo;
    const float sc = (hi - lo) / 3.0f;
    for (size_t i = 0; i < n; ++i) codes[i] = 0;
    if (sc > 0.0f) {
        for (size_t i = 0; i < n; ++i) {
            const float qv = roundf((values[i] - zp) / sc);
            const float cl = qv < 0.0f ? 0.0f : (qv > 3.0f ? 3.0f : qv);
            codes[i] = (uint8_t)cl;
        }
    }
    *scale = sc;
    *zero_point = zp;
    return MKO_OK;
}

/* quantizer.cpp:55-65 */
int mko_dequantize_group(const uint8_t* codes, size_t n, float scale, float zero_point,
                         float* out) {
    for (size_t i = 0; i < n; ++i) {
        if (codes[i] > 3) return MKO_DOMAIN;
        float p = (float)codes[i] * scale;
        out[i] = p + zero_point;
    }
    return MKO_OK;
}

/* quantizer.cpp:67-77: 16 codes per word, code i at bits 2*(i%16). */
int mko_pack_codes(const uint8_t* codes, size_t n, uint32_t* words) {
    const size_t nw = (n + 15) / 16;
    for (size_t w = 0; w < nw; ++w) words[w] = 0;
    for (size_t i = 0; i < n; ++i) {
        if (codes[i] > 3) return MKO_DOMAIN;
        words[i / 16] |= (uint32_t)codes[i] << (2 * (i % 16));
    }
    return MKO_OK;
}

/* quantizer.cpp:79-88 */
int mko_unpack_codes(const uint32_t* words, size_t n_words, size_t count, uint8_t* codes) {
    if (count > n_words * 16) return MKO_INVALID;
    for (size_t i = 0; i < count; ++i) codes[i] = (uint8_t)((words[i / 16] >> (2 * (i % 16))) & 3u);
    return MKO_OK;
}

/* append_block, quantizer.cpp:102-136 (append_group :92-98). */
int mko_quantize_block(const float* block, size_t rows, size_t cols, int axis,
                       size_t group_size, uint8_t* codes, float* params, size_t* n_groups_out) {
    if (rows == 0 || cols == 0) return MKO_INVALID;
    if (group_size < 1) return MKO_INVALID;
    const size_t gs = group_size;
    float* scratch = (float*)malloc(sizeof(float) * gs);
    size_t code_idx = 0, g_idx = 0;
    int st = MKO_OK;
    if (axis == 0) { /* PerChannel: channel-major, token groups within the block */
        for (size_t c = 0; c < cols && st == MKO_OK; ++c) {
            for (size_t g0 = 0; g0 < rows; g0 += gs) {
                const size_t glen = (gs < rows - g0) ? gs : rows - g0;
                for (size_t i = 0; i < glen; ++i) scratch[i] = block[(g0 + i) * cols + c];
                st = mko_quantize_group(scratch, glen, codes + code_idx, &params[2 * g_idx],
                                        &params[2 * g_idx + 1]);
                if (st != MKO_OK) break;
                code_idx += glen;
                ++g_idx;
            }
        }
    } else { /* PerToken: token-major, channel groups */
        for (size_t r = 0; r < rows && st == MKO_OK; ++r) {
            for (size_t g0 = 0; g0 < cols; g0 += gs) {
                const size_t glen = (gs < cols - g0) ? gs : cols - g0;
                st = mko_quantize_group(block + r * cols + g0, glen, codes + code_idx,
                                        &params[2 * g_idx], &params[2 * g_idx + 1]);
                if (st != MKO_OK) break;
                code_idx += glen;
                ++g_idx;
            }
        }
    }
    free(scratch);
    if (n_groups_out) *n_groups_out = g_idx;
    return st;
}

/* dequantize_matrix, quantizer.cpp:153-195, for one block. */
int mko_dequantize_block(const uint8_t* codes, const float* params, size_t rows, size_t cols,
                         int axis, size_t group_size, int param_fp16, float* out) {
    const size_t gs = group_size;
    size_t code_idx = 0, g_idx = 0;
    if (axis == 0) {
        for (size_t c = 0; c < cols; ++c) {
            for (size_t g0 = 0; g0 < rows; g0 += gs) {
                const size_t glen = (gs < rows - g0) ? gs : rows - g0;
                float sc = params[2 * g_idx], zp = params[2 * g_idx + 1];
                if (param_fp16) { sc = mko_round_fp16(sc); zp = mko_round_fp16(zp); }
                ++g_idx;
                for (size_t i = 0; i < glen; ++i) {
                    float p = (float)codes[code_idx++] * sc;
                    out[(g0 + i) * cols + c] = p + zp;
                }
            }
        }
    } else {
        for (size_t r = 0; r < rows; ++r) {
            for (size_t g0 = 0; g0 < cols; g0 += gs) {
                const size_t glen = (gs < cols - g0) ? gs : cols - g0;
                float sc = params[2 * g_idx], zp = params[2 * g_idx + 1];
                if (param_fp16) { sc = mko_round_fp16(sc); zp = mko_round_fp16(zp); }
                ++g_idx;
                for (size_t i = 0; i < glen; ++i) {
                    float p = (float)codes[code_idx++] * sc;
                    out[r * cols + g0 + i] = p + zp;
                }
            }
        }
    }
    return MKO_OK;
}

/* ------------------------------------------------------------------ */
/* selection (selection.cpp)                                          */
/* ------------------------------------------------------------------ */

static const float* g_sort_scores; /* qsort has no context argument; oracle is single-threaded */

/* score desc, index asc: identical to stable_sort by score desc over an iota (selection.cpp:22-27). */
static int cmp_desc_idx(const void* pa, const void* pb) {
    const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    const float sa = g_sort_scores[a], sb = g_sort_scores[b];
    if (sa > sb) return -1;
    if (sb > sa) return 1;
    return (a < b) ? -1 : (a > b);
}

static int cmp_i64(const void* pa, const void* pb) {
    const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    return (a < b) ? -1 : (a > b);
}

/* selection.cpp:10-33 */
int mko_select_token_counts(const float* a_cumul, size_t l, size_t hh_count, size_t rw_count,
                            int64_t* kept, size_t* n_kept, int64_t* hh_out, size_t* n_hh,
                            int64_t* rw_out, size_t* n_rw, int* clamped) {
    int cl = 0;
    if (hh_count + rw_count >= l) {
        cl = hh_count + rw_count > l;
        rw_count = rw_count < l ? rw_count : l;
        hh_count = l - rw_count;
    }
    const size_t pool = l - rw_count;
    const size_t nh = hh_count < pool ? hh_count : pool;
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (pool ? pool : 1));
    for (size_t i = 0; i < pool; ++i) order[i] = (int64_t)i;
    g_sort_scores = a_cumul;
    qsort(order, pool, sizeof(int64_t), cmp_desc_idx);
    qsort(order, nh, sizeof(int64_t), cmp_i64);
    for (size_t i = 0; i < nh; ++i) kept[i] = order[i];
    for (size_t i = 0; i < rw_count; ++i) kept[nh + i] = (int64_t)(l - rw_count + i);
    if (hh_out) memcpy(hh_out, order, sizeof(int64_t) * nh);
    if (n_hh) *n_hh = nh;
    if (rw_out) for (size_t i = 0; i < rw_count; ++i) rw_out[i] = (int64_t)(l - rw_count + i);
    if (n_rw) *n_rw = rw_count;
    *n_kept = nh + rw_count;
    if (clamped) *clamped = cl;
    free(order);
    return MKO_OK;
}

/* selection.cpp:35-46: floor(alpha * l) counts. */
int mko_select_tokens(const float* a_cumul, size_t l, double alpha_hh, double alpha_rw,
                      int64_t* kept, size_t* n_kept, int* clamped) {
    if (alpha_hh < 0 || alpha_rw < 0) return MKO_INVALID;
    const size_t hh = (size_t)floor(alpha_hh * (double)l);
    const size_t rw = (size_t)floor(alpha_rw * (double)l);
    return mko_select_token_counts(a_cumul, l, hh, rw, kept, n_kept, NULL, NULL, NULL, NULL,
                                   clamped);
}

/* selection.cpp:48-59 */
int mko_allocate_uniform(size_t total_hh, size_t layers, int64_t* out) {
    if (layers < 1) return MKO_INVALID;
    for (size_t i = 0; i < layers; ++i) out[i] = (int64_t)(total_hh / layers);
    for (size_t i = 0; i < total_hh % layers; ++i) ++out[i];
    return MKO_OK;
}

/* selection.cpp:61-83: linear interpolation first -> last, llround(max(v, 0)). */
int mko_allocate_pyramid(size_t mean_x, size_t layers, size_t depth, int bottom_heavy,
                         int64_t* out) {
    if (layers < 1 || depth < 1) return MKO_INVALID;
    const double x = (double)mean_x;
    const double small_end = x / (double)depth;
    const double large_end = 2.0 * x - small_end;
    const double first = bottom_heavy ? large_end : small_end;
    const double last = bottom_heavy ? small_end : large_end;
    for (size_t i = 0; i < layers; ++i) {
        const double t = (layers == 1) ? 0.0 : (double)i / (double)(layers - 1);
        const double span = (last - first) * t;
        const double vv = first + span;
        out[i] = (int64_t)llround(vv > 0.0 ? vv : 0.0);
    }
    return MKO_OK;
}

/* selection.cpp:85-128 */
typedef struct {
    double frac;
    size_t idx;
} mko_frac;

int mko_allocate_variance(const float* variance, size_t layers, size_t total_hh, int inverse,
                          int64_t* out, int* uniform_fallback) {
    if (layers < 1) return MKO_INVALID;
    const double eps = 1e-6;
    double* shares = (double*)malloc(layers * sizeof(double));
    mko_frac* fr = (mko_frac*)malloc(layers * sizeof(mko_frac));
    if (!shares || !fr) { free(shares); free(fr); return MKO_RUNTIME; }
    double sum = 0.0;
    int all_zero = 1;
    for (size_t i = 0; i < layers; ++i) {
        if (variance[i] < 0) { free(shares); free(fr); return MKO_INVALID; }
        if (variance[i] > 0) all_zero = 0;
        shares[i] = inverse ? 1.0 / ((double)variance[i] + eps) : (double)variance[i];
        sum += shares[i];
    }
    *uniform_fallback = 0;
    if (all_zero && !inverse) {
        free(shares); free(fr);
        *uniform_fallback = 1;
        return mko_allocate_uniform(total_hh, layers, out);
    }
    size_t assigned = 0;
    for (size_t i = 0; i < layers; ++i) {
        const double target = (double)total_hh * shares[i] / sum;
        out[i] = (int64_t)floor(target);
        assigned += (size_t)out[i];
        fr[i].frac = target - floor(target);
        fr[i].idx = i;
    }
    /* stable sort by fraction, descending (insertion sort keeps equal fractions in index order) */
    for (size_t i = 1; i < layers; ++i) {
        mko_frac x = fr[i];
        size_t j = i;
        while (j > 0 && fr[j - 1].frac < x.frac) { fr[j] = fr[j - 1]; --j; }
        fr[j] = x;
    }
    for (size_t r = 0; assigned < total_hh; ++r, ++assigned) ++out[fr[r % layers].idx];
    free(shares);
    free(fr);
    return MKO_OK;
}

/* selection.cpp:130-146 */
int mko_layer_score_variance(const float* a, size_t n, float* out) {
    if (n == 0) return MKO_INVALID;
    double mean = 0.0;
    for (size_t i = 0; i < n; ++i) mean += a[i];
    mean /= (double)n;
    double var = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double d = a[i] - mean;
        var += d * d;
    }
    *out = (float)(var / (double)n);
    return MKO_OK;
}

/* ------------------------------------------------------------------ */
/* H2O comparison baseline (harness.cpp:75-150)                        */
/* ------------------------------------------------------------------ */

/* evict_to_budget (harness.cpp:83-106): drop the first lowest score outside the rw most
   recent entries until n <= budget; the kept list holds original positions in order */
static size_t h2o_evict(size_t* pos, const double* score, size_t n, size_t budget, size_t rw) {
    while (n > budget) {
        const size_t protect_from = n > rw ? n - rw : 0;
        size_t victim = n;
        double best = INFINITY;
        for (size_t i = 0; i < protect_from; ++i)
            if (score[pos[i]] < best) {
                best = score[pos[i]];
                victim = i;
            }
        if (victim == n) break;
        memmove(pos + victim, pos + victim + 1, (n - victim - 1) * sizeof(size_t));
        --n;
    }
    return n;
}

/* h2o_dynamic_baseline (harness.cpp:108-150): scores per original position in double;
   attn = scale * dot (matrix.cpp:60-66), softmax_inplace (matrix.cpp:83-99) with expf */
int mko_h2o_dynamic_baseline(const float* pk, size_t l, size_t d, const float* scores, const float* qs,
                             const float* ks, size_t steps, size_t hh, size_t rw, float scale, int32_t* kept,
                             size_t stride, int32_t* counts) {
    if (hh + rw < 1) return MKO_INVALID;
    const size_t total = l + steps, budget = hh + rw;
    size_t* pos = (size_t*)malloc((total + 1) * sizeof(size_t));
    double* score = (double*)malloc((total + 1) * sizeof(double));
    float* attn = (float*)malloc((total + 1) * sizeof(float));
    if (!pos || !score || !attn) {
        free(pos); free(score); free(attn);
        return MKO_INVALID;
    }
    for (size_t i = 0; i < l; ++i) {
        pos[i] = i;
        score[i] = (double)scores[i];
    }
    size_t n = h2o_evict(pos, score, l, budget, rw);
    for (size_t i = 0; i < n; ++i) kept[i] = (int32_t)pos[i];
    counts[0] = (int32_t)n;
    for (size_t s = 0; s < steps; ++s) {
        pos[n] = l + s;
        score[l + s] = 0.0;
        ++n;
        const float* q = qs + s * d;
        for (size_t j = 0; j < n; ++j) {
            const size_t p = pos[j];
            const float* key = p < l ? pk + p * d : ks + (p - l) * d;
            float acc = 0.0f;
            for (size_t c = 0; c < d; ++c) acc += q[c] * key[c];
            attn[j] = scale * acc;
        }
        float m = attn[0];
        for (size_t j = 1; j < n; ++j) m = attn[j] > m ? attn[j] : m;
        float sum = 0.0f;
        for (size_t j = 0; j < n; ++j) {
            attn[j] = expf(attn[j] - m);
            sum += attn[j];
        }
        for (size_t j = 0; j < n; ++j) score[pos[j]] += (double)(attn[j] / sum);
        n = h2o_evict(pos, score, n, budget, rw);
        for (size_t i = 0; i < n; ++i) kept[(s + 1) * stride + i] = (int32_t)pos[i];
        counts[s + 1] = (int32_t)n;
    }
    free(pos); free(score); free(attn);
    return MKO_OK;
}

/* ------------------------------------------------------------------ */
/* cache engine (cache_engine.cpp)                                    */
/* ------------------------------------------------------------------ */

typedef struct {
    uint8_t* codes; /* one byte per code, stream order */
    size_t n_codes, cap_codes;
    float* params; /* (scale, zero) pairs */
    size_t n_groups, cap_groups;
    int64_t* block_rows;
    size_t n_blocks, cap_blocks;
} qtensor;

struct mko_cache {
    size_t d, n_r, gs;
    qtensor key, value;   /* PerChannel keys, PerToken values */
    float* r_key;         /* n_r x d residual */
    float* r_value;
    size_t n_res;
    size_t tokens_quantized;
};

static void* grow(void* p, size_t* cap, size_t need, size_t elem) {
    if (need <= *cap) return p;
    size_t nc = *cap ? *cap : 64;
    while (nc < need) nc *= 2;
    *cap = nc;
    return realloc(p, nc * elem);
}

/* append_block on a qtensor (quantizer.cpp:102-136). */
static int qt_append(qtensor* t, const float* block, size_t rows, size_t cols, int axis,
                     size_t gs) {
    if (rows == 0) return MKO_INVALID; /* "append_block: empty block" */
    const size_t groups = axis == 0 ? cols * ((rows + gs - 1) / gs) : rows * ((cols + gs - 1) / gs);
    t->codes = (uint8_t*)grow(t->codes, &t->cap_codes, t->n_codes + rows * cols, 1);
    t->params = (float*)grow(t->params, &t->cap_groups, t->n_groups + groups, 2 * sizeof(float));
    t->block_rows = (int64_t*)grow(t->block_rows, &t->cap_blocks, t->n_blocks + 1, sizeof(int64_t));
    size_t ng = 0;
    int st = mko_quantize_block(block, rows, cols, axis, gs, t->codes + t->n_codes,
                                t->params + 2 * t->n_groups, &ng);
    if (st != MKO_OK) return st;
    t->n_codes += rows * cols;
    t->n_groups += ng;
    t->block_rows[t->n_blocks++] = (int64_t)rows;
    return MKO_OK;
}

/* dequantize_matrix (quantizer.cpp:153-195): all blocks, row-major [rows x cols]. */
static void qt_dequant(const qtensor* t, size_t cols, int axis, size_t gs, int param_fp16,
                       float* out) {
    size_t code_off = 0, group_off = 0, row0 = 0;
    for (size_t b = 0; b < t->n_blocks; ++b) {
        const size_t rows = (size_t)t->block_rows[b];
        mko_dequantize_block(t->codes + code_off, t->params + 2 * group_off, rows, cols, axis, gs,
                             param_fp16, out + row0 * cols);
        code_off += rows * cols;
        group_off += axis == 0 ? cols * ((rows + gs - 1) / gs) : rows * ((cols + gs - 1) / gs);
        row0 += rows;
    }
}

/* make_cache, cache_engine.cpp:9-30 */
int mko_cache_create(size_t d, size_t n_r, size_t group_size, mko_cache** out) {
    if (d == 0) return MKO_INVALID;
    if (group_size < 1 || n_r == 0 || n_r % group_size != 0) return MKO_INVALID;
    mko_cache* c = (mko_cache*)calloc(1, sizeof(mko_cache));
    c->d = d;
    c->n_r = n_r;
    c->gs = group_size;
    c->r_key = (float*)calloc(n_r * d, sizeof(float));
    c->r_value = (float*)calloc(n_r * d, sizeof(float));
    *out = c;
    return MKO_OK;
}

void mko_cache_destroy(mko_cache* c) {
    if (!c) return;
    free(c->key.codes); free(c->key.params); free(c->key.block_rows);
    free(c->value.codes); free(c->value.params); free(c->value.block_rows);
    free(c->r_key); free(c->r_value);
    free(c);
}

/* store_block, cache_engine.cpp:34-52 (TwoBit mode). */
static int store_block(mko_cache* c, const float* kb, const float* vb, size_t rows) {
    int st = qt_append(&c->key, kb, rows, c->d, 0, c->gs);
    if (st != MKO_OK) return st;
    st = qt_append(&c->value, vb, rows, c->d, 1, c->gs);
    if (st != MKO_OK) return st;
    c->tokens_quantized += rows;
    return MKO_OK;
}

/* prefill, cache_engine.cpp:56-77 (shape checks :60-68 are the caller's l/d contract). */
int mko_cache_prefill(mko_cache* c, const float* k, const float* v, const float* a_cumul,
                      size_t l, size_t hh_count, size_t rw_count) {
    if (hh_count + rw_count == 0) return MKO_RUNTIME;
    int64_t* kept = (int64_t*)malloc(sizeof(int64_t) * (l ? l : 1));
    size_t nk = 0;
    mko_select_token_counts(a_cumul, l, hh_count, rw_count, kept, &nk, NULL, NULL, NULL, NULL,
                            NULL);
    const size_t d = c->d;
    float* kg = (float*)malloc(sizeof(float) * (nk ? nk : 1) * d);
    float* vg = (float*)malloc(sizeof(float) * (nk ? nk : 1) * d);
    for (size_t i = 0; i < nk; ++i) { /* gather_rows, matrix.cpp:38-47 */
        memcpy(kg + i * d, k + (size_t)kept[i] * d, sizeof(float) * d);
        memcpy(vg + i * d, v + (size_t)kept[i] * d, sizeof(float) * d);
    }
    int st = store_block(c, kg, vg, nk);
    free(kept); free(kg); free(vg);
    return st;
}

/* decode_append, cache_engine.cpp:79-90 */
int mko_cache_append(mko_cache* c, const float* t_k, const float* t_v) {
    memcpy(c->r_key + c->n_res * c->d, t_k, sizeof(float) * c->d);
    memcpy(c->r_value + c->n_res * c->d, t_v, sizeof(float) * c->d);
    ++c->n_res;
    if (c->n_res == c->n_r) {
        int st = store_block(c, c->r_key, c->r_value, c->n_r);
        if (st != MKO_OK) return st;
        c->n_res = 0;
    }
    return MKO_OK;
}

/* decode_step body after the append (cache_engine.cpp:110-137). */
int mko_cache_attend(const mko_cache* c, const float* t_q, float scale, int param_fp16,
                     float* out) {
    const size_t d = c->d, nq = c->tokens_quantized, nr = c->n_res, n = nq + nr;
    if (n == 0) return MKO_RUNTIME;
    float* keys = (float*)malloc(sizeof(float) * (nq ? nq : 1) * d);
    float* vals = (float*)malloc(sizeof(float) * (nq ? nq : 1) * d);
    float* attn = (float*)malloc(sizeof(float) * n);
    qt_dequant(&c->key, d, 0, c->gs, param_fp16, keys);
    qt_dequant(&c->value, d, 1, c->gs, param_fp16, vals);
    for (size_t j = 0; j < nq; ++j) attn[j] = scale * mko_dot(t_q, keys + j * d, d);
    for (size_t j = 0; j < nr; ++j) attn[nq + j] = scale * mko_dot(t_q, c->r_key + j * d, d);
    mko_softmax_inplace(attn, n);
    for (size_t ch = 0; ch < d; ++ch) out[ch] = 0.0f;
    for (size_t j = 0; j < nq; ++j)
        for (size_t ch = 0; ch < d; ++ch) { float p = attn[j] * vals[j * d + ch]; out[ch] += p; }
    for (size_t j = 0; j < nr; ++j)
        for (size_t ch = 0; ch < d; ++ch) { float p = attn[nq + j] * c->r_value[j * d + ch]; out[ch] += p; }
    free(keys); free(vals); free(attn);
    return MKO_OK;
}

/* decode_step, cache_engine.cpp:100-138: empty check, append (flush first), attend. */
int mko_cache_decode_step(mko_cache* c, const float* t_q, const float* t_k, const float* t_v,
                          float scale, int param_fp16, float* out) {
    if (c->tokens_quantized + c->n_res == 0) return MKO_RUNTIME;
    int st = mko_cache_append(c, t_k, t_v);
    if (st != MKO_OK) return st;
    return mko_cache_attend(c, t_q, scale, param_fp16, out);
}

size_t mko_cache_tokens_quantized(const mko_cache* c) { return c->tokens_quantized; }
size_t mko_cache_tokens_residual(const mko_cache* c) { return c->n_res; }
size_t mko_cache_n_blocks(const mko_cache* c) { return c->key.n_blocks; }
size_t mko_cache_total_codes(const mko_cache* c, int which) {
    return which ? c->value.n_codes : c->key.n_codes;
}
size_t mko_cache_n_params(const mko_cache* c, int which) {
    return which ? c->value.n_groups : c->key.n_groups;
}

int mko_cache_export(const mko_cache* c, int which, uint32_t* packed_words, float* params,
                     int64_t* block_rows) {
    const qtensor* t = which ? &c->value : &c->key;
    if (packed_words) mko_pack_codes(t->codes, t->n_codes, packed_words);
    if (params) memcpy(params, t->params, sizeof(float) * 2 * t->n_groups);
    if (block_rows) memcpy(block_rows, t->block_rows, sizeof(int64_t) * t->n_blocks);
    return MKO_OK;
}

int mko_cache_residual(const mko_cache* c, float* r_key, float* r_value) {
    memcpy(r_key, c->r_key, sizeof(float) * c->n_res * c->d);
    memcpy(r_value, c->r_value, sizeof(float) * c->n_res * c->d);
    return MKO_OK;
}

/* ------------------------------------------------------------------ */
/* synthetic inputs                                     */
/* ------------------------------------------------------------------ */

uint64_t mko_synth_mix(uint64_t seed, uint64_t stream, uint64_t index) {
    uint64_t z = seed + stream * 0xD1B54A32D192ED03ull + (index + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void mko_synth_fp16(uint64_t seed, uint64_t stream, size_t n, uint16_t* out_half_bits) {
    for (size_t i = 0; i < n; ++i) {
        const uint64_t z = mko_synth_mix(seed, stream, i);
        const int32_t s = (int32_t)(z & 0xFFFFu) + (int32_t)((z >> 16) & 0xFFFFu) +
                          (int32_t)((z >> 32) & 0xFFFFu) + (int32_t)(z >> 48) - 131070;
        const float f = (float)s * 2.6428997e-05f;
        out_half_bits[i] = mko_float_to_half_bits(f);
    }
}
