/*
 * minikv_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the MiniKV reference hot path (the CPU reference in
 * /root/reference/proj/core/src), used as the parity checker for the B200
 * kernels.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product path never links it.
 *
 * Every function cites the reference file:line it restates.  Arithmetic is
 * fp32 in the reference's exact operation order (compile with
 * -ffp-contract=off and no -march so no FMA contraction happens, matching the
 * reference's Release build), so results are bit-identical to the reference
 * compiled the same way; tests/test_oracle_vs_reference.py pins that against
 * oracle/_ref (the reference itself, compiled from its own sources).
 *
 * Status codes mirror the reference's exception classes:
 *   0 ok, 1 std::invalid_argument, 2 std::domain_error,
 *   3 std::runtime_error, 4 std::out_of_range.
 */
#ifndef MINIKV_ORACLE_H
#define MINIKV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { MKO_OK = 0, MKO_INVALID = 1, MKO_DOMAIN = 2, MKO_RUNTIME = 3, MKO_RANGE = 4 };

/* ---- numerics helpers (matrix.cpp) ---- */
float mko_dot(const float* a, const float* b, size_t n);             /* matrix.cpp:60-66 */
int mko_softmax_inplace(float* x, size_t n);                          /* matrix.cpp:83-99 */
float mko_round_fp16(float x);                                        /* IEEE RNE to binary16 and back */
uint16_t mko_float_to_half_bits(float x);
float mko_half_bits_to_float(uint16_t h);

/* ---- attention (attention.cpp) ---- */
/* attention.cpp:29-117.  q[lq*d], k[lk*d], v[lk*dv] row-major; out[lq*dv], lse[lq], a_cumul[lk]. */
int mko_selective_flash_attn(const float* q, const float* k, const float* v, size_t lq, size_t lk,
                             size_t d, size_t dv, float scale, int causal, size_t block_m,
                             size_t block_n, float* out, float* lse, float* a_cumul,
                             size_t* aux_elements);
/* attention.cpp:119-143.  keys[n*d], values[n*dv]; out[dv], attn[n]. */
int mko_decode_attention(const float* q, const float* keys, const float* values, size_t n,
                         size_t d, size_t dv, float scale, float* out, float* attn);

/* ---- quantizer (quantizer.cpp) ---- */
int mko_quantize_group(const float* values, size_t n, uint8_t* codes, float* scale,
                       float* zero_point);                                         /* :28-53 */
int mko_dequantize_group(const uint8_t* codes, size_t n, float scale, float zero_point,
                         float* out);                                              /* :55-65 */
int mko_pack_codes(const uint8_t* codes, size_t n, uint32_t* words);              /* :67-77 */
int mko_unpack_codes(const uint32_t* words, size_t n_words, size_t count,
                     uint8_t* codes);                                              /* :79-88 */
/* Quantize one block (append_block, quantizer.cpp:102-136) into the continuous code stream.
 * axis 0 = PerChannel (keys), 1 = PerToken (values).  codes[rows*cols] in stream order;
 * params[2*n_groups] as (scale, zero) pairs in stream order.  *n_groups_out receives the
 * number of groups written. */
int mko_quantize_block(const float* block, size_t rows, size_t cols, int axis,
                       size_t group_size, uint8_t* codes, float* params, size_t* n_groups_out);
/* dequantize_matrix for one block (quantizer.cpp:153-195).  param_fp16 != 0 rounds each
 * scale/zero to binary16 first (the device stores fp16 params). */
int mko_dequantize_block(const uint8_t* codes, const float* params, size_t rows, size_t cols,
                         int axis, size_t group_size, int param_fp16, float* out);

/* ---- selection (selection.cpp) ---- */
/* selection.cpp:10-33.  kept[] receives sort(hh) ++ rw (size n_kept), hh_out/rw_out optional. */
int mko_select_token_counts(const float* a_cumul, size_t l, size_t hh_count, size_t rw_count,
                            int64_t* kept, size_t* n_kept, int64_t* hh_out, size_t* n_hh,
                            int64_t* rw_out, size_t* n_rw, int* clamped);
int mko_select_tokens(const float* a_cumul, size_t l, double alpha_hh, double alpha_rw,
                      int64_t* kept, size_t* n_kept, int* clamped);               /* :35-46 */
int mko_allocate_uniform(size_t total_hh, size_t layers, int64_t* out);            /* :48-59 */
/* selection.cpp:85-128: shares var (Prop) or 1/(var + 1e-6) (Inv) in double, all-zero Prop
 * falls back to uniform (flag), largest-remainder rounding, remainder ties to the lower layer. */
int mko_allocate_variance(const float* variance, size_t layers, size_t total_hh, int inverse,
                          int64_t* out, int* uniform_fallback);
/* selection.cpp:130-146: population variance, two double passes in index order. */
int mko_layer_score_variance(const float* a_cumul, size_t n, float* out);
/* harness.cpp:108-150: kept [(steps + 1) x stride] ascending positions, counts [steps + 1] */
int mko_h2o_dynamic_baseline(const float* prompt_k, size_t l, size_t d, const float* prompt_scores,
                             const float* qs, const float* ks, size_t steps, size_t hh, size_t rw, float scale,
                             int32_t* kept, size_t stride, int32_t* counts);
int mko_allocate_pyramid(size_t mean_x, size_t layers, size_t depth, int bottom_heavy,
                         int64_t* out);                                            /* :61-83 */

/* ---- cache engine (cache_engine.cpp) for one (seq, layer, kv-head) unit ---- */
typedef struct mko_cache mko_cache;
/* make_cache, cache_engine.cpp:9-30 */
int mko_cache_create(size_t d, size_t n_r, size_t group_size, mko_cache** out);
void mko_cache_destroy(mko_cache* c);
/* prefill, cache_engine.cpp:56-77 (select -> gather -> quantize) */
int mko_cache_prefill(mko_cache* c, const float* k, const float* v, const float* a_cumul,
                      size_t l, size_t hh_count, size_t rw_count);
/* decode_append, cache_engine.cpp:79-90 */
int mko_cache_append(mko_cache* c, const float* t_k, const float* t_v);
/* decode_step, cache_engine.cpp:100-138 (append first, one softmax over [deq ; residual]). */
int mko_cache_decode_step(mko_cache* c, const float* t_q, const float* t_k, const float* t_v,
                          float scale, int param_fp16, float* out);
/* Single-query attention of an extra query over the current cache state without appending
 * (GQA composition: decode_attention over vstack(stored, residual)). */
int mko_cache_attend(const mko_cache* c, const float* t_q, float scale, int param_fp16,
                     float* out);
size_t mko_cache_tokens_quantized(const mko_cache* c);
size_t mko_cache_tokens_residual(const mko_cache* c);
size_t mko_cache_n_blocks(const mko_cache* c);
size_t mko_cache_total_codes(const mko_cache* c, int which); /* which 0 = keys, 1 = values */
size_t mko_cache_n_params(const mko_cache* c, int which);
/* Export in the reference QuantizedTensor format: packed_words (ceil(codes/16) u32),
 * params (2 floats per group), block_rows[n_blocks]. */
int mko_cache_export(const mko_cache* c, int which, uint32_t* packed_words, float* params,
                     int64_t* block_rows);
int mko_cache_residual(const mko_cache* c, float* r_key, float* r_value);

/* ---- synthetic inputs: integer-exact approximate N(0,1) rounded to fp16 ----
 * value(seed, stream, i) = RN_fp16( (float)(sum of four 16-bit lanes of
 * splitmix_mix(seed, stream, i)) - 131070) * 2.6429605e-5f )
 * Every step is exactly rounded, so the device generator reproduces the same bits. */
uint64_t mko_synth_mix(uint64_t seed, uint64_t stream, uint64_t index);
void mko_synth_fp16(uint64_t seed, uint64_t stream, size_t n, uint16_t* out_half_bits);

#ifdef __cplusplus
}
#endif
#endif
