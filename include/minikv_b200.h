/*
 * minikv_b200.h -- C ABI of the B200-native MiniKV attention hot path.
 *
 * Drop-in boundary for the reference C++ core (namespace minikv in
 * /root/reference/proj/core/include/minikv).  Every entry point names the
 * reference interface it replaces.  Plain pointers and sizes only; device
 * pointers are CUDA global memory on the current device; `stream` is a
 * cudaStream_t passed as void*.  All compute calls are stream-ordered and
 * asynchronous; a cache handle is single-writer (the reference's
 * KVCacheLayer contract): distinct caches may be driven concurrently.
 *
 * Errors never throw across the ABI.  Every call returns an mkv_status whose
 * value maps 1:1 onto the reference's exception class; the
 * message is available from mkv_last_error() on the calling thread.
 *
 * Device data layout:
 *   Q/K/V/X_O   fp16, [.., tokens, head_dim] with unit-stride channels
 *   LSE         fp32 [B, Hq, Lq]       A_cumul fp32 [B, Hkv, Lk] (GQA-summed)
 *   cache       16-token pages of 16*head_dim bytes: 2-bit K codes (per-channel
 *               groups of 16 tokens) + fp16 (scale, zero), 2-bit V codes
 *               (per-token groups of 16 channels) + fp16 (scale, zero), in an
 *               mma-fragment-native order; fp16 residual ring of n_r tokens.
 */
#ifndef MINIKV_B200_H
#define MINIKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MKV_ABI_VERSION 1

typedef enum {
    MKV_OK = 0,
    MKV_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    MKV_ERR_DOMAIN = 2,           /* std::domain_error (non-finite input, code > 3) */
    MKV_ERR_RUNTIME = 3,          /* std::runtime_error (zero kept, empty cache) */
    MKV_ERR_OUT_OF_RANGE = 4,     /* std::out_of_range */
    MKV_ERR_CUDA = 5,             /* CUDA runtime / launch failure */
    MKV_ERR_UNSUPPORTED = 6       /* not an sm_100 device, or an unsupported shape */
} mkv_status;

/* Thread-local text of the last error on this thread ("" if none). */
const char* mkv_last_error(void);
int mkv_abi_version(void);
/* Succeeds only on a compute-capability 10.0 device (the kernels are sm_100a). */
int mkv_device_check(int device);

/* ------------------------------------------------------------------------ */
/* K1  selective flash-attention prefill                                     */
/* replaces: AttentionResult selective_flash_attn(q, k, v, scale, causal,     */
/*           TileConfig)        attention.hpp:38-39, attention.cpp:29-117     */
/* ------------------------------------------------------------------------ */
typedef struct {
    const void* q;       /* fp16 [B, Hq, Lq, d]: element (b,h,t,c) at b*q_sb + h*q_sh + t*q_st + c */
    int64_t q_sb, q_sh, q_st;
    const void* k;       /* fp16 [B, Hkv, Lk, d] */
    int64_t k_sb, k_sh, k_st;
    const void* v;       /* fp16 [B, Hkv, Lk, d] */
    int64_t v_sb, v_sh, v_st;
    void* out;           /* fp16 X_O [B, Hq, Lq, d] */
    int64_t o_sb, o_sh, o_st;
    float* lse;          /* fp32 [B, Hq, Lq] contiguous (natural log, attention.cpp:98) */
    float* a_cumul;      /* fp32 [B, Hkv, Lk] contiguous; sum over the G q-heads of each kv-head */
    int batch, n_q_heads, n_kv_heads, len_q, len_k, head_dim;
    float scale;
    int causal;          /* query i sees keys 0 .. len_k - len_q + i (attention.cpp:42,60) */
} mkv_prefill_args;
int mkv_prefill_attn(const mkv_prefill_args* args, void* stream);

/* ------------------------------------------------------------------------ */
/* K2  rectified top-k token selection                                       */
/* replaces: SelectionResult select_token_counts(a_cumul, hh, rw)            */
/*           selection.hpp:34-35, selection.cpp:10-33                        */
/* kept[u] = sort(top-hh of a_cumul[u][0, L-rw) by value desc, ties to the   */
/* lower index) ++ [L-rw, L).  n_kept[u] = min(hh[u] + rw, L).               */
/* ------------------------------------------------------------------------ */
typedef struct {
    const float* a_cumul;      /* device fp32 [n_units, a_stride] */
    int64_t a_stride;
    int n_units, length;
    const int32_t* hh_count;   /* host int32 [n_units] */
    int rw_count;
    int32_t* kept;             /* device int32 [n_units, kept_stride] ascending */
    int64_t kept_stride;
    int32_t* n_kept;           /* device int32 [n_units] (optional) */
} mkv_select_args;
int mkv_select(const mkv_select_args* args, void* stream);

/* Host helpers with the reference's exact arithmetic (selection.cpp:48-83). */
int mkv_allocate_pyramid(size_t mean_budget_x, size_t layers, size_t depth, int bottom_heavy,
                         int64_t* per_layer_hh);
int mkv_allocate_uniform(size_t total_hh, size_t layers, int64_t* per_layer_hh);
/* replaces: LayerAllocation allocate_variance(per_layer_variance, total_hh, mode)      */
/*           selection.hpp:52-56, selection.cpp:85-128 (host arithmetic, bit-exact);    */
/* inverse = 0: VarianceMode::Prop, 1: VarianceMode::Inv; *uniform_fallback as the     */
/* reference's LayerAllocation::uniform_fallback.                                       */
int mkv_allocate_variance(const float* per_layer_variance, size_t layers, size_t total_hh,
                          int inverse, int64_t* per_layer_hh, int* uniform_fallback);
/* replaces: float layer_score_variance(a_cumul)  selection.hpp:58-59,                */
/*           selection.cpp:130-146 -- on the device, for n_units rows of A_cumul at    */
/* once (fp32 [n_units, length], row stride a_stride): population variance with two   */
/* fp64 passes per row -> out fp32 [n_units] (device), stream-ordered.                 */
int mkv_score_variance(const float* a_cumul, int64_t a_stride, int n_units, int length, float* out,
                       void* stream);

/* replaces: H2OBaselineTrace h2o_dynamic_baseline(prompt_k, prompt_scores, decode_qs,    */
/*           decode_ks, hh_budget, rw_budget, scale)  harness.hpp:33-43,              */
/*           harness.cpp:83-150 -- the step-wise greedy H2O comparison policy on the    */
/* device (one CTA).  All pointers are device fp32: prompt_k [l_prompt, d] (row stride   */
/* ld_k), prompt_scores [l_prompt], qs / ks [steps, d].  Output kept [steps + 1,         */
/* kept_stride] int32 (ascending original positions; row 0 = after the prompt eviction)  */
/* and kept_count [steps + 1]; kept_stride >= min(l_prompt + steps, hh + rw).  Same      */
/* arithmetic order as the reference, so the kept sets are bit-identical to it.         */
typedef struct {
    const float* prompt_k;
    int64_t ld_k;
    const float* prompt_scores;
    const float* qs;
    const float* ks;
    int l_prompt, d, steps;
    int64_t hh_budget, rw_budget;
    float scale;
    int32_t* kept;
    int64_t kept_stride;
    int32_t* kept_count;
} mkv_h2o_args;
int mkv_h2o_dynamic_baseline(const mkv_h2o_args* args, void* stream);

/* ------------------------------------------------------------------------ */
/* Device KV cache: one handle owns n_units (seq, layer, kv-head) caches.    */
/* replaces: KVCacheLayer make_cache(d, n_r, gs, mode)  cache_engine.hpp:44-46 */
/* ------------------------------------------------------------------------ */
typedef struct mkv_cache mkv_cache;

typedef struct {
    int n_units;
    int head_dim;               /* 128 (the device layout; other values: MKV_ERR_UNSUPPORTED) */
    int n_r;                    /* residual flush period; multiple of group_size (cache_engine.cpp:13-15) */
    int group_size;             /* 16 (the only device grouping) */
    const int32_t* prefill_capacity; /* host [n_units]: max kept tokens at prefill */
    int max_decode_tokens;      /* decode growth reserved per unit */
    int keep_fp32_params;       /* also keep fp32 (scale, zero) for bit-exact export */
} mkv_cache_config;

/* Allocates the page pool, residual rows and the page plan of calls over all n_units (its
 * device buffers and pinned staging buffer), so the first decode call after a prefill does no
 * allocation; a call over another unit range allocates that range's plan on first use. */
int mkv_cache_create(const mkv_cache_config* cfg, mkv_cache** out);
int mkv_cache_destroy(mkv_cache* cache);
/* Device bytes held: quantized pages, residual ring, metadata. */
int mkv_cache_bytes(const mkv_cache* cache, uint64_t* page_bytes, uint64_t* residual_bytes,
                    uint64_t* total_bytes);
/* Host mirror of one unit's state (exact: updated in call order). */
int mkv_cache_unit_info(const mkv_cache* cache, int unit, int64_t* tokens_quantized,
                        int64_t* tokens_residual, int64_t* n_pages, int64_t* n_blocks);

/* ------------------------------------------------------------------------ */
/* K3  gather + 2-bit quantize + pack of the kept tokens                     */
/* replaces: prefill(k, v, a_cumul, hh, rw, n_r, gs) after selection,        */
/*           i.e. gather_rows + append_block(PerChannel K / PerToken V)      */
/*           cache_engine.cpp:56-77, quantizer.cpp:102-136                   */
/* ------------------------------------------------------------------------ */
typedef struct {
    int unit_begin, n_units;
    const void* k;              /* fp16: unit i token t row at k + i*k_su + t*k_st (elements) */
    int64_t k_su, k_st;
    const void* v;
    int64_t v_su, v_st;
    const int32_t* kept;        /* device int32 [n_units, kept_stride], ascending */
    int64_t kept_stride;
    const int32_t* n_kept_host; /* host int32 [n_units] (= min(hh + rw, L), known without a sync) */
} mkv_cache_prefill_args;
int mkv_cache_prefill(mkv_cache* cache, const mkv_cache_prefill_args* args, void* stream);

/* Select + gather + quantize in one call (prefill, cache_engine.cpp:56-77). */
typedef struct {
    int unit_begin, n_units, length;
    const float* a_cumul;       /* device fp32 [n_units, a_stride] */
    int64_t a_stride;
    const int32_t* hh_count;    /* host [n_units] */
    int rw_count;
    const void* k;
    int64_t k_su, k_st;
    const void* v;
    int64_t v_su, v_st;
} mkv_prefill_select_args;
int mkv_cache_prefill_select(mkv_cache* cache, const mkv_prefill_select_args* args, void* stream);

/* ------------------------------------------------------------------------ */
/* K4  fused unpack-and-multiply 2-bit decode attention                      */
/* replaces: Vector decode_step(cache, t_q, t_k, t_v, scale)                 */
/*           cache_engine.hpp:63-64, cache_engine.cpp:100-138 (GQA-batched)  */
/* Appends (t_k, t_v) to each unit's residual (flushing a full n_r block to  */
/* 2-bit pages first, cache_engine.cpp:79-90), then attends [pages ; residual]*/
/* with one softmax.  k_new == NULL attends without appending.               */
/* ------------------------------------------------------------------------ */
typedef struct {
    int unit_begin, n_units;
    int group;                  /* q-heads per unit (G = Hq / Hkv), 1..8 */
    const void* q;              /* fp16 [n_units, G, d] */
    const void* k_new;          /* fp16 [n_units, d] or NULL */
    const void* v_new;          /* fp16 [n_units, d] or NULL */
    void* out;                  /* fp16 [n_units, G, d] */
    float scale;
} mkv_decode_args;
int mkv_decode_step(mkv_cache* cache, const mkv_decode_args* args, void* stream);
/* decode_append only (cache_engine.cpp:79-90). */
int mkv_cache_append(mkv_cache* cache, int unit_begin, int n_units, const void* k_new,
                     const void* v_new, void* stream);
/* Profiling entry: ONLY the fused page kernel of K4 (pages -> partials -> merge),
 * reusing the residual partials of the previous mkv_decode_step on the same
 * units.  Used by bench.py to time the dominant kernel for its roofline. */
int mkv_decode_pages_only(mkv_cache* cache, const mkv_decode_args* args, void* stream);
/* Diagnostics: per-warp timeline of the latest K4 page kernel (only when the process
 * runs with MKV_DECODE_TRACE set): 4 globaltimer stamps per warp {start, after
 * griddepcontrol.wait, pages done, 0}.  Returns words written. */
int mkv_debug_decode_trace(const mkv_cache* cache, uint64_t* out, int max_words);
/* Diagnostics: how many decode-path kernels (page / finish / residual / merge / append / plan
 * build / steps) this library has launched so far in the process (host-side counter). */
uint64_t mkv_debug_launch_count(void);
/* Multi-layer decode step: n_layers consecutive mkv_decode_step calls in one FFI crossing.
 * Layers that continue each other -- adjacent unit ranges, the same group and scale, and
 * q / out / k_new / v_new back to back as in one [layers][units] array -- are coalesced into ONE
 * pass over all their units (one page kernel + one finish step for the run): bit-identical
 * to one mkv_decode_step over those units, equal to per-layer calls up to the fp32 rounding of
 * a different split-K partition (MKV_LAYERS_SPLIT=1 disables coalescing).  Any other layer
 * list (overlapping ranges included) gives the per-layer calls' results bit for bit.
 * Precondition -- every layer's q / k_new / v_new is already written when the call is made
 * (stream-ordered before it), and none of them aliases an earlier layer's `out`: a layer whose
 * unit range is disjoint from every earlier layer's may start its page pass (reading its q)
 * while the previous layer's finish kernel is still merging (calls of at most one unit per SM;
 * larger calls split their finish step and start each page pass after the previous merges).
 * This is the "all q known" form (a
 * benchmark/driver that has every layer's q up front); a model whose q of layer l+1 depends on
 * layer l's output calls mkv_decode_step once per layer (bench.py reports both). */
int mkv_decode_step_layers(mkv_cache* cache, int n_layers, const mkv_decode_args* args,
                           void* stream);
/* n_steps consecutive decode steps of units [unit_begin, unit_begin + n_units) over a prepared
 * token stream -- the decode loop of the reference's pipeline / CLI chain
 * (minikv_cli.cpp:180-201, pipeline.cpp:199-215: decode_step per step, cache_engine.cpp:100-138)
 * in one FFI crossing.  Step s reads q + s * q_step, k_new + s * kv_step, v_new + s * kv_step
 * and writes out + s * out_step (strides in fp16 ELEMENTS; k_new / v_new may be null: attend
 * only).  Every step's inputs must be written before the call.  Few short units (at most one
 * per SM, <= 1024 pages each by the last step) are served by one launch that keeps each unit on
 * one cluster of CTAs for all the steps: outputs equal n_steps mkv_decode_step calls up to the fp32
 * accumulation order of a different split of the pages, the cache state bit for bit; other
 * calls run the per-step kernels and are bit-identical to mkv_decode_step calls
 * (MKV_STEPS=off forces that path). */
typedef struct {
    int unit_begin, n_units, group, n_steps;
    const void* q;              /* fp16, step s at q + s * q_step: [n_units, G, d] */
    int64_t q_step;
    const void* k_new;          /* fp16, step s at k_new + s * kv_step: [n_units, d] (or null) */
    const void* v_new;
    int64_t kv_step;
    void* out;                  /* fp16, step s at out + s * out_step: [n_units, G, d] */
    int64_t out_step;
    float scale;
} mkv_decode_steps_args;
int mkv_decode_steps(mkv_cache* cache, const mkv_decode_steps_args* args, void* stream);

/* ------------------------------------------------------------------------ */
/* Reference-format export (synchronous): the unit's QuantizedTensor for     */
/* keys (which = 0, PerChannel) or values (which = 1, PerToken) exactly as   */
/* quantizer.hpp:30-42 lays it out (continuous 16-codes-per-word stream,     */
/* per-block grouping, (scale, zero) per group, block_rows), plus the fp16   */
/* residual rows.  Sizes come from mkv_cache_export_sizes.                   */
/* ------------------------------------------------------------------------ */
int mkv_cache_export_sizes(const mkv_cache* cache, int unit, int which, int64_t* n_words,
                           int64_t* n_params, int64_t* n_blocks);
int mkv_cache_export_reference(const mkv_cache* cache, int unit, int which,
                               uint32_t* packed_words, float* params, int64_t* block_rows);
int mkv_cache_export_residual(const mkv_cache* cache, int unit, uint16_t* r_key_fp16,
                              uint16_t* r_value_fp16);
/* Synchronizes and reports device-side input faults (non-finite values met by
 * the quantizer -> MKV_ERR_DOMAIN, like quantize_group, quantizer.cpp:35-37). */
int mkv_cache_check(mkv_cache* cache);

/* ------------------------------------------------------------------------ */
/* MKVC snapshots of one unit (the reference's on-disk cache format).        */
/* replaces: save_cache(const KVCacheLayer&, path) / load_cache(path)        */
/*           snapshot.hpp:11-24, snapshot.cpp:71-198 (little-endian "MKVC" */
/*           v1: d, n_r, group_size, mode, tokens_quantized, K then V        */
/*           QuantizedTensor streams, identity stores, fp32 residuals).      */
/* save: synchronous; byte-identical to the reference's save_cache for the  */
/* same cache when the handle keeps fp32 params (else fp16 params widened). */
/* load: replaces unit `unit` with the snapshot (2-bit mode; d, n_r and     */
/* group_size must match the handle; pages rebuilt in the device layout;    */
/* residual rows rounded to fp16).  Errors as the reference: bad magic /    */
/* version / truncation -> MKV_ERR_RUNTIME.                                 */
/* ------------------------------------------------------------------------ */
int mkv_cache_save_mkvc(const mkv_cache* cache, int unit, const char* path);
int mkv_cache_load_mkvc(mkv_cache* cache, int unit, const char* path);

/* ------------------------------------------------------------------------ */
/* Reference-format fp32 entries: the reference's own fp32 matrices and its   */
/* QuantizedTensor stream, for ANY head dim and group size (refmt.cu).  They  */
/* back the value-type reference signatures of the C++ drop-in; arithmetic    */
/* follows the reference's order (sequential no-FMA dots, quantize_group's    */
/* IEEE division and rounding): scores, codes and params are bit-identical,   */
/* outputs differ from the host only through exp/log ulps.  Device pointers,  */
/* stream-ordered; mkv_quantize_block_f32 synchronizes (it reports non-finite */
/* input as the reference's std::domain_error).                               */
/* ------------------------------------------------------------------------ */
/* replaces: selective_flash_attn(q, k, v, scale, causal, TileConfig) on fp32   */
/*           matrices (attention.hpp:38-39, attention.cpp:29-117): pass 1 (out, */
/*           lse) one CTA per query row, pass 2 (a_cumul, optional) one thread  */
/*           per key column accumulating in row order.  dv <= 512.             */
typedef struct {
    const float* q;     /* [len_q, d], row stride ld_q */
    int64_t ld_q;
    const float* k;     /* [len_k, d] */
    int64_t ld_k;
    const float* v;     /* [len_k, dv] */
    int64_t ld_v;
    float* out;         /* [len_q, dv] */
    int64_t ld_o;
    float* lse;         /* [len_q] natural log */
    float* a_cumul;     /* [len_k] or NULL */
    int len_q, len_k, d, dv;
    float scale;
    int causal;
} mkv_attention_f32_args;
int mkv_attention_f32(const mkv_attention_f32_args* args, void* stream);
/* replaces: decode_attention(q_row, keys, values, scale) (attention.hpp:43-44,            */
/*           attention.cpp:119-143): out[dv], attn[n] (the softmax row).                  */
int mkv_decode_attention_f32(const float* q, const float* keys, int64_t ld_k, const float* values, int64_t ld_v,
                             int n, int d, int dv, float scale, float* out, float* attn, void* stream);
/* replaces: append_block(t, block) / quantize_matrix(m, axis, gs) (quantizer.hpp:61-65,     */
/*           quantizer.cpp:102-151): quantizes the rows x cols block (rows gathered through   */
/*           row_idx when non-NULL: prefill's gather_rows + append_block in one pass), axis 0 */
/*           PerChannel / 1 PerToken, groups of group_size, appended to a stream that already */
/*           holds code_offset codes.  words_out receives the words [code_offset / 16,        */
/*           (code_offset + rows * cols + 15) / 16) -- the first one keeps first_word's low    */
/*           codes when code_offset % 16 != 0 -- and params_out the block's (scale, zero)     */
/*           pairs in group order.  Synchronous.                                              */
int mkv_quantize_block_f32(const float* src, int64_t ld, const int32_t* row_idx, int rows, int cols,
                           int group_size, int axis, int64_t code_offset, uint32_t first_word,
                           uint32_t* words_out, float* params_out, void* stream);
/* replaces: dequantize_matrix(t) (quantizer.hpp:67-68, quantizer.cpp:153-195): words / params */
/*           (device) of a stream whose blocks have block_rows (host [n_blocks]) rows of cols    */
/*           channels -> out [sum(block_rows), cols] (row stride ld_out).  The caller checks the */
/*           group count (std::runtime_error) as the reference does.                             */
int mkv_dequantize_f32(const uint32_t* words, const float* params, const int64_t* block_rows, int n_blocks,
                       int cols, int group_size, int axis, float* out, int64_t ld_out, void* stream);

/* ------------------------------------------------------------------------ */
/* Synthetic inputs (benchmarks/tests): the integer-exact approximate-N(0,1) */
/* fp16 generator of oracle/minikv_oracle.h, bit-identical on device.        */
/* ------------------------------------------------------------------------ */
int mkv_synth_fp16(void* out, int64_t n, uint64_t seed, uint64_t stream_id, void* stream);
/* Rows: out row r (of n_rows, row_len elements, row stride ld) uses stream
 * stream_base + r * stream_step. */
int mkv_synth_fp16_rows(void* out, int64_t n_rows, int64_t row_len, int64_t ld, uint64_t seed,
                        uint64_t stream_base, uint64_t stream_step, void* stream);
int mkv_synth_uniform_f32(float* out, int64_t n_rows, int64_t row_len, int64_t ld, uint64_t seed,
                          uint64_t stream_base, uint64_t stream_step, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MINIKV_B200_H */
