// mkv_kernels.h -- host-side launch interface between the C ABI (capi.cu) and
// the kernel translation units.  Internal; not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mkv_common.cuh"

namespace mkv {

constexpr int kMaxG = 8;  // q-heads per kv-head handled by one mma N=8 tile

// ---- K3: prefill pages (quant_pack.cu) ----
struct PrefillPagesParams {
    const __half* k;
    int64_t k_su, k_st;
    const __half* v;
    int64_t v_su, v_st;
    const int32_t* kept;
    int64_t kept_stride;
    UnitMeta* meta;     // global unit meta array
    int unit_begin, n_units, max_pages;
    uint8_t* pool;
    float* shadow;      // may be null
    uint32_t* status;
};
cudaError_t launch_prefill_pages(const PrefillPagesParams& p, cudaStream_t s);

// ---- K2: selection (select.cu) ----
struct SelectParams {
    const float* a;
    int64_t a_stride;
    int n_units, length;
    const int32_t* hh;  // device [n_units], or null: every unit keeps hh_uniform
    int hh_uniform;
    int rw;
    int32_t* kept;
    int64_t kept_stride;
    int32_t* n_kept;    // may be null
};
cudaError_t launch_select(const SelectParams& p, cudaStream_t s);
// layer_score_variance (selection.cpp:130-146) of n rows, fp64 two-pass, deterministic
cudaError_t launch_score_variance(const float* a, int64_t a_stride, int n, int length, float* out, cudaStream_t s);

// ---- K4: decode (decode.cu) ----
// Balanced worker ranges: the plan's padded page sequence is T = total_pages / batch whole
// batches; worker w of W owns batches [range_begin(w), range_begin(w + 1)) -- range sizes
// differ by at most one batch, so every SM gets the same share of pages (a fixed chunk rounded
// up to whole batches left up to 1/16 of the SMs' capacity idle).
__host__ __device__ inline int range_begin(int w, int T, int W) { return (int)(((int64_t)w * T) / W); }
// the worker whose range holds batch b (the largest w with range_begin(w) <= b)
__host__ __device__ inline int worker_of_batch(int b, int T, int W) { return (int)((((int64_t)b + 1) * W - 1) / T); }
struct WorkerRanges {
    int workers;        // W
    int total_batches;  // T
    int batch;          // pages per batch
};
struct ResidualParams {
    UnitMeta* meta;
    int unit_begin, n_units, group, n_r;
    const __half* q;      // [n_units][G][d]
    const __half* k_new;  // [n_units][d] or null (no append)
    const __half* v_new;
    __half* res_k;        // [total_units][n_r][d]
    __half* res_v;
    uint8_t* pool;
    float* shadow;
    const float* part_ml; // page partials (pages_kernel), merged by finish_kernel
    const float* part_o;
    __half* out;          // [n_units][G][d]
    float scale_log2;
    uint32_t* status;
    uint64_t* trace;      // diagnostics: per CTA {start, residual done, wait released, end}, or null
    int fused_flush;      // finish_kernel quantizes a residual block this append fills (no append_kernel)
    // split finish (launch_resid_merge): per-unit arrival counters (page segments + the residual
    // partial) and the residual partial of every unit, indexed by the global unit
    int* unit_cnt;
    float* res_ml;        // [total_units][2][kMaxG]
    float* res_o;         // [total_units][kMaxG][d]
};
constexpr int kTraceFinishCtas = 8192;  // finish-kernel CTAs recorded per trace slot
cudaError_t launch_append(const ResidualParams& p, cudaStream_t s);
// every layer of one multi-layer decode call appended (and flushed) by one launch
constexpr int kMaxAppendSegs = 32;
struct AppendSegs {
    int n_seg;
    int block_begin[kMaxAppendSegs + 1];
    int unit_begin[kMaxAppendSegs];
    const __half* k_new[kMaxAppendSegs];
    const __half* v_new[kMaxAppendSegs];
};
cudaError_t launch_append_segments(const ResidualParams& p, const AppendSegs& segs, cudaStream_t s);
cudaError_t launch_finish(const ResidualParams& p, const int32_t* pref, WorkerRanges wr, bool after_pages,
                          cudaStream_t s);
// The split form of launch_finish: a persistent residual kernel (resid_ctas CTAs, one beside each
// page CTA: append + residual attention of every unit during the page pass, the residual partial
// to global memory) and a merge kernel (one CTA per unit: waits on the unit's arrival counter,
// merges, writes out), so the merges do not queue behind residual attention after the page pass.
cudaError_t launch_resid_merge(const ResidualParams& p, const int32_t* pref, WorkerRanges wr, bool after_pages,
                               int resid_ctas, cudaStream_t s);

// Per-unit page-run record of a K4 plan (host-computed from the cache mirror).
struct UnitRec {
    int64_t base;       // pool page index of the unit's page 0 minus pbeg
    int32_t pbeg, pend; // the unit's [begin, end) in the plan's padded page sequence
    int32_t rend;       // pbeg + real pages
    int32_t n_prefill;  // tokens of the prefill block (its last page may be partial)
    int32_t pad[2];
};
// device-side plan construction (flush steps of a multi-layer call)
struct PlanBuildJob {
    int unit_begin, n, warps, batch;
    int32_t* pref;    // [n + 1]
    int32_t* wstart;  // [warps]
    UnitRec* rec;     // [n]
};
constexpr int kMaxPlanJobs = 32;
struct PlanBuildJobs {
    int n_jobs;
    PlanBuildJob job[kMaxPlanJobs];
};
cudaError_t launch_plan_build(const UnitMeta* meta, const PlanBuildJobs& jobs, cudaStream_t s);

struct PagesParams {
    const uint8_t* pool;
    const UnitMeta* meta;
    int unit_begin, n_units, group;
    const __half* q;
    const int32_t* pref;    // [n_units + 1] local page prefix
    const int32_t* wstart;  // [n_warps] first (non-empty) unit of each warp's page range
    const UnitRec* rec;     // [n_units]
    int total_pages, n_warps;  // padded pages of the plan; W = workers with a (balanced) range
    float* part_ml;         // [slots][2][kMaxG]   slot = warp + unit
    float* part_o;          // [slots][kMaxG][d]
    float scale_log2;
    uint64_t* trace;        // diagnostics: per warp {start, after wait, done} (globaltimer), or null
    int early;              // q may be read before griddepcontrol.wait (see pages_kernel)
    int* unit_cnt;          // split finish: +1 per (warp, unit) segment whose partial is written, or null
};
constexpr int kMaxPagesWarps = 12;  // partial-slot sizing
// pages_tc_kernel trace (MKV_DECODE_TRACE): per worker, batches 4..7: 8 stamps of compute warp 0,
// 8 of compute warp 1, 4 of the control warp
constexpr int kTcTraceWords = 80;
struct PagesConfig {
    int warps, stages;  // workers (page-range owners) per CTA, ring stages
    int batch;          // pages per batch: units are padded to whole batches in the plan
    int tc;             // 1: pages_tc_kernel (tcgen05), 0: pages_kernel (mma.sync)
};
PagesConfig pages_config();
// pdl = false: a full stream dependency (the previous kernel wrote the plan this kernel reads
// before its griddepcontrol.wait, e.g. plan_build_kernel on a fused flush step)
cudaError_t launch_pages(const PagesParams& p, int grid, cudaStream_t s, bool pdl = true);
// A prepared token stream's decode steps, one CTA per unit for all steps (few short units:
// mkv_decode_steps picks it when every unit's pages fit one CTA's share; see steps_kernel).
struct StepsParams {
    UnitMeta* meta;
    int unit_begin, n_units, group, n_r, n_steps;
    const __half* q;          // step st, unit i, head h: q + st * q_step + (i * G + h) * d
    int64_t q_step;
    const __half* k_new;      // step st, unit i: k_new + st * kv_step + i * d (null: attend only)
    const __half* v_new;
    int64_t kv_step;
    __half* out;              // like q
    int64_t out_step;
    __half* res_k;
    __half* res_v;
    uint8_t* pool;
    float* shadow;
    float scale_log2;
    uint32_t* status;
};
cudaError_t launch_steps(const StepsParams& p, cudaStream_t s);
// host-side count of decode-path kernel launches (diagnostics: mkv_debug_launch_count)
void count_launch(int n);
uint64_t launch_count();
cudaError_t launch_pages_tc(const PagesParams& p, int grid, cudaStream_t s, bool pdl);

// ---- H2O baseline (h2o.cu) ----
struct H2OParams {
    const float* prompt_k;
    int64_t ld_k;
    const float* prompt_scores;
    const float* qs;
    const float* ks;
    int l_prompt, d, steps, hh_budget, rw_budget;
    float scale;
    int32_t* kept;
    int64_t kept_stride;
    int32_t* kept_count;
    int* ws_pos;       // [l_prompt + steps]
    double* ws_score;  // [l_prompt + steps]
    float* ws_attn;    // [l_prompt + steps]
};
cudaError_t launch_h2o(const H2OParams& p, cudaStream_t s);

// ---- utilities (synth.cu) ----
cudaError_t launch_synth_fp16(__half* out, int64_t n_rows, int64_t row_len, int64_t ld,
                              uint64_t seed, uint64_t stream_base, uint64_t stream_step,
                              cudaStream_t s);
cudaError_t launch_synth_uniform(float* out, int64_t n_rows, int64_t row_len, int64_t ld,
                                 uint64_t seed, uint64_t stream_base, uint64_t stream_step,
                                 cudaStream_t s);

// ---- K1: prefill attention (prefill.cu) ----
struct PrefillAttnParams {
    const __half* q;
    int64_t q_sb, q_sh, q_st;
    const __half* k;
    int64_t k_sb, k_sh, k_st;
    const __half* v;
    int64_t v_sb, v_sh, v_st;
    __half* out;
    int64_t o_sb, o_sh, o_st;
    float* lse;
    float* a_cumul;
    int batch, hq, hkv, lq, lk;
    float scale;
    int causal;
};
cudaError_t launch_prefill_attn(const PrefillAttnParams& p, cudaStream_t s);

// ---- reference-format fp32 kernels (refmt.cu): the value-type reference signatures ----
struct AttnF32Params {
    const float* q;
    const float* k;
    const float* v;
    int64_t ld_q, ld_k, ld_v, ld_o;
    float* out;      // [lq][dv]
    float* lse;      // [lq]
    float* a_cumul;  // [lk] or null (pass 1 only)
    int lq, lk, d, dv;
    float scale;
    int causal;
};
cudaError_t launch_attn_f32(const AttnF32Params& p, cudaStream_t s);
int attn_f32_max_dv();
struct DecodeF32Params {
    const float* q;       // [d]
    const float* keys;    // [n][ld_k]
    const float* values;  // [n][ld_v]
    int64_t ld_k, ld_v;
    int n, d, dv;
    float scale;
    float* out;           // [dv]
    float* attn;          // [n]
};
cudaError_t launch_decode_attn_f32(const DecodeF32Params& p, cudaStream_t s);
struct QuantBlockParams {
    const float* src;       // block rows (optionally gathered through row_idx) x cols, row stride ld
    int64_t ld;
    const int32_t* row_idx; // null: rows 0 .. rows - 1
    int rows, cols, gs;
    int axis;               // 0 = PerChannel, 1 = PerToken
    uint8_t* codes;         // [rows * cols] in the block's stream order
    float* params;          // [n_groups][2] (scale, zero)
    uint32_t* status;       // |= 1: non-finite input
};
cudaError_t launch_quantize_block(const QuantBlockParams& p, cudaStream_t s);
cudaError_t launch_pack_codes(const uint8_t* codes, int64_t n, int64_t code_off, uint32_t init, uint32_t* words,
                              uint32_t* status, cudaStream_t s);
struct DequantBlock {
    int64_t code_off, group_off, row0;
    int rows;
    int pad;
};
struct DequantParams {
    const uint32_t* words;
    const float* params;
    const DequantBlock* blk;
    int n_blocks;
    int64_t total_codes;
    int cols, gs, axis;
    float* out;
    int64_t ld_out;
};
cudaError_t launch_dequantize(const DequantParams& p, cudaStream_t s);

}  // namespace mkv
