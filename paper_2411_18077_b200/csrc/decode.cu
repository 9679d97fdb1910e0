// decode.cu -- K4: fused unpack-and-multiply 2-bit decode attention.
//
// Restates decode_step (cache_engine.cpp:100-138) for a batch of units with
// GQA: append the new token (flushing a full n_r residual block to 2-bit pages
// first, cache_engine.cpp:79-90), then ONE softmax over
// [dequant(K_q) ; R_K] and out = attn . [dequant(V_q) ; R_V].
//
// Kernels (per call = one layer's units):
//   append_kernel  (only on steps where some unit's residual fills up)
//                  decode_append + flush of the n_r block through the K3 page
//                  builder, so the new pages are visible to pages_kernel.
//   pages_kernel   persistent, 8 warps/CTA, each warp an independent worker
//                  over a contiguous range of the global page sequence; pages
//                  stream HBM -> smem with cp.async.bulk (2-stage ring of
//                  4-page batches per warp), are dequantized in registers and
//                  multiplied on the tensor cores (mma.sync m16n8k16), four
//                  pages interleaved for ILP -> one partial (m, l, o) per
//                  (warp, unit) segment.
//   finish_kernel  one CTA per unit: decode_append (non-flush steps), exact
//                  attention over the fp16 residual (mma, one warp per 16-token
//                  tile), and the split-K merge of every partial into out.  With
//                  more units than SMs: finish_kernel<true> (persistent, residual
//                  work beside the page pass) + merge_kernel (per-unit arrival
//                  counters).
//   steps_kernel   mkv_decode_steps for few short units: a cluster of CTAs per
//                  unit runs every step (append, flush, pages, residual, merge).
//
// Dequantization never materialises fp16 K/V: each 2-bit code becomes an fp16
// *subnormal* code * 4^s * 2^-24 with one LOP3 (s = position for the first five codes of a
// word, after one 10-bit shift for the last three), the 4^-s and the per-channel key scale are folded into the query
// fragment, the per-token value scale into the probability fragment, and the
// zero points enter through one extra mma per page (keys: sum_c q_c z_c over a
// 4-page batch; values: sum_t p_t z_t).  See DESIGN.md.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <atomic>

#include "mkv_kernels.h"
#include "mkv_page.cuh"

namespace mkv {

// Host-side count of this library's decode-path kernel launches (mkv_debug_launch_count: bench.py
// reports the launches of its timed region from it).
static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

namespace {

constexpr int kBatch = 4;  // pages per bulk copy / per K-bias mma / per softmax update
constexpr float kTwo24 = 16777216.0f;
constexpr float kLazy = 3.0f;  // log2 units: P <= 8 keeps fp16 P and P*s far from overflow
constexpr int kQBytes = kMaxG * kHeadDim * 2;  // per-warp q staging
constexpr int kRecSlots = 8;  // unit records staged per warp (the units its page range touches)
template <int kStages>
__host__ __device__ constexpr int warp_smem() {
    return kStages * kBatch * kPageBytes + kQBytes + kRecSlots * (int)sizeof(UnitRec);
}

__device__ __forceinline__ uint4 lds128(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ uint2 lds64(const uint8_t* p) { return *reinterpret_cast<const uint2*>(p); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Code position k (0..7) of a word: k < 5 is read in place (bits 2k, 16+2k lie in the fp16
// mantissa: value code * 4^k * 2^-24); k >= 5 after one shift by 10 (value code * 4^(k-5) * 2^-24).
__host__ __device__ constexpr int code_class(int k) { return k < 5 ? k : k - 5; }
__host__ __device__ constexpr int code_shift(int k) { return k < 5 ? 0 : 10; }
__host__ __device__ constexpr float pow4_neg(int s) {  // 4^-s, exact
    return s == 0 ? 1.0f : (s == 1 ? 0.25f : (s == 2 ? 0.0625f : (s == 3 ? 0.015625f : 0.00390625f)));
}
__device__ __forceinline__ float extract_scale(int k) { return kTwo24 * pow4_neg(code_class(k)); }

// q of local unit i, head gid (zero for gid >= G), staged in smem, -> B fragments
__device__ __forceinline__ void load_q_frags(const __half* qs_smem, int G, int gid, int tig, uint32_t (&qb)[8][2],
                                             uint32_t (&qsc)[8][2]) {
#pragma unroll
    for (int kc = 0; kc < 8; ++kc) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            uint32_t v = 0;
            if (gid < G) v = *reinterpret_cast<const uint32_t*>(qs_smem + gid * kHeadDim + 16 * kc + 2 * tig + 8 * p);
            qb[kc][p] = v;
            const float f = pow4_neg(code_class(kc));
            qsc[kc][p] = hmul2_u32(v, pack_half2(f, f));
        }
    }
}

// launch with programmatic dependent launch (PDL): the kernel may start while the
// previous kernel on the stream drains; it must execute griddepcontrol.wait before
// touching that kernel's outputs.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    count_launch(1);
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// The page kernel (146 KB) and a finish CTA (33 KB) share an SM only under the largest
// shared-memory carveout; left to the driver, an SM may be configured for the page CTA alone,
// and a finish CTA placed there waits for the page CTA to exit (its residual attention then
// lands on the layer's critical path).  MKV_CARVEOUT=<percent> (-1: driver default) for A/B.
static cudaError_t set_carveout(const void* fn) {
    static const int pct = [] {
        const char* e = getenv("MKV_CARVEOUT");
        return e ? atoi(e) : 100;
    }();
    if (pct < 0) return cudaSuccess;
    return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

}  // namespace

// ---------------------------------------------------------------------------
// pages kernel
// ---------------------------------------------------------------------------
// kCount: the split finish's per-segment arrival count (P.unit_cnt) is compiled in only where it
// is used -- even unused, its epilogue code cost the pass ~1% (584 vs 578 us per headline launch).
template <int kWarps, int kStages, bool kCount>
// <= 208 registers (x 256 threads = 53248): leaves 12288 registers of the SM's 65536 for one
// co-resident finish CTA (4 warps x 96).
__global__ void __maxnreg__(208) pages_kernel(const PagesParams P) {
    constexpr int kWarpSmem = warp_smem<kStages>();
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int gid = lane >> 2, tig = lane & 3;
    uint8_t* wsm = smem + (size_t)warp * kWarpSmem;
    uint8_t* ring = wsm;
    __half* qsm = reinterpret_cast<__half*>(wsm + kStages * kBatch * kPageBytes);
    UnitRec* srec = reinterpret_cast<UnitRec*>(wsm + kStages * kBatch * kPageBytes + kQBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kWarps * kWarpSmem) + warp * kStages;

    const int wg = blockIdx.x * kWarps + warp;
    auto stamp = [&](int k) {
        if (P.trace != nullptr && lane == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            P.trace[(size_t)wg * 4 + k] = t;
        }
    };
    stamp(0);
    const int T = P.total_pages / kBatch;
    if (wg >= P.n_warps) return;
    const int start = kBatch * range_begin(wg, T, P.n_warps);
    const int end = kBatch * range_begin(wg + 1, T, P.n_warps);
    if (start >= end) return;
    const int G = P.group;
    const int qchunks = G * kHeadDim * 2 / 16;

    int ci = 0;
    auto prefetch_q = [&](int unit) {
        const uint8_t* src = reinterpret_cast<const uint8_t*>(P.q + (size_t)unit * G * kHeadDim);
        for (int e = lane; e < qchunks; e += 32) cp_async16(reinterpret_cast<uint8_t*>(qsm) + 16 * e, src + 16 * e);
        cp_async_commit();
    };

    // zero the ring once: slots past a short batch then hold finite stale data, so the
    // batch body runs branch-free (invalid pages are masked with selects, not branches)
    for (int e = lane; e < kStages * kBatch * kPageBytes / 16; e += 32)
        reinterpret_cast<uint4*>(ring)[e] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    ci = __ldg(P.wstart + wg);  // first unit of this warp's range (host plan)
    // Stage the records of the first kRecSlots units of the range in shared memory (one
    // round trip at start instead of dependent global loads at every unit boundary).
    const int ci0 = ci;
    for (int e = lane; e < kRecSlots * 2; e += 32)
        if (ci0 + (e >> 1) < P.n_units)
            cp_async16(reinterpret_cast<uint8_t*>(srec) + 16 * e, reinterpret_cast<const uint8_t*>(P.rec + ci0) + 16 * e);
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
    auto rec_pend = [&](int i) { return i - ci0 < kRecSlots ? srec[i - ci0].pend : __ldg(&P.rec[i].pend); };
    auto rec_pbeg = [&](int i) { return i - ci0 < kRecSlots ? srec[i - ci0].pbeg : __ldg(&P.rec[i].pbeg); };
    auto rec_rend = [&](int i) { return i - ci0 < kRecSlots ? srec[i - ci0].rend : __ldg(&P.rec[i].rend); };
    auto rec_base = [&](int i) { return i - ci0 < kRecSlots ? srec[i - ci0].base : __ldg(&P.rec[i].base); };
    auto rec_npre = [&](int i) { return i - ci0 < kRecSlots ? srec[i - ci0].n_prefill : __ldg(&P.rec[i].n_prefill); };
    // ---- producer cursor (warp-uniform) ----
    int pi = ci;
    int pg = start;
    int p_uend = rec_pend(pi);  // units start at multiples of kBatch (padded prefix)
    int p_rend = rec_rend(pi);  // end of its real pages
    // pool address of "global page 0" of unit pi (its first page minus its prefix)
    const uint8_t* p_base = P.pool + rec_base(pi) * kPageBytes;
    auto issue = [&](int stage) {
        if (pg >= end) return;
        const int n = min(kBatch, p_rend - pg);  // batches never straddle units or warp ranges
#ifdef MKV_AB_COMPUTE_ONLY  // A/B probe: after the first ring fill, batches reuse stale smem
        if (pg >= start + kStages * kBatch) {
            if (lane == 0) mbar_expect_tx(&bars[stage], 0);
        } else
#endif
        if (lane == 0) {
            mbar_expect_tx(&bars[stage], n * kPageBytes);
            bulk_g2s(ring + (size_t)stage * kBatch * kPageBytes, p_base + (size_t)pg * kPageBytes, n * kPageBytes,
                     &bars[stage]);
        }
        pg += kBatch;
        if (pg == p_uend && pg < end) {
            while (pg == p_uend) {  // next unit that has pages
                ++pi;
                p_uend = rec_pend(pi);
            }
            p_base = P.pool + rec_base(pi) * kPageBytes;
            p_rend = rec_rend(pi);
        }
    };
    // The first kStages batches are requested before griddepcontrol.wait: under PDL they
    // overlap the previous kernel's tail.  Safe because no kernel that may still be running
    // writes these pages or the plan read above (the append kernel of a flush step is a
    // full-dependency launch, and a page kernel whose plan was just written by
    // plan_build_kernel is launched without PDL -- capi.cu decode_impl `after_plan_build`);
    // q is read and partials are written after the wait.
    for (int s = 0; s < kStages; ++s) issue(s);
    // P.early (every layer of a multi-layer call but the first): q is an input of the call and
    // the partial buffers belong to this layer's plan, so the whole page pass may run while the
    // previous layer's finish kernel is still merging; the wait moves to the kernel's end (it
    // orders this grid's completion after that kernel's, which keeps the launch chain from
    // running ahead and makes the next call's first kernel wait for every merge).  Otherwise
    // wait here, before touching q.
    if (!P.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    stamp(1);
    prefetch_q(ci);

    int cg = start;
    int n_segments = 0;  // diagnostics (trace word 3)
    int stage = 0;
    uint32_t phase = 0;
    const float sl2 = P.scale_log2;
    const float sk = kTwo24 * sl2;

    while (cg < end) {
        ++n_segments;
        const int unit = ci;
        const int upre = rec_pbeg(unit);
        const int uend_g = rec_pend(unit);
        const int seg_end = min(uend_g, end);
        const int n_prefill = rec_npre(unit);
        const int partial_page = (n_prefill & 15) ? ((n_prefill + 15) >> 4) - 1 : -1;
        const int partial_valid = n_prefill & 15;

        uint32_t qb[8][2], qsc[8][2];
        cp_async_wait_all();
        __syncwarp();
        load_q_frags(qsm, G, gid, tig, qb, qsc);
        __syncwarp();
        {  // K-bias query copy carries the softmax scale: Kb comes out in log2 units
            const uint32_t s2 = pack_half2(P.scale_log2, P.scale_log2);
#pragma unroll
            for (int kc = 0; kc < 8; ++kc) {
                qb[kc][0] = hmul2_u32(qb[kc][0], s2);
                qb[kc][1] = hmul2_u32(qb[kc][1], s2);
            }
        }
        uint32_t qa[8][4];  // K-bias A operand: rows = heads (gid), k = channels, rows 8-15 zero
#pragma unroll
        for (int kc = 0; kc < 8; ++kc) {
            qa[kc][0] = qb[kc][0]; qa[kc][1] = 0u; qa[kc][2] = qb[kc][1]; qa[kc][3] = 0u;
        }
        if (seg_end < end) {
            int nu = unit + 1;
            while (rec_pend(nu) == seg_end) ++nu;
            prefetch_q(nu);
        }

        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
        float O[8][4];
#pragma unroll
        for (int g = 0; g < 8; ++g) O[g][0] = O[g][1] = O[g][2] = O[g][3] = 0.0f;
        float Dvb[4] = {0.0f, 0.0f, 0.0f, 0.0f};

        const int uend_real = rec_rend(unit);
        while (cg < seg_end) {
            const int n = min(kBatch, uend_real - cg);
            const int pfirst = cg - upre;
            mbar_wait(&bars[stage], phase);
#ifdef MKV_AB_STREAM_ONLY  // A/B probe (tools/abbuild.sh): data movement only, no compute
            __syncwarp();
            issue(stage);
            cg += kBatch;
            if (++stage == kStages) { stage = 0; phase ^= 1u; }
            continue;
#endif
            const uint8_t* buf = ring + (size_t)stage * kBatch * kPageBytes;

            // ---- scores for the 4 pages, interleaved: S[j][t][h] = sum_c code * q'' ----
            float S[kBatch][4];
            uint4 kw[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                kw[j] = lds128(buf + j * kPageBytes + kKC + lane * 16);
                S[j][0] = S[j][1] = S[j][2] = S[j][3] = 0.0f;
            }
#pragma unroll
            for (int kc = 0; kc < 8; ++kc) {
                const int sh = code_shift(kc);
                const uint32_t mask = 0x00030003u << (2 * code_class(kc));
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    const uint2 ks = lds64(buf + j * kPageBytes + kKS + ((kc >> 1) * 4 + tig) * 16 + (kc & 1) * 8);
                    const uint32_t a[4] = {(kw[j].x >> sh) & mask, (kw[j].y >> sh) & mask,
                                           (kw[j].z >> sh) & mask, (kw[j].w >> sh) & mask};
                    mma_16816(S[j], a, hmul2_u32(qsc[kc][0], ks.x), hmul2_u32(qsc[kc][1], ks.y));
                }
            }
            // ---- key zero-point bias Kb^T[h][page] = sum_c q[h][c] z[page][c]: A = the unit's q
            // fragments (built once per unit), B = z pairs straight from LDS (no fragment
            // assembly per batch); columns are pages gid & 3.  Issued after the scores: their
            // four independent chains start the tensor pipe sooner (measured ~0.4%). ----
            float Kb[4] = {0.0f, 0.0f, 0.0f, 0.0f}, Kb2[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            {
                uint4 z[4];
                const uint8_t* zp = buf + (gid & (kBatch - 1)) * kPageBytes + kKZ + tig * 16;
#pragma unroll
                for (int j = 0; j < 4; ++j) z[j] = lds128(zp + 64 * j);  // columns >= kBatch: unused
                const uint32_t* zz = reinterpret_cast<const uint32_t*>(z);
#pragma unroll
                for (int kc = 0; kc < 8; kc += 2) {
                    mma_16816(Kb, qa[kc], zz[2 * kc], zz[2 * kc + 1]);
                    mma_16816(Kb2, qa[kc + 1], zz[2 * kc + 2], zz[2 * kc + 3]);
                }
                Kb[0] += Kb2[0];
                Kb[1] += Kb2[1];
            }

            // ---- online softmax over the batch (log2 domain) ----
            const bool special = (n < kBatch) || (partial_page >= pfirst && partial_page < pfirst + n);
            float x[kBatch][4];
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                // Kb^T[h][page = 2 t + e] sits in Kb[e] of lane 4 h + t
                const float kb0 = __shfl_sync(0xffffffffu, Kb[j & 1], 8 * tig + (j >> 1));
                const float kb1 = __shfl_sync(0xffffffffu, Kb[j & 1], 8 * tig + 4 + (j >> 1));
                x[j][0] = fmaf(S[j][0], sk, kb0);
                x[j][1] = fmaf(S[j][1], sk, kb1);
                x[j][2] = fmaf(S[j][2], sk, kb0);
                x[j][3] = fmaf(S[j][3], sk, kb1);
            }
            if (special) {  // one branch per batch: short batch or the prefill block's partial page
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    const int lp = pfirst + j;
                    const int valid = (j >= n) ? 0 : ((lp == partial_page) ? partial_valid : 16);
                    if (gid >= valid) { x[j][0] = -INFINITY; x[j][1] = -INFINITY; }
                    if (gid + 8 >= valid) { x[j][2] = -INFINITY; x[j][3] = -INFINITY; }
                }
            }
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                mx0 = fmaxf(mx0, fmaxf(x[j][0], x[j][2]));
                mx1 = fmaxf(mx1, fmaxf(x[j][1], x[j][3]));
            }
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
            }
            // lazy rescale: keep the running max unless it grows by > kLazy (then P <= 2^kLazy)
            const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
            if (__any_sync(0xffffffffu, (mn0 > m0 + kLazy) | (mn1 > m1 + kLazy))) {
                const float a0 = fast_exp2(m0 - mn0), a1 = fast_exp2(m1 - mn1);
                l0 *= a0; l1 *= a1;
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    O[g][0] *= a0; O[g][1] *= a1; O[g][2] *= a0; O[g][3] *= a1;
                }
                Dvb[0] *= a0; Dvb[1] *= a1;
                m0 = mn0; m1 = mn1;
            }
            uint32_t pb0[kBatch], pb1[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const float p0 = fast_exp2(x[j][0] - m0), p1 = fast_exp2(x[j][1] - m1);
                const float p2 = fast_exp2(x[j][2] - m0), p3 = fast_exp2(x[j][3] - m1);
                l0 += p0 + p2;
                l1 += p1 + p3;
                pb0[j] = movmatrix_trans(pack_half2(p0, p1));
                pb1[j] = movmatrix_trans(pack_half2(p2, p3));
            }
            // ---- values: Dvb[g][h] += sum_t z[t][g] p[h][t];  O_g[c][h] += sum_t code * p * s ----
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const uint8_t* page = buf + j * kPageBytes;
                const uint2 vz = lds64(page + kVZ + lane * 8);
                const uint32_t az[4] = {vz.x, 0u, vz.y, 0u};
                mma_16816(Dvb, az, pb0[j], pb1[j]);
                const uint4 vw = lds128(page + kVC + lane * 16);
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const int sh = code_shift(g);
                    const uint32_t mask = 0x00030003u << (2 * code_class(g));
                    const uint2 vs = lds64(page + kVS + ((g >> 1) * 4 + tig) * 16 + (g & 1) * 8);
                    const uint32_t a[4] = {(vw.x >> sh) & mask, (vw.y >> sh) & mask, (vw.z >> sh) & mask,
                                           (vw.w >> sh) & mask};
                    mma_16816(O[g], a, hmul2_u32(pb0[j], vs.x), hmul2_u32(pb1[j], vs.y));
                }
            }
            __syncwarp();
            issue(stage);  // refill this stage with the batch kStages ahead
            cg += kBatch;
            if (++stage == kStages) { stage = 0; phase ^= 1u; }
        }
        if (cg == uend_g) {
            ++ci;
            while (cg < end && rec_pend(ci) == cg) ++ci;
        }

        // ---- segment epilogue: partial (m, l, o) for slot (warp wg, unit) ----
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, o);
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        }
        const int slot = wg + unit;
        float* pml = P.part_ml + (size_t)slot * 2 * kMaxG;
        float* po = P.part_o + (size_t)slot * kMaxG * kHeadDim;
        const int h0 = 2 * tig, h1 = 2 * tig + 1;
        if (gid == 0) {
            if (h0 < G) { pml[h0] = m0; pml[kMaxG + h0] = l0; }
            if (h1 < G) { pml[h1] = m1; pml[kMaxG + h1] = l1; }
        }
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const float dv0 = __shfl_sync(0xffffffffu, Dvb[0], 4 * g + tig);
            const float dv1 = __shfl_sync(0xffffffffu, Dvb[1], 4 * g + tig);
            const float f = extract_scale(g);
            const int c = 16 * g + gid;
            if (h0 < G) {
                po[h0 * kHeadDim + c] = fmaf(O[g][0], f, dv0);
                po[h0 * kHeadDim + c + 8] = fmaf(O[g][2], f, dv0);
            }
            if (h1 < G) {
                po[h1 * kHeadDim + c] = fmaf(O[g][1], f, dv1);
                po[h1 * kHeadDim + c + 8] = fmaf(O[g][3], f, dv1);
            }
        }
        // (the runtime test is kept in the counting variant: as `if constexpr` alone the pass
        // compiled ~1% slower -- code layout, measured)
        if (kCount && P.unit_cnt != nullptr) {  // split finish: count this segment's partial
            // bar.warp.sync orders every lane's partial stores before lane 0's release add
            // (release is cumulative); merge_kernel acquires the counter before reading them
            __syncwarp();
            if (lane == 0)
                asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(P.unit_cnt + P.unit_begin + unit) : "memory");
        }
    }
    stamp(2);
    if (P.trace != nullptr && lane == 0) P.trace[(size_t)wg * 4 + 3] = (uint64_t)n_segments;
    if (P.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

template <int W, int S, bool C>
static cudaError_t launch_pages_c(const PagesParams& p, int grid, cudaStream_t s, bool pdl) {
    const size_t smem = (size_t)W * warp_smem<S>() + (size_t)W * S * sizeof(uint64_t);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(pages_kernel<W, S, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) e = set_carveout(reinterpret_cast<const void*>(pages_kernel<W, S, C>));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    if (!pdl) {
        count_launch(1);
        pages_kernel<W, S, C><<<grid, W * 32, smem, s>>>(p);
        return cudaGetLastError();
    }
    return launch_pdl(pages_kernel<W, S, C>, dim3(grid), dim3(W * 32), smem, s, p);
}
template <int W, int S>
static cudaError_t launch_pages_t(const PagesParams& p, int grid, cudaStream_t s, bool pdl) {
    return p.unit_cnt != nullptr ? launch_pages_c<W, S, true>(p, grid, s, pdl) : launch_pages_c<W, S, false>(p, grid, s, pdl);
}

// The page pass: the mma.sync pages_kernel above (8 warps x 2 stages, 4-page batches;
// MKV_PAGES_CFG=8x3 for 3 stages) by default.  MKV_PAGES_IMPL=tc selects pages_tc_kernel
// (decode_tc.cu: tcgen05 + TMEM, 2 workers per CTA, 8-page batches) -- parity-green, but measured
// 2.4x slower on the bench shapes, so it stays an A/B
// variant.
PagesConfig pages_config() {
    static PagesConfig cfg = [] {
        // 8 warps: a 12-warp CTA ran the page pass ~2% faster (same SM sub-partition
        // throughput) but needs the whole register file, so no finish CTA could share its SM
        PagesConfig c{8, 2, 4, 0};
        if (const char* e = getenv("MKV_PAGES_CFG")) {
            int w = 0, st = 0;
            if (sscanf(e, "%dx%d", &w, &st) == 2 && (w == 8 || w == 4) && (st == 2 || st == 3)) {
                c.warps = w;
                c.stages = st;
            }
        }
        const char* impl = getenv("MKV_PAGES_IMPL");
        if (impl && impl[0] == 't') c = PagesConfig{2, 3, 8, 1};
        return c;
    }();
    return cfg;
}

cudaError_t launch_pages(const PagesParams& p, int grid, cudaStream_t s, bool pdl) {
    const PagesConfig c = pages_config();
    if (c.tc) return launch_pages_tc(p, grid, s, pdl);
    if (c.warps == 4) return c.stages == 3 ? launch_pages_t<4, 3>(p, grid, s, pdl) : launch_pages_t<4, 2>(p, grid, s, pdl);
    if (c.stages == 3) return launch_pages_t<8, 3>(p, grid, s, pdl);
    return launch_pages_t<8, 2>(p, grid, s, pdl);
}

// ---------------------------------------------------------------------------
// append kernel: decode_append with flush (flush steps only)
// ---------------------------------------------------------------------------
constexpr int kAppendThreads = 32;  // one warp per unit: at a flush usually one group (of n_r / 16) is left to quantize

// One CTA per unit.  S.n_seg == 0: the units of P (unit_begin + block, tokens P.k_new /
// P.v_new); otherwise segment s covers blocks [S.block_begin[s], S.block_begin[s + 1]) with its
// own unit range and token arrays (every layer of a multi-layer call in one launch).
constexpr size_t kAppendSmem = (kAppendThreads / 32) * (sizeof(PageRows) + sizeof(PageParams));

__global__ void __launch_bounds__(kAppendThreads) append_kernel(const ResidualParams P, const AppendSegs S) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
    int i = blockIdx.x, u = P.unit_begin + i;
    const __half* k_new = P.k_new;
    const __half* v_new = P.v_new;
    if (S.n_seg > 0) {
        int sg = 0;
        while (sg + 1 < S.n_seg && S.block_begin[sg + 1] <= (int)blockIdx.x) ++sg;
        i = blockIdx.x - S.block_begin[sg];
        u = S.unit_begin[sg] + i;
        k_new = S.k_new[sg];
        v_new = S.v_new[sg];
    }
    const int d = kHeadDim;
    const UnitMeta meta = P.meta[u];
    __half* rk = P.res_k + (size_t)u * P.n_r * d;
    __half* rv = P.res_v + (size_t)u * P.n_r * d;
    const int n = meta.n_res + 1;
    if (tid < 16) {
        reinterpret_cast<uint4*>(rk + (size_t)meta.n_res * d)[tid] = reinterpret_cast<const uint4*>(k_new + (size_t)i * d)[tid];
    } else if (tid < 32) {
        reinterpret_cast<uint4*>(rv + (size_t)meta.n_res * d)[tid - 16] =
            reinterpret_cast<const uint4*>(v_new + (size_t)i * d)[tid - 16];
    }
    __threadfence();  // the new row is read back below by cp.async.cg (through L2)
    __syncthreads();
    // (the K3 staged page builder: rows by cp.async, codes from fp16 pairs)
    PageRows& rows = reinterpret_cast<PageRows*>(smem_raw)[warp];
    PageParams& prm = reinterpret_cast<PageParams*>(smem_raw + (kAppendThreads / 32) * sizeof(PageRows))[warp];
    if (n < P.n_r) {
        // a filled 16-row group is quantized now into the page it occupies after the flush (as
        // finish_kernel does on decode steps), so the flush builds only the groups still open
        const bool early = (n & 15) == 0 && meta.n_built == (n >> 4) - 1 && meta.n_pages + (n >> 4) <= meta.cap_pages;
        if (early && warp == 0) {
            const int j = (n >> 4) - 1;
            stage_rows_contig(rows, rk + (size_t)16 * j * d, rv + (size_t)16 * j * d);
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            __syncwarp();
            const int64_t page = meta.page_base + meta.n_pages + j;
            if (!build_page_staged(rows, prm, 16, P.pool + (size_t)page * kPageBytes,
                                   P.shadow ? P.shadow + (size_t)page * (kShadowBytes / 4) : nullptr) &&
                lane == 0)
                atomicOr(P.status, kStatusNonFinite);
        }
        if (tid == 0) {
            P.meta[u].n_res = n;
            if (early) P.meta[u].n_built = n >> 4;
        }
        return;
    }
    // store_block (cache_engine.cpp:34-52): quantize the full block into n_r/16 pages
    const int npg = P.n_r / kGroup;
    bool ok = true;
    // groups [0, n_built) were quantized when they filled (finish_kernel): only the rest
    for (int j = warp + meta.n_built; j < npg; j += kAppendThreads / 32) {
        stage_rows_contig(rows, rk + (size_t)16 * j * d, rv + (size_t)16 * j * d);
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
        const int64_t page = meta.page_base + meta.n_pages + j;
        ok &= build_page_staged(rows, prm, 16, P.pool + (size_t)page * kPageBytes,
                                P.shadow ? P.shadow + (size_t)page * (kShadowBytes / 4) : nullptr);
    }
    if (!ok && lane == 0) atomicOr(P.status, kStatusNonFinite);
    __syncthreads();
    if (tid == 0) {
        P.meta[u].n_pages = meta.n_pages + npg;
        P.meta[u].n_res = 0;
        P.meta[u].n_built = 0;
    }
}

static cudaError_t append_configure(size_t smem) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(append_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    return cudaSuccess;
}

cudaError_t launch_append(const ResidualParams& p, cudaStream_t s) {
    const size_t smem = kAppendSmem;
    if (cudaError_t e = append_configure(smem)) return e;
    AppendSegs none{};
    count_launch(1);
    append_kernel<<<p.n_units, kAppendThreads, smem, s>>>(p, none);
    return cudaGetLastError();
}

cudaError_t launch_append_segments(const ResidualParams& p, const AppendSegs& segs, cudaStream_t s) {
    const size_t smem = kAppendSmem;
    if (cudaError_t e = append_configure(smem)) return e;
    const int blocks = segs.block_begin[segs.n_seg];
    if (blocks == 0) return cudaSuccess;
    count_launch(1);
    append_kernel<<<blocks, kAppendThreads, smem, s>>>(p, segs);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// plan build: a layer's page plan (prefix, per-warp first unit, unit records) from the device
// meta, one CTA per plan, so a flush step uploads nothing between its kernels.  Same
// arithmetic as the host (capi.cu get_plan): units padded to whole batches.
// ---------------------------------------------------------------------------
constexpr int kPlanThreads = 256;

__global__ void __launch_bounds__(kPlanThreads) plan_build_kernel(const UnitMeta* __restrict__ meta,
                                                                  const PlanBuildJobs J) {
    __shared__ int part[kPlanThreads + 1];
    const PlanBuildJob& jb = J.job[blockIdx.x];
    const int n = jb.n, tid = threadIdx.x;
    const int per = (n + kPlanThreads - 1) / kPlanThreads;
    const int i0 = min(n, tid * per), i1 = min(n, i0 + per);
    int local = 0;
    const int bm = jb.batch - 1;  // units padded to whole batches
    for (int i = i0; i < i1; ++i) local += (meta[jb.unit_begin + i].n_pages + bm) & ~bm;
    part[tid] = local;
    __syncthreads();
    if (tid == 0) {  // exclusive scan of the per-thread sums
        int acc = 0;
        for (int t = 0; t < kPlanThreads; ++t) {
            const int v = part[t];
            part[t] = acc;
            acc += v;
        }
        part[kPlanThreads] = acc;
    }
    __syncthreads();
    int pf = part[tid];
    for (int i = i0; i < i1; ++i) {
        const UnitMeta m = meta[jb.unit_begin + i];
        const int next = pf + ((m.n_pages + bm) & ~bm);
        jb.pref[i] = pf;
        UnitRec r;
        r.base = m.page_base - pf;
        r.pbeg = pf;
        r.pend = next;
        r.rend = pf + m.n_pages;
        r.n_prefill = m.n_prefill;
        r.pad[0] = r.pad[1] = 0;
        jb.rec[i] = r;
        pf = next;
    }
    if (tid == 0) jb.pref[n] = part[kPlanThreads];
    __syncthreads();
    // first unit of warp w's range: the smallest i with pref[i + 1] > w * chunk (n - 1 at most)
    const int T = part[kPlanThreads] / jb.batch;
    for (int w = tid; w < jb.warps; w += kPlanThreads) {
        const int p = jb.batch * range_begin(w, T, jb.warps);
        int lo = 0, hi = n - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (jb.pref[mid + 1] > p) hi = mid;
            else lo = mid + 1;
        }
        jb.wstart[w] = lo;
    }
}

cudaError_t launch_plan_build(const UnitMeta* meta, const PlanBuildJobs& jobs, cudaStream_t s) {
    if (jobs.n_jobs == 0) return cudaSuccess;
    count_launch(1);
    plan_build_kernel<<<jobs.n_jobs, kPlanThreads, 0, s>>>(meta, jobs);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// finish kernel: (append) + residual attention on tensor cores + split-K merge
// ---------------------------------------------------------------------------
// Finish kernel (one CTA per unit, launched with PDL): decode_append and the exact fp16
// residual attention first, then -- after griddepcontrol.wait -- the split-K merge of the
// residual and page partials (online max over kMergeBatch partials at a time, no extra barriers).
// 4 warps at <= 96 registers and 33 KB of shared memory: a finish CTA fits on an SM beside a
// page-kernel CTA (<= 208 x 256 registers, 150 KB), so layer l's finish runs its residual
// attention while layer l's pages are still in flight and layer l + 1's pages overlap its merge.
constexpr int kFinishWarps = 4;
constexpr int kMergeBatch = 12;  // page partials folded per online-max round (one L2 round trip)
constexpr int kFinishThreads = kFinishWarps * 32;

// Shared memory: one slot per warp -- 16 K rows + 16 V rows (swizzled 16-byte chunks, 8 KB;
// afterwards the warp's residual partial o[G][128] fp32 reuses the same bytes) -- then the warp
// (m, l) partials.  A launch that may fuse a flush (ResidualParams::fused_flush) uses
// PageScratch-sized slots (its k / v rows are the tile); the others stay at 8 KB per warp, so a
// finish CTA keeps fitting beside a page-kernel CTA.
constexpr int kFinishSlot = 8192;
constexpr int kFinishSlotFlush = (int)sizeof(PageScratch);
// + one PageParams (1 KB): the page a filled 16-row group becomes (finish_kernel, early build)
__host__ __device__ constexpr int finish_smem_bytes(int slot) {
    return kFinishWarps * slot + kFinishWarps * 2 * kMaxG * 4 + (int)sizeof(PageParams);
}
static_assert(offsetof(PageScratch, k) == 0 && offsetof(PageScratch, v) == 4096, "tile = PageScratch k, v");

// The early page build as a real call: inlined, the builder's registers would raise the finish
// kernel's (capped at 96 so a finish CTA fits beside a page CTA) and spill in its hot loop.
__device__ __noinline__ bool build_page_call(PageRows& rows, PageParams& prm, uint8_t* dst, float* shadow) {
    return build_page_staged(rows, prm, 16, dst, shadow);
}

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}

// kSplit = false: one CTA per unit (residual attention, griddepcontrol.wait, merge).
// kSplit = true (the residual kernel of launch_resid_merge): a persistent grid, CTA b attends the
// residuals of units b, b + gridDim.x, ... and stores each unit's combined residual partial to
// P.res_ml / P.res_o, then counts it on P.unit_cnt; merge_kernel does the rest.
template <bool kSplit>
__global__ void __launch_bounds__(kFinishThreads, 5) finish_kernel(const ResidualParams P, const int32_t* __restrict__ pref,
                                                                   const WorkerRanges wr) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int slot = P.fused_flush ? kFinishSlotFlush : kFinishSlot;
    float (*wml)[2][kMaxG] = reinterpret_cast<float (*)[2][kMaxG]>(smem_raw + kFinishWarps * slot);
    const int tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
    const int gid = lane >> 2, tig = lane & 3;
    // the next kernel may start its prologue on SMs this grid leaves free (the page kernel of the
    // next layer reads nothing this kernel writes before its own griddepcontrol.wait; the merge
    // kernel waits on the per-unit counters)
    if (tid == 0) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    for (int i = blockIdx.x; i < P.n_units; i += kSplit ? gridDim.x : P.n_units) {
        const int u = P.unit_begin + i;
        const int d = kHeadDim;
        const int G = P.group;
        // pre-wait prologue: meta / plan were produced before the page kernel started
        const int n_old = P.meta[u].n_res;
        const bool app = P.k_new != nullptr;
        const int n = n_old + (app ? 1 : 0);
        const bool flush = app && P.fused_flush && n == P.n_r;  // this append fills the residual block
        const int ntiles = (n + 15) >> 4;
        const int upre = pref[i], uend = pref[i + 1];
        const int w_first = uend > upre ? worker_of_batch(upre / wr.batch, wr.total_batches, wr.workers) : 0;
        const int w_last = uend > upre ? worker_of_batch((uend - 1) / wr.batch, wr.total_batches, wr.workers) : -1;
        const int n_part = w_last - w_first + 1;
        __half* rk = P.res_k + (size_t)u * P.n_r * d;
        __half* rv = P.res_v + (size_t)u * P.n_r * d;
        const float sl2 = P.scale_log2;
        const int h0 = 2 * tig, h1 = 2 * tig + 1;
        // the next layer's page kernel may start its prologue and first page loads on SMs this
        // grid leaves free (it reads nothing this kernel writes before its own griddepcontrol.wait)
        auto fstamp = [&](int k) {
            if (P.trace != nullptr && tid == 0 && i < kTraceFinishCtas) {
                uint64_t t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                P.trace[(size_t)i * 4 + k] = t;
            }
        };
        fstamp(0);

        // ---- residual attention (overlaps the page kernel): warp w owns tiles w, w + kFinishWarps, ... ----
        uint32_t qb[8][2];
    #pragma unroll
        for (int kc = 0; kc < 8; ++kc)
    #pragma unroll
            for (int p = 0; p < 2; ++p)
                qb[kc][p] = (gid < G) ? __ldg(reinterpret_cast<const uint32_t*>(P.q + ((size_t)i * G + gid) * d + 16 * kc +
                                                                                  2 * tig + 8 * p))
                                      : 0u;
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
        float O[8][4];
    #pragma unroll
        for (int g = 0; g < 8; ++g) O[g][0] = O[g][1] = O[g][2] = O[g][3] = 0.0f;
        uint8_t* tile = smem_raw + warp * slot;
        // rows past the residual count are multiplied by p = 0: they must hold finite values
        for (int e = lane; e < 8192 / 16; e += 32) reinterpret_cast<uint4*>(tile)[e] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        // scores, online softmax and P V of one 16-row tile (rows >= valid masked)
        auto attend_tile = [&](int valid) {
            float Sx[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    #pragma unroll
            for (int kc = 0; kc < 8; ++kc) {
                uint32_t a[4];
                a[0] = *reinterpret_cast<const uint32_t*>(tile + gid * 256 + (((2 * kc) ^ gid) << 4) + 4 * tig);
                a[1] = *reinterpret_cast<const uint32_t*>(tile + (gid + 8) * 256 + (((2 * kc) ^ gid) << 4) + 4 * tig);
                a[2] = *reinterpret_cast<const uint32_t*>(tile + gid * 256 + (((2 * kc + 1) ^ gid) << 4) + 4 * tig);
                a[3] = *reinterpret_cast<const uint32_t*>(tile + (gid + 8) * 256 + (((2 * kc + 1) ^ gid) << 4) + 4 * tig);
                mma_16816(Sx, a, qb[kc][0], qb[kc][1]);
            }
            float x0 = Sx[0] * sl2, x1 = Sx[1] * sl2, x2 = Sx[2] * sl2, x3 = Sx[3] * sl2;
            if (gid >= valid) { x0 = -INFINITY; x1 = -INFINITY; }
            if (gid + 8 >= valid) { x2 = -INFINITY; x3 = -INFINITY; }
            float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
    #pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
            }
            const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
            const float a0 = fast_exp2(m0 - mn0), a1 = fast_exp2(m1 - mn1);
            m0 = mn0; m1 = mn1;
            l0 *= a0; l1 *= a1;
    #pragma unroll
            for (int g = 0; g < 8; ++g) { O[g][0] *= a0; O[g][1] *= a1; O[g][2] *= a0; O[g][3] *= a1; }
            const float p0 = fast_exp2(x0 - m0), p1 = fast_exp2(x1 - m1);
            const float p2 = fast_exp2(x2 - m0), p3 = fast_exp2(x3 - m1);
            l0 += p0 + p2;
            l1 += p1 + p3;
            const uint32_t pb0 = movmatrix_trans(pack_half2(p0, p1));
            const uint32_t pb1 = movmatrix_trans(pack_half2(p2, p3));
            // O[c][h] += sum_t V^T[c][t] P[t][h]; ldmatrix.trans of the swizzled V rows:
            // m0 (t0-7, c0-7) m1 (t0-7, c8-15) m2 (t8-15, c0-7) m3 (t8-15, c8-15) = a0 a1 a2 a3
            const int mi = lane >> 3, ri = lane & 7;
            const int vr = ri + 8 * (mi >> 1);
    #pragma unroll
            for (int g = 0; g < 8; ++g) {
                uint32_t a[4];
                ldmatrix_x4_trans(a, tile + 4096 + vr * 256 + ((((2 * g) + (mi & 1)) ^ (vr & 7)) << 4));
                mma_16816(O[g], a, pb0, pb1);
            }
            __syncwarp();
        };
        if (flush) {
            // ---- fused flush (decode_append's store_block, cache_engine.cpp:34-52,79-90): the new
            // token completes the n_r-row residual block; quantize it into n_r / 16 pages here (the
            // K3 page builder, same pages as append_kernel) and attend the block in its DEQUANTIZED
            // form, as decode_step does after a flush (cache_engine.cpp:108-136).  This step's page
            // pass covers the older pages only. ----
            if (tid < 16) {
                reinterpret_cast<uint4*>(rk + (size_t)n_old * d)[tid] = reinterpret_cast<const uint4*>(P.k_new + (size_t)i * d)[tid];
            } else if (tid < 32) {
                reinterpret_cast<uint4*>(rv + (size_t)n_old * d)[tid - 16] =
                    reinterpret_cast<const uint4*>(P.v_new + (size_t)i * d)[tid - 16];
            }
            __threadfence_block();
            __syncthreads();
            const UnitMeta meta = P.meta[u];
            PageScratch& ps = *reinterpret_cast<PageScratch*>(tile);
            bool ok = true;
            for (int t = warp; t < P.n_r / kGroup; t += kFinishWarps) {
                for (int e = lane; e < 16 * 16; e += 32) {
                    const int r = e >> 4, c16 = e & 15;
                    reinterpret_cast<uint4*>(ps.k[r])[c16] = reinterpret_cast<const uint4*>(rk + (size_t)(16 * t + r) * d)[c16];
                    reinterpret_cast<uint4*>(ps.v[r])[c16] = reinterpret_cast<const uint4*>(rv + (size_t)(16 * t + r) * d)[c16];
                }
                __syncwarp();
                const int64_t page = meta.page_base + meta.n_pages + t;
                ok &= build_page(ps, 16, P.pool + (size_t)page * kPageBytes,
                                 P.shadow ? P.shadow + (size_t)page * (kShadowBytes / 4) : nullptr);
                // dequantize the page into the tile: v = fl(code * scale) + zero with the page's fp16
                // (scale, zero), rounded to fp16 (the page pass's values, up to that rounding)
                const __half* ks = reinterpret_cast<const __half*>(ps.page + kKS);
                const __half* kz = reinterpret_cast<const __half*>(ps.page + kKZ);
                const __half* vs = reinterpret_cast<const __half*>(ps.page + kVS);
                const __half* vz = reinterpret_cast<const __half*>(ps.page + kVZ);
                for (int e = lane; e < 16 * 16; e += 32) {
                    const int r = e >> 4, cc = e & 15, g = cc >> 1;
                    uint32_t kq[4], vq[4];
                    const float vsc = __half2float(vs[vs_param_idx(r, g)]), vzp = __half2float(vz[vz_param_idx(r, g)]);
    #pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int c0 = 8 * cc + 2 * j, c1 = c0 + 1;
                        const float k0 = __fadd_rn(__fmul_rn((float)ps.kc[r][c0], __half2float(ks[k_param_idx(c0)])),
                                                   __half2float(kz[k_param_idx(c0)]));
                        const float k1 = __fadd_rn(__fmul_rn((float)ps.kc[r][c1], __half2float(ks[k_param_idx(c1)])),
                                                   __half2float(kz[k_param_idx(c1)]));
                        kq[j] = pack_half2(k0, k1);
                        vq[j] = pack_half2(__fadd_rn(__fmul_rn((float)ps.vc[r][c0], vsc), vzp),
                                           __fadd_rn(__fmul_rn((float)ps.vc[r][c1], vsc), vzp));
                    }
                    __syncwarp();  // (ps.k / ps.v are overwritten: every lane has read its codes first)
                    *reinterpret_cast<uint4*>(tile + r * 256 + ((cc ^ (r & 7)) << 4)) = make_uint4(kq[0], kq[1], kq[2], kq[3]);
                    *reinterpret_cast<uint4*>(tile + 4096 + r * 256 + ((cc ^ (r & 7)) << 4)) =
                        make_uint4(vq[0], vq[1], vq[2], vq[3]);
                }
                __syncwarp();
                attend_tile(16);
            }
            if (!ok && lane == 0) atomicOr(P.status, kStatusNonFinite);
        }
        for (int t = warp; t < (flush ? 0 : ntiles); t += kFinishWarps) {
            const int row0 = 16 * t;
            const int nrows = min(16, n_old - row0);  // rows already in the residual buffer
            for (int e = lane; e < 256; e += 32) {
                const int r = e >> 4, cc = e & 15;
                if (r < nrows) {
                    const int off = r * 256 + ((cc ^ (r & 7)) << 4);
                    cp_async16(tile + off, rk + (size_t)(row0 + r) * d + cc * 8);
                    cp_async16(tile + 4096 + off, rv + (size_t)(row0 + r) * d + cc * 8);
                }
            }
            cp_async_commit();
            if (app && n_old >= row0 && n_old < row0 + 16) {  // decode_append (cache_engine.cpp:79-90)
                const int r = n_old - row0, cc = lane & 15;
                const bool is_v = lane >= 16;
                const uint4 x = reinterpret_cast<const uint4*>((is_v ? P.v_new : P.k_new) + (size_t)i * d)[cc];
                reinterpret_cast<uint4*>((is_v ? rv : rk) + (size_t)n_old * d)[cc] = x;
                *reinterpret_cast<uint4*>(tile + (is_v ? 4096 : 0) + r * 256 + ((cc ^ (r & 7)) << 4)) = x;
            }
            cp_async_wait_all();
            __syncwarp();
            attend_tile(n - row0);
        }
        // Early page build: when this append fills a 16-row group of the residual block (and the
        // block is not flushed now), the warp that attended that group's tile -- its 16 rows are in
        // the tile, in the staged builder's swizzled layout -- quantizes it into the page it will
        // occupy after the flush (store_block groups, cache_engine.cpp:34-52: each 16-row group is
        // its own page, so the result is the flush's), so the flush step builds only the last one.
        const bool early_build = app && !flush && (n & 15) == 0 && n < P.n_r && P.meta[u].n_built == (n >> 4) - 1 &&
                                 P.meta[u].n_pages + (n >> 4) <= P.meta[u].cap_pages;
        if (early_build && warp == ((n >> 4) - 1) % kFinishWarps) {
            PageParams& prm = *reinterpret_cast<PageParams*>(smem_raw + finish_smem_bytes(slot) - (int)sizeof(PageParams));
            const int64_t page = P.meta[u].page_base + P.meta[u].n_pages + (n >> 4) - 1;
            __syncwarp();
            const bool ok = build_page_call(*reinterpret_cast<PageRows*>(tile), prm, P.pool + (size_t)page * kPageBytes,
                                            P.shadow ? P.shadow + (size_t)page * (kShadowBytes / 4) : nullptr);
            if (!ok && lane == 0) atomicOr(P.status, kStatusNonFinite);
        }
    #pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, o);
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        }
        // warp partial -> smem over the warp's (now idle) tile buffer (l = 0 for warps without tiles)
        float* wo = reinterpret_cast<float*>(tile);  // [kMaxG][128]
        __syncwarp();
    #pragma unroll
        for (int g = 0; g < 8; ++g) {
            const int c = 16 * g + gid;
            if (h0 < G) { wo[h0 * kHeadDim + c] = O[g][0]; wo[h0 * kHeadDim + c + 8] = O[g][2]; }
            if (h1 < G) { wo[h1 * kHeadDim + c] = O[g][1]; wo[h1 * kHeadDim + c + 8] = O[g][3]; }
        }
        if (gid == 0) {
            if (h0 < G) { wml[warp][0][h0] = m0; wml[warp][1][h0] = l0; }
            if (h1 < G) { wml[warp][0][h1] = m1; wml[warp][1][h1] = l1; }
        }
        __syncthreads();  // every read of this unit's meta above is done before it changes
        if (app && tid == 0) {  // only this CTA reads this unit's meta after the append
            if (flush) {
                P.meta[u].n_pages += P.n_r / kGroup;
                P.meta[u].n_res = 0;
                P.meta[u].n_built = 0;
            } else {
                P.meta[u].n_res = n;
                if (early_build) P.meta[u].n_built = n >> 4;
            }
        }
        if constexpr (kSplit) {
            // combine the warps' residual partials into the unit's (online max over 4), store it,
            // then count it: merge_kernel reads it once the unit's counter is complete
            for (int e = tid; e < G * (d / 4); e += kFinishThreads) {
                const int h = e / (d / 4), c4 = e % (d / 4);
                float M = -INFINITY, L = 0.0f;
                float4 a = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                for (int w = 0; w < kFinishWarps; ++w) {
                    const float lw = wml[w][1][h];
                    if (lw > 0.0f) {
                        const float mw = wml[w][0][h];
                        const float nm = fmaxf(M, mw);
                        const float f = fast_exp2(M - nm), sc = fast_exp2(mw - nm);
                        const float4 wv = reinterpret_cast<const float4*>(smem_raw + w * slot)[h * (kHeadDim / 4) + c4];
                        a.x = fmaf(wv.x, sc, a.x * f);
                        a.y = fmaf(wv.y, sc, a.y * f);
                        a.z = fmaf(wv.z, sc, a.z * f);
                        a.w = fmaf(wv.w, sc, a.w * f);
                        L = fmaf(lw, sc, L * f);
                        M = nm;
                    }
                }
                reinterpret_cast<float4*>(P.res_o + ((size_t)u * kMaxG + h) * d)[c4] = a;
                if (c4 == 0) {
                    P.res_ml[(size_t)u * 2 * kMaxG + h] = M;
                    P.res_ml[(size_t)u * 2 * kMaxG + kMaxG + h] = L;
                }
            }
            __syncthreads();  // (also: the next unit reuses the tiles and the warp partials)
            // bar.sync orders every thread's partial stores before thread 0's release add
            if (tid == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(P.unit_cnt + u) : "memory");
            fstamp(3);
        } else {
            // ---- the page partials are complete past this point ----
            fstamp(1);
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            fstamp(2);
            __syncthreads();  // residual warp partials visible
            // Merge: every thread owns 4 consecutive channels of one head (float4: one chunk per thread
            // at G = 4) and loads (m, l, o) of kMergeBatch page partials at once -- one L2 round trip
            // for a unit split over up to kMergeBatch page warps -- folded with an online max (no
            // global-max pass, no further barriers).  h is warp-uniform: the (m, l) loads broadcast.
            for (int e = tid; e < G * (d / 4); e += kFinishThreads) {
                const int h = e / (d / 4), c4 = e % (d / 4);
                float M = -INFINITY, L = 0.0f;
                float4 a = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                for (int w = 0; w < kFinishWarps; ++w) {
                    const float lw = wml[w][1][h];
                    if (lw > 0.0f) {
                        const float mw = wml[w][0][h];
                        const float nm = fmaxf(M, mw);
                        const float f = fast_exp2(M - nm), s = fast_exp2(mw - nm);
                        const float4 wv = reinterpret_cast<const float4*>(smem_raw + w * slot)[h * (kHeadDim / 4) + c4];
                        a.x = fmaf(wv.x, s, a.x * f);
                        a.y = fmaf(wv.y, s, a.y * f);
                        a.z = fmaf(wv.z, s, a.z * f);
                        a.w = fmaf(wv.w, s, a.w * f);
                        L = fmaf(lw, s, L * f);
                        M = nm;
                    }
                }
                for (int p0 = 0; p0 < n_part; p0 += kMergeBatch) {
                    float pm[kMergeBatch], pl[kMergeBatch];
                    float4 po[kMergeBatch];
        #pragma unroll
                    for (int k = 0; k < kMergeBatch; ++k) {
                        const int slot = w_first + p0 + k + i;
                        const bool ok = p0 + k < n_part;
                        pm[k] = ok ? __ldcg(P.part_ml + (size_t)slot * 2 * kMaxG + h) : -INFINITY;
                        pl[k] = ok ? __ldcg(P.part_ml + (size_t)slot * 2 * kMaxG + kMaxG + h) : 0.0f;
                        po[k] = ok ? __ldcg(reinterpret_cast<const float4*>(P.part_o + ((size_t)slot * kMaxG + h) * d) + c4)
                                   : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                    }
                    float cm = pm[0];
        #pragma unroll
                    for (int k = 1; k < kMergeBatch; ++k) cm = fmaxf(cm, pm[k]);
                    const float nm = fmaxf(M, cm);
                    const float f = fast_exp2(M - nm);
                    a.x *= f; a.y *= f; a.z *= f; a.w *= f; L *= f;
        #pragma unroll
                    for (int k = 0; k < kMergeBatch; ++k) {
                        const float s = fast_exp2(pm[k] - nm);  // 0 for absent partials (m = -inf)
                        a.x = fmaf(po[k].x, s, a.x);
                        a.y = fmaf(po[k].y, s, a.y);
                        a.z = fmaf(po[k].z, s, a.z);
                        a.w = fmaf(po[k].w, s, a.w);
                        L = fmaf(pl[k], s, L);
                    }
                    M = nm;
                }
                const float li = 1.0f / L;
                __half2* o2 = reinterpret_cast<__half2*>(P.out + ((size_t)i * G + h) * d) + 2 * c4;
                o2[0] = __floats2half2_rn(a.x * li, a.y * li);
                o2[1] = __floats2half2_rn(a.z * li, a.w * li);
            }
            __syncthreads();
            fstamp(3);
        }  // !kSplit
    }  // units
    // split: the residual CTAs stay resident until the page grid completes (their SM slot beside
    // the page CTA is not released to merge CTAs, which would only poll their counters there)
    if constexpr (kSplit) asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

// Merge kernel of launch_resid_merge: one CTA per unit; waits until the unit's page segments and
// its residual partial have been counted, merges them (as finish_kernel does), writes out and
// resets the counter (its next increment comes from a kernel that waits for this grid).
// kB page partials per L2 round trip: 12 for calls whose units spread over many page warps, 4
// when units outnumber the page warps (~1-2 partials per unit; fewer registers, more resident
// merge CTAs for the merge wave after the page pass).
template <int kB>
__global__ void __launch_bounds__(kFinishThreads) merge_kernel(const ResidualParams P, const int32_t* __restrict__ pref,
                                                               const WorkerRanges wr) {
    const int tid = threadIdx.x;
    const int i = blockIdx.x, u = P.unit_begin + i;
    const int d = kHeadDim, G = P.group;
    if (tid == 0) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int upre = pref[i], uend = pref[i + 1];
    const int w_first = uend > upre ? worker_of_batch(upre / wr.batch, wr.total_batches, wr.workers) : 0;
    const int w_last = uend > upre ? worker_of_batch((uend - 1) / wr.batch, wr.total_batches, wr.workers) : -1;
    const int n_part = w_last - w_first + 1;
    if (tid == 0) {
        const int want = n_part + 1;
        int got;
        // bounded: a lost arrival (an internal error) is reported through the status word
        // instead of hanging the device
        for (uint32_t spin = 0;; ++spin) {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(got) : "l"(P.unit_cnt + u) : "memory");
            if (got >= want) break;
            if (spin > (1u << 23)) {
                atomicOr(P.status, kStatusMergeTimeout);
                break;
            }
            __nanosleep(128);
        }
    }
    __syncthreads();
    for (int e = tid; e < G * (d / 4); e += kFinishThreads) {
        const int h = e / (d / 4), c4 = e % (d / 4);
        float M = __ldcg(P.res_ml + (size_t)u * 2 * kMaxG + h), L = __ldcg(P.res_ml + (size_t)u * 2 * kMaxG + kMaxG + h);
        float4 a = __ldcg(reinterpret_cast<const float4*>(P.res_o + ((size_t)u * kMaxG + h) * d) + c4);
        if (!(L > 0.0f)) {
            M = -INFINITY;
            L = 0.0f;
            a = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
        for (int p0 = 0; p0 < n_part; p0 += kB) {
            float pm[kB], pl[kB];
            float4 po[kB];
#pragma unroll
            for (int k = 0; k < kB; ++k) {
                const int slot = w_first + p0 + k + i;
                const bool ok = p0 + k < n_part;
                pm[k] = ok ? __ldcg(P.part_ml + (size_t)slot * 2 * kMaxG + h) : -INFINITY;
                pl[k] = ok ? __ldcg(P.part_ml + (size_t)slot * 2 * kMaxG + kMaxG + h) : 0.0f;
                po[k] = ok ? __ldcg(reinterpret_cast<const float4*>(P.part_o + ((size_t)slot * kMaxG + h) * d) + c4)
                           : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            }
            float cm = pm[0];
#pragma unroll
            for (int k = 1; k < kB; ++k) cm = fmaxf(cm, pm[k]);
            const float nm = fmaxf(M, cm);
            const float f = fast_exp2(M - nm);
            a.x *= f; a.y *= f; a.z *= f; a.w *= f; L *= f;
#pragma unroll
            for (int k = 0; k < kB; ++k) {
                const float sc = fast_exp2(pm[k] - nm);
                a.x = fmaf(po[k].x, sc, a.x);
                a.y = fmaf(po[k].y, sc, a.y);
                a.z = fmaf(po[k].z, sc, a.z);
                a.w = fmaf(po[k].w, sc, a.w);
                L = fmaf(pl[k], sc, L);
            }
            M = nm;
        }
        const float li = 1.0f / L;
        __half2* o2 = reinterpret_cast<__half2*>(P.out + ((size_t)i * G + h) * d) + 2 * c4;
        o2[0] = __floats2half2_rn(a.x * li, a.y * li);
        o2[1] = __floats2half2_rn(a.z * li, a.w * li);
    }
    __syncthreads();
    if (tid == 0) P.unit_cnt[u] = 0;
    // No griddepcontrol.wait: every write of the page and residual grids this call makes has been
    // consumed through the counters, so the next kernel may start as soon as the merges are done
    // (the residual grid's CTAs may still sit in their final wait for the page grid).
}

cudaError_t launch_finish(const ResidualParams& p, const int32_t* pref, WorkerRanges wr, bool after_pages,
                          cudaStream_t s) {
    const size_t smem = finish_smem_bytes(p.fused_flush ? kFinishSlotFlush : kFinishSlot);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(finish_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             finish_smem_bytes(kFinishSlotFlush));
        if (e == cudaSuccess) e = set_carveout(reinterpret_cast<const void*>(finish_kernel<false>));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    // PDL only behind a page kernel: a finish that follows another finish (no pages) reads
    // the n_res / residual rows that kernel writes, so it needs the full dependency
    if (!after_pages) {
        count_launch(1);
        finish_kernel<false><<<p.n_units, kFinishThreads, smem, s>>>(p, pref, wr);
        return cudaGetLastError();
    }
    return launch_pdl(finish_kernel<false>, dim3(p.n_units), dim3(kFinishThreads), smem, s, p, pref, wr);
}

cudaError_t launch_resid_merge(const ResidualParams& p, const int32_t* pref, WorkerRanges wr, bool after_pages,
                               int resid_ctas, cudaStream_t s) {
    const size_t smem = finish_smem_bytes(p.fused_flush ? kFinishSlotFlush : kFinishSlot);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(finish_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             finish_smem_bytes(kFinishSlotFlush));
        if (e == cudaSuccess) e = set_carveout(reinterpret_cast<const void*>(finish_kernel<true>));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int grid = std::max(1, std::min(resid_ctas, p.n_units));
    cudaError_t e;
    if (!after_pages) {
        count_launch(1);
        finish_kernel<true><<<grid, kFinishThreads, smem, s>>>(p, pref, wr);
        e = cudaGetLastError();
    } else {
        e = launch_pdl(finish_kernel<true>, dim3(grid), dim3(kFinishThreads), smem, s, p, pref, wr);
    }
    if (e != cudaSuccess) return e;
    if (p.n_units >= 2 * wr.workers)
        return launch_pdl(merge_kernel<4>, dim3(p.n_units), dim3(kFinishThreads), 0, s, p, pref, wr);
    return launch_pdl(merge_kernel<kMergeBatch>, dim3(p.n_units), dim3(kFinishThreads), 0, s, p, pref, wr);
}


// ---------------------------------------------------------------------------
// steps kernel: a prepared token stream's decode steps for few, short units in ONE launch
// ---------------------------------------------------------------------------
// mkv_decode_steps over few units with few pages (configs[0]: 8 units of ~60 pages, 256 steps)
// is latency-bound as two kernels per step (~17 us a step).  Here one CTA owns one unit for all
// the steps: per step it appends the token (quantizing the n_r block into pages with the K3
// builder when it fills: store_block, cache_engine.cpp:34-52,79-90), attends its pages (8 warps,
// contiguous 4-page batches each, the page kernel's batch arithmetic: same subnormal
// dequantization, folded scales and zero-point mmas) and then its residual tiles in the same
// online softmax, merges the 8 warp partials in shared memory and writes the step's output
// (decode_step, cache_engine.cpp:100-138).  Units are independent: no grid synchronization.
constexpr int kStepsWarps = 8;
constexpr int kStepsThreads = kStepsWarps * 32;
constexpr int kStepsRing = 2 * kBatch * kPageBytes;  // per warp: 2 stages of one 4-page batch (16 KB)
static_assert(kStepsRing >= (int)sizeof(PageRows), "ring doubles as the residual tile / flush row buffer");
constexpr size_t kStepsSmem = (size_t)kStepsWarps * (kStepsRing + sizeof(PageParams)) + 2 * kQBytes +
                              (size_t)kStepsWarps * (2 * kMaxG + kMaxG * kHeadDim) * sizeof(float) +
                              2 * (2 * kMaxG + kMaxG * kHeadDim) * sizeof(float) + 64;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float4 ld_dsmem_f4(const void* local, uint32_t rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(local)), "r"(rank));
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ float ld_dsmem_f(const void* local, uint32_t rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(local)), "r"(rank));
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}

// kC > 1: a cluster of kC CTAs per unit (kC x 8 warps share its pages and residual tiles); each
// CTA merges its 8 warp partials, rank 0 merges the kC CTA partials through distributed shared
// memory and writes out; rank 0 alone appends / builds the flushed block's pages.
template <int kC>
__global__ void __launch_bounds__(kStepsThreads, 1) steps_kernel(const StepsParams P) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
    const int gid = lane >> 2, tig = lane & 3;
    const uint32_t crank = kC > 1 ? cluster_rank() : 0u;
    constexpr int kGW = kC * kStepsWarps;  // warps sharing one unit
    const int gw = (int)crank * kStepsWarps + warp;
    const int i = blockIdx.x / kC, u = P.unit_begin + i;
    const int d = kHeadDim, G = P.group;
    uint8_t* ring = smem_raw + (size_t)warp * kStepsRing;
    PageParams& prm = reinterpret_cast<PageParams*>(smem_raw + (size_t)kStepsWarps * kStepsRing)[warp];
    __half* qbuf = reinterpret_cast<__half*>(smem_raw + (size_t)kStepsWarps * (kStepsRing + sizeof(PageParams)));
    float* parts = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(qbuf) + 2 * kQBytes);  // [warp][2][kMaxG] then o
    float (*pml)[2][kMaxG] = reinterpret_cast<float (*)[2][kMaxG]>(parts);
    float* po_all = parts + kStepsWarps * 2 * kMaxG;  // [warp][kMaxG][d]
    float* cta_part = po_all + kStepsWarps * kMaxG * kHeadDim;  // [2 step parities][ml 2*kMaxG | o kMaxG*d]
    const UnitMeta meta0 = P.meta[u];
    const int64_t page_base = meta0.page_base;
    int n_pages = meta0.n_pages, n_res = meta0.n_res, n_built = meta0.n_built;
    const int n_prefill = meta0.n_prefill;
    const int partial_page = (n_prefill & 15) ? ((n_prefill + 15) >> 4) - 1 : -1;
    const int partial_valid = n_prefill & 15;
    __half* rk = P.res_k + (size_t)u * P.n_r * d;
    __half* rv = P.res_v + (size_t)u * P.n_r * d;
    const float sl2 = P.scale_log2;
    const float sk = kTwo24 * sl2;
    const int h0 = 2 * tig, h1 = 2 * tig + 1;
    // stale ring slots past a short batch must hold finite values (masked by selects)
    for (int e = lane; e < kStepsRing / 16; e += 32) reinterpret_cast<uint4*>(ring)[e] = make_uint4(0, 0, 0, 0);
    bool ok = true;

    auto load_batch = [&](int b, int stage) {
        const int n = min(kBatch, n_pages - kBatch * b);
        const uint8_t* src = P.pool + (size_t)(page_base + kBatch * b) * kPageBytes;
        uint8_t* dst = ring + (size_t)stage * kBatch * kPageBytes;
        for (int e = lane; e < n * kPageBytes / 16; e += 32) cp_async16(dst + 16 * e, src + 16 * e);
        cp_async_commit();
    };
    // step inputs are loaded one step ahead into registers (q: <= one 16-byte chunk per thread,
    // the token: one chunk per thread of warp 0) and staged at the end of the previous step
    auto q_chunk = [&](int st) {
        const __half* q = P.q + (size_t)st * P.q_step + (size_t)i * G * d;
        return tid < G * d / 8 ? __ldg(reinterpret_cast<const uint4*>(q) + tid) : make_uint4(0, 0, 0, 0);
    };
    auto tok_chunk = [&](int st) {
        if (P.k_new == nullptr || tid >= 32) return make_uint4(0, 0, 0, 0);
        const __half* src = (tid < 16 ? P.k_new : P.v_new) + (size_t)st * P.kv_step + (size_t)i * d;
        return __ldg(reinterpret_cast<const uint4*>(src) + (tid & 15));
    };
    static_assert(kMaxG * kHeadDim / 8 <= kStepsThreads, "q chunk per thread");
    if (tid < G * d / 8) reinterpret_cast<uint4*>(qbuf)[tid] = q_chunk(0);
    uint4 tok = tok_chunk(0);
    __syncthreads();
    for (int st = 0; st < P.n_steps; ++st) {
        const __half* qsm = qbuf + (st & 1) * (kQBytes / 2);
        // the warp's first page batch is requested before the append unless this step flushes
        // (then the new pages are built first): its latency overlaps the append
        const bool flushes = P.k_new != nullptr && n_res + 1 == P.n_r;
        int nb = (n_pages + kBatch - 1) / kBatch;
        int b0 = (int)(((int64_t)gw * nb) / kGW), b1 = (int)(((int64_t)(gw + 1) * nb) / kGW);
        if (!flushes && b0 < b1) load_batch(b0, 0);
        const bool more = st + 1 < P.n_steps;
        const uint4 q_next = more ? q_chunk(st + 1) : make_uint4(0, 0, 0, 0);
        const uint4 tok_next = more ? tok_chunk(st + 1) : make_uint4(0, 0, 0, 0);
        // ---- decode_append (+ store_block of a full residual block) ----
        if (P.k_new != nullptr) {
            if (crank == 0 && tid < 32) reinterpret_cast<uint4*>((tid < 16 ? rk : rv) + (size_t)n_res * d)[tid & 15] = tok;
            ++n_res;
            if (n_res == P.n_r) {
                __threadfence();  // the rows are read back through L2 (cp.async.cg)
                __syncthreads();
                PageRows& rows = *reinterpret_cast<PageRows*>(ring);
                for (int j = warp + n_built; crank == 0 && j < P.n_r / kGroup; j += kStepsWarps) {
                    stage_rows_contig(rows, rk + (size_t)16 * j * d, rv + (size_t)16 * j * d);
                    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
                    __syncwarp();
                    const int64_t page = page_base + n_pages + j;
                    ok &= build_page_staged(rows, prm, 16, P.pool + (size_t)page * kPageBytes,
                                            P.shadow ? P.shadow + (size_t)page * (kShadowBytes / 4) : nullptr);
                    __syncwarp();
                }
                for (int e = lane; e < kStepsRing / 16; e += 32) reinterpret_cast<uint4*>(ring)[e] = make_uint4(0, 0, 0, 0);
                n_pages += P.n_r / kGroup;
                n_res = 0;
                n_built = 0;
            }
        }
        // pages built above are read back through L2 (cp.async.cg) below; the new residual row is
        // staged from the step's input instead, and reaches L2 for later steps through the fence
        // at the end of this step
        if (flushes) __threadfence();
        if constexpr (kC > 1) {
            if (flushes) cluster_sync_all();  // rank 0's new pages, before any CTA loads them
            else __syncthreads();
        } else {
            __syncthreads();
        }

        // ---- q fragments (as pages_kernel: scales folded in, K-bias copy carries the softmax scale) ----
        uint32_t qb[8][2], qsc[8][2];
        load_q_frags(qsm, G, gid, tig, qb, qsc);
        uint32_t qa[8][4];
        {
            const uint32_t s2 = pack_half2(sl2, sl2);
#pragma unroll
            for (int kc = 0; kc < 8; ++kc) {
                qa[kc][0] = hmul2_u32(qb[kc][0], s2); qa[kc][1] = 0u;
                qa[kc][2] = hmul2_u32(qb[kc][1], s2); qa[kc][3] = 0u;
            }
        }
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
        float O[8][4];
#pragma unroll
        for (int g = 0; g < 8; ++g) O[g][0] = O[g][1] = O[g][2] = O[g][3] = 0.0f;
        float Dvb[4] = {0.0f, 0.0f, 0.0f, 0.0f};

        // ---- this warp's pages: batches [b0, b1) of the unit's ceil(n_pages / 4) ----
        if (flushes) {
            nb = (n_pages + kBatch - 1) / kBatch;
            b0 = (int)(((int64_t)gw * nb) / kGW);
            b1 = (int)(((int64_t)(gw + 1) * nb) / kGW);
            if (b0 < b1) load_batch(b0, 0);
        }
        for (int b = b0; b < b1; ++b) {
            const int stage = (b - b0) & 1;
            if (b + 1 < b1) {
                load_batch(b + 1, stage ^ 1);
                asm volatile("cp.async.wait_group 1;\n" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            }
            __syncwarp();
            const uint8_t* buf = ring + (size_t)stage * kBatch * kPageBytes;
            const int n = min(kBatch, n_pages - kBatch * b);
            const int pfirst = kBatch * b;
            float S[kBatch][4];
            uint4 kw[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                kw[j] = lds128(buf + j * kPageBytes + kKC + lane * 16);
                S[j][0] = S[j][1] = S[j][2] = S[j][3] = 0.0f;
            }
#pragma unroll
            for (int kc = 0; kc < 8; ++kc) {
                const int sh = code_shift(kc);
                const uint32_t mask = 0x00030003u << (2 * code_class(kc));
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    const uint2 ks = lds64(buf + j * kPageBytes + kKS + ((kc >> 1) * 4 + tig) * 16 + (kc & 1) * 8);
                    const uint32_t a[4] = {(kw[j].x >> sh) & mask, (kw[j].y >> sh) & mask,
                                           (kw[j].z >> sh) & mask, (kw[j].w >> sh) & mask};
                    mma_16816(S[j], a, hmul2_u32(qsc[kc][0], ks.x), hmul2_u32(qsc[kc][1], ks.y));
                }
            }
            float Kb[4] = {0.0f, 0.0f, 0.0f, 0.0f}, Kb2[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            {
                uint4 z[4];
                const uint8_t* zp = buf + (gid & (kBatch - 1)) * kPageBytes + kKZ + tig * 16;
#pragma unroll
                for (int j = 0; j < 4; ++j) z[j] = lds128(zp + 64 * j);
                const uint32_t* zz = reinterpret_cast<const uint32_t*>(z);
#pragma unroll
                for (int kc = 0; kc < 8; kc += 2) {
                    mma_16816(Kb, qa[kc], zz[2 * kc], zz[2 * kc + 1]);
                    mma_16816(Kb2, qa[kc + 1], zz[2 * kc + 2], zz[2 * kc + 3]);
                }
                Kb[0] += Kb2[0];
                Kb[1] += Kb2[1];
            }
            const bool special = (n < kBatch) || (partial_page >= pfirst && partial_page < pfirst + n);
            float x[kBatch][4];
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const float kb0 = __shfl_sync(0xffffffffu, Kb[j & 1], 8 * tig + (j >> 1));
                const float kb1 = __shfl_sync(0xffffffffu, Kb[j & 1], 8 * tig + 4 + (j >> 1));
                x[j][0] = fmaf(S[j][0], sk, kb0);
                x[j][1] = fmaf(S[j][1], sk, kb1);
                x[j][2] = fmaf(S[j][2], sk, kb0);
                x[j][3] = fmaf(S[j][3], sk, kb1);
            }
            if (special) {
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    const int lp = pfirst + j;
                    const int valid = (j >= n) ? 0 : ((lp == partial_page) ? partial_valid : 16);
                    if (gid >= valid) { x[j][0] = -INFINITY; x[j][1] = -INFINITY; }
                    if (gid + 8 >= valid) { x[j][2] = -INFINITY; x[j][3] = -INFINITY; }
                }
            }
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                mx0 = fmaxf(mx0, fmaxf(x[j][0], x[j][2]));
                mx1 = fmaxf(mx1, fmaxf(x[j][1], x[j][3]));
            }
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
            }
            const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
            if (__any_sync(0xffffffffu, (mn0 > m0 + kLazy) | (mn1 > m1 + kLazy))) {
                const float a0 = fast_exp2(m0 - mn0), a1 = fast_exp2(m1 - mn1);
                l0 *= a0; l1 *= a1;
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    O[g][0] *= a0; O[g][1] *= a1; O[g][2] *= a0; O[g][3] *= a1;
                }
                Dvb[0] *= a0; Dvb[1] *= a1;
                m0 = mn0; m1 = mn1;
            }
            uint32_t pb0[kBatch], pb1[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const float p0 = fast_exp2(x[j][0] - m0), p1 = fast_exp2(x[j][1] - m1);
                const float p2 = fast_exp2(x[j][2] - m0), p3 = fast_exp2(x[j][3] - m1);
                l0 += p0 + p2;
                l1 += p1 + p3;
                pb0[j] = movmatrix_trans(pack_half2(p0, p1));
                pb1[j] = movmatrix_trans(pack_half2(p2, p3));
            }
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const uint8_t* page = buf + j * kPageBytes;
                const uint2 vz = lds64(page + kVZ + lane * 8);
                const uint32_t az[4] = {vz.x, 0u, vz.y, 0u};
                mma_16816(Dvb, az, pb0[j], pb1[j]);
                const uint4 vw = lds128(page + kVC + lane * 16);
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const int sh = code_shift(g);
                    const uint32_t mask = 0x00030003u << (2 * code_class(g));
                    const uint2 vs = lds64(page + kVS + ((g >> 1) * 4 + tig) * 16 + (g & 1) * 8);
                    const uint32_t a[4] = {(vw.x >> sh) & mask, (vw.y >> sh) & mask, (vw.z >> sh) & mask,
                                           (vw.w >> sh) & mask};
                    mma_16816(O[g], a, hmul2_u32(pb0[j], vs.x), hmul2_u32(pb1[j], vs.y));
                }
            }
            __syncwarp();
        }
        // page partial -> plain (m, l, o[c][h]) form: o = O * 2^24 * 4^s + value zero-point bias
        // (Dvb[g][h] of lane 4 g + tig); l summed over the lane quads below
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const float dv0 = __shfl_sync(0xffffffffu, Dvb[0], 4 * g + tig);
            const float dv1 = __shfl_sync(0xffffffffu, Dvb[1], 4 * g + tig);
            const float f = extract_scale(g);
            O[g][0] = fmaf(O[g][0], f, dv0);
            O[g][2] = fmaf(O[g][2], f, dv0);
            O[g][1] = fmaf(O[g][1], f, dv1);
            O[g][3] = fmaf(O[g][3], f, dv1);
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, o);
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        }

        // ---- residual tiles (exact fp16 attention, as finish_kernel), same online softmax ----
        // tile t goes to warp kGW - 1 - t % kGW of the unit (the page ranges differ by <= 1 batch)
        for (int t = kGW - 1 - gw; 16 * t < n_res; t += kGW) {
            const int nrows = min(16, n_res - 16 * t);
            uint8_t* tile = ring;  // this warp's page batches are done: its ring holds the tile
            const bool fresh = P.k_new != nullptr && !flushes;  // row n_res - 1 came with this step
            for (int e = lane; e < 256; e += 32) {
                const int r = e >> 4, cc = e & 15;
                const int off = r * 256 + ((cc ^ (r & 7)) << 4);
                if (r < nrows) {
                    const int row = 16 * t + r;
                    const bool tokrow = fresh && row == n_res - 1;
                    cp_async16(tile + off, tokrow ? P.k_new + (size_t)st * P.kv_step + (size_t)i * d + cc * 8
                                                  : rk + (size_t)row * d + cc * 8);
                    cp_async16(tile + 4096 + off, tokrow ? P.v_new + (size_t)st * P.kv_step + (size_t)i * d + cc * 8
                                                         : rv + (size_t)row * d + cc * 8);
                } else {  // rows past the residual are multiplied by p = 0: keep them finite
                    *reinterpret_cast<uint4*>(tile + off) = make_uint4(0, 0, 0, 0);
                    *reinterpret_cast<uint4*>(tile + 4096 + off) = make_uint4(0, 0, 0, 0);
                }
            }
            cp_async_commit();
            cp_async_wait_all();
            __syncwarp();
            float Sx[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int kc = 0; kc < 8; ++kc) {
                uint32_t a[4];
                a[0] = *reinterpret_cast<const uint32_t*>(tile + gid * 256 + (((2 * kc) ^ gid) << 4) + 4 * tig);
                a[1] = *reinterpret_cast<const uint32_t*>(tile + (gid + 8) * 256 + (((2 * kc) ^ gid) << 4) + 4 * tig);
                a[2] = *reinterpret_cast<const uint32_t*>(tile + gid * 256 + (((2 * kc + 1) ^ gid) << 4) + 4 * tig);
                a[3] = *reinterpret_cast<const uint32_t*>(tile + (gid + 8) * 256 + (((2 * kc + 1) ^ gid) << 4) + 4 * tig);
                mma_16816(Sx, a, qb[kc][0], qb[kc][1]);
            }
            float x0 = Sx[0] * sl2, x1 = Sx[1] * sl2, x2 = Sx[2] * sl2, x3 = Sx[3] * sl2;
            if (gid >= nrows) { x0 = -INFINITY; x1 = -INFINITY; }
            if (gid + 8 >= nrows) { x2 = -INFINITY; x3 = -INFINITY; }
            float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
            }
            const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
            const float a0 = fast_exp2(m0 - mn0), a1 = fast_exp2(m1 - mn1);
            m0 = mn0; m1 = mn1;
            l0 *= a0; l1 *= a1;
#pragma unroll
            for (int g = 0; g < 8; ++g) { O[g][0] *= a0; O[g][1] *= a1; O[g][2] *= a0; O[g][3] *= a1; }
            const float p0 = fast_exp2(x0 - m0), p1 = fast_exp2(x1 - m1);
            const float p2 = fast_exp2(x2 - m0), p3 = fast_exp2(x3 - m1);
            float ls0 = p0 + p2, ls1 = p1 + p3;
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {  // l is kept quad-reduced in this phase
                ls0 += __shfl_xor_sync(0xffffffffu, ls0, o);
                ls1 += __shfl_xor_sync(0xffffffffu, ls1, o);
            }
            l0 += ls0;
            l1 += ls1;
            const uint32_t pb0 = movmatrix_trans(pack_half2(p0, p1));
            const uint32_t pb1 = movmatrix_trans(pack_half2(p2, p3));
            const int mi = lane >> 3, ri = lane & 7;
            const int vr = ri + 8 * (mi >> 1);
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                uint32_t a[4];
                ldmatrix_x4_trans(a, tile + 4096 + vr * 256 + ((((2 * g) + (mi & 1)) ^ (vr & 7)) << 4));
                mma_16816(O[g], a, pb0, pb1);
            }
            __syncwarp();
        }

        // ---- warp partial -> shared memory, merge of the 8 partials, out ----
        float* wo = po_all + (size_t)warp * kMaxG * d;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const int c = 16 * g + gid;
            if (h0 < G) { wo[h0 * d + c] = O[g][0]; wo[h0 * d + c + 8] = O[g][2]; }
            if (h1 < G) { wo[h1 * d + c] = O[g][1]; wo[h1 * d + c + 8] = O[g][3]; }
        }
        if (gid == 0) {
            if (h0 < G) { pml[warp][0][h0] = m0; pml[warp][1][h0] = l0; }
            if (h1 < G) { pml[warp][0][h1] = m1; pml[warp][1][h1] = l1; }
        }
        __syncthreads();
        for (int e = tid; e < G * (d / 4); e += kStepsThreads) {
            const int h = e / (d / 4), c4 = e % (d / 4);
            float M = -INFINITY, L = 0.0f;
            float4 a = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            for (int w = 0; w < kStepsWarps; ++w) {
                const float lw = pml[w][1][h];
                if (lw > 0.0f) {
                    const float mw = pml[w][0][h];
                    const float nm = fmaxf(M, mw);
                    const float f = fast_exp2(M - nm), sc = fast_exp2(mw - nm);
                    const float4 wv = reinterpret_cast<const float4*>(po_all + ((size_t)w * kMaxG + h) * d)[c4];
                    a.x = fmaf(wv.x, sc, a.x * f);
                    a.y = fmaf(wv.y, sc, a.y * f);
                    a.z = fmaf(wv.z, sc, a.z * f);
                    a.w = fmaf(wv.w, sc, a.w * f);
                    L = fmaf(lw, sc, L * f);
                    M = nm;
                }
            }
            if constexpr (kC == 1) {
                const float li = 1.0f / L;
                __half2* o2 = reinterpret_cast<__half2*>(P.out + (size_t)st * P.out_step + ((size_t)i * G + h) * d) + 2 * c4;
                o2[0] = __floats2half2_rn(a.x * li, a.y * li);
                o2[1] = __floats2half2_rn(a.z * li, a.w * li);
            } else {
                float* cp = cta_part + (size_t)(st & 1) * (2 * kMaxG + kMaxG * kHeadDim);
                reinterpret_cast<float4*>(cp + 2 * kMaxG + h * d)[c4] = a;
                if (c4 == 0) { cp[h] = M; cp[kMaxG + h] = L; }
            }
        }
        if constexpr (kC > 1) {
            // every CTA's partial of this step is in its shared memory; rank 0 merges them.  The
            // buffers alternate by step: a CTA writes the same buffer again two steps later, after
            // the next step's barrier, which rank 0 reaches only when this merge is done.
            cluster_sync_all();
            if (crank == 0) {
                const float* cp = cta_part + (size_t)(st & 1) * (2 * kMaxG + kMaxG * kHeadDim);
                for (int e = tid; e < G * (d / 4); e += kStepsThreads) {
                    const int h = e / (d / 4), c4 = e % (d / 4);
                    float M = -INFINITY, L = 0.0f;
                    float4 a = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
                    for (int r = 0; r < kC; ++r) {
                        const float lr = ld_dsmem_f(cp + kMaxG + h, (uint32_t)r);
                        if (lr > 0.0f) {
                            const float mr = ld_dsmem_f(cp + h, (uint32_t)r);
                            const float4 v = ld_dsmem_f4(cp + 2 * kMaxG + h * d + 4 * c4, (uint32_t)r);
                            const float nm = fmaxf(M, mr);
                            const float f = fast_exp2(M - nm), sc = fast_exp2(mr - nm);
                            a.x = fmaf(v.x, sc, a.x * f);
                            a.y = fmaf(v.y, sc, a.y * f);
                            a.z = fmaf(v.z, sc, a.z * f);
                            a.w = fmaf(v.w, sc, a.w * f);
                            L = fmaf(lr, sc, L * f);
                            M = nm;
                        }
                    }
                    const float li = 1.0f / L;
                    __half2* o2 = reinterpret_cast<__half2*>(P.out + (size_t)st * P.out_step + ((size_t)i * G + h) * d) + 2 * c4;
                    o2[0] = __floats2half2_rn(a.x * li, a.y * li);
                    o2[1] = __floats2half2_rn(a.z * li, a.w * li);
                }
            }
        }
        // next step's q into the other buffer; the appended row reaches L2 for later steps
        if (more && tid < G * d / 8) reinterpret_cast<uint4*>(qbuf + ((st + 1) & 1) * (kQBytes / 2))[tid] = q_next;
        tok = tok_next;
        if (tid < 32) __threadfence();
        __syncthreads();  // partials / q staging are reused by the next step
    }
    if (!ok && lane == 0) atomicOr(P.status, kStatusNonFinite);
    if constexpr (kC > 1) cluster_sync_all();  // no CTA exits while rank 0 may still read its partials
    if (crank == 0 && tid == 0) {
        P.meta[u].n_pages = n_pages;
        P.meta[u].n_res = n_res;
        P.meta[u].n_built = n_built;
    }
}

template <int kC>
static cudaError_t launch_steps_c(const StepsParams& p, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(steps_kernel<kC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStepsSmem);
        if (e == cudaSuccess && kC > 1) e = cudaFuncSetAttribute(steps_kernel<kC>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    count_launch(1);
    if constexpr (kC == 1) {
        steps_kernel<1><<<p.n_units, kStepsThreads, kStepsSmem, s>>>(p);
        return cudaGetLastError();
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(p.n_units * kC);
        cfg.blockDim = dim3(kStepsThreads);
        cfg.dynamicSmemBytes = kStepsSmem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kC;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, steps_kernel<kC>, p);
    }
}

// CTAs per unit: as many as fit one CTA per SM (4, 2 or 1; 8 measured no faster than 4);
// MKV_STEPS_CLUSTER=1|2|4|8 forces it.
cudaError_t launch_steps(const StepsParams& p, cudaStream_t s) {
    static const int forced = [] {
        const char* e = getenv("MKV_STEPS_CLUSTER");
        return e ? atoi(e) : 0;
    }();
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int c = forced == 1 || forced == 2 || forced == 4 || forced == 8 ? forced
                                                                     : (p.n_units * 4 <= sms ? 4 : (p.n_units * 2 <= sms ? 2 : 1));
    if (c == 8) return launch_steps_c<8>(p, s);
    if (c == 4) return launch_steps_c<4>(p, s);
    if (c == 2) return launch_steps_c<2>(p, s);
    return launch_steps_c<1>(p, s);
}

}  // namespace mkv
