// decode_tc.cu -- K4 page pass on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Same contract as pages_kernel (decode.cu): every (worker, unit) segment of the step's global
// page sequence -> one split-K partial (m, l, o) in the log2 domain, merged by finish_kernel.
// What changes is where the products run.  Per 8-page batch (128 tokens of one unit):
//
//   S[t][(j, h)] = sum_c codeK[t][c] * 4^cls(c) 2^-24 * (q_h[c] 4^-cls(c) s_j[c])      (tcgen05)
//                  A = the 2-bit key codes as fp16 subnormals, stored to TMEM straight from the
//                  page's mma-fragment words (tcgen05.st.16x256b: lanes = tokens); B = q scaled by
//                  each page's per-channel key scales, K-major SW128 in shared memory, N = 8 pages
//                  x GP heads (only page j's block is read back for a token of page j).
//   O[c][(g, h)] += sum_t codeV[c][t] * 4^cls(g) 2^-24 * (p_h[t] sV[t][g])               (tcgen05)
//                  A = the value codes transposed (lanes = channels), B = the probabilities scaled
//                  by each token's per-group value scale, N = 8 groups x GP heads (channel c reads
//                  its group's block); accumulated in TMEM across the segment's batches.
//   key / value zero points: Kb[j][h] = sum_c z_j[c] q_h[c] and Vb[g][h] = sum_t zV[t][g] p_h[t]
//                  on mma.sync (8 resp. 2 per warp per batch, fp32-exact products).
//
// TMEM stores put fragment register pairs at (lane, column) so that a 16-column K step reads the
// k-pairs in the order 0 4 1 5 2 6 3 7 (tools/probes/probe_ts.cu); the B operands are written in
// that permuted K order (kpos below).  The 4^cls(g) of the value codes is a per-row factor and is
// applied in the epilogue; the key one is folded into B.
//
// CTA = one SM: two independent workers (warpgroups 0 and 1, each 4 compute warps + one control
// warp that issues the bulk copies of its 3-stage ring and its tcgen05.mma).  A worker's batches:
//   compute: K codes -> TMEM, B_K -> smem, key bias (warp 0)  --opK-->  control: S = A_K B_K
//            V codes -> TMEM (after the previous PV)
//            S -> regs (thread = token), lazy online softmax (rescale of O in TMEM only when a
//            head's max grows by > 2^kLazy), p -> smem, B_V -> smem, value bias  --opV-->
//                                                                       control: O += A_V B_V
// so one worker's MMAs run under the other worker's (and its own next batch's) CUDA-core work.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "mkv_kernels.h"
#include "mkv_sm100.cuh"

namespace mkv {

using namespace sm100;

namespace {

constexpr int kTcBatch = 8;                      // pages per batch (one M = 128 token tile)
constexpr int kTcStages = 3;                     // ring stages per worker
// pages sit 2048 + 16 bytes apart in a stage: the same field of the 8 pages falls in different
// shared-memory banks (the per-page parameter loads of one warp instruction span pages)
constexpr int kPgStride = kPageBytes + 16;
constexpr int kStageBytes = kTcBatch * kPgStride;
constexpr int kTcWarps = 10;                     // 2 x (4 compute + 1 control)
constexpr float kTwo24 = 16777216.0f;
constexpr float kLazy = 3.0f;                    // log2 units: p <= 8 keeps fp16 p * s far from overflow

__host__ __device__ constexpr int code_class(int k) { return k < 5 ? k : k - 5; }
__host__ __device__ constexpr int code_shift(int k) { return k < 5 ? 0 : 10; }
__host__ __device__ constexpr float pow4_neg(int s) {
    return s == 0 ? 1.0f : (s == 1 ? 0.25f : (s == 2 ? 0.0625f : (s == 3 ? 0.015625f : 0.00390625f)));
}
// position of token / channel i (0..15) of a 16-wide K step in the MMA's K order
__host__ __device__ constexpr int kpos(int i) { return (i < 8 ? 4 * (i >> 1) : 4 * ((i - 8) >> 1) + 2) + (i & 1); }

template <int GP>
struct TcLayout {
    static constexpr int N = 8 * GP;               // MMA N (pages x heads, groups x heads)
    static constexpr int kB = N * 256;             // one K-major SW128 B tile: 2 halves x N rows x 128 B
    static constexpr int kRing = 0;
    static constexpr int kBK = (kRing + kTcStages * kStageBytes + 1023) & ~1023;  // SW128 tiles: 1024-aligned
    static constexpr int kBV = kBK + kB;
    static constexpr int kP = kBV + kB;            // p [GP][128] fp16 (K order)
    static constexpr int kQsl = kP + GP * 256;     // q * scale_log2 [GP][128] fp16 (natural order)
    static constexpr int kQsc = kQsl + GP * 256;   // q * 4^-cls [GP][128] fp16 (K order)
    static constexpr int kKb = kQsc + GP * 256;    // key-bias partials [4 warps][8 pages][GP] fp32
    static constexpr int kRed = kKb + 4 * 8 * GP * 4;  // [4 warps][GP] fp32
    static constexpr int kDvb = kRed + 4 * GP * 4; // [4 warps][8 groups][GP] fp32
    static constexpr int kFlag = kDvb + 4 * 8 * GP * 4;
    static constexpr int kBars = (kFlag + 16 + 7) & ~7;
    static constexpr int kBarCount = 2 * kTcStages + 4;
    static constexpr int kWorker = (kBars + kBarCount * 8 + 1023) & ~1023;
    static constexpr int kSmem = 2 * kWorker + 1024 + 16;  // + alignment slack + TMEM base word
    // TMEM columns of a worker (256 each): A_K, A_V (64 each), D_S, D_O (N each)
    static constexpr int kTAK = 0, kTAV = 64, kTDS = 128, kTDO = 128 + N;
};

__device__ __forceinline__ void tmem_st_16x256_x8(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
template <int X>
__device__ __forceinline__ void tmem_ld_32x32(uint32_t taddr, uint32_t (&r)[X]);
template <>
__device__ __forceinline__ void tmem_ld_32x32<8>(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld_32x32<16>(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
template <int X>
__device__ __forceinline__ void tmem_st_32x32(uint32_t taddr, const uint32_t (&r)[X]);
template <>
__device__ __forceinline__ void tmem_st_32x32<8>(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
template <>
__device__ __forceinline__ void tmem_st_32x32<16>(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__device__ __forceinline__ uint4 lds128(const uint8_t* p) { return *reinterpret_cast<const uint4*>(p); }

// value codes of groups 2Q, 2Q+1 of the batch's 8 pages -> TMEM A_V (lanes = channels 32Q..32Q+31);
// compile-time class shifts / masks
template <int Q>
__device__ __forceinline__ void store_v_codes(const uint8_t* stage, int lane, uint32_t taddr) {
    constexpr int g0 = 2 * Q, g1 = 2 * Q + 1;
    constexpr int sh0 = code_shift(g0), sh1 = code_shift(g1);
    constexpr uint32_t m0 = 0x00030003u << (2 * code_class(g0)), m1 = 0x00030003u << (2 * code_class(g1));
    uint32_t r0[32], r1[32];
#pragma unroll
    for (int j = 0; j < kTcBatch; ++j) {
        const uint4 vw = lds128(stage + j * kPgStride + kVC + lane * 16);
        r0[4 * j + 0] = (vw.x >> sh0) & m0; r0[4 * j + 1] = (vw.z >> sh0) & m0;
        r0[4 * j + 2] = (vw.y >> sh0) & m0; r0[4 * j + 3] = (vw.w >> sh0) & m0;
        r1[4 * j + 0] = (vw.x >> sh1) & m1; r1[4 * j + 1] = (vw.z >> sh1) & m1;
        r1[4 * j + 2] = (vw.y >> sh1) & m1; r1[4 * j + 3] = (vw.w >> sh1) & m1;
    }
    tmem_st_16x256_x8(taddr, r0);
    tmem_st_16x256_x8(taddr + ((uint32_t)16 << 16), r1);
}
__device__ __forceinline__ uint2 lds64(const uint8_t* p) { return *reinterpret_cast<const uint2*>(p); }

// byte offset of element (row n, K index kk) of a K-major SW128 B tile with N rows
template <int N>
__device__ __forceinline__ int bk_off(int n, int kk) {
    const int half = kk >> 6, chunk = (kk & 63) >> 3;
    return half * (N * 128) + n * 128 + ((chunk ^ (n & 7)) << 4) + (kk & 7) * 2;
}

// Batch cursor over a worker's page range [start, end) of the plan's padded page sequence
// (units padded to whole batches, so batches never straddle units).
struct Cursor {
    const UnitRec* rec;
    int n_units, end;
    int unit, pg;          // current batch: unit, first padded page index
    int pbeg, pend, rend;  // the unit's record
    int64_t base;
    // record fields broadcast from lane 0: provably warp-uniform, so the .sync.aligned tcgen05 /
    // shuffle instructions under this control flow need no divergence handling (ENDCOLLECTIVE)
    __device__ void load_unit() {
        const UnitRec r = rec[unit];
        pbeg = __shfl_sync(0xffffffffu, r.pbeg, 0);
        pend = __shfl_sync(0xffffffffu, r.pend, 0);
        rend = __shfl_sync(0xffffffffu, r.rend, 0);
        base = (int64_t)(((uint64_t)(uint32_t)__shfl_sync(0xffffffffu, (int)(r.base >> 32), 0) << 32) |
                         (uint32_t)__shfl_sync(0xffffffffu, (int)(uint32_t)r.base, 0));
    }
    __device__ void init(const UnitRec* rec_, int n_units_, int first_unit, int start, int end_) {
        rec = rec_; n_units = n_units_; end = end_; unit = first_unit; pg = start;
        load_unit();
        while (pg >= pend && unit + 1 < n_units) { ++unit; load_unit(); }
    }
    __device__ bool valid() const { return pg < end; }
    __device__ void next() {
        pg += kTcBatch;
        if (pg >= pend && pg < end) {
            do { ++unit; load_unit(); } while (pg >= pend && unit + 1 < n_units);
        }
    }
    __device__ int n_real() const { return min(kTcBatch, rend - pg); }
    __device__ bool seg_first(int start) const { return pg == pbeg || pg == start; }
    __device__ bool seg_last() const { return pg + kTcBatch >= min(pend, end); }
};

}  // namespace

template <int GP>
// <= 160 registers (x 320 threads = 51200): a finish CTA (128 threads x 96) still fits beside it
__global__ void __maxnreg__(160) pages_tc_kernel(const PagesParams P) {
    using Lay = TcLayout<GP>;
    constexpr int N = Lay::N;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned base derived by pointer arithmetic on the shared array itself, so every
    // access below stays a shared-memory (LDS/STS) access rather than a generic one
    uint8_t* sm_base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint32_t* tmem_word = reinterpret_cast<uint32_t*>(sm_base + 2 * Lay::kWorker);
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // provably warp-uniform
    const int wg = warp < 8 ? (warp >> 2) : (warp - 8);  // worker of this warp
    uint8_t* sw = sm_base + wg * Lay::kWorker;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sw + Lay::kBars);
    uint64_t* full = bars;                 // [stages]  bulk copy landed
    uint64_t* empty = bars + kTcStages;    // [stages]  the compute warps are done with the stage
    uint64_t* opK = bars + 2 * kTcStages;  // A_K, B_K ready (128 arrivals)
    uint64_t* opV = opK + 1;               // A_V, B_V ready (128 arrivals)
    uint64_t* sFull = opK + 2;             // S = A_K B_K complete (commit)
    uint64_t* pvDone = opK + 3;            // O += A_V B_V complete (commit)

    // Dependents (this layer's finish kernel) may launch only once the previous kernel on the
    // stream has completed, unless this is an early page pass (P.early): the finish kernel's
    // pre-wait prologue appends to the residual of units the previous finish kernel may own.
    if (threadIdx.x == 0) {
        if (!P.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    }
    // ---- setup: TMEM, barriers, zeroed rings (stale slots of short batches stay finite) ----
    if (warp == 8) {
        tmem_alloc(tmem_word, 512);
        tmem_relinquish();
    }
    if (warp < 8) {
        uint8_t* ring = sw + Lay::kRing;
        for (int e = tid & 127; e < kTcStages * kStageBytes / 16; e += 128)
            reinterpret_cast<uint4*>(ring)[e] = make_uint4(0, 0, 0, 0);
    }
    if (lane == 0 && warp >= 8) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 128);
        }
        mbar_init(opK, 128);
        mbar_init(opV, 128);
        mbar_init(sFull, 1);
        mbar_init(pvDone, 1);
        fence_mbar_init();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_word + (uint32_t)(wg * 256);

    const int worker = blockIdx.x * 2 + wg;
    const int Tb = P.total_pages / kTcBatch;
    const int start = worker < P.n_warps ? kTcBatch * range_begin(worker, Tb, P.n_warps) : 0;
    const int end = worker < P.n_warps ? kTcBatch * range_begin(worker + 1, Tb, P.n_warps) : 0;
    const bool active = start < end;
    // diagnostics (P.trace): globaltimer stamps of batches 4..7 of this worker
    auto stamp = [&](int b, int base, int per, int k) {
        if (P.trace != nullptr && lane == 0 && b >= 4 && b < 8) {
            uint64_t tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            P.trace[(size_t)worker * kTcTraceWords + base + (b - 4) * per + k] = tt;
        }
    };

    if (warp >= 8) {
        // ================= control warp: bulk copies + tcgen05.mma =================
        // The whole warp walks the batch sequence (uniform control flow); lane 0 issues.
        if (active) {
            const int first_unit = __shfl_sync(0xffffffffu, __ldg(P.wstart + worker), 0);
            Cursor cc, pc;  // consumer (MMA) and producer (copies) cursors
            cc.init(P.rec, P.n_units, first_unit, start, end);
            pc = cc;
            int pb = 0;     // batches issued
            auto produce = [&](int upto) {
                while (pc.valid() && pb < upto) {
                    const int s = pb % kTcStages;
                    if (pb >= kTcStages) mbar_wait_sleep(&empty[s], ((pb / kTcStages) - 1) & 1);
                    if (lane == 0) {
                        const int n = pc.n_real();
                        mbar_expect_tx(&full[s], n * kPageBytes);
                        for (int j = 0; j < n; ++j)
                            bulk_g2s(sw + Lay::kRing + s * kStageBytes + j * kPgStride,
                                     P.pool + (pc.base + pc.pg + j) * kPageBytes, kPageBytes, &full[s]);
                    }
                    __syncwarp();
                    ++pb;
                    pc.next();
                }
            };
            constexpr uint32_t kIdesc = idesc_f16(128, N, false);
            const uint32_t bk = smem_u32(sw + Lay::kBK), bv = smem_u32(sw + Lay::kBV);
            for (int b = 0; cc.valid(); ++b) {
                produce(b + kTcStages);
                const uint32_t ph = b & 1;
                mbar_wait_sleep(opK, ph);
                tc_fence_after();
                stamp(b, 64, 4, 0);
                if (lane == 0) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        umma_f16_ts(tmem + Lay::kTDS, tmem + Lay::kTAK + 8 * k,
                                    desc_kmajor_sw128(bk + (k >> 2) * (N * 128) + (k & 3) * 32), kIdesc, k > 0 ? 1u : 0u);
                    umma_commit(sFull);
                }
                __syncwarp();
                stamp(b, 64, 4, 1);
                const bool first = cc.seg_first(start);
                mbar_wait_sleep(opV, ph);
                tc_fence_after();
                stamp(b, 64, 4, 2);
                if (lane == 0) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        umma_f16_ts(tmem + Lay::kTDO, tmem + Lay::kTAV + 8 * k,
                                    desc_kmajor_sw128(bv + (k >> 2) * (N * 128) + (k & 3) * 32), kIdesc,
                                    (k > 0 || !first) ? 1u : 0u);
                    umma_commit(pvDone);
                }
                __syncwarp();
                stamp(b, 64, 4, 3);
                cc.next();
            }
        }
    } else if (active) {
        // ================= compute warpgroup =================
        const int q = warp & 3;              // TMEM lane quarter: tokens / channels 32q .. 32q + 31
        const int t = 32 * q + lane;         // token of the batch (S rows) / channel (O rows)
        const int gid = lane >> 2, tig = lane & 3;
        const int G = P.group;
        const float sl2 = P.scale_log2;
        const float sk = kTwo24 * sl2;
        const int wbar = 1 + wg;             // named barrier of this warpgroup
        __half* sP = reinterpret_cast<__half*>(sw + Lay::kP);
        __half* sQsl = reinterpret_cast<__half*>(sw + Lay::kQsl);
        __half* sQsc = reinterpret_cast<__half*>(sw + Lay::kQsc);
        float* sKb = reinterpret_cast<float*>(sw + Lay::kKb);
        float* sRed = reinterpret_cast<float*>(sw + Lay::kRed);
        float* sDvb = reinterpret_cast<float*>(sw + Lay::kDvb);
        int* sFlag = reinterpret_cast<int*>(sw + Lay::kFlag);
        uint8_t* sBK = sw + Lay::kBK;
        uint8_t* sBV = sw + Lay::kBV;
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;

        if (!P.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
        Cursor cc;
        cc.init(P.rec, P.n_units, __shfl_sync(0xffffffffu, __ldg(P.wstart + worker), 0), start, end);
        float m[GP], l[GP];
        float dvb[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        uint32_t qa[2][2];  // key-bias A fragments of channel chunks 2q, 2q+1 (q * scale_log2; rows = heads)
        int seg_batches = 0;
        for (int b = 0; cc.valid(); ++b) {
            const int s = b % kTcStages;
            const uint32_t ph = b & 1;
            const uint8_t* stage = sw + Lay::kRing + s * kStageBytes;
            const int unit = cc.unit;
            const int n_real = cc.n_real();
            const int pfirst = cc.pg - cc.pbeg;
            const bool first = cc.seg_first(start), last = cc.seg_last();
            if (first) {
                // ---- segment start: stage q (this unit, G heads) ----
                named_bar_sync(wbar, 128);  // the previous segment's readers of q are done
                const int c = t;            // thread = channel
#pragma unroll
                for (int h = 0; h < GP; ++h) {
                    __half qv = __float2half(0.0f);
                    if (h < G) qv = P.q[((size_t)unit * G + h) * kHeadDim + c];
                    sQsl[h * kHeadDim + c] = __hmul(qv, __float2half(sl2));
                    sQsc[h * kHeadDim + 16 * (c >> 4) + kpos(c & 15)] = __hmul(qv, __float2half(pow4_neg(code_class(c >> 4))));
                    m[h] = -INFINITY;
                    l[h] = 0.0f;
                }
                dvb[0] = dvb[1] = dvb[2] = dvb[3] = 0.0f;
                seg_batches = 0;
                named_bar_sync(wbar, 128);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int kc = 2 * q + e;
                    qa[e][0] = gid < GP ? *reinterpret_cast<const uint32_t*>(sQsl + gid * kHeadDim + 16 * kc + 2 * tig) : 0u;
                    qa[e][1] = gid < GP ? *reinterpret_cast<const uint32_t*>(sQsl + gid * kHeadDim + 16 * kc + 2 * tig + 8) : 0u;
                }
            }
            const int tb = q < 2 ? 32 * q : -1000;  // trace base of compute warps 0 and 1
            if (q < 2) stamp(b, tb, 8, 0);
            mbar_wait(&full[s], (b / kTcStages) & 1);
            if (q < 2) stamp(b, tb, 8, 1);

            // ---- K codes -> TMEM A_K (this warp's pages 2q, 2q+1; lanes = tokens) ----
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const uint4 kw = lds128(stage + (2 * q + jj) * kPgStride + kKC + lane * 16);
                uint32_t r[32];
#pragma unroll
                for (int kc = 0; kc < 8; ++kc) {
                    const int sh = code_shift(kc);
                    const uint32_t mask = 0x00030003u << (2 * code_class(kc));
                    r[4 * kc + 0] = (kw.x >> sh) & mask;  // a0
                    r[4 * kc + 1] = (kw.z >> sh) & mask;  // a2
                    r[4 * kc + 2] = (kw.y >> sh) & mask;  // a1
                    r[4 * kc + 3] = (kw.w >> sh) & mask;  // a3
                }
                tmem_st_16x256_x8(tmem + lane_base + ((uint32_t)(16 * jj) << 16) + Lay::kTAK, r);
            }
            // ---- B_K[(j, h)][kk] = q_h[c] 4^-cls(c) s_j[c]  (K order) ----
#pragma unroll
            for (int it = 0; it < N * 16 / 128; ++it) {
                const int task = it * 128 + t;
                const int n = task >> 4, cg = task & 15;  // row, 16-byte chunk (8 K entries)
                const int j = n / GP, h = n % GP;
                const int kc = cg >> 1, hb = cg & 1;
                const uint4 qv = lds128(reinterpret_cast<const uint8_t*>(sQsc + h * kHeadDim + 8 * cg));
                const uint8_t* ks = stage + j * kPgStride + kKS + ((((kc >> 1) * 4 + 2 * hb) * 2 + (kc & 1)) * 4) * 2;
                const uint2 s0 = lds64(ks), s1 = lds64(ks + 16);
                uint4 o;
                o.x = hmul2_u32(qv.x, s0.x);
                o.y = hmul2_u32(qv.y, s0.y);
                o.z = hmul2_u32(qv.z, s1.x);
                o.w = hmul2_u32(qv.w, s1.y);
                *reinterpret_cast<uint4*>(sBK + bk_off<N>(n, 8 * cg)) = o;
            }
            // ---- key bias Kb[j][h] = sum_c z_j[c] q_h[c] sl2: warp q sums channel chunks 2q, 2q+1 of
            //      all 8 pages (mma.sync, rows = heads, columns = pages) -> partial sKb[q] ----
            {
                float kb[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int kc = 2 * q + e;
                    const uint2 z = lds64(stage + gid * kPgStride + kKZ + (q * 4 + tig) * 16 + e * 8);
                    const uint32_t a[4] = {qa[e][0], 0u, qa[e][1], 0u};
                    (void)kc;
                    mma_16816(kb, a, z.x, z.y);
                }
                if (gid < GP) {  // row = head gid, columns = pages 2 tig, 2 tig + 1
                    sKb[(q * 8 + 2 * tig) * GP + gid] = kb[0];
                    sKb[(q * 8 + 2 * tig + 1) * GP + gid] = kb[1];
                }
            }
            tmem_wait_st();
            fence_proxy_async_smem();
            tc_fence_before();
            if (q < 2) stamp(b, tb, 8, 2);
            mbar_arrive(opK);

            // ---- V codes -> TMEM A_V (groups 2q, 2q+1; lanes = channels), after the previous PV ----
            if (b > 0) mbar_wait(pvDone, (b - 1) & 1);
            switch (q) {
                case 0: store_v_codes<0>(stage, lane, tmem + lane_base + Lay::kTAV); break;
                case 1: store_v_codes<1>(stage, lane, tmem + lane_base + Lay::kTAV); break;
                case 2: store_v_codes<2>(stage, lane, tmem + lane_base + Lay::kTAV); break;
                default: store_v_codes<3>(stage, lane, tmem + lane_base + Lay::kTAV); break;
            }

            // ---- scores of this thread's token ----
            if (q < 2) stamp(b, tb, 8, 3);
            mbar_wait(sFull, ph);
            tc_fence_after();
            if (q < 2) stamp(b, tb, 8, 4);
            uint32_t sr[2 * GP];
            tmem_ld_32x32<2 * GP>(tmem + lane_base + Lay::kTDS + GP * 2 * q, sr);
            tmem_wait_ld();
            named_bar_sync(wbar, 128);  // sKb visible
            const int j = t >> 4, i = t & 15;
            const int n_prefill = __shfl_sync(0xffffffffu, __ldg(&P.rec[unit].n_prefill), 0);
            const int partial_page = (n_prefill & 15) ? ((n_prefill + 15) >> 4) - 1 : -1;
            const bool tok_ok = j < n_real && !(pfirst + j == partial_page && i >= (n_prefill & 15));
            float x[GP];
            bool grow = false;
#pragma unroll
            for (int h = 0; h < GP; ++h) {
                const float sv = __uint_as_float((lane >> 4) ? sr[GP + h] : sr[h]);
                const float kbias = sKb[(0 * 8 + j) * GP + h] + sKb[(1 * 8 + j) * GP + h] + sKb[(2 * 8 + j) * GP + h] +
                                    sKb[(3 * 8 + j) * GP + h];
                x[h] = (tok_ok && h < G) ? fmaf(sv, sk, kbias) : -INFINITY;
                grow |= x[h] > m[h] + kLazy;
            }
            // ---- lazy online softmax: a new max only when some head grows by > 2^kLazy ----
            const unsigned any = __ballot_sync(0xffffffffu, grow);
            if (lane == 0) sFlag[q] = any != 0u;
            named_bar_sync(wbar, 128);
            if (__shfl_sync(0xffffffffu, sFlag[0] | sFlag[1] | sFlag[2] | sFlag[3], 0)) {
                float bm[GP];
#pragma unroll
                for (int h = 0; h < GP; ++h) {
                    float v = x[h];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
                    bm[h] = v;
                }
                named_bar_sync(wbar, 128);  // every thread has read sFlag
                if (lane == 0)
#pragma unroll
                    for (int h = 0; h < GP; ++h) sRed[q * GP + h] = bm[h];
                named_bar_sync(wbar, 128);
                float alpha[GP];
                bool rescale = false;
#pragma unroll
                for (int h = 0; h < GP; ++h) {
                    const float mx = fmaxf(fmaxf(sRed[h], sRed[GP + h]), fmaxf(sRed[2 * GP + h], sRed[3 * GP + h]));
                    const float mn = fmaxf(m[h], mx);
                    alpha[h] = (mn == -INFINITY) ? 1.0f : exp2f(m[h] - mn);
                    rescale |= mn > m[h] && m[h] != -INFINITY;
                    m[h] = mn;
                    l[h] *= alpha[h];
                }
                if (rescale && seg_batches > 0) {
                    // O (TMEM, thread = channel) *= alpha after the previous PV completed
                    mbar_wait(pvDone, (b - 1) & 1);
                    tc_fence_after();
                    uint32_t orr[2 * GP];
                    const uint32_t oaddr = tmem + lane_base + Lay::kTDO + GP * 2 * q;
                    tmem_ld_32x32<2 * GP>(oaddr, orr);
                    tmem_wait_ld();
#pragma unroll
                    for (int h = 0; h < GP; ++h) {  // only this channel's group block is meaningful
                        orr[h] = __float_as_uint(__uint_as_float(orr[h]) * alpha[h]);
                        orr[GP + h] = __float_as_uint(__uint_as_float(orr[GP + h]) * alpha[h]);
                    }
                    tmem_st_32x32<2 * GP>(oaddr, orr);
                    tmem_wait_st();
                }
                // value-bias accumulator fragment: d[0] = (group gid, head 2 tig), d[1] = (gid, 2 tig + 1)
                if (2 * tig < GP) dvb[0] *= alpha[2 * tig];
                if (2 * tig + 1 < GP) dvb[1] *= alpha[2 * tig + 1];
            } else {
                named_bar_sync(wbar, 128);  // keep the barrier count uniform: every thread has read sFlag
            }
            // ---- probabilities ----
            {
                __half* pc = sP + 16 * j + kpos(i);
#pragma unroll
                for (int h = 0; h < GP; ++h) {
                    const float p = h < G ? fast_exp2(x[h] - m[h]) : 0.0f;
                    l[h] += p;
                    pc[h * 128] = __float2half_rn(p);
                }
            }
            named_bar_sync(wbar, 128);  // p complete
            if (q < 2) stamp(b, tb, 8, 5);
            // ---- B_V[(g, h)][kk] = p_h[t] sV[t][g]  (K = tokens in K order) ----
#pragma unroll
            for (int it = 0; it < N * 16 / 128; ++it) {
                const int task = it * 128 + t;
                const int n = task % N, cg = task / N;  // rows fastest: one (page, half) per 32 rows
                const int g = n / GP, h = n % GP;
                const int jp = cg >> 1, hb = cg & 1;
                const uint4 pv = lds128(reinterpret_cast<const uint8_t*>(sP + h * 128 + 8 * cg));
                const uint8_t* vs = stage + jp * kPgStride + kVS + (((((g >> 1) * 4 + 2 * hb) * 2 + (g & 1)) * 4) * 2);
                const uint2 s0 = lds64(vs), s1 = lds64(vs + 16);
                uint4 o;
                o.x = hmul2_u32(pv.x, s0.x);
                o.y = hmul2_u32(pv.y, s0.y);
                o.z = hmul2_u32(pv.z, s1.x);
                o.w = hmul2_u32(pv.w, s1.y);
                *reinterpret_cast<uint4*>(sBV + bk_off<N>(n, 8 * cg)) = o;
            }
#ifdef MKV_TC_TRACE_FINE
            if (q < 2) stamp(b, tb, 8, 6);
#endif
            // ---- value bias Vb[g][h] += sum_t zV[t][g] p_h[t] (this warp's pages; mma.sync) ----
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const int jp = 2 * q + jj;
                const uint2 vz = lds64(stage + jp * kPgStride + kVZ + lane * 8);
                const uint32_t a[4] = {vz.x, 0u, vz.y, 0u};
                const uint2 pb = gid < GP ? lds64(reinterpret_cast<const uint8_t*>(sP + gid * 128 + 16 * jp + 4 * tig))
                                          : make_uint2(0u, 0u);
                mma_16816(dvb, a, pb.x, pb.y);
            }
            tmem_wait_st();
            fence_proxy_async_smem();
#ifdef MKV_TC_TRACE_FINE
            if (q < 2) stamp(b, tb, 8, 7);
#endif
            tc_fence_before();
            mbar_arrive(opV);
            mbar_arrive(&empty[s]);
#ifndef MKV_TC_TRACE_FINE
            if (q < 2) stamp(b, tb, 8, 6);
#endif
            ++seg_batches;

            if (last) {
                // ---- segment epilogue: partial (m, l, o) for slot (worker, unit) ----
                float lt[GP];
#pragma unroll
                for (int h = 0; h < GP; ++h) {
                    float v = l[h];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    lt[h] = v;
                }
                named_bar_sync(wbar, 128);  // sRed / sDvb free
                if (lane == 0)
#pragma unroll
                    for (int h = 0; h < GP; ++h) sRed[q * GP + h] = lt[h];
                if (gid < 8) {
                    if (2 * tig < GP) sDvb[(q * 8 + gid) * GP + 2 * tig] = dvb[0];
                    if (2 * tig + 1 < GP) sDvb[(q * 8 + gid) * GP + 2 * tig + 1] = dvb[1];
                }
                mbar_wait(pvDone, ph);
                tc_fence_after();
                uint32_t orr[2 * GP];
                tmem_ld_32x32<2 * GP>(tmem + lane_base + Lay::kTDO + GP * 2 * q, orr);
                tmem_wait_ld();
                named_bar_sync(wbar, 128);
                const int slot = worker + unit;  // the finish kernel's slot of (worker, local unit)
                float* pml = P.part_ml + (size_t)slot * 2 * kMaxG;
                float* po = P.part_o + (size_t)slot * kMaxG * kHeadDim;
                const int c = t, g = c >> 4;
                const float f = kTwo24 * pow4_neg(code_class(g));
#pragma unroll
                for (int h = 0; h < GP; ++h) {
                    if (h < G) {
                        const float vb = sDvb[(0 * 8 + g) * GP + h] + sDvb[(1 * 8 + g) * GP + h] +
                                         sDvb[(2 * 8 + g) * GP + h] + sDvb[(3 * 8 + g) * GP + h];
                        po[h * kHeadDim + c] = fmaf(__uint_as_float((lane >> 4) ? orr[GP + h] : orr[h]), f, vb);
                        if (t == 0) {
                            pml[h] = m[h];
                            pml[kMaxG + h] = sRed[h] + sRed[GP + h] + sRed[2 * GP + h] + sRed[3 * GP + h];
                        }
                    }
                }
            }
#ifndef MKV_TC_TRACE_FINE
            if (q < 2) stamp(b, tb, 8, 7);
#endif
            cc.next();
        }
    }
    if (P.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    tc_fence_before();
    __syncthreads();
    if (warp == 8) tmem_dealloc(*tmem_word, 512);
}

template <int GP>
static cudaError_t launch_tc_t(const PagesParams& p, int grid, cudaStream_t s, bool pdl) {
    const size_t smem = TcLayout<GP>::kSmem;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(pages_tc_kernel<GP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kTcWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    count_launch(1);
    return cudaLaunchKernelEx(&cfg, pages_tc_kernel<GP>, p);
}

cudaError_t launch_pages_tc(const PagesParams& p, int grid, cudaStream_t s, bool pdl) {
    if (p.group <= 4) return launch_tc_t<4>(p, grid, s, pdl);
    return launch_tc_t<8>(p, grid, s, pdl);
}

}  // namespace mkv
