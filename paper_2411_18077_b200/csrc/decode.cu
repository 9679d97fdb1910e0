// decode.cu -- K4: fused unpack-and-multiply 2-bit decode attention.
//
// Restates decode_step (cache_engine.cpp:100-138) for a batch of units with
// GQA: append the new token (flushing a full n_r residual block to 2-bit pages
// first, cache_engine.cpp:79-90), then ONE softmax over
// [dequant(K_q) ; R_K] and out = attn . [dequant(V_q) ; R_V].
//
// Two kernels per call:
//   residual_kernel  one CTA per unit: append (+flush via the K3 page builder),
//                    attention over the fp16 residual -> partial (m, l, o)
//   pages_kernel     persistent, 8 warps/CTA, each warp an independent worker
//                    over a contiguous range of the global page sequence; pages
//                    stream HBM -> smem with cp.async.bulk (3-stage ring per
//                    warp), are dequantized in registers and multiplied on the
//                    tensor cores (mma.sync m16n8k16) -> per-(warp, unit)
//                    partials; the last warp to finish a unit merges all
//                    partials (split-K / flash-decoding combine) into out.
//
// Dequantization never materialises fp16 K/V: the 2-bit code is extracted
// into an fp16 *subnormal* (code * 4^s * 2^-24) with one LOP3, the per-channel
// key scale is folded into the query fragment, the per-token value scale into
// the probability fragment, and the zero points enter through one extra mma
// per page (sum_c q_c z_c for keys, sum_t p_t z_t for values).  See DESIGN.md.
#include <math.h>

#include "mkv_kernels.h"
#include "mkv_page.cuh"

namespace mkv {

namespace {

constexpr int kStages = 3;
constexpr int kBatch = 4;  // pages per bulk copy / per K-bias mma
constexpr float kTwo24 = 16777216.0f;

__device__ __forceinline__ uint4 lds128(const uint8_t* p) {
    return *reinterpret_cast<const uint4*>(p);
}
__device__ __forceinline__ uint2 lds64(const uint8_t* p) {
    return *reinterpret_cast<const uint2*>(p);
}

// Binary search: largest i in [0, n) with pref[i] <= x.
__device__ __forceinline__ int find_unit(const int32_t* pref, int n, int x) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(pref + mid) <= x) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Merge every partial of local unit i (pages partial slots + residual) into out.
__device__ void merge_unit(const PagesParams& P, int i, int w_first, int w_last) {
    const int lane = lane_id();
    const int G = P.group;
    const float* rml = P.res_ml + (size_t)i * 2 * kMaxG;
    const float* ro = P.res_o + (size_t)i * kMaxG * kHeadDim;
    for (int h = 0; h < G; ++h) {
        float M = __ldcg(rml + h);
        for (int w = w_first; w <= w_last; ++w) {
            const float* ml = P.part_ml + (size_t)(w + i) * 2 * kMaxG;
            M = fmaxf(M, __ldcg(ml + h));
        }
        const float rs = (__ldcg(rml + kMaxG + h) > 0.0f) ? fast_exp2(__ldcg(rml + h) - M) : 0.0f;
        float L = __ldcg(rml + kMaxG + h) * rs;
        float4 acc = __ldcg(reinterpret_cast<const float4*>(ro + h * kHeadDim) + lane);
        acc.x *= rs; acc.y *= rs; acc.z *= rs; acc.w *= rs;
        for (int w = w_first; w <= w_last; ++w) {
            const float* ml = P.part_ml + (size_t)(w + i) * 2 * kMaxG;
            const float* po = P.part_o + (size_t)(w + i) * kMaxG * kHeadDim;
            const float sc = fast_exp2(__ldcg(ml + h) - M);
            L += __ldcg(ml + kMaxG + h) * sc;
            const float4 o = __ldcg(reinterpret_cast<const float4*>(po + h * kHeadDim) + lane);
            acc.x += o.x * sc; acc.y += o.y * sc; acc.z += o.z * sc; acc.w += o.w * sc;
        }
        const float inv = 1.0f / L;
        __half2 lo = __floats2half2_rn(acc.x * inv, acc.y * inv);
        __half2 hi = __floats2half2_rn(acc.z * inv, acc.w * inv);
        uint2 st;
        st.x = *reinterpret_cast<uint32_t*>(&lo);
        st.y = *reinterpret_cast<uint32_t*>(&hi);
        reinterpret_cast<uint2*>(P.out + ((size_t)i * G + h) * kHeadDim)[lane] = st;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// pages kernel
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kPagesWarps * 32, 1) pages_kernel(const PagesParams P) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int gid = lane >> 2, tig = lane & 3;
    uint8_t* ring = smem + (size_t)warp * kStages * kBatch * kPageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kPagesWarps * kStages * kBatch * kPageBytes) +
                     warp * kStages;

    const int wg = blockIdx.x * kPagesWarps + warp;
    const int start = wg * P.chunk;
    const int end = min(start + P.chunk, P.total_pages);
    if (start >= end) return;

    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();

    // ---- producer cursor (warp-uniform) ----
    int pi = find_unit(P.pref, P.n_units, start);
    int pg = start;
    auto issue = [&](int stage) {
        // next batch: [pg, pg + n) inside unit pi
        if (pg >= end) return;
        const int uend = __ldg(P.pref + pi + 1);
        const int n = min(min(kBatch, uend - pg), end - pg);
        if (lane == 0) {
            const UnitMeta& m = P.meta[P.unit_begin + pi];
            const uint8_t* src = P.pool + (size_t)(m.page_base + (pg - __ldg(P.pref + pi))) * kPageBytes;
            mbar_expect_tx(&bars[stage], n * kPageBytes);
            bulk_g2s(ring + (size_t)stage * kBatch * kPageBytes, src, n * kPageBytes, &bars[stage]);
        }
        pg += n;
        if (pg == uend) ++pi;
    };
    for (int s = 0; s < kStages; ++s) issue(s);

    // ---- consumer state ----
    int ci = find_unit(P.pref, P.n_units, start);
    int cg = start;
    int stage = 0;
    uint32_t phase = 0;
    const int G = P.group;
    const float sl2 = P.scale_log2;
    const float sk = kTwo24 * sl2;

    while (cg < end) {
        // ---- new unit segment: load query fragments ----
        const int unit = ci;
        const int upre = __ldg(P.pref + unit);
        const int uend_g = __ldg(P.pref + unit + 1);
        const int seg_end = min(uend_g, end);
        const UnitMeta meta = P.meta[P.unit_begin + unit];
        const int prefill_pages = (meta.n_prefill + 15) >> 4;
        const int partial_valid = meta.n_prefill & 15;  // 0 -> last prefill page is full

        uint32_t qb[8][2], qs[8][2];
        {
            const __half* qh = P.q + ((size_t)unit * G + gid) * kHeadDim;
#pragma unroll
            for (int kc = 0; kc < 8; ++kc) {
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    uint32_t v = 0;
                    if (gid < G) v = *reinterpret_cast<const uint32_t*>(qh + 16 * kc + 2 * tig + 8 * p);
                    qb[kc][p] = v;
                    // fold 4^-(kc mod 3) (the code-extraction scale) into the query
                    const float f = (kc % 3 == 0) ? 1.0f : ((kc % 3 == 1) ? 0.25f : 0.0625f);
                    const uint32_t fs = pack_half2(f, f);
                    qs[kc][p] = hmul2_u32(v, fs);
                }
            }
        }
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
        float O[8][4];
#pragma unroll
        for (int g = 0; g < 8; ++g) O[g][0] = O[g][1] = O[g][2] = O[g][3] = 0.0f;
        float Dvb[4] = {0.0f, 0.0f, 0.0f, 0.0f};

        while (cg < seg_end) {
            const int n = min(min(kBatch, uend_g - cg), end - cg);
            const int pfirst = cg - upre;  // local page index within the unit
            mbar_wait(&bars[stage], phase);
            const uint8_t* buf = ring + (size_t)stage * kBatch * kPageBytes;

            // K zero-point bias for the batch: Kb[page][h] = sum_c z[page][c] q[h][c]
            float Kb[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            {
                uint4 z[4];
                if (gid < n) {
                    const uint8_t* zp = buf + gid * kPageBytes + kKZ + tig * 64;
#pragma unroll
                    for (int j = 0; j < 4; ++j) z[j] = lds128(zp + 16 * j);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) z[j] = make_uint4(0, 0, 0, 0);
                }
                const uint32_t* zz = reinterpret_cast<const uint32_t*>(z);
#pragma unroll
                for (int kc = 0; kc < 8; ++kc) {
                    const uint32_t a[4] = {zz[2 * kc], 0u, zz[2 * kc + 1], 0u};
                    mma_16816(Kb, a, qb[kc][0], qb[kc][1]);
                }
            }

            for (int j = 0; j < n; ++j) {
                const uint8_t* page = buf + j * kPageBytes;
                const int lp = pfirst + j;
                // ---- scores S[t][h] = sum_c code[t][c] * q''[h][c] ----
                const uint4 kw = lds128(page + kKC + lane * 16);
                uint4 ksv[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) ksv[r] = lds128(page + kKS + tig * 64 + 16 * r);
                const uint32_t* ks = reinterpret_cast<const uint32_t*>(ksv);  // [kc][p]
                const uint32_t w0[4] = {kw.x, kw.y, kw.z, kw.w};
                const uint32_t w6[4] = {kw.x >> 6, kw.y >> 6, kw.z >> 6, kw.w >> 6};
                const uint32_t w12[4] = {kw.x >> 12, kw.y >> 12, kw.z >> 12, kw.w >> 12};
                float S[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int kc = 0; kc < 8; ++kc) {
                    const uint32_t* src = (kc < 3) ? w0 : ((kc < 6) ? w6 : w12);
                    const uint32_t mask = 0x00030003u << (2 * (kc % 3));
                    const uint32_t a[4] = {src[0] & mask, src[1] & mask, src[2] & mask, src[3] & mask};
                    const uint32_t b0 = hmul2_u32(qs[kc][0], ks[2 * kc]);
                    const uint32_t b1 = hmul2_u32(qs[kc][1], ks[2 * kc + 1]);
                    mma_16816(S, a, b0, b1);
                }
                const float kb0 = __shfl_sync(0xffffffffu, Kb[0], 4 * j + tig);
                const float kb1 = __shfl_sync(0xffffffffu, Kb[1], 4 * j + tig);
                float x0 = fmaf(S[0], sk, kb0 * sl2);
                float x1 = fmaf(S[1], sk, kb1 * sl2);
                float x2 = fmaf(S[2], sk, kb0 * sl2);
                float x3 = fmaf(S[3], sk, kb1 * sl2);
                if (partial_valid != 0 && lp == prefill_pages - 1) {
                    if (gid >= partial_valid) { x0 = -INFINITY; x1 = -INFINITY; }
                    if (gid + 8 >= partial_valid) { x2 = -INFINITY; x3 = -INFINITY; }
                }
                // ---- online softmax (log2 domain) ----
                float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) {
                    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
                    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
                }
                const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
                if (__any_sync(0xffffffffu, (mn0 != m0) | (mn1 != m1))) {
                    const float a0 = fast_exp2(m0 - mn0), a1 = fast_exp2(m1 - mn1);
                    l0 *= a0; l1 *= a1;
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        O[g][0] *= a0; O[g][1] *= a1; O[g][2] *= a0; O[g][3] *= a1;
                    }
                    Dvb[0] *= a0; Dvb[1] *= a1;
                    m0 = mn0; m1 = mn1;
                }
                const float p0 = fast_exp2(x0 - m0), p1 = fast_exp2(x1 - m1);
                const float p2 = fast_exp2(x2 - m0), p3 = fast_exp2(x3 - m1);
                l0 += p0 + p2;
                l1 += p1 + p3;
                const uint32_t pb0 = movmatrix_trans(pack_half2(p0, p1));
                const uint32_t pb1 = movmatrix_trans(pack_half2(p2, p3));
                // ---- value zero-point bias: Dvb[g][h] += sum_t z[t][g] p[h][t] ----
                {
                    const uint2 vz = lds64(page + kVZ + lane * 8);
                    const uint32_t a[4] = {vz.x, 0u, vz.y, 0u};
                    mma_16816(Dvb, a, pb0, pb1);
                }
                // ---- O_g[c][h] += sum_t code[t][c] * p[h][t] * s[t][g] ----
                const uint4 vw = lds128(page + kVC + lane * 16);
                uint4 vsv[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) vsv[r] = lds128(page + kVS + tig * 64 + 16 * r);
                const uint32_t* vs = reinterpret_cast<const uint32_t*>(vsv);  // [g][pt]
                const uint32_t v0[4] = {vw.x, vw.y, vw.z, vw.w};
                const uint32_t v6[4] = {vw.x >> 6, vw.y >> 6, vw.z >> 6, vw.w >> 6};
                const uint32_t v12[4] = {vw.x >> 12, vw.y >> 12, vw.z >> 12, vw.w >> 12};
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const uint32_t* src = (g < 3) ? v0 : ((g < 6) ? v6 : v12);
                    const uint32_t mask = 0x00030003u << (2 * (g % 3));
                    const uint32_t a[4] = {src[0] & mask, src[1] & mask, src[2] & mask, src[3] & mask};
                    const uint32_t b0 = hmul2_u32(pb0, vs[2 * g]);
                    const uint32_t b1 = hmul2_u32(pb1, vs[2 * g + 1]);
                    mma_16816(O[g], a, b0, b1);
                }
            }
            __syncwarp();
            issue(stage);  // refill this stage with the batch kStages ahead
            cg += n;
            if (++stage == kStages) { stage = 0; phase ^= 1u; }
        }
        if (cg == uend_g) ++ci;

        // ---- segment epilogue: partial (m, l, o) for (warp wg, unit) ----
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
            const float f = kTwo24 * ((g % 3 == 0) ? 1.0f : ((g % 3 == 1) ? 0.25f : 0.0625f));
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
        __threadfence();
        __syncwarp();
        const int w_first = upre / P.chunk;
        const int w_last = (uend_g - 1) / P.chunk;
        int last = 0;
        if (lane == 0) {
            const int old = atomicAdd(P.counters + unit, 1);
            last = (old == w_last - w_first);
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
            __threadfence();
            merge_unit(P, unit, w_first, w_last);
            if (lane == 0) P.counters[unit] = 0;
        }
    }
}

cudaError_t launch_pages(const PagesParams& p, int grid, cudaStream_t s) {
    const size_t smem = (size_t)kPagesWarps * kStages * kBatch * kPageBytes +
                        (size_t)kPagesWarps * kStages * sizeof(uint64_t);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(pages_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    pages_kernel<<<grid, kPagesWarps * 32, smem, s>>>(p);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// residual kernel: append (+flush) and attention over the fp16 residual
// ---------------------------------------------------------------------------
constexpr int kResThreads = 256;
constexpr int kResRowStride = kHeadDim + 2;  // halves; odd word stride -> conflict-free row reads

struct ResSmem {
    union {
        PageScratch scratch[kResThreads / 32];
        struct {
            __half k[128][kResRowStride];
            __half v[128][kHeadDim];
            float q[kMaxG][kHeadDim];
            float s[kMaxG][128];
            float red[kMaxG][2];
        } att;
    };
};

__global__ void __launch_bounds__(kResThreads) residual_kernel(const ResidualParams P) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    ResSmem& S = *reinterpret_cast<ResSmem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
    const int i = blockIdx.x;
    const int u = P.unit_begin + i;
    const int d = kHeadDim;
    UnitMeta meta = P.meta[u];
    __half* rk = P.res_k + (size_t)u * P.n_r * d;
    __half* rv = P.res_v + (size_t)u * P.n_r * d;
    int n = meta.n_res;

    if (P.k_new) {  // decode_append (cache_engine.cpp:79-90)
        if (tid < 16) {
            reinterpret_cast<uint4*>(rk + (size_t)n * d)[tid] =
                reinterpret_cast<const uint4*>(P.k_new + (size_t)i * d)[tid];
        } else if (tid < 32) {
            reinterpret_cast<uint4*>(rv + (size_t)n * d)[tid - 16] =
                reinterpret_cast<const uint4*>(P.v_new + (size_t)i * d)[tid - 16];
        }
        ++n;
        __threadfence_block();
        __syncthreads();
    }
    const bool flush = (n == P.n_r);
    if (flush) {
        // quantize the full block into n_r/16 new pages (store_block, cache_engine.cpp:34-52)
        const int npg = P.n_r / kGroup;
        bool ok = true;
        for (int j = warp; j < npg; j += kResThreads / 32) {
            PageScratch& ps = S.scratch[warp];
            for (int e = lane; e < 16 * 16; e += 32) {
                const int r = e >> 4, c16 = e & 15;
                reinterpret_cast<uint4*>(ps.k[r])[c16] = reinterpret_cast<const uint4*>(rk + (size_t)(16 * j + r) * d)[c16];
                reinterpret_cast<uint4*>(ps.v[r])[c16] = reinterpret_cast<const uint4*>(rv + (size_t)(16 * j + r) * d)[c16];
            }
            __syncwarp();
            const int64_t page = meta.page_base + meta.n_pages + j;
            ok &= build_page(ps, 16, P.pool + (size_t)page * kPageBytes,
                             P.shadow ? P.shadow + (size_t)page * (kShadowBytes / 4) : nullptr);
        }
        if (!ok && lane == 0) atomicOr(P.status, kStatusNonFinite);
        __syncthreads();
        if (tid == 0) {
            P.meta[u].n_pages = meta.n_pages + npg;
            P.meta[u].n_res = 0;
        }
        meta.n_pages += npg;
        n = 0;
    } else if (P.k_new && tid == 0) {
        P.meta[u].n_res = n;
    }
    if (!P.attend) return;

    const int G = P.group;
    float* rml = P.res_ml + (size_t)i * 2 * kMaxG;
    float* ro = P.res_o + (size_t)i * kMaxG * d;
    if (n == 0) {  // empty residual: neutral partial
        if (tid < G) { rml[tid] = -INFINITY; rml[kMaxG + tid] = 0.0f; }
        for (int e = tid; e < G * d; e += kResThreads) ro[(e / d) * d + (e % d)] = 0.0f;
        return;
    }
    // stage residual rows and q
    for (int e = tid; e < n * 16; e += kResThreads) {
        const int r = e >> 4, c16 = e & 15;
        const uint4 kv = reinterpret_cast<const uint4*>(rk + (size_t)r * d)[c16];
        const uint32_t* kw = reinterpret_cast<const uint32_t*>(&kv);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&S.att.k[r][c16 * 8]);
        dst[0] = kw[0]; dst[1] = kw[1]; dst[2] = kw[2]; dst[3] = kw[3];
        reinterpret_cast<uint4*>(S.att.v[r])[c16] = reinterpret_cast<const uint4*>(rv + (size_t)r * d)[c16];
    }
    for (int e = tid; e < G * d; e += kResThreads)
        S.att.q[e / d][e % d] = __half2float(P.q[(size_t)i * G * d + e]);
    __syncthreads();
    // scores (log2 domain)
    for (int e = tid; e < n * G; e += kResThreads) {
        const int t = e / G, h = e % G;
        float acc = 0.0f;
        const __half2* kr = reinterpret_cast<const __half2*>(S.att.k[t]);
#pragma unroll 8
        for (int c2 = 0; c2 < d / 2; ++c2) {
            const float2 kf = __half22float2(kr[c2]);
            acc = fmaf(S.att.q[h][2 * c2], kf.x, acc);
            acc = fmaf(S.att.q[h][2 * c2 + 1], kf.y, acc);
        }
        S.att.s[h][t] = acc * P.scale_log2;
    }
    __syncthreads();
    if (warp < G) {  // per-head max / exp / sum
        const int h = warp;
        float mx = -INFINITY;
        for (int t = lane; t < n; t += 32) mx = fmaxf(mx, S.att.s[h][t]);
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float sum = 0.0f;
        for (int t = lane; t < n; t += 32) {
            const float p = fast_exp2(S.att.s[h][t] - mx);
            S.att.s[h][t] = p;
            sum += p;
        }
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) { S.att.red[h][0] = mx; S.att.red[h][1] = sum; }
    }
    __syncthreads();
    const bool final_out = (meta.n_pages == 0);
    for (int e = tid; e < G * (d / 2); e += kResThreads) {
        const int h = e / (d / 2), c2 = e % (d / 2);
        float a0 = 0.0f, a1 = 0.0f;
        for (int t = 0; t < n; ++t) {
            const float p = S.att.s[h][t];
            const float2 vf = __half22float2(reinterpret_cast<const __half2*>(S.att.v[t])[c2]);
            a0 = fmaf(p, vf.x, a0);
            a1 = fmaf(p, vf.y, a1);
        }
        if (final_out) {
            const float inv = 1.0f / S.att.red[h][1];
            reinterpret_cast<__half2*>(P.out + ((size_t)i * G + h) * d)[c2] = __floats2half2_rn(a0 * inv, a1 * inv);
        } else {
            ro[h * d + 2 * c2] = a0;
            ro[h * d + 2 * c2 + 1] = a1;
        }
    }
    if (tid < G) { rml[tid] = S.att.red[tid][0]; rml[kMaxG + tid] = S.att.red[tid][1]; }
}

cudaError_t launch_residual(const ResidualParams& p, cudaStream_t s) {
    const size_t smem = sizeof(ResSmem);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(residual_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    residual_kernel<<<p.n_units, kResThreads, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace mkv
