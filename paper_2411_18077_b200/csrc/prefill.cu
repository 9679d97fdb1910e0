// prefill.cu -- K1: two-pass selective flash-attention prefill on tcgen05.
//
// Restates selective_flash_attn (attention.cpp:29-117) for [B, H, L, 128]
// fp16 tensors with GQA:
//   pass 1  attn_fwd_kernel   one CTA per (pair of 128-query tiles, q-head, batch):
//           online softmax over 128-key tiles -> X_O (fp16) and LSE (fp32,
//           natural log, attention.cpp:98).  S = Q K^T and O += P V are
//           tcgen05.mma (M = N = 128, K = 16 steps) with K/V staged by TMA
//           (SWIZZLE_128B, shared by both query tiles) and S / O in TMEM; the two
//           tiles ping-pong (one's MMAs run under the other's softmax) and P is
//           written back over S in TMEM as the A operand of P V (TS-MMA).
//   pass 2  acumul_kernel     one CTA per (128-key block, kv-head, batch): the
//           paper's column-parallel pass.  S^T = K_blk Q^T
//           is recomputed on tcgen05 into TMEM, each thread owns ONE key row and
//           sums exp(s - lse_q) over every visible query of every q-head of its
//           kv-head, in a fixed order -> A_cumul[b, kv-head, key] with no atomics
//           and memory linear in L (LSE + A_cumul only).
// Causal convention: query i sees keys 0 .. lk - lq + i (attention.cpp:42,60);
// masked pairs contribute exactly 0.
//
// Warp roles: pass 1 (320 threads) -- warps 0-3 / 4-7 softmax of query tile A / B
// (thread = TMEM lane = row), warp 8 TMA producer, warp 9 TMEM allocator +
// single-thread MMA issuer; pass 2 (448 threads) -- warps 0-11 three exp warpgroups
// taking query tiles round-robin (thread = key row, one 128-column S^T buffer each, the
// key block held in TMEM as the A operand), warp 12 TMA, warp 13 MMA.
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include <type_traits>

#include "mkv_kernels.h"
#include "mkv_sm100.cuh"

namespace mkv {

using namespace sm100;

namespace {

constexpr int kTile = 128;
constexpr int kHalf = kTile * 128;   // one [128 rows x 64 fp16] swizzled TMA box = 16 KB
constexpr int kTileB = 2 * kHalf;    // [128 x 128] fp16 tile = 32 KB
constexpr uint32_t kIdescS = idesc_f16(128, 128, false);   // S = A[K-major] * B[K-major]
constexpr uint32_t kIdescPV = idesc_f16(128, 128, true);   // O += P[K-major] * V[MN-major]
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;  // lazy rescale (log2 units): P <= 2^8 in fp16

// slot c of every 8 exponentials runs on the FMA pipe when it is one of kPoly spread slots
template <int kPoly>
__host__ __device__ constexpr bool poly_slot(int c) {
    return kPoly <= 0 ? false : ((c & 7) * kPoly) % 8 + kPoly >= 8;
}

// pair p of every 4 exponential PAIRS runs on the FMA pipe when it is one of kPoly spread slots
template <int kPoly>
__host__ __device__ constexpr bool poly_pair(int p) {
    return kPoly <= 0 ? false : ((p & 3) * kPoly) % 4 + kPoly >= 4;
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// k-th K=16 slice of a K-major [128 x 128] fp16 tile made of two 64-column swizzled halves
__device__ __forceinline__ uint64_t kslice(const uint8_t* tile, int k) {
    return desc_kmajor_sw128(smem_u32(tile + (k >> 2) * kHalf + (k & 3) * 32));
}

// exp2 on the FMA pipe (offloads the MUFU unit): round-to-nearest split x = j + f,
// f in [-0.5, 0.5], 2^f by a degree-4 polynomial (rel. err < 5e-5), 2^j into the exponent.
__device__ __forceinline__ float exp2_fma(float x) {
    x = fmaxf(x, -127.0f);
    const float xr = x + 12582912.0f;  // 1.5 * 2^23: rounds x to an integer in the low mantissa bits
    const float f = x - (xr - 12582912.0f);
    float p = fmaf(0.0096181291f, f, 0.0555041087f);
    p = fmaf(p, f, 0.2402265070f);
    p = fmaf(p, f, 0.6931471806f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + ((__float_as_int(xr) - 0x4B400000) << 23));
}

// Two exp2's on the FMA pipe with packed fp32 (FADD2 / FFMA2: one issue slot per PAIR).
// Same split and polynomial as exp2_fma.  2^j goes into the exponent with one shift-add
// per element: bits(xr) = 0x4B400000 + j and (0x4B400000 << 23) == 0 mod 2^32, so
// bits(2^j * p) = bits(p) + (bits(xr) << 23).
__device__ __forceinline__ float2 exp2_fma2(float2 x) {
    x.x = fmaxf(x.x, -127.0f);  // ALU pipe
    x.y = fmaxf(x.y, -127.0f);
    const float2 xr = __fadd2_rn(x, make_float2(12582912.0f, 12582912.0f));
    const float2 t = __fadd2_rn(xr, make_float2(-12582912.0f, -12582912.0f));
    const float2 f = __ffma2_rn(t, make_float2(-1.0f, -1.0f), x);  // x - t, exact
    float2 p = __ffma2_rn(make_float2(0.0096181291f, 0.0096181291f), f, make_float2(0.0555041087f, 0.0555041087f));
    p = __ffma2_rn(p, f, make_float2(0.2402265070f, 0.2402265070f));
    p = __ffma2_rn(p, f, make_float2(0.6931471806f, 0.6931471806f));
    p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(xr.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(xr.y) << 23)));
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

// ---------------------------------------------------------------------------
// pass 1
// ---------------------------------------------------------------------------
// Two query tiles (A, B) per CTA ping-pong on the tensor core (FA4-style): while
// warpgroup A runs softmax on S_A(j), the MMA warp computes P_B(j-1)V / S_B(j)
// and vice versa.  K/V tiles are loaded once for both query tiles.  P never
// touches shared memory: softmax writes fp16 P over the first 64 TMEM columns
// of its own S buffer and the PV product reads A from TMEM.
// TMEM (512 cols): tile h: S_h / P_h at 256h, O_h at 256h + 128.
struct FwdBars {
    uint64_t q_full, kv_full[2], kv_empty[2], s_full[2], p_full[2], o_full[2];
    uint32_t tmem;
};
constexpr int kFwdThreads = 320;  // warps 0-3 softmax A, 4-7 softmax B, 8 TMA, 9 MMA
constexpr int kFwdSmem = 6 * kTileB + 1024 + 256;  // Q[2], K[2], V[2] + alignment slack + barriers

__device__ __forceinline__ float fmax3(float a, float b, float c) {  // FMNMX3 (sm_100)
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

template <int kPoly>
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const PrefillAttnParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = align1024(smem_raw);
    uint8_t* sQ = sm;                // 2 query tiles
    uint8_t* sK = sm + 2 * kTileB;   // 2 stages
    uint8_t* sV = sm + 4 * kTileB;   // 2 stages
    FwdBars& B = *reinterpret_cast<FwdBars*>(sm + 6 * kTileB);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_qt = (P.lq + kTile - 1) / kTile;
    const int n_pairs = (n_qt + 1) / 2;
    // grid (hq * batch, n_pairs): every head's longest causal pair is scheduled before any
    // head's next one (longest-processing-time-first across the whole grid)
    const int pair = n_pairs - 1 - blockIdx.y;
    const int hq = blockIdx.x % P.hq, b = blockIdx.x / P.hq;
    const int G = P.hq / P.hkv;
    const int hk = hq / G;
    const int offset = P.causal ? P.lk - P.lq : 0;
    // per query tile h: first row, number of KV tiles it needs
    int q0[2], nkv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int qt = 2 * pair + h;
        q0[h] = qt * kTile;
        if (qt < n_qt) {
            const int last_row = min(q0[h] + kTile, P.lq) - 1;
            const int kmax = P.causal ? min(P.lk - 1, offset + last_row) : P.lk - 1;
            nkv[h] = kmax / kTile + 1;
        } else {
            nkv[h] = 0;
        }
    }
    const int nmax = max(nkv[0], nkv[1]);

    if (warp == 9) {
        tmem_alloc(&B.tmem, 512);
        tmem_relinquish();
    }
    if (tid == 256) {
        mbar_init(&B.q_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&B.kv_full[s], 1);
            mbar_init(&B.kv_empty[s], 1);
            mbar_init(&B.s_full[s], 1);
            mbar_init(&B.p_full[s], 128);
            mbar_init(&B.o_full[s], 1);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tq);
        tma_prefetch_desc(&tk);
        tma_prefetch_desc(&tv);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = B.tmem;

    if (warp == 8) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            const int ntiles = nkv[1] > 0 ? 2 : 1;
            mbar_expect_tx(&B.q_full, ntiles * kTileB);
            tma_load_4d(sQ, &tq, 0, q0[0], hq, b, &B.q_full);
            tma_load_4d(sQ + kHalf, &tq, 64, q0[0], hq, b, &B.q_full);
            if (ntiles == 2) {
                tma_load_4d(sQ + kTileB, &tq, 0, q0[1], hq, b, &B.q_full);
                tma_load_4d(sQ + kTileB + kHalf, &tq, 64, q0[1], hq, b, &B.q_full);
            }
            for (int j = 0; j < nmax; ++j) {
                const int s = j & 1;
                if (j >= 2) mbar_wait(&B.kv_empty[s], ((j >> 1) - 1) & 1);
                mbar_expect_tx(&B.kv_full[s], 2 * kTileB);
                uint8_t* k_dst = sK + s * kTileB;
                uint8_t* v_dst = sV + s * kTileB;
                tma_load_4d(k_dst, &tk, 0, j * kTile, hk, b, &B.kv_full[s]);
                tma_load_4d(k_dst + kHalf, &tk, 64, j * kTile, hk, b, &B.kv_full[s]);
                tma_load_4d(v_dst, &tv, 0, j * kTile, hk, b, &B.kv_full[s]);
                tma_load_4d(v_dst + kHalf, &tv, 64, j * kTile, hk, b, &B.kv_full[s]);
            }
        }
    } else if (warp == 9) {
        // ---------------- MMA issuer (one thread) ----------------
        if (lane == 0) {
            auto issue_s = [&](int h, int j) {  // S_h = Q_h K_j^T  (M = N = 128, 8 K-steps)
                const uint8_t* k = sK + (j & 1) * kTileB;
                const uint8_t* q = sQ + h * kTileB;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_f16(tmem + 256 * h, kslice(q, kk), kslice(k, kk), kIdescS, kk > 0 ? 1u : 0u);
                umma_commit(&B.s_full[h]);
            };
            auto issue_pv = [&](int h, int j) {  // O_h += P_h V_j, P from TMEM (16 keys = 8 columns)
                const uint8_t* v = sV + (j & 1) * kTileB;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_f16_ts(tmem + 256 * h + 128, tmem + 256 * h + 8 * kk,
                                desc_mnmajor_sw128(smem_u32(v + kk * 2048), kHalf), kIdescPV,
                                (j > 0 || kk > 0) ? 1u : 0u);
            };
            mbar_wait(&B.q_full, 0);
            mbar_wait(&B.kv_full[0], 0);
            tc_fence_after();
            issue_s(0, 0);
            if (nkv[1] > 0) issue_s(1, 0);
            for (int j = 0; j < nmax; ++j) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (j >= nkv[h]) continue;
                    mbar_wait(&B.p_full[h], j & 1);
                    tc_fence_after();
                    issue_pv(h, j);
                    if (j + 1 < nkv[h]) {
                        mbar_wait(&B.kv_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
                        tc_fence_after();
                        issue_s(h, j + 1);  // in-order tensor pipe: overwrites S_h/P_h after PV_h(j) read it
                    } else {
                        umma_commit(&B.o_full[h]);
                    }
                }
                umma_commit(&B.kv_empty[j & 1]);
            }
        }
    } else {
        // ---------------- softmax warpgroups: thread = query row of tile h ----------------
        const int h = warp >> 2;
        const int r = tid & 127;
        const int row_g = (h ? q0[1] : q0[0]) + r;
        const int n = h ? nkv[1] : nkv[0];
        const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 256 * h;
        const float sl2 = P.scale * kLog2e;
        const int lim = P.causal ? min(P.lk - 1, offset + row_g) : P.lk - 1;
        float m = -INFINITY, l = 0.0f;
        for (int j = 0; j < n; ++j) {
            mbar_wait(&B.s_full[h], j & 1);  // also implies PV_h(j-1) completed (commit order)
            tc_fence_after();
#ifdef MKV_AB_MMA_ONLY  // A/B probe (tools/abbuild_prefill.sh): the MMA / TMA pipeline without the softmax
            tc_fence_before();
            mbar_arrive(&B.p_full[h]);
            continue;
#endif
            // one TMEM read of the 128 scores; P is packed in place over x (x[c/2] <- c, c+1)
            uint32_t x[128];
            tmem_ld32(trow + 0, *reinterpret_cast<uint32_t(*)[32]>(x + 0));
            tmem_ld32(trow + 32, *reinterpret_cast<uint32_t(*)[32]>(x + 32));
            tmem_ld32(trow + 64, *reinterpret_cast<uint32_t(*)[32]>(x + 64));
            tmem_ld32(trow + 96, *reinterpret_cast<uint32_t(*)[32]>(x + 96));
            tmem_wait_ld();
            const int cut = lim - j * kTile;  // columns c > cut are masked
            const bool nomask = __all_sync(0xffffffffu, cut >= kTile - 1);
            float mt = -INFINITY;
            if (!nomask) {
#pragma unroll
                for (int c = 0; c < 128; ++c)
                    if (c > cut) x[c] = __float_as_uint(-INFINITY);
            }
            {  // row max with the 3-input FMNMX3 (half the max instructions), 4 chains
                float mc[4] = {__uint_as_float(x[0]), __uint_as_float(x[1]), __uint_as_float(x[2]), __uint_as_float(x[3])};
#pragma unroll
                for (int c = 4; c < 128; c += 8) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) mc[k] = fmax3(mc[k], __uint_as_float(x[c + 2 * k]), __uint_as_float(x[c + 2 * k + 1]));
                }
                mt = fmax3(fmaxf(mc[0], mc[1]), mc[2], mc[3]);
            }
            mt *= sl2;
            const float m_new = fmaxf(m, mt);
            float alpha = 1.0f;
            bool rescale = false;
            if (m == -INFINITY) {
                m = m_new;  // nothing accumulated yet for this row (all earlier P were 0)
            } else if (m_new > m + kRescaleThreshold) {
                alpha = fast_exp2(m - m_new);
                m = m_new;
                l *= alpha;
                rescale = true;
            }
            // P = 2^(s*scale*log2e - m) -> fp16 pairs packed in place, then written over S in TMEM
            float ls = 0.0f;
#pragma unroll
            for (int cc = 0; cc < 128; cc += 2) {
                const float a0 = fmaf(__uint_as_float(x[cc]), sl2, -m), a1 = fmaf(__uint_as_float(x[cc + 1]), sl2, -m);
                const float p0 = poly_slot<kPoly>(cc) ? exp2_fma(a0) : fast_exp2(a0);
                const float p1 = poly_slot<kPoly>(cc + 1) ? exp2_fma(a1) : fast_exp2(a1);
                ls += p0 + p1;
                x[cc >> 1] = pack_half2(p0, p1);
            }
            tmem_st32(trow + 0, *reinterpret_cast<uint32_t(*)[32]>(x + 0));
            tmem_st32(trow + 32, *reinterpret_cast<uint32_t(*)[32]>(x + 32));
            // O_h is stable (PV_h(j-1) done, PV_h(j) not issued yet); rescale after P is out of registers; tcgen05.ld/st are warp-collective
            if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    uint32_t o[32];
                    tmem_ld32(trow + 128 + 32 * cc, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                    tmem_st32(trow + 128 + 32 * cc, o);
                }
            }
            l += ls;
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&B.p_full[h]);
        }
        // ---------------- epilogue ----------------
        if (n > 0) {
            mbar_wait(&B.o_full[h], 0);
            tc_fence_after();
            const float inv = 1.0f / l;
            const bool valid = row_g < P.lq;
            __half* orow = P.out + (size_t)b * P.o_sb + (size_t)hq * P.o_sh + (size_t)row_g * P.o_st;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                uint32_t o[32];
                tmem_ld32(trow + 128 + 32 * cc, o);
                tmem_wait_ld();
                if (valid) {
#pragma unroll
                    for (int e = 0; e < 32; e += 8) {
                        uint4 v;
                        v.x = pack_half2(__uint_as_float(o[e]) * inv, __uint_as_float(o[e + 1]) * inv);
                        v.y = pack_half2(__uint_as_float(o[e + 2]) * inv, __uint_as_float(o[e + 3]) * inv);
                        v.z = pack_half2(__uint_as_float(o[e + 4]) * inv, __uint_as_float(o[e + 5]) * inv);
                        v.w = pack_half2(__uint_as_float(o[e + 6]) * inv, __uint_as_float(o[e + 7]) * inv);
                        *reinterpret_cast<uint4*>(orow + 32 * cc + e) = v;
                    }
                }
            }
            if (valid) P.lse[((size_t)b * P.hq + hq) * P.lq + row_g] = (m + __log2f(l)) * kLn2;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------------------
// pass 2: column-parallel A_cumul
// ---------------------------------------------------------------------------
constexpr int kQStages = 4;
constexpr int kAcWG = 3;                           // exp warpgroups: item it goes to warpgroup it % kAcWG
constexpr int kAcThreads = kAcWG * 128 + 64;       // + TMA warp + MMA warp
constexpr int kAcTma = kAcWG * 4, kAcMma = kAcWG * 4 + 1;
// The key block is the A operand of every S^T MMA of the CTA: it is copied once into TMEM
// (columns kAcKCol .. + 63, fp16 pairs, lane = key row) so the MMAs read only the Q tile from
// shared memory -- an SS MMA at M = N = 128 reads 8 KB of shared memory per 64-clk K step, the
// whole 128 B/clk, a TS MMA half of it.
constexpr int kAcKCol = 128 * kAcWG;
// kNB = kAcWG (default): one S^T buffer per warpgroup, the key block in TMEM (TS MMAs).
// kNB = 4 (MKV_ACUMUL_BUFS=4, A/B): the key block stays in shared memory (SS MMAs) and its 64
// TMEM columns become a fourth S^T buffer -- a ring of 4 buffers over the 3 warpgroups, so the
// MMA of item it + 1 may run while every warpgroup still holds its current S^T.
constexpr int kAcMaxBufs = 4;
static_assert(kAcKCol + 64 <= 512 && 128 * kAcMaxBufs <= 512, "TMEM: S^T buffers + key block");
struct AcBars {
    uint64_t k_full, k_tmem, q_full[kQStages], q_empty[kQStages], s_full[kAcMaxBufs], s_free[kAcMaxBufs];
    uint32_t tmem;
    alignas(16) float lse2[kAcWG][2][kTile];  // [warpgroup][item parity][query], -lse*log2e (ld.shared.v4)
    float part[kAcWG - 1][kTile];             // partial sums of warpgroups 1..
};
constexpr int kAcSmem = (1 + kQStages) * kTileB + 1024 + (int)sizeof(AcBars) + 64;

// item -> (q-head g of the kv-head, query tile t); items run g-major from the block's first
// visible query tile.  Advanced incrementally (no integer division per item).
struct ItemPos {
    int g, t;
    __device__ __forceinline__ void advance(int by, int t_first, int n_qt) {
        t += by;
        while (t >= n_qt) {
            t -= n_qt - t_first;
            ++g;
        }
    }
};

// kPoly of every 4 exponential PAIRS run as a polynomial on the FMA pipe (FFMA2, the rest
// on MUFU.EX2).  Per element the pass costs 1 exponential + half an FFMA2 + half an FADD2.
// kDirect (MKV_ACUMUL_LSE=direct, A/B; needs lq % 4 == 0): every thread reads the item's 128
// LSE values straight from global memory (L1 broadcast, ld.global.nc.v4) instead of the
// warpgroup staging them in shared memory behind a named barrier per item.
template <int kPoly, int kNB, bool kDirect = false>
__global__ void __launch_bounds__(kAcThreads, 1)
    acumul_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                  const PrefillAttnParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = align1024(smem_raw);
    uint8_t* sK = sm;
    uint8_t* sQ = sm + kTileB;  // kQStages stages
    AcBars& B = *reinterpret_cast<AcBars*>(sm + (1 + kQStages) * kTileB);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // grid (hkv * batch, n_kt): key block 0 (seen by every query) of every head first -- the
    // causal work per CTA falls with kt, so this is longest-processing-time-first
    const int kt = blockIdx.y, hk = blockIdx.x % P.hkv, b = blockIdx.x / P.hkv;
    const int G = P.hq / P.hkv;
    const int key0 = kt * kTile;
    const int offset = P.causal ? P.lk - P.lq : 0;
    const int n_qt = (P.lq + kTile - 1) / kTile;
    const int i_min = P.causal ? max(0, key0 - offset) : 0;  // first query that sees any key of the block
    const int t_first = i_min / kTile;
    const int per_head = n_qt - t_first;
    const int n_items = G * per_head;

    if (warp == kAcMma) {
        tmem_alloc(&B.tmem, 512);
        tmem_relinquish();
    }
    if (tid == kAcTma * 32) {
        mbar_init(&B.k_full, 1);
        mbar_init(&B.k_tmem, 128);
        for (int s = 0; s < kQStages; ++s) {
            mbar_init(&B.q_full[s], 1);
            mbar_init(&B.q_empty[s], 1);
        }
        for (int s = 0; s < kNB; ++s) {
            mbar_init(&B.s_full[s], 1);
            mbar_init(&B.s_free[s], 128);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tq);
        tma_prefetch_desc(&tk);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = B.tmem;

    if (warp == kAcTma) {
        if (lane == 0) {
            mbar_expect_tx(&B.k_full, kTileB);
            tma_load_4d(sK, &tk, 0, key0, hk, b, &B.k_full);
            tma_load_4d(sK + kHalf, &tk, 64, key0, hk, b, &B.k_full);
            ItemPos pos{0, t_first};
            for (int it = 0; it < n_items; ++it, pos.advance(1, t_first, n_qt)) {
                const int s = it % kQStages;
                if (it >= kQStages) mbar_wait(&B.q_empty[s], ((it / kQStages) - 1) & 1);
                const int hq = hk * G + pos.g;
                mbar_expect_tx(&B.q_full[s], kTileB);
                tma_load_4d(sQ + s * kTileB, &tq, 0, pos.t * kTile, hq, b, &B.q_full[s]);
                tma_load_4d(sQ + s * kTileB + kHalf, &tq, 64, pos.t * kTile, hq, b, &B.q_full[s]);
            }
        }
    } else if (warp == kAcMma) {
        if (lane == 0) {
            if constexpr (kNB == kAcWG)
                mbar_wait(&B.k_tmem, 0);  // the key block is in TMEM (A operand of every S^T MMA)
            else
                mbar_wait(&B.k_full, 0);
            for (int it = 0; it < n_items; ++it) {
                // S^T(item) = K_blk Q_t^T into TMEM buffer it % kNB.  (Split into two N = 64
                // halves with their own barriers it measured 1.46x slower.)
                const int s = it % kQStages, bb = it % kNB;
                mbar_wait(&B.q_full[s], (it / kQStages) & 1);
                if (it >= kNB) mbar_wait(&B.s_free[bb], ((it / kNB) - 1) & 1);
                tc_fence_after();
                const uint8_t* q = sQ + s * kTileB;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    if constexpr (kNB == kAcWG)  // A = K_blk from TMEM (8 columns = 16 d per step), B = Q tile
                        umma_f16_ts(tmem + 128 * bb, tmem + kAcKCol + 8 * kk, kslice(q, kk), kIdescS, kk > 0 ? 1u : 0u);
                    else
                        umma_f16(tmem + 128 * bb, kslice(sK, kk), kslice(q, kk), kIdescS, kk > 0 ? 1u : 0u);
                }
                umma_commit(&B.s_full[bb]);
                umma_commit(&B.q_empty[s]);
            }
        }
    } else {
        // warpgroup wg handles items it = wg, wg + kAcWG, ...; thread = key row; each
        // warpgroup accumulates in a fixed order and the partial sums are added in a fixed order.
        const int wg = warp >> 2;
        const int kr = tid & 127;
        const int kj = key0 + kr;
        const uint32_t trow0 = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        const float sl2 = P.scale * kLog2e;
        // the LSE of the query row this thread stages is loaded one item ahead: its global
        // latency hides behind the current item's exponentials (consumed only at the next one)
        const float* lse_b = P.lse + ((size_t)b * P.hq + hk * G) * P.lq;
        auto load_lse = [&](int item, const ItemPos& ps) -> float {
            const int i = ps.t * kTile + kr;
            return (item < n_items && i < P.lq) ? __ldg(lse_b + (size_t)ps.g * P.lq + i) : INFINITY;
        };
        // packed fp32: one FFMA2 per 2 scores (s * scale*log2e - lse*log2e), one FADD2 per 2
        // exponentials into four pair accumulators
        const float2 s2 = make_float2(sl2, sl2);
        float2 a0 = make_float2(0.0f, 0.0f), a1 = a0, a2 = a0, a3 = a0;
        if (kNB == kAcWG && wg == 0) {
            // key row kr (SW128 tile: two 64-column halves, 16-byte chunk c of row r at
            // r * 128 + ((c ^ (r & 7)) << 4)) -> TMEM lane kr, columns kAcKCol + d / 2
            mbar_wait(&B.k_full, 0);
            uint32_t kv[64];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf)
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    *reinterpret_cast<uint4*>(kv + 32 * hf + 4 * c) =
                        *reinterpret_cast<const uint4*>(sK + hf * kHalf + kr * 128 + ((c ^ (kr & 7)) << 4));
            const uint32_t tk = tmem + ((uint32_t)((warp & 3) * 32) << 16) + kAcKCol;
            tmem_st32(tk, *reinterpret_cast<uint32_t(*)[32]>(kv));
            tmem_st32(tk + 32, *reinterpret_cast<uint32_t(*)[32]>(kv + 32));
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&B.k_tmem);
        }
        ItemPos pos{0, t_first};
        pos.advance(wg, t_first, n_qt);
        ItemPos nxt = pos;
        nxt.advance(kAcWG, t_first, n_qt);
        float lse_next = load_lse(wg, pos);
        for (int it = wg, k = 0; it < n_items; it += kAcWG, ++k) {
            float* l2 = B.lse2[wg][k & 1];
            const float* lrow = lse_b + (size_t)pos.g * P.lq + (size_t)pos.t * kTile;
            if constexpr (!kDirect) {
                l2[kr] = lse_next * -kLog2e;  // INFINITY -> -inf: masked rows add exact zeros
                named_bar_sync(1 + wg, 128);
                lse_next = load_lse(it + kAcWG, nxt);
            }
            const int t = pos.t;
            const int c_lim = P.lq - t * kTile;  // columns >= c_lim are past the last query
            pos = nxt;
            nxt.advance(kAcWG, t_first, n_qt);
            const uint32_t l2a = smem_u32(l2);
            const int bb = it % kNB;
            const uint32_t trow = trow0 + 128 * bb;
            mbar_wait(&B.s_full[bb], (it / kNB) & 1);
            tc_fence_after();
            // query i = t*128 + c visible iff kj <= offset + i  <=>  c >= kj - offset - t*128
            const int c_min = P.causal ? (kj - offset - t * kTile) : -1;
            const bool full = __all_sync(0xffffffffu, c_min <= 0) && (!kDirect || c_lim >= kTile);
            // the two loops differ only in the causal mask (diagonal items): separate copies keep
            // the full-tile loop free of per-column compares
            auto tile = [&](auto masked) {
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    uint32_t x[64];
                    tmem_ld32(trow + 64 * half, *reinterpret_cast<uint32_t(*)[32]>(x));
                    tmem_ld32(trow + 64 * half + 32, *reinterpret_cast<uint32_t(*)[32]>(x + 32));
                    tmem_wait_ld();
                    if (half == 1) {
                        tc_fence_before();
                        mbar_arrive(&B.s_free[bb]);  // TMEM buffer free for the next MMA into it
                    }
#pragma unroll
                    for (int c = 0; c < 64; c += 4) {
                        float4 nl;
                        if constexpr (kDirect) {
                            const int col = 64 * half + c;
                            const float4 lv = (!decltype(masked)::value || col < c_lim)
                                                  ? __ldg(reinterpret_cast<const float4*>(lrow + col))
                                                  : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                            const float2 m2 = make_float2(-kLog2e, -kLog2e);
                            const float2 n0 = __fmul2_rn(make_float2(lv.x, lv.y), m2);
                            const float2 n1 = __fmul2_rn(make_float2(lv.z, lv.w), m2);
                            nl = make_float4(n0.x, n0.y, n1.x, n1.y);
                        } else {
                            nl = lds128(l2a + (64 * half + c) * 4);
                        }
                        const float2 v0 = __ffma2_rn(make_float2(__uint_as_float(x[c]), __uint_as_float(x[c + 1])),
                                                     s2, make_float2(nl.x, nl.y));
                        const float2 v1 = __ffma2_rn(
                            make_float2(__uint_as_float(x[c + 2]), __uint_as_float(x[c + 3])), s2,
                            make_float2(nl.z, nl.w));
                        float2 e0 = poly_pair<kPoly>(c >> 1) ? exp2_fma2(v0)
                                                              : make_float2(fast_exp2(v0.x), fast_exp2(v0.y));
                        float2 e1 = poly_pair<kPoly>((c >> 1) + 1) ? exp2_fma2(v1)
                                                                    : make_float2(fast_exp2(v1.x), fast_exp2(v1.y));
                        if constexpr (decltype(masked)::value) {
                            const int col = 64 * half + c;
                            const int lo = c_min, hi = kDirect ? c_lim : kTile;  // visible: lo <= col < hi
                            e0.x = (col >= lo && col < hi) ? e0.x : 0.0f;
                            e0.y = (col + 1 >= lo && col + 1 < hi) ? e0.y : 0.0f;
                            e1.x = (col + 2 >= lo && col + 2 < hi) ? e1.x : 0.0f;
                            e1.y = (col + 3 >= lo && col + 3 < hi) ? e1.y : 0.0f;
                        }
                        if ((c & 4) == 0) {
                            a0 = __fadd2_rn(a0, e0);
                            a1 = __fadd2_rn(a1, e1);
                        } else {
                            a2 = __fadd2_rn(a2, e0);
                            a3 = __fadd2_rn(a3, e1);
                        }
                    }
                }
            };
            if (full)
                tile(std::false_type{});
            else
                tile(std::true_type{});
        }
        const float acc = ((a0.x + a1.x) + (a0.y + a1.y)) + ((a2.x + a3.x) + (a2.y + a3.y));
        if (wg > 0) B.part[wg - 1][kr] = acc;
        named_bar_sync(1 + kAcWG, kAcWG * 128);
        if (wg == 0 && kj < P.lk) {
            float sum = acc;
#pragma unroll
            for (int w = 1; w < kAcWG; ++w) sum += B.part[w - 1][kr];
            P.a_cumul[((size_t)b * P.hkv + hk) * P.lk + kj] = sum;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kAcMma) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------------------
// host: TMA descriptors + launches
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 get_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

bool make_map(CUtensorMap* m, const __half* base, int64_t sb, int64_t sh, int64_t st, int L, int H, int Bn) {
    auto enc = get_encoder();
    if (!enc) return false;
    cuuint64_t dims[4] = {128, (cuuint64_t)L, (cuuint64_t)H, (cuuint64_t)Bn};
    cuuint64_t strides[3] = {(cuuint64_t)st * 2, (cuuint64_t)sh * 2, (cuuint64_t)sb * 2};
    cuuint32_t box[4] = {64, 128, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<__half*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace

template <int KF, int KA, int NB = kAcWG, bool DIRECT = false>
static cudaError_t launch_prefill_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                                   const PrefillAttnParams& p, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<KF>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(acumul_kernel<KA, NB, DIRECT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kAcSmem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int n_qt = (p.lq + kTile - 1) / kTile, n_kt = (p.lk + kTile - 1) / kTile;
    attn_fwd_kernel<KF><<<dim3(p.hq * p.batch, (n_qt + 1) / 2), kFwdThreads, kFwdSmem, s>>>(tq, tk, tv, p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    acumul_kernel<KA, NB, DIRECT><<<dim3(p.hkv * p.batch, n_kt), kAcThreads, kAcSmem, s>>>(tq, tk, p);
    return cudaGetLastError();
}

cudaError_t launch_prefill_attn(const PrefillAttnParams& p, cudaStream_t s) {
    CUtensorMap tq, tk, tv;
    if (!make_map(&tq, p.q, p.q_sb, p.q_sh, p.q_st, p.lq, p.hq, p.batch) ||
        !make_map(&tk, p.k, p.k_sb, p.k_sh, p.k_st, p.lk, p.hkv, p.batch) ||
        !make_map(&tv, p.v, p.v_sb, p.v_sh, p.v_st, p.lk, p.hkv, p.batch))
        return cudaErrorInvalidValue;
    // exponentials on the FMA pipe: fwd per 8, A_cumul pairs per 4; MKV_PREFILL_POLY="f,a"
    // default: no pass-1 exponentials on the FMA pipe (since the FMNMX3 row max the softmax
    // warps' issue slots, not MUFU, bound pass 1: 0 of 8 measured 1-2.5% faster than 1 of 8),
    // one A_cumul exponential pair in four
    static int kf = 0, ka = 1, nb = kAcWG;
    static bool direct = false;
    static bool parsed = false;
    if (!parsed) {
        if (const char* e = getenv("MKV_PREFILL_POLY")) sscanf(e, "%d,%d", &kf, &ka);
        if (const char* e = getenv("MKV_ACUMUL_BUFS")) nb = atoi(e);
        if (const char* e = getenv("MKV_ACUMUL_LSE")) direct = e[0] == 'd';
        parsed = true;
    }
    if (direct && kf == 0 && ka == 1 && nb == kAcWG && p.lq % 4 == 0)
        return launch_prefill_t<0, 1, kAcWG, true>(tq, tk, tv, p, s);
    if (nb == 4 && kf == 0 && ka == 1) return launch_prefill_t<0, 1, 4>(tq, tk, tv, p, s);
    if (kf == 1 && ka == 1) return launch_prefill_t<1, 1>(tq, tk, tv, p, s);
    if (kf == 1 && ka == 0) return launch_prefill_t<1, 0>(tq, tk, tv, p, s);
    if (kf == 1 && ka == 2) return launch_prefill_t<1, 2>(tq, tk, tv, p, s);
    if (kf == 2 && ka == 1) return launch_prefill_t<2, 1>(tq, tk, tv, p, s);
    return launch_prefill_t<0, 1>(tq, tk, tv, p, s);
}

}  // namespace mkv