// mkv_common.cuh -- shared device/host helpers for the MiniKV B200 kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "minikv_b200.h"

namespace mkv {

constexpr int kWarp = 32;
constexpr int kGroup = 16;  // quantization group = tokens per page (quantizer.hpp:23)

// ---------------------------------------------------------------------------
// Page layout (one 16-token page of one (seq, layer, kv-head) unit, d = 128).
// All offsets in bytes.  Lane L = 4*gid + tig is the mma.sync m16n8k16 lane.
//
//  KC  u32[32][4]    lane L word r = tt + 2p: token t = gid + 8tt; bits 2kc (lo)
//                    = code(t, 16kc + 2tig + 8p), bits 16 + 2kc (hi) = code(t, ch + 1)
//  KS  half2[4][4][2][2] (kc/2, tig, kc%2, p) = (scale[16kc+2tig+8p], scale[..+1])   K per-channel
//  KZ  same order, zero points      (a lane's (kc, kc+1) pair is one conflict-free 16-byte load)
//  VC  u32[32][4]    lane L word r = cc + 2pt: channel c = 16g + gid + 8cc, token
//                    t = 2tig + 8pt; bits 2g (lo) = code(t, c), bits 16 + 2g (hi) = code(t + 1, c)
//  VS  half2[4][4][2][2] (g/2, tig, g%2, pt) = (scale[t=2tig+8pt][g], scale[t+1][g])  V per-token
//  VZ  half2[8][4][2] (g, tig, pt) = (zero[2tig+8pt][g], zero[2tig+8pt+1][g])
//
// The reference stream (quantizer.cpp:102-136) is recovered by
// mkv_cache_export_reference; these indices are the single source of truth.
// ---------------------------------------------------------------------------
constexpr int kHeadDim = 128;
constexpr int kPageBytes = 16 * kHeadDim;  // 2048
constexpr int kKC = 0, kKS = 512, kKZ = 768, kVC = 1024, kVS = 1536, kVZ = 1792;
// fp32 shadow params (optional, for bit-exact export): per page
//   K: float2[128] (scale, zero) by channel; V: float2[16][8] by (token, group).
constexpr int kShadowBytes = 128 * 8 + 16 * 8 * 8;  // 2048

struct CodePos {
    int word;   // u32 index inside the KC or VC block
    int shift;  // bit position
};

__host__ __device__ inline CodePos k_code_pos(int t, int c) {
    const int kc = c >> 4, w = c & 15, p = w >> 3, tig = (w & 7) >> 1, e = w & 1;
    const int gid = t & 7, tt = t >> 3;
    return CodePos{(4 * gid + tig) * 4 + tt + 2 * p, 2 * kc + 16 * e};
}
__host__ __device__ inline CodePos v_code_pos(int t, int c) {
    const int g = c >> 4, cin = c & 15, gid = cin & 7, cc = cin >> 3;
    const int pt = t >> 3, w = t & 7, tig = w >> 1, e = w & 1;
    return CodePos{(4 * gid + tig) * 4 + cc + 2 * pt, 2 * g + 16 * e};
}
// half index (not byte) inside KS / KZ for channel c
__host__ __device__ inline int k_param_idx(int c) {
    const int kc = c >> 4, w = c & 15, p = w >> 3, tig = (w & 7) >> 1, e = w & 1;
    return (((((kc >> 1) * 4 + tig) * 2 + (kc & 1)) * 2 + p) * 2) + e;
}
// half index inside VS for (token t, group g)
__host__ __device__ inline int vs_param_idx(int t, int g) {
    const int pt = t >> 3, w = t & 7, tig = w >> 1, e = w & 1;
    return (((((g >> 1) * 4 + tig) * 2 + (g & 1)) * 2 + pt) * 2) + e;
}
// half index inside VZ for (token t, group g)
__host__ __device__ inline int vz_param_idx(int t, int g) {
    const int pt = t >> 3, w = t & 7, tig = w >> 1, e = w & 1;
    return ((g * 4 + tig) * 2 + pt) * 2 + e;
}

// ---------------------------------------------------------------------------
// Device-side cache metadata (one entry per unit).
// ---------------------------------------------------------------------------
struct UnitMeta {
    int64_t page_base;  // first page of this unit in the pool
    int32_t n_pages;    // pages written (prefill pages + flushed blocks)
    int32_t n_prefill;  // tokens in the prefill block (its last page may be partial)
    int32_t n_res;      // residual tokens
    int32_t cap_pages;
    int32_t n_built;    // 16-row groups of the residual block already quantized into their pages
                        // (pool pages n_pages .. n_pages + n_built - 1, not yet attended as pages:
                        // the flush makes them visible and builds only the rest); device-side only
};

// Device status word bits
constexpr uint32_t kStatusNonFinite = 1u;
constexpr uint32_t kStatusOverflow = 2u;
constexpr uint32_t kStatusMergeTimeout = 4u;  // a merge waited > ~1 s for its unit's arrivals (internal error)

#if defined(__CUDACC__)
// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mma_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
    return y;
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t hmul2_u32(uint32_t a, uint32_t b) {
    __half2 r = __hmul2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// mbarrier + bulk async copy (TMA 1-D bulk engine)
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra.uni DONE;\n"
        "bra.uni LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// as mbar_wait, but each try suspends the warp up to ~1 us until the phase completes (fewer
// spinning issue slots for waiters that are rarely on the critical path)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAITS:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000;\n"
        "@p bra.uni DONES;\n"
        "bra.uni LAB_WAITS;\n"
        "DONES:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Exact code thresholds of one quantization group (quantize_group, quantizer.cpp:28-53):
// scale = fl((hi - lo) / 3) and code = round_half_away(fl(fl(v - lo) / scale)), clamped to
// [0, 3].  fl(dv / sc) is monotone in dv, so code = #{k in 1..3 : dv >= T_k} with T_k the
// smallest float whose IEEE quotient reaches c = k - 0.5.  fl(y) >= c  <=>  y > m  or
// (y == m and c has an even mantissa -- 0.5, 1.5, 2.5 all do), m = the midpoint of c and its
// predecessor, so T_k = the smallest float >= m * sc, where m * sc (25 x 24 significant bits)
// is exact in double.  Returns false (and T = +inf: every code 0) when the scale is not a
// positive finite number (a constant group).
__device__ __forceinline__ bool group_thresholds(float lo, float hi, float* sc_out, float (&T)[3]) {
    const float sc = __fdiv_rn(__fsub_rn(hi, lo), 3.0f);
    const bool ok = sc > 0.0f && isfinite(sc);
    T[0] = T[1] = T[2] = INFINITY;
    if (ok && sc >= 0x1p-100f && sc <= 0x1p100f) {
        // fp32 only (no FP64): m_k = c_k - d_k with d_k = 2^-26, 2^-24, 2^-23; ds = sc * d_k is
        // exact, y = fma(c_k, sc, -ds) = fl(m_k * sc), r = fma(-c_k, sc, y) = y - c_k * sc
        // exactly, so y >= m_k * sc  <=>  r >= -ds.  Bit-identical to the double form below for
        // every scale in [2^-100, 2^100] (tools/threshold_fp32_check.c: all 5.0e9 (scale, k)).
        const float cs[3] = {0.5f, 1.5f, 2.5f}, ds_[3] = {0x1p-26f, 0x1p-24f, 0x1p-23f};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float ds = sc * ds_[k];
            const float y = __fmaf_rn(cs[k], sc, -ds);
            const float r = __fmaf_rn(-cs[k], sc, y);
            T[k] = (r >= -ds) ? y : __int_as_float(__float_as_int(y) + 1);
        }
    } else if (ok) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float c = static_cast<float>(k) + 0.5f;
            const double m = 0.5 * (static_cast<double>(nextafterf(c, 0.0f)) + static_cast<double>(c));
            const double prod = m * static_cast<double>(sc);  // exact
            float x = __double2float_rn(prod);
            if (static_cast<double>(x) < prod) x = nextafterf(x, INFINITY);
            T[k] = x;
        }
    }
    *sc_out = sc;
    return ok;
}

// Reference-exact group quantization of n (<= 16) fp32 values (quantizer.cpp:28-53):
// zero = min, scale = (max - min) / 3.0f (IEEE division), code = clamp(roundf((v-zero)/scale)).
// Returns false if a value is non-finite (the reference throws std::domain_error).
__device__ __forceinline__ bool quantize_group16(const float* v, int n, uint8_t* codes,
                                                 float* scale_out, float* zero_out) {
    // fixed 16-trip loops (entries past n are ignored / produce unused codes): the value and
    // code arrays stay in registers instead of local memory
    float lo = v[0], hi = v[0];
    bool finite = true;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        if (i < n) {
            const float x = v[i];
            finite &= isfinite(x);
            lo = (x < lo) ? x : lo;
            hi = (hi < x) ? x : hi;
        }
    }
    float sc, T[3];
    const bool thr_ok = group_thresholds(lo, hi, &sc, T);
    if (thr_ok) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float dv = __fsub_rn(v[i], lo);
            codes[i] = static_cast<uint8_t>((dv >= T[0]) + (dv >= T[1]) + (dv >= T[2]));
        }
    } else {  // scale 0 (constant group) -> codes 0; non-finite scale -> the reference's formula
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            uint8_t c = 0;
            if (sc > 0.0f) {
                float q = roundf(__fdiv_rn(__fsub_rn(v[i], lo), sc));
                c = static_cast<uint8_t>(q < 0.0f ? 0.0f : (q > 3.0f ? 3.0f : q));
            }
            codes[i] = c;
        }
    }
    *scale_out = sc;
    *zero_out = lo;
    return finite;
}
#endif  // __CUDACC__

}  // namespace mkv
