// mkv_page.cuh -- build one 16-token 2-bit page (K3 core), shared by the
// prefill quantizer and the decode-time residual flush.
//
// Restates append_block (quantizer.cpp:102-136) for one 16-token group:
//   keys   PerChannel: per channel, one group over the page's valid tokens
//   values PerToken:   per token, 8 groups of 16 channels
// with the exact fp32 arithmetic of quantize_group (quantizer.cpp:28-53), so
// codes are bit-identical to the reference; (scale, zero) are stored as fp16
// in the page (the paper's format) and optionally as fp32 in a
// shadow page for bit-exact export.
#pragma once

#include "mkv_common.cuh"

namespace mkv {

// Per-warp scratch for building one page.
struct PageScratch {
    __half k[16][kHeadDim];  // token rows (fp16 inputs, widened exactly to fp32)
    __half v[16][kHeadDim];
    uint8_t kc[16][kHeadDim];  // codes (t, c)
    uint8_t vc[16][kHeadDim];
    alignas(16) uint8_t page[kPageBytes];
};

// One warp.  `valid` tokens (1..16) of s.k / s.v are meaningful.  Writes the
// page to `dst` (global, 16-byte aligned) and, if non-null, fp32 params to
// `shadow`.  Returns (warp-uniform) false if any input was non-finite.
__device__ __forceinline__ bool build_page(PageScratch& s, int valid, uint8_t* __restrict__ dst,
                                           float* __restrict__ shadow) {
    const int lane = lane_id();
    __half* ks = reinterpret_cast<__half*>(s.page + kKS);
    __half* kz = reinterpret_cast<__half*>(s.page + kKZ);
    __half* vs = reinterpret_cast<__half*>(s.page + kVS);
    __half* vz = reinterpret_cast<__half*>(s.page + kVZ);
    bool finite = true;

    // keys: channel c = lane + 32 j
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
        const int c = lane + 32 * j;
        float vals[16];
        uint8_t codes[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) vals[t] = __half2float(s.k[t][c]);
        float sc, zp;
        finite &= quantize_group16(vals, valid, codes, &sc, &zp);
#pragma unroll
        for (int t = 0; t < 16; ++t) s.kc[t][c] = (t < valid) ? codes[t] : 0;
        ks[k_param_idx(c)] = __float2half_rn(sc);
        kz[k_param_idx(c)] = __float2half_rn(zp);
        if (shadow) {
            shadow[2 * c] = sc;
            shadow[2 * c + 1] = zp;
        }
    }
    // values: (token t, group g) = idx >> 3, idx & 7 with idx = lane + 32 j
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
        const int idx = lane + 32 * j, t = idx >> 3, g = idx & 7;
        float vals[16];
        uint8_t codes[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) vals[i] = __half2float(s.v[t][16 * g + i]);
        float sc = 0.0f, zp = 0.0f;
        if (t < valid) {
            finite &= quantize_group16(vals, 16, codes, &sc, &zp);
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) codes[i] = 0;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) s.vc[t][16 * g + i] = codes[i];
        vs[vs_param_idx(t, g)] = __float2half_rn(sc);
        vz[vz_param_idx(t, g)] = __float2half_rn(zp);
        if (shadow) {
            shadow[256 + 2 * (t * 8 + g)] = sc;
            shadow[256 + 2 * (t * 8 + g) + 1] = zp;
        }
    }
    __syncwarp();
    // pack: lane builds its 4 KC words and 4 VC words
    const int gid = lane >> 2, tig = lane & 3;
    uint32_t kw[4], vw[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int tt = r & 1, p = r >> 1;
        const int t = gid + 8 * tt;
        uint32_t w = 0;
#pragma unroll
        for (int kc = 0; kc < 8; ++kc) {
            const int c = 16 * kc + 2 * tig + 8 * p;
            w |= static_cast<uint32_t>(s.kc[t][c]) << (2 * kc);
            w |= static_cast<uint32_t>(s.kc[t][c + 1]) << (16 + 2 * kc);
        }
        kw[r] = w;
        const int cc = r & 1, pt = r >> 1;
        const int cin = gid + 8 * cc, tv = 2 * tig + 8 * pt;
        uint32_t u = 0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const int c = 16 * g + cin;
            u |= static_cast<uint32_t>(s.vc[tv][c]) << (2 * g);
            u |= static_cast<uint32_t>(s.vc[tv + 1][c]) << (16 + 2 * g);
        }
        vw[r] = u;
    }
    reinterpret_cast<uint4*>(s.page + kKC)[lane] = make_uint4(kw[0], kw[1], kw[2], kw[3]);
    reinterpret_cast<uint4*>(s.page + kVC)[lane] = make_uint4(vw[0], vw[1], vw[2], vw[3]);
    __syncwarp();
    // coalesced 2 KB write-out
    const uint4* src = reinterpret_cast<const uint4*>(s.page);
    uint4* out = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int i = 0; i < kPageBytes / 16 / 32; ++i) out[lane + 32 * i] = src[lane + 32 * i];
    __syncwarp();
    return __all_sync(0xffffffffu, finite);
}

// ---------------------------------------------------------------------------
// Prefill variant (K3): the page's 16 kept tokens are read straight from K/V in
// global memory -- keys as 64-byte coalesced column runs (lane = channel), values
// as 16-channel 32-byte runs (lane = (token, group)) -- so only codes and the page
// are staged (6 KB per warp instead of 14 KB: four times the resident warps to hide
// the gather latency).  Same arithmetic and layout as build_page.
// ---------------------------------------------------------------------------
struct PageScratchLite {
    uint8_t kc[16][kHeadDim];
    uint8_t vc[16][kHeadDim];
    alignas(16) uint8_t page[kPageBytes];
};

__device__ __forceinline__ bool build_page_gather(PageScratchLite& s, int valid, const __half* __restrict__ kbase,
                                                  int64_t k_st, const __half* __restrict__ vbase, int64_t v_st,
                                                  const int32_t* __restrict__ kept16, uint8_t* __restrict__ dst,
                                                  float* __restrict__ shadow) {
    const int lane = lane_id();
    __half* ks = reinterpret_cast<__half*>(s.page + kKS);
    __half* kz = reinterpret_cast<__half*>(s.page + kKZ);
    __half* vs = reinterpret_cast<__half*>(s.page + kVS);
    __half* vz = reinterpret_cast<__half*>(s.page + kVZ);
    bool finite = true;
    const int my_tok = lane < valid ? __ldg(kept16 + (lane & 15)) : 0;
    int64_t krow[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) krow[t] = (int64_t)__shfl_sync(0xffffffffu, my_tok, t) * k_st;
    // keys: channel c = lane + 32 j, its 16 tokens (PerChannel group)
#pragma unroll 1  // rolled: smaller code, fewer instruction-cache misses (measured 4-10% faster)
    for (int j = 0; j < 4; ++j) {
        const int c = lane + 32 * j;
        float vals[16];
        uint8_t codes[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) vals[t] = t < valid ? __half2float(__ldg(kbase + krow[t] + c)) : 0.0f;
        float sc, zp;
        finite &= quantize_group16(vals, valid, codes, &sc, &zp);
#pragma unroll
        for (int t = 0; t < 16; ++t) s.kc[t][c] = (t < valid) ? codes[t] : 0;
        ks[k_param_idx(c)] = __float2half_rn(sc);
        kz[k_param_idx(c)] = __float2half_rn(zp);
        if (shadow) {
            shadow[2 * c] = sc;
            shadow[2 * c + 1] = zp;
        }
    }
    // values: (token t, group g) = idx >> 3, idx & 7 with idx = lane + 32 j (PerToken groups)
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
        const int idx = lane + 32 * j, t = idx >> 3, g = idx & 7;
        float vals[16];
        uint8_t codes[16];
        float sc = 0.0f, zp = 0.0f;
        const int vt = __shfl_sync(0xffffffffu, my_tok, t);
        if (t < valid) {
            const uint4* src = reinterpret_cast<const uint4*>(vbase + (int64_t)vt * v_st + 16 * g);
            const uint4 a = __ldg(src), b = __ldg(src + 1);
            const __half2* h2a = reinterpret_cast<const __half2*>(&a);
            const __half2* h2b = reinterpret_cast<const __half2*>(&b);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 fa = __half22float2(h2a[e]), fb = __half22float2(h2b[e]);
                vals[2 * e] = fa.x; vals[2 * e + 1] = fa.y;
                vals[8 + 2 * e] = fb.x; vals[8 + 2 * e + 1] = fb.y;
            }
            finite &= quantize_group16(vals, 16, codes, &sc, &zp);
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) codes[i] = 0;
        }
        *reinterpret_cast<uint4*>(&s.vc[t][16 * g]) = *reinterpret_cast<const uint4*>(codes);
        vs[vs_param_idx(t, g)] = __float2half_rn(sc);
        vz[vz_param_idx(t, g)] = __float2half_rn(zp);
        if (shadow) {
            shadow[256 + 2 * (t * 8 + g)] = sc;
            shadow[256 + 2 * (t * 8 + g) + 1] = zp;
        }
    }
    __syncwarp();
    const int gid = lane >> 2, tig = lane & 3;
    uint32_t kw[4], vw[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int tt = r & 1, p = r >> 1;
        const int t = gid + 8 * tt;
        uint32_t w = 0;
#pragma unroll
        for (int kc = 0; kc < 8; ++kc) {
            const int c = 16 * kc + 2 * tig + 8 * p;
            w |= static_cast<uint32_t>(s.kc[t][c]) << (2 * kc);
            w |= static_cast<uint32_t>(s.kc[t][c + 1]) << (16 + 2 * kc);
        }
        kw[r] = w;
        const int cc = r & 1, pt = r >> 1;
        const int cin = gid + 8 * cc, tv = 2 * tig + 8 * pt;
        uint32_t u = 0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const int c = 16 * g + cin;
            u |= static_cast<uint32_t>(s.vc[tv][c]) << (2 * g);
            u |= static_cast<uint32_t>(s.vc[tv + 1][c]) << (16 + 2 * g);
        }
        vw[r] = u;
    }
    reinterpret_cast<uint4*>(s.page + kKC)[lane] = make_uint4(kw[0], kw[1], kw[2], kw[3]);
    reinterpret_cast<uint4*>(s.page + kVC)[lane] = make_uint4(vw[0], vw[1], vw[2], vw[3]);
    __syncwarp();
    const uint4* src = reinterpret_cast<const uint4*>(s.page);
    uint4* out = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int i = 0; i < kPageBytes / 16 / 32; ++i) out[lane + 32 * i] = src[lane + 32 * i];
    __syncwarp();
    return __all_sync(0xffffffffu, finite);
}

}  // namespace mkv
