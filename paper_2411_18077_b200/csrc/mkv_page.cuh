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

// ---------------------------------------------------------------------------
// Staged variant (K3, round 2).  The page's 16 K rows and 16 V rows are first copied into
// shared memory (prefill: cp.async of the gathered kept rows, one round trip; rows past
// `valid` zero-filled), 16-byte chunks XOR-swizzled by row so that both read patterns below
// are bank-conflict-free.  Codes are then computed from fp16 PAIRS -- the pair a code word
// holds: two channels of one token for keys, two tokens of one channel for values -- with one
// packed fp32 subtraction (FADD2) and compares against the three exact thresholds
// (group_thresholds), and OR-ed straight into their fragment-order bit positions; the four
// lanes that hold parts of one word combine them through a 2 KB partial-word buffer.  No
// per-code byte staging, min / max on packed fp16 (HMNMX2, NaN-propagating), the code words
// are stored to global straight from registers.  Same codes and params as build_page.
// ---------------------------------------------------------------------------
struct PageRows {
    alignas(16) __half k[16 * kHeadDim];  // swizzled rows (stage_row_offset); after the keys are
                                          // coded, reused as the [4][128] partial code words
    alignas(16) __half v[16 * kHeadDim];
};
struct PageParams {
    alignas(16) uint8_t b[1024];  // KS | KZ | VS | VZ (page bytes 512..1023, 1536..2047)
};

// byte offset of 16-byte chunk `chunk` (0..15) of row t
__device__ __forceinline__ int stage_row_offset(int t, int chunk) { return t * 256 + ((chunk ^ (t & 7)) << 4); }

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
__device__ __forceinline__ __half2 u2h2(uint32_t x) { return *reinterpret_cast<__half2*>(&x); }

// (fl32(v.lo - lo.x), fl32(v.hi - lo.y)) of an fp16 pair: one mixed-precision subtraction each
// (FHADD: the fp16 operand is exact in fp32, one rounding)
__device__ __forceinline__ float2 sub_h2(uint32_t v, float2 lo) {
    float2 r;
    asm("{.reg .f16 l, h;\n mov.b32 {l, h}, %2;\n sub.rn.f32.f16 %0, l, %3;\n sub.rn.f32.f16 %1, h, %4;}"
        : "=f"(r.x), "=f"(r.y)
        : "r"(v), "f"(lo.x), "f"(lo.y));
    return r;
}

// code = #{k : dv >= T_k} (T_0 < T_1 < T_2, so the compares are nested): bit 1 = (dv >= T_1),
// bit 0 = (dv >= T_2) if bit 1 else (dv >= T_0) -- two compares; placed at the bits of mlo / mhi
__device__ __forceinline__ uint32_t code_bits(float dv, const float (&T)[3], uint32_t mlo, uint32_t mhi) {
    const bool hi = dv >= T[1];
    const bool lo = dv >= (hi ? T[2] : T[0]);
    return (lo ? mlo : 0u) | (hi ? mhi : 0u);
}

// The reference's min / max keep the FIRST element equal to the extreme (std::min / std::max);
// equal fp16 values have equal bits except +-0, so only a zero extreme needs the scan.
// vals(i) yields element i of the group in the reference's order.
// vals(i) reads element i from shared memory (rolled loop: rare path, small code).
template <typename F>
__device__ __forceinline__ float first_zero(float ext, F vals) {
    if (ext != 0.0f) return ext;
#pragma unroll 1
    for (int i = 0; i < 16; ++i) {
        const float x = vals(i);
        if (x == 0.0f) return x;
    }
    return ext;
}

// One warp, rows already staged in s.k / s.v.  Writes the page to `dst` (global) and the fp32
// params to `shadow` if non-null.  Returns (warp-uniform) false if any input was non-finite.
__device__ __forceinline__ bool build_page_staged(PageRows& s, PageParams& pr_, int valid, uint8_t* __restrict__ dst,
                                                  float* __restrict__ shadow) {
    const int lane = lane_id();
    const uint8_t* sk = reinterpret_cast<const uint8_t*>(s.k);
    const uint8_t* sv = reinterpret_cast<const uint8_t*>(s.v);
    uint32_t (*part)[128] = reinterpret_cast<uint32_t (*)[128]>(s.k);  // after the keys
    __half* ks = reinterpret_cast<__half*>(pr_.b + (kKS - 512));
    __half* kz = reinterpret_cast<__half*>(pr_.b + (kKZ - 512));
    __half* vs = reinterpret_cast<__half*>(pr_.b + (kVS - 1024));
    __half* vz = reinterpret_cast<__half*>(pr_.b + (kVZ - 1024));
    bool finite = true;
    const int m = lane >> 3;  // lane quarter: the partial-word buffer it writes

    // ---- keys (PerChannel): lane owns channel pairs q = lane + 32 j, i.e. channels 2q, 2q+1
    // (kc = q >> 3).  Their codes for token t belong to word (4 (t & 7) + tig) * 4 + (t >> 3) +
    // 2 p (tig = q & 3, p = (q >> 2) & 1 -- the same for both j) at bits 2 kc / 16 + 2 kc. ----
    {
        uint32_t cw[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) cw[t] = 0u;
#pragma unroll 1  // rolled: half the code (instruction-cache misses were 14% of stalls)
        for (int j = 0; j < 2; ++j) {
            const int q = lane + 32 * j;
            uint32_t h[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) h[t] = *reinterpret_cast<const uint32_t*>(sk + stage_row_offset(t, q >> 2) + 4 * (q & 3));
            if (valid < 16) {  // (last page of a prefill block) tokens past `valid`: repeat token 0
#pragma unroll
                for (int t = 1; t < 16; ++t) h[t] = t < valid ? h[t] : h[0];
            }
            __half2 mn = u2h2(h[0]), mx = mn;
#pragma unroll
            for (int t = 1; t < 16; ++t) {
                mn = __hmin2_nan(mn, u2h2(h[t]));
                mx = __hmax2_nan(mx, u2h2(h[t]));
            }
            float lo[2] = {__low2float(mn), __high2float(mn)}, hi[2] = {__low2float(mx), __high2float(mx)};
            float T[2][3], sc[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                auto val = [&](int t) {  // (rows past `valid` hold token 0's values in h; same here)
                    const int tt = t < valid ? t : 0;
                    return __half2float(*reinterpret_cast<const __half*>(sk + stage_row_offset(tt, q >> 2) + 4 * (q & 3) + 2 * e));
                };
                lo[e] = first_zero(lo[e], val);
                hi[e] = first_zero(hi[e], val);
                finite &= isfinite(lo[e]) && isfinite(hi[e]);
                group_thresholds(lo[e], hi[e], &sc[e], T[e]);
                const int c = 2 * q + e;
                ks[k_param_idx(c)] = __float2half_rn(sc[e]);
                kz[k_param_idx(c)] = __float2half_rn(lo[e]);
                if (shadow) {
                    shadow[2 * c] = sc[e];
                    shadow[2 * c + 1] = lo[e];
                }
            }
            const int sh = 2 * (q >> 3);
            const uint32_t mlx = 1u << sh, mhx = 2u << sh, mly = 0x10000u << sh, mhy = 0x20000u << sh;
            const float2 lo2 = make_float2(lo[0], lo[1]);
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const float2 dv = sub_h2(h[t], lo2);  // fl(v - lo), both channels
                cw[t] |= code_bits(dv.x, T[0], mlx, mhx) | code_bits(dv.y, T[1], mly, mhy);
            }
        }
        if (valid < 16) {
#pragma unroll
            for (int t = 1; t < 16; ++t) cw[t] = t < valid ? cw[t] : 0u;
        }
        const int tig = lane & 3, p = (lane >> 2) & 1;
        __syncwarp();  // every lane is done with the key rows: they become the partial words
#pragma unroll
        for (int t = 0; t < 16; ++t) part[m][(4 * (t & 7) + tig) * 4 + (t >> 3) + 2 * p] = cw[t];
        __syncwarp();
        uint4 w = reinterpret_cast<const uint4*>(part[0])[lane];
#pragma unroll
        for (int mm = 1; mm < 4; ++mm) {
            const uint4 x = reinterpret_cast<const uint4*>(part[mm])[lane];
            w.x |= x.x; w.y |= x.y; w.z |= x.z; w.w |= x.w;
        }
        reinterpret_cast<uint4*>(dst + kKC)[lane] = w;
        __syncwarp();
    }

    // ---- values (PerToken): lane owns tokens t0 = 2 tp, t1 = t0 + 1 (tp = lane & 7) of the
    // groups g = m + 4 j; the fp16 pair (v[t0][c], v[t1][c]) of channel c = 16 g + cin is the
    // pair of word (4 (cin & 7) + (tp & 3)) * 4 + (cin >> 3) + 2 (tp >> 2) at bits 2 g / 16 + 2 g. ----
    {
        const int tp = lane & 7, t0 = 2 * tp;
        uint32_t cv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) cv[i] = 0u;
#pragma unroll 1  // rolled: half the code (instruction-cache misses were 14% of stalls)
        for (int j = 0; j < 2; ++j) {
            const int g = m + 4 * j;
            uint32_t a[8], b[8];  // channels 16 g + 2 i, + 1 of token t0 (a) / t1 (b)
            *reinterpret_cast<uint4*>(a) = *reinterpret_cast<const uint4*>(sv + stage_row_offset(t0, 2 * g));
            *reinterpret_cast<uint4*>(a + 4) = *reinterpret_cast<const uint4*>(sv + stage_row_offset(t0, 2 * g + 1));
            *reinterpret_cast<uint4*>(b) = *reinterpret_cast<const uint4*>(sv + stage_row_offset(t0 + 1, 2 * g));
            *reinterpret_cast<uint4*>(b + 4) = *reinterpret_cast<const uint4*>(sv + stage_row_offset(t0 + 1, 2 * g + 1));
            uint32_t pr[16];  // pr[cin] = (v[t0][16 g + cin], v[t1][16 g + cin])
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                pr[2 * i] = prmt(a[i], b[i], 0x5410);
                pr[2 * i + 1] = prmt(a[i], b[i], 0x7632);
            }
            __half2 mn = u2h2(pr[0]), mx = mn;
#pragma unroll
            for (int i = 1; i < 16; ++i) {
                mn = __hmin2_nan(mn, u2h2(pr[i]));
                mx = __hmax2_nan(mx, u2h2(pr[i]));
            }
            float lo[2] = {__low2float(mn), __high2float(mn)}, hi[2] = {__low2float(mx), __high2float(mx)};
            float T[2][3], sc[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                auto val = [&](int i) {
                    return __half2float(*reinterpret_cast<const __half*>(sv + stage_row_offset(t0 + e, 2 * g + (i >> 3)) + 2 * (i & 7)));
                };
                lo[e] = first_zero(lo[e], val);
                hi[e] = first_zero(hi[e], val);
                finite &= isfinite(lo[e]) && isfinite(hi[e]);
                group_thresholds(lo[e], hi[e], &sc[e], T[e]);  // rows past `valid` are zeros: scale 0
                const int t = t0 + e;
                vs[vs_param_idx(t, g)] = __float2half_rn(sc[e]);
                vz[vz_param_idx(t, g)] = __float2half_rn(lo[e]);
                if (shadow) {
                    shadow[256 + 2 * (t * 8 + g)] = sc[e];
                    shadow[256 + 2 * (t * 8 + g) + 1] = lo[e];
                }
            }
            const int sh = 2 * g;
            const uint32_t mlx = 1u << sh, mhx = 2u << sh, mly = 0x10000u << sh, mhy = 0x20000u << sh;
            const float2 lo2 = make_float2(lo[0], lo[1]);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float2 dv = sub_h2(pr[i], lo2);
                cv[i] |= code_bits(dv.x, T[0], mlx, mhx) | code_bits(dv.y, T[1], mly, mhy);
            }
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) part[m][(4 * (i & 7) + (tp & 3)) * 4 + (i >> 3) + 2 * (tp >> 2)] = cv[i];
        __syncwarp();
        uint4 w = reinterpret_cast<const uint4*>(part[0])[lane];
#pragma unroll
        for (int mm = 1; mm < 4; ++mm) {
            const uint4 x = reinterpret_cast<const uint4*>(part[mm])[lane];
            w.x |= x.x; w.y |= x.y; w.z |= x.z; w.w |= x.w;
        }
        reinterpret_cast<uint4*>(dst + kVC)[lane] = w;
    }
    __syncwarp();
    // params: KS / KZ (bytes 512..1023) and VS / VZ (1536..2047), 16-byte coalesced
    {
        reinterpret_cast<uint4*>(dst + kKS)[lane] = reinterpret_cast<const uint4*>(pr_.b)[lane];  // 2 x 32 chunks
        reinterpret_cast<uint4*>(dst + kVS)[lane] = reinterpret_cast<const uint4*>(pr_.b + 512)[lane];
    }
    __syncwarp();
    return __all_sync(0xffffffffu, finite);
}

// Flush staging: rows k0[t * 128 ..], v0[t * 128 ..] (t = 0..15, contiguous residual rows) into
// s.k / s.v as one cp.async commit group.
__device__ __forceinline__ void stage_rows_contig(PageRows& s, const __half* __restrict__ k0, const __half* __restrict__ v0) {
    const int lane = lane_id();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int e = lane + 32 * i, t = e >> 4, c = e & 15;
        const uint32_t off = stage_row_offset(t, c);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(reinterpret_cast<uint8_t*>(s.k) + off)),
                     "l"(k0 + (size_t)t * kHeadDim + 8 * c)
                     : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(reinterpret_cast<uint8_t*>(s.v) + off)),
                     "l"(v0 + (size_t)t * kHeadDim + 8 * c)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// Prefill staging: issue cp.async copies of the `valid` kept rows of a page (token indices
// kept16[0..valid)) into s.k / s.v (rows past `valid` zero-filled) as one commit group.
__device__ __forceinline__ void stage_page_rows(PageRows& s, int valid, const __half* __restrict__ kbase, int64_t k_st,
                                                const __half* __restrict__ vbase, int64_t v_st,
                                                const int32_t* __restrict__ kept16) {
    const int lane = lane_id();
    const int my_tok = lane < valid ? __ldg(kept16 + (lane & 15)) : 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int e = lane + 32 * i, t = e >> 4, c = e & 15;  // row t, chunk c
        const int tok = __shfl_sync(0xffffffffu, my_tok, t);
        const uint32_t src_bytes = t < valid ? 16u : 0u;      // 0: zero-fill
        const uint32_t off = stage_row_offset(t, c);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(reinterpret_cast<uint8_t*>(s.k) + off)),
                     "l"(kbase + (int64_t)tok * k_st + 8 * c), "r"(src_bytes)
                     : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(reinterpret_cast<uint8_t*>(s.v) + off)),
                     "l"(vbase + (int64_t)tok * v_st + 8 * c), "r"(src_bytes)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

}  // namespace mkv
