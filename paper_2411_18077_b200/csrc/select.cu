// select.cu -- K2: rectified top-k token selection (select_token_counts,
// selection.cpp:10-33) as a radix select over A_cumul.
//
// Per unit: RW = the last rw positions; HH = the top-hh of [0, L - rw) by
// a_cumul descending with ties to the LOWER index (stable_sort, :22-27);
// kept = sort(HH) ++ RW; if hh + rw >= L everything is kept (:14-18).
// The k-th largest key T is found with four 8-bit MSB-first radix passes
// (per-warp shared-memory histograms, so ties never serialise a whole CTA on
// one bin); a two-pass order-preserving compaction (each warp owns a
// contiguous slice: count, one block scan, write) then emits every index with
// key > T plus the first (k - #greater) indices with key == T in index order --
// exactly the stable_sort tie rule, so indices are bit-identical to the
// reference for identical inputs.
//
// Keys are the order-preserving u32 image of the float (-0 folded onto +0, as
// the reference's operator> treats them equal); NaN sorts below everything
// (the reference's comparator is undefined for NaN).
#include <cooperative_groups.h>
#include <stdlib.h>

#include "mkv_kernels.h"

namespace cg = cooperative_groups;

namespace mkv {

constexpr int kSelThreads = 1024;
constexpr int kSelWarps = kSelThreads / 32;

__device__ __forceinline__ uint32_t order_key(float f) {
    uint32_t b = __float_as_uint(f);
    if ((b & 0x7fffffffu) == 0u) b = 0u;
    if ((b & 0x7f800000u) == 0x7f800000u && (b & 0x007fffffu)) return 0u;
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(const SelectParams P) {
    __shared__ int hist[kSelWarps][256];
    __shared__ int tot[256];
    __shared__ int s_digit, s_k;
    __shared__ int w_gt[kSelWarps], w_eq[kSelWarps], w_sel[kSelWarps];
    const int u = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int L = P.length;
    const float* a = P.a + (size_t)u * P.a_stride;
    int32_t* kept = P.kept + (size_t)u * P.kept_stride;
    int hh = P.hh ? P.hh[u] : P.hh_uniform, rw = P.rw;
    if (hh + rw >= L) {
        rw = min(rw, L);
        hh = L - rw;
    }
    const int pool = L - rw;
    const int nh = min(hh, pool);
    for (int j = tid; j < rw; j += kSelThreads) kept[nh + j] = L - rw + j;
    if (P.n_kept && tid == 0) P.n_kept[u] = nh + rw;
    if (nh == 0) return;
    if (nh == pool) {
        for (int j = tid; j < pool; j += kSelThreads) kept[j] = j;
        return;
    }
    // ---- key range: bits shared by min and max need no radix pass ----
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (int j = tid; j < pool; j += kSelThreads) {
        const uint32_t key = order_key(__ldg(a + j));
        kmin = min(kmin, key);
        kmax = max(kmax, key);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) { w_gt[warp] = (int)kmin; w_eq[warp] = (int)kmax; }
    __syncthreads();
    if (warp == 0) {
        uint32_t mn = (uint32_t)w_gt[lane], mx = (uint32_t)w_eq[lane];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) { w_sel[0] = (int)mn; w_sel[1] = (int)mx; }
    }
    __syncthreads();
    const uint32_t gmin = (uint32_t)w_sel[0], gmax = (uint32_t)w_sel[1];
    const int free_bits = (gmin == gmax) ? 0 : 32 - __clz(gmin ^ gmax);  // low bits that still vary
    uint32_t prefix = gmin & ~((free_bits == 32) ? 0xffffffffu : ((1u << free_bits) - 1u));
    uint32_t pmask = (free_bits == 32) ? 0u : ~((1u << free_bits) - 1u);
    int k = nh;
    // ---- radix select of the nh-th largest key over the varying bits, 8 at a time ----
    for (int top = free_bits; top > 0; top -= 8) {
        const int shift = max(top - 8, 0), width = top - shift;
        const uint32_t dmask = (1u << width) - 1u;
        for (int j = lane; j < 256; j += 32) hist[warp][j] = 0;
        __syncthreads();
        for (int base = warp * 32; base < pool; base += kSelThreads) {  // warp-uniform trip count
            const int j = base + lane;
            const uint32_t key = j < pool ? order_key(__ldg(a + j)) : 0u;
            const bool inp = j < pool && (key & pmask) == prefix;
            const unsigned act = __ballot_sync(0xffffffffu, inp);
            if (inp) {  // warp-aggregated: one shared atomic per distinct digit in the warp
                const uint32_t dg = (key >> shift) & dmask;
                const unsigned same = __match_any_sync(act, dg);
                if ((__ffs(same) - 1) == lane) atomicAdd(&hist[warp][dg], __popc(same));
            }
        }
        __syncthreads();
        if (tid < 256) {
            int s = 0;
#pragma unroll 8
            for (int w = 0; w < kSelWarps; ++w) s += hist[w][tid];
            tot[tid] = s;
        }
        __syncthreads();
        if (warp == 0) {
            // digit d with greater < k <= greater + tot[d], scanning 255 -> 0
            int greater = 0, found = -1, kk = k;
            for (int base = 255; base >= 0 && found < 0; base -= 32) {
                const int cnt = tot[base - lane];
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int n = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += n;
                }
                const int excl = incl - cnt;
                const unsigned ball = __ballot_sync(0xffffffffu, (greater + excl < kk) && (kk <= greater + incl));
                if (ball) {
                    const int src = __ffs(ball) - 1;
                    found = base - src;
                    kk -= greater + __shfl_sync(0xffffffffu, excl, src);
                } else {
                    greater += __shfl_sync(0xffffffffu, incl, 31);
                }
            }
            if (lane == 0) { s_digit = found; s_k = kk; }
        }
        __syncthreads();
        prefix |= static_cast<uint32_t>(s_digit) << shift;
        pmask |= dmask << shift;
        k = s_k;
    }
    const uint32_t T = prefix;
    const int take_eq = k;  // equal keys to take, lowest indices first
    // ---- order-preserving compaction: warp w owns the contiguous slice [w*span, (w+1)*span) ----
    const int span = (pool + kSelWarps - 1) / kSelWarps;
    const int lo = min(warp * span, pool), hi = min(lo + span, pool);
    int c_gt = 0, c_eq = 0;
    for (int j = lo + lane; j < hi; j += 32) {
        const uint32_t key = order_key(__ldg(a + j));
        c_gt += key > T;
        c_eq += key == T;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        c_gt += __shfl_xor_sync(0xffffffffu, c_gt, o);
        c_eq += __shfl_xor_sync(0xffffffffu, c_eq, o);
    }
    if (lane == 0) { w_gt[warp] = c_gt; w_eq[warp] = c_eq; }
    __syncthreads();
    if (warp == 0) {  // exclusive scans over warps: equal-key rank base, then output base
        const int g = w_gt[lane], e = w_eq[lane];
        int ie = e;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xffffffffu, ie, o);
            if (lane >= o) ie += n;
        }
        const int eq_base = ie - e;
        const int take = max(0, min(e, take_eq - eq_base));  // equal keys this warp emits
        const int sel = g + take;
        int is = sel;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xffffffffu, is, o);
            if (lane >= o) is += n;
        }
        w_eq[lane] = eq_base;
        w_sel[lane] = is - sel;
    }
    __syncthreads();
    int eq_rank = w_eq[warp], out = w_sel[warp];
    for (int base = lo; base < hi; base += 32) {
        const int j = base + lane;
        const bool in = j < hi;
        const uint32_t key = in ? order_key(__ldg(a + j)) : 0u;
        const bool eq = in && key == T;
        const unsigned beq = __ballot_sync(0xffffffffu, eq);
        const int my_eq = eq_rank + __popc(beq & ((1u << lane) - 1u));
        const bool sel = (in && key > T) || (eq && my_eq < take_eq);
        const unsigned bsel = __ballot_sync(0xffffffffu, sel);
        if (sel) kept[out + __popc(bsel & ((1u << lane) - 1u))] = j;
        eq_rank += __popc(beq);
        out += __popc(bsel);
    }
}

// ---------------------------------------------------------------------------
// Cluster variant for few, long units (configs[3]: 8 kv-head units of 128K keys): a
// thread-block cluster of C CTAs per unit, each CTA owning a contiguous slice of the
// pool.  Key range, the per-pass 256-bin histograms and the compaction counts are
// combined through distributed shared memory (every CTA reads its peers' partials and
// derives the same digit), so the selection is the same deterministic radix select as
// the single-CTA kernel -- identical indices -- spread over C SMs.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSelThreads) select_cluster_kernel(const SelectParams P) {
    __shared__ int hist[kSelWarps][256];
    __shared__ int tot[2][256];  // this CTA's histogram, double-buffered by pass parity
    __shared__ int totg[256];    // cluster-wide histogram
    __shared__ uint32_t s_mm[2];
    __shared__ int s_cnt[2];
    __shared__ int s_digit, s_k;
    __shared__ int w_gt[kSelWarps], w_eq[kSelWarps], w_sel[kSelWarps];
    cg::cluster_group cluster = cg::this_cluster();
    const int C = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
    const int u = blockIdx.x / C;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int L = P.length;
    const float* a = P.a + (size_t)u * P.a_stride;
    int32_t* kept = P.kept + (size_t)u * P.kept_stride;
    int hh = P.hh ? P.hh[u] : P.hh_uniform, rw = P.rw;
    if (hh + rw >= L) {
        rw = min(rw, L);
        hh = L - rw;
    }
    const int pool = L - rw;
    const int nh = min(hh, pool);
    for (int j = rank * kSelThreads + tid; j < rw; j += C * kSelThreads) kept[nh + j] = L - rw + j;
    if (P.n_kept && rank == 0 && tid == 0) P.n_kept[u] = nh + rw;
    if (nh == 0) return;  // uniform across the cluster: no DSMEM traffic follows
    if (nh == pool) {
        for (int j = rank * kSelThreads + tid; j < pool; j += C * kSelThreads) kept[j] = j;
        return;
    }
    const int cspan = (((pool + C - 1) / C) + 31) & ~31;
    const int c_lo = min(rank * cspan, pool), c_hi = min(c_lo + cspan, pool);
    // ---- key range over the cluster ----
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (int j = c_lo + tid; j < c_hi; j += kSelThreads) {
        const uint32_t key = order_key(__ldg(a + j));
        kmin = min(kmin, key);
        kmax = max(kmax, key);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) { w_gt[warp] = (int)kmin; w_eq[warp] = (int)kmax; }
    __syncthreads();
    if (warp == 0) {
        uint32_t mn = (uint32_t)w_gt[lane], mx = (uint32_t)w_eq[lane];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) { s_mm[0] = mn; s_mm[1] = mx; }
    }
    cluster.sync();
    if (warp == 0) {
        uint32_t mn = 0xffffffffu, mx = 0u;
        if (lane < C) {
            const uint32_t* pm = cluster.map_shared_rank(s_mm, lane);
            mn = pm[0];
            mx = pm[1];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) { w_sel[0] = (int)mn; w_sel[1] = (int)mx; }
    }
    __syncthreads();
    const uint32_t gmin = (uint32_t)w_sel[0], gmax = (uint32_t)w_sel[1];
    const int free_bits = (gmin == gmax) ? 0 : 32 - __clz(gmin ^ gmax);
    uint32_t prefix = gmin & ~((free_bits == 32) ? 0xffffffffu : ((1u << free_bits) - 1u));
    uint32_t pmask = (free_bits == 32) ? 0u : ~((1u << free_bits) - 1u);
    int k = nh;
    int par = 0;
    for (int top = free_bits; top > 0; top -= 8, par ^= 1) {
        const int shift = max(top - 8, 0), width = top - shift;
        const uint32_t dmask = (1u << width) - 1u;
        for (int j = lane; j < 256; j += 32) hist[warp][j] = 0;
        __syncthreads();
        for (int base = c_lo + warp * 32; base < c_hi; base += kSelThreads) {
            const int j = base + lane;
            const uint32_t key = j < c_hi ? order_key(__ldg(a + j)) : 0u;
            const bool inp = j < c_hi && (key & pmask) == prefix;
            const unsigned act = __ballot_sync(0xffffffffu, inp);
            if (inp) {
                const uint32_t dg = (key >> shift) & dmask;
                const unsigned same = __match_any_sync(act, dg);
                if ((__ffs(same) - 1) == lane) atomicAdd(&hist[warp][dg], __popc(same));
            }
        }
        __syncthreads();
        if (tid < 256) {
            int sm = 0;
#pragma unroll 8
            for (int w = 0; w < kSelWarps; ++w) sm += hist[w][tid];
            tot[par][tid] = sm;
        }
        cluster.sync();  // every CTA's histogram of this pass is published
        if (tid < 256) {
            int sm = 0;
            for (int r = 0; r < C; ++r) sm += cluster.map_shared_rank(&tot[par][0], r)[tid];
            totg[tid] = sm;
        }
        __syncthreads();
        if (warp == 0) {
            int greater = 0, found = -1, kk = k;
            for (int base = 255; base >= 0 && found < 0; base -= 32) {
                const int cnt = totg[base - lane];
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int n = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += n;
                }
                const int excl = incl - cnt;
                const unsigned ball = __ballot_sync(0xffffffffu, (greater + excl < kk) && (kk <= greater + incl));
                if (ball) {
                    const int src = __ffs(ball) - 1;
                    found = base - src;
                    kk -= greater + __shfl_sync(0xffffffffu, excl, src);
                } else {
                    greater += __shfl_sync(0xffffffffu, incl, 31);
                }
            }
            if (lane == 0) { s_digit = found; s_k = kk; }
        }
        __syncthreads();
        prefix |= static_cast<uint32_t>(s_digit) << shift;
        pmask |= dmask << shift;
        k = s_k;
    }
    const uint32_t T = prefix;
    const int take_eq = k;
    // ---- order-preserving compaction: CTA slices in rank order, warps in slice order ----
    const int span = (c_hi - c_lo + kSelWarps - 1) / kSelWarps;
    const int lo = min(c_lo + warp * span, c_hi), hi = min(lo + span, c_hi);
    int c_gt = 0, c_eq = 0;
    for (int j = lo + lane; j < hi; j += 32) {
        const uint32_t key = order_key(__ldg(a + j));
        c_gt += key > T;
        c_eq += key == T;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        c_gt += __shfl_xor_sync(0xffffffffu, c_gt, o);
        c_eq += __shfl_xor_sync(0xffffffffu, c_eq, o);
    }
    if (lane == 0) { w_gt[warp] = c_gt; w_eq[warp] = c_eq; }
    __syncthreads();
    if (tid == 0) {
        int g = 0, e = 0;
        for (int w = 0; w < kSelWarps; ++w) { g += w_gt[w]; e += w_eq[w]; }
        s_cnt[0] = g;
        s_cnt[1] = e;
    }
    cluster.sync();
    __shared__ int cta_eq_base, cta_gt_base;
    if (warp == 0) {  // bases from lower-ranked CTAs of the cluster
        int g = 0, e = 0;
        if (lane < rank) {
            const int* pc = cluster.map_shared_rank(s_cnt, lane);
            g = pc[0];
            e = pc[1];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            g += __shfl_xor_sync(0xffffffffu, g, o);
            e += __shfl_xor_sync(0xffffffffu, e, o);
        }
        if (lane == 0) { cta_gt_base = g; cta_eq_base = e; }
    }
    cluster.sync();  // no peer reads this CTA's shared memory past this point
    if (warp == 0) {
        const int g = w_gt[lane], e = w_eq[lane];
        int ie = e;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xffffffffu, ie, o);
            if (lane >= o) ie += n;
        }
        const int eq_base = cta_eq_base + ie - e;
        const int take = max(0, min(e, take_eq - eq_base));
        // selected before this warp: greater keys of lower CTAs + their taken equals
        const int sel = g + take;
        int is = sel;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xffffffffu, is, o);
            if (lane >= o) is += n;
        }
        const int lower_taken = max(0, min(cta_eq_base, take_eq));
        w_eq[lane] = eq_base;
        w_sel[lane] = cta_gt_base + lower_taken + is - sel;
    }
    __syncthreads();
    int eq_rank = w_eq[warp], out = w_sel[warp];
    for (int base = lo; base < hi; base += 32) {
        const int j = base + lane;
        const bool in = j < hi;
        const uint32_t key = in ? order_key(__ldg(a + j)) : 0u;
        const bool eq = in && key == T;
        const unsigned beq = __ballot_sync(0xffffffffu, eq);
        const int my_eq = eq_rank + __popc(beq & ((1u << lane) - 1u));
        const bool sel = (in && key > T) || (eq && my_eq < take_eq);
        const unsigned bsel = __ballot_sync(0xffffffffu, sel);
        if (sel) kept[out + __popc(bsel & ((1u << lane) - 1u))] = j;
        eq_rank += __popc(beq);
        out += __popc(bsel);
    }
}

// ---------------------------------------------------------------------------
// layer_score_variance (selection.cpp:130-146): population variance of A_cumul, the
// per-layer statistic of variance-based budget allocation (allocate_variance,
// selection.cpp:85-128).  One CTA per row; two fp64 passes (mean, then squared
// deviations) like the reference, reduced in a fixed tree order (deterministic).
// ---------------------------------------------------------------------------
constexpr int kVarThreads = 512;

__device__ __forceinline__ double block_sum_f64(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < kVarThreads / 32 ? red[lane] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) red[32] = t;
    }
    __syncthreads();
    t = red[32];
    __syncthreads();
    return t;
}

__global__ void __launch_bounds__(kVarThreads) score_variance_kernel(const float* __restrict__ a, int64_t stride,
                                                                     int length, float* __restrict__ out) {
    __shared__ double red[33];
    const float* row = a + (size_t)blockIdx.x * stride;
    double s = 0.0;
    for (int j = threadIdx.x; j < length; j += kVarThreads) s += (double)__ldg(row + j);
    const double mean = block_sum_f64(s, red) / (double)length;
    double q = 0.0;
    for (int j = threadIdx.x; j < length; j += kVarThreads) {
        const double d = (double)__ldg(row + j) - mean;
        q = __dadd_rn(q, __dmul_rn(d, d));  // multiply then add, as the reference (no FMA)
    }
    const double var = block_sum_f64(q, red);
    if (threadIdx.x == 0) out[blockIdx.x] = (float)(var / (double)length);
}

cudaError_t launch_score_variance(const float* a, int64_t a_stride, int n, int length, float* out, cudaStream_t s) {
    score_variance_kernel<<<n, kVarThreads, 0, s>>>(a, a_stride, length, out);
    return cudaGetLastError();
}

// cluster size per unit: spread few long units over the SMs (0 = single-CTA kernel)
static int select_cluster_size(const SelectParams& p) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    if (const char* e = getenv("MKV_SELECT_CLUSTER")) return atoi(e);
    for (int c : {16, 8, 4, 2})
        if ((int64_t)p.n_units * c <= 2 * sms && p.length / c >= 4096) return c;
    return 0;
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t s) {
    if (p.n_units == 0) return cudaSuccess;
    const int C = select_cluster_size(p);
    if (C > 1) {
        static bool configured = false;
        if (!configured) {
            cudaError_t e = cudaFuncSetAttribute(select_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
            configured = true;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(p.n_units * C);
        cfg.blockDim = dim3(kSelThreads);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, select_cluster_kernel, p);
    }
    select_kernel<<<p.n_units, kSelThreads, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace mkv
