// select.cu -- K2: rectified top-k token selection (select_token_counts,
// selection.cpp:10-33) as a radix select over A_cumul.
//
// Per unit: RW = the last rw positions; HH = the top-hh of [0, L - rw) by
// a_cumul descending with ties to the LOWER index (stable_sort, :22-27);
// kept = sort(HH) ++ RW; if hh + rw >= L everything is kept (:14-18).
// The k-th largest key T is found with four 8-bit MSB-first radix passes
// (shared-memory histograms); an order-preserving ballot compaction then
// emits every index with key > T plus the first (k - #greater) indices with
// key == T in index order -- exactly the stable_sort tie rule, so indices are
// bit-identical to the reference for identical inputs.
//
// Keys are the order-preserving u32 image of the float (-0 folded onto +0, as
// the reference's operator> treats them equal); NaN sorts below everything
// (the reference's comparator is undefined for NaN).
#include "mkv_kernels.h"

namespace mkv {

constexpr int kSelThreads = 1024;

__device__ __forceinline__ uint32_t order_key(float f) {
    uint32_t b = __float_as_uint(f);
    if ((b & 0x7fffffffu) == 0u) b = 0u;
    if ((b & 0x7f800000u) == 0x7f800000u && (b & 0x007fffffu)) return 0u;
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// inclusive block scan of one int per warp (warp totals in sm[0..31])
__device__ __forceinline__ void scan_warp_totals(int* sm, int nwarps) {
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        int v = lane < nwarps ? sm[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += n;
        }
        sm[lane] = v;
    }
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(const SelectParams P) {
    __shared__ int hist[256];
    __shared__ int s_digit, s_k;
    __shared__ int wtot_eq[32], wtot_sel[32];
    const int u = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int L = P.length;
    const float* a = P.a + (size_t)u * P.a_stride;
    int32_t* kept = P.kept + (size_t)u * P.kept_stride;
    int hh = P.hh[u], rw = P.rw;
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
    // ---- radix select of the nh-th largest key ----
    uint32_t prefix = 0, pmask = 0;
    int k = nh;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int j = tid; j < 256; j += kSelThreads) hist[j] = 0;
        __syncthreads();
        for (int j = tid; j < pool; j += kSelThreads) {
            const uint32_t key = order_key(__ldg(a + j));
            if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 0xffu], 1);
        }
        __syncthreads();
        if (warp == 0) {
            // find digit d with greater < k <= greater + hist[d], scanning 255 -> 0
            int greater = 0;
            int found = -1, kk = k;
            for (int base = 255; base >= 0 && found < 0; base -= 32) {
                const int dgt = base - lane;
                const int c = hist[dgt];
                int incl = c;  // inclusive suffix sum within this chunk (from high digits)
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int n = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += n;
                }
                const int excl = incl - c;
                const bool hit = (greater + excl < kk) && (kk <= greater + incl);
                const unsigned ball = __ballot_sync(0xffffffffu, hit);
                if (ball) {
                    const int src = __ffs(ball) - 1;
                    found = base - src;
                    const int ex = __shfl_sync(0xffffffffu, excl, src);
                    kk -= greater + ex;
                } else {
                    greater += __shfl_sync(0xffffffffu, incl, 31);
                }
            }
            if (lane == 0) { s_digit = found; s_k = kk; }
        }
        __syncthreads();
        prefix |= static_cast<uint32_t>(s_digit) << shift;
        pmask |= 0xffu << shift;
        k = s_k;
        __syncthreads();
    }
    const uint32_t T = prefix;
    const int take_eq = k;  // equal keys to take, lowest indices first
    // ---- order-preserving compaction ----
    int carry_eq = 0, carry_sel = 0;
    for (int base = 0; base < pool; base += kSelThreads) {
        const int j = base + tid;
        uint32_t key = 0;
        const bool in = j < pool;
        if (in) key = order_key(__ldg(a + j));
        const bool gt = in && key > T;
        const bool eq = in && key == T;
        const unsigned beq = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) wtot_eq[warp] = __popc(beq);
        __syncthreads();
        scan_warp_totals(wtot_eq, kSelThreads / 32);
        __syncthreads();
        const int eq_rank = carry_eq + (warp ? wtot_eq[warp - 1] : 0) + __popc(beq & ((1u << lane) - 1u));
        const bool sel = gt || (eq && eq_rank < take_eq);
        const unsigned bsel = __ballot_sync(0xffffffffu, sel);
        if (lane == 0) wtot_sel[warp] = __popc(bsel);
        __syncthreads();
        scan_warp_totals(wtot_sel, kSelThreads / 32);
        __syncthreads();
        if (sel) kept[carry_sel + (warp ? wtot_sel[warp - 1] : 0) + __popc(bsel & ((1u << lane) - 1u))] = j;
        carry_eq += wtot_eq[kSelThreads / 32 - 1];
        carry_sel += wtot_sel[kSelThreads / 32 - 1];
        __syncthreads();
    }
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t s) {
    if (p.n_units == 0) return cudaSuccess;
    select_kernel<<<p.n_units, kSelThreads, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace mkv
