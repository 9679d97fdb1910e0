// quant_pack.cu -- K3: gather the selected tokens and 2-bit quantize + pack them.
//
// Restates the tail of prefill (cache_engine.cpp:56-77): gather_rows of the
// kept indices (ascending) followed by append_block for keys (PerChannel) and
// values (PerToken) as ONE block of n_kept rows (quantizer.cpp:102-136).  Key
// groups are 16 consecutive *kept* tokens; the last group of the
// block may be short and is quantized over its own tokens only.  No gathered
// intermediate is materialised: each warp reads its page's 16 kept rows straight
// from K/V in global memory (keys as coalesced column runs, values as 32-byte
// group runs), stages only the codes, and writes one finished 2 KB page with
// 16-byte coalesced stores.
#include <stdlib.h>

#include "mkv_kernels.h"
#include "mkv_page.cuh"

namespace mkv {

constexpr int kQuantWarps = 8;
constexpr int kStageWarps = 6;   // staged kernel: 6 warps x (2 x 8 KB rows + 1 KB params), 2 CTAs / SM
constexpr int kStagePages = 4;   // consecutive pages per warp, the next one's rows in flight
constexpr int kStageSmem = kStageWarps * (2 * (int)sizeof(PageRows) + (int)sizeof(PageParams));

// round 2: rows staged by cp.async (double-buffered across the warp's pages), codes from fp16
// pairs (build_page_staged)
__global__ void __launch_bounds__(kStageWarps * 32, 2) prefill_pages_kernel(const PrefillPagesParams P) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    PageRows* rows = reinterpret_cast<PageRows*>(smem_raw) + 2 * warp;
    PageParams& prm = reinterpret_cast<PageParams*>(smem_raw + kStageWarps * 2 * sizeof(PageRows))[warp];
    const int i = blockIdx.y;
    const int u = P.unit_begin + i;
    const int p0 = (blockIdx.x * kStageWarps + warp) * kStagePages;
    const UnitMeta meta = P.meta[u];
    const int n_kept = meta.n_prefill;
    const int pages = (n_kept + 15) >> 4;
    const int pend = min(p0 + kStagePages, pages);
    if (p0 >= pend) return;
    const __half* kb = P.k + (size_t)i * P.k_su;
    const __half* vb = P.v + (size_t)i * P.v_su;
    const int32_t* kept = P.kept + (size_t)i * P.kept_stride;
    auto stage = [&](int p) { stage_page_rows(rows[p & 1], min(16, n_kept - 16 * p), kb, P.k_st, vb, P.v_st, kept + 16 * p); };
    stage(p0);
    bool ok = true;
    for (int p = p0; p < pend; ++p) {
        if (p + 1 < pend) {
            stage(p + 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncwarp();
        const int64_t page = meta.page_base + p;
        ok &= build_page_staged(rows[p & 1], prm, min(16, n_kept - 16 * p), P.pool + (size_t)page * kPageBytes,
                                P.shadow ? P.shadow + (size_t)page * (kShadowBytes / 4) : nullptr);
    }
    if (!ok && lane == 0) atomicOr(P.status, kStatusNonFinite);
}

// round 1 (MKV_K3=gather, A/B): rows read per channel / group straight from global
__global__ void __launch_bounds__(kQuantWarps * 32, 4) prefill_pages_gather_kernel(const PrefillPagesParams P) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    PageScratchLite* scratch = reinterpret_cast<PageScratchLite*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int i = blockIdx.y;
    const int u = P.unit_begin + i;
    const int p = blockIdx.x * kQuantWarps + warp;
    const UnitMeta meta = P.meta[u];
    const int n_kept = meta.n_prefill;
    const int pages = (n_kept + 15) >> 4;
    if (p >= pages) return;
    const int valid = min(16, n_kept - 16 * p);
    const int64_t page = meta.page_base + p;
    const bool ok = build_page_gather(scratch[warp], valid, P.k + (size_t)i * P.k_su, P.k_st, P.v + (size_t)i * P.v_su,
                                      P.v_st, P.kept + (size_t)i * P.kept_stride + 16 * p,
                                      P.pool + (size_t)page * kPageBytes,
                                      P.shadow ? P.shadow + (size_t)page * (kShadowBytes / 4) : nullptr);
    if (!ok && lane == 0) atomicOr(P.status, kStatusNonFinite);
}

cudaError_t launch_prefill_pages(const PrefillPagesParams& p, cudaStream_t s) {
    if (p.n_units == 0 || p.max_pages == 0) return cudaSuccess;
    static const bool gather = [] {
        const char* e = getenv("MKV_K3");
        return e && e[0] == 'g';
    }();
    auto kern = gather ? prefill_pages_gather_kernel : prefill_pages_kernel;
    const size_t smem = gather ? sizeof(PageScratchLite) * kQuantWarps : (size_t)kStageSmem;
    const int pages_per_cta = gather ? kQuantWarps : kStageWarps * kStagePages;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    for (int u0 = 0; u0 < p.n_units; u0 += 65535) {  // grid.y limit
        PrefillPagesParams q = p;
        q.unit_begin = p.unit_begin + u0;
        q.n_units = min(65535, p.n_units - u0);
        q.k = p.k + (size_t)u0 * p.k_su;
        q.v = p.v + (size_t)u0 * p.v_su;
        q.kept = p.kept + (size_t)u0 * p.kept_stride;
        dim3 grid((p.max_pages + pages_per_cta - 1) / pages_per_cta, q.n_units);
        kern<<<grid, (gather ? kQuantWarps : kStageWarps) * 32, smem, s>>>(q);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace mkv
