// refmt.cu -- reference-format device kernels: the reference's own fp32 matrices and its
// QuantizedTensor stream (quantizer.hpp:30-42), for ANY head dim and group size.
//
// These serve the value-type reference signatures (selective_flash_attn, decode_attention,
// quantize_matrix / append_block / dequantize_matrix, and the KVCacheLayer state machine of
// make_cache / prefill / decode_append / decode_step) through the C++ drop-in
// (include/minikv_b200.hpp, namespace minikv_b200::value; dropin/).  They compute in fp32 with
// the reference's operation order where it defines bits:
//   * dot products are sequential fl(fl(a*b) + acc) with no FMA contraction (matrix.cpp:60-66),
//     so scores are bit-identical to the reference's;
//   * the quantizer is quantize_group (quantizer.cpp:28-53) exactly: std::min/std::max
//     semantics for lo/hi (signed zeros), IEEE (hi - lo) / 3.0f, roundf((v - lo) / scale)
//     with IEEE division, clamp -- codes and params are bit-identical;
//   * dequantization is fl(fl(code * scale) + zero) (quantizer.cpp:55-65, no FMA);
//   * decode_attention follows attention.cpp:119-143 / softmax_inplace (matrix.cpp:83-99):
//     one max, exp, a sequential sum, IEEE division, out += attn * v in key order;
//   * A_cumul accumulates every column in row order 0 .. lq-1 (attention.cpp:101-115).
// Only exp/log differ from the host libm by ulps.  The batched fp16 tensor-core path (K1-K4,
// the page layout) is the throughput path; this is the exact-fp32 reference-signature path.
#include <math.h>

#include "mkv_kernels.h"

namespace mkv {

namespace {

__device__ __forceinline__ float dot_ref(const float* __restrict__ a, const float* __restrict__ b, int n) {
    float acc = 0.0f;
    for (int k = 0; k < n; ++k) acc = __fadd_rn(acc, __fmul_rn(a[k], b[k]));
    return acc;
}

template <int kThreads>
__device__ float block_max(float v, float* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    float r = red[0];
    for (int i = 1; i < kThreads / 32; ++i) r = fmaxf(r, red[i]);
    return r;
}

constexpr int kRowThreads = 128;
constexpr int kMaxDvPerThread = 4;  // dv <= 512

// pass 1, one CTA per query row i: max of the visible scores, then exp weights in key chunks
// (staged in shared memory), out[c] accumulated in key order by the channel threads, the
// denominator summed in key order; out *= 1 / sum, lse = m + log(sum).
__global__ void __launch_bounds__(kRowThreads) attn_rows_f32_kernel(const AttnF32Params P) {
    __shared__ float w[kRowThreads];
    __shared__ float red[kRowThreads / 32];
    __shared__ float ssum;
    const int i = blockIdx.x, tid = threadIdx.x;
    const int limit = P.causal ? (P.lk - P.lq + i + 1) : P.lk;
    const float* qi = P.q + (size_t)i * P.ld_q;
    float mx = -INFINITY;
    for (int j = tid; j < limit; j += kRowThreads)
        mx = fmaxf(mx, __fmul_rn(P.scale, dot_ref(qi, P.k + (size_t)j * P.ld_k, P.d)));
    const float m = block_max<kRowThreads>(mx, red);
    float acc[kMaxDvPerThread];
#pragma unroll
    for (int e = 0; e < kMaxDvPerThread; ++e) acc[e] = 0.0f;
    if (tid == 0) ssum = 0.0f;
    for (int j0 = 0; j0 < limit; j0 += kRowThreads) {
        const int j = j0 + tid;
        __syncthreads();
        if (j < limit) w[tid] = expf(__fmul_rn(P.scale, dot_ref(qi, P.k + (size_t)j * P.ld_k, P.d)) - m);
        __syncthreads();
        const int n = min(kRowThreads, limit - j0);
        if (tid == 0) {
            float s = ssum;
            for (int t = 0; t < n; ++t) s = __fadd_rn(s, w[t]);
            ssum = s;
        }
#pragma unroll
        for (int e = 0; e < kMaxDvPerThread; ++e) {
            const int c = tid + e * kRowThreads;
            if (c < P.dv) {
                float a = acc[e];
                for (int t = 0; t < n; ++t) a = __fadd_rn(a, __fmul_rn(w[t], P.v[(size_t)(j0 + t) * P.ld_v + c]));
                acc[e] = a;
            }
        }
    }
    __syncthreads();
    const float sum = ssum;
    const float inv = 1.0f / sum;
#pragma unroll
    for (int e = 0; e < kMaxDvPerThread; ++e) {
        const int c = tid + e * kRowThreads;
        if (c < P.dv) P.out[(size_t)i * P.ld_o + c] = __fmul_rn(acc[e], inv);
    }
    if (tid == 0) P.lse[i] = m + logf(sum);
}

// pass 2, one thread per key column j: sum over the rows that see j, in row order.
__global__ void acumul_f32_kernel(const AttnF32Params P) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= P.lk) return;
    const float* kj = P.k + (size_t)j * P.ld_k;
    const int i0 = P.causal ? max(0, j - (P.lk - P.lq)) : 0;
    float acc = 0.0f;
    for (int i = i0; i < P.lq; ++i) {
        const float s = __fmul_rn(P.scale, dot_ref(P.q + (size_t)i * P.ld_q, kj, P.d));
        acc = __fadd_rn(acc, expf(s - P.lse[i]));
    }
    P.a_cumul[j] = acc;
}

constexpr int kDecThreads = 256;

// decode_attention (attention.cpp:119-143), one CTA: scores -> attn; softmax_inplace with a
// sequential sum (matrix.cpp:83-99); out[c] += attn[j] * v[j][c] in key order.
__global__ void __launch_bounds__(kDecThreads) decode_attn_f32_kernel(const DecodeF32Params P) {
    __shared__ float red[kDecThreads / 32];
    __shared__ float ssum;
    const int tid = threadIdx.x;
    float mx = -INFINITY;
    for (int j = tid; j < P.n; j += kDecThreads) {
        const float s = __fmul_rn(P.scale, dot_ref(P.q, P.keys + (size_t)j * P.ld_k, P.d));
        P.attn[j] = s;
        mx = fmaxf(mx, s);
    }
    const float m = block_max<kDecThreads>(mx, red);
    for (int j = tid; j < P.n; j += kDecThreads) P.attn[j] = expf(P.attn[j] - m);
    __syncthreads();
    if (tid == 0) {
        float s = 0.0f;
        for (int j = 0; j < P.n; ++j) s = __fadd_rn(s, P.attn[j]);
        ssum = s;
    }
    __syncthreads();
    const float sum = ssum;
    for (int j = tid; j < P.n; j += kDecThreads) P.attn[j] = P.attn[j] / sum;
    __syncthreads();
    for (int c = tid; c < P.dv; c += kDecThreads) {
        float a = 0.0f;
        for (int j = 0; j < P.n; ++j) a = __fadd_rn(a, __fmul_rn(P.attn[j], P.values[(size_t)j * P.ld_v + c]));
        P.out[c] = a;
    }
}

// quantize_group (quantizer.cpp:28-53) for every group of one appended block (append_block,
// quantizer.cpp:102-136): one thread per group; codes in the block's stream order.
__global__ void quantize_block_kernel(const QuantBlockParams P) {
    const int per = P.axis == 0 ? (P.rows + P.gs - 1) / P.gs : (P.cols + P.gs - 1) / P.gs;
    const int64_t ng = (int64_t)(P.axis == 0 ? P.cols : P.rows) * per;
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= ng) return;
    // PerChannel: channel `outer`, tokens g0 .. g0 + glen of this block (stream c * rows + t);
    // PerToken: token `outer`, channels g0 .. g0 + glen (stream r * cols + c)
    const int outer = (int)(g / per), g0 = (int)(g % per) * P.gs;
    const int glen = min(P.gs, (P.axis == 0 ? P.rows : P.cols) - g0);
    const int64_t code0 = (int64_t)outer * (P.axis == 0 ? P.rows : P.cols) + g0;
    auto val = [&](int t) {
        if (P.axis == 0) {
            const int r = P.row_idx ? P.row_idx[g0 + t] : g0 + t;
            return P.src[(size_t)r * P.ld + outer];
        }
        const int r = P.row_idx ? P.row_idx[outer] : outer;
        return P.src[(size_t)r * P.ld + g0 + t];
    };
    float lo = val(0), hi = lo;
    bool finite = true;
    for (int t = 0; t < glen; ++t) {
        const float v = val(t);
        finite &= isfinite(v);
        lo = (v < lo) ? v : lo;  // std::min(lo, v)
        hi = (hi < v) ? v : hi;  // std::max(hi, v)
    }
    if (!finite) {  // std::domain_error (quantizer.cpp:35-37)
        atomicOr(P.status, 1u);
        return;
    }
    const float scale = (hi - lo) / 3.0f;
    P.params[2 * g] = scale;
    P.params[2 * g + 1] = lo;
    for (int t = 0; t < glen; ++t) {
        uint8_t code = 0;
        if (scale > 0.0f) code = (uint8_t)fminf(fmaxf(roundf(__fdiv_rn(__fsub_rn(val(t), lo), scale)), 0.0f), 3.0f);
        P.codes[code0 + t] = code;
    }
}

// pack_codes (quantizer.cpp:67-77) of n codes appended at stream position code_off: one thread
// per output word; the first word keeps the existing low codes (init) when code_off % 16 != 0.
__global__ void pack_codes_kernel(const uint8_t* __restrict__ codes, int64_t n, int64_t code_off, uint32_t init,
                                  uint32_t* __restrict__ words, uint32_t* status) {
    const int64_t w0 = code_off / 16;
    const int64_t nw = (code_off + n + 15) / 16 - w0;
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w >= nw) return;
    uint32_t word = (w == 0 && (code_off % 16)) ? init : 0u;
    for (int k = 0; k < 16; ++k) {
        const int64_t pos = (w0 + w) * 16 + k;   // stream position
        const int64_t i = pos - code_off;        // index into this block's codes
        if (i < 0 || i >= n) continue;
        const uint32_t c = codes[i];
        if (c > 3u) atomicOr(status, 2u);
        word |= (c & 3u) << (2 * k);
    }
    words[w] = word;
}

// dequantize_matrix (quantizer.cpp:153-195): one thread per code of the stream; blocks from the
// host table (code offset, group offset, first row, rows per block).
__global__ void dequantize_kernel(const DequantParams P) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= P.total_codes) return;
    int lo = 0, hi = P.n_blocks - 1;
    while (lo < hi) {  // last block whose code offset <= idx
        const int mid = (lo + hi + 1) >> 1;
        if (P.blk[mid].code_off <= idx) lo = mid;
        else hi = mid - 1;
    }
    const DequantBlock b = P.blk[lo];
    const int64_t local = idx - b.code_off;
    int t, c;
    int64_t g;
    if (P.axis == 0) {
        c = (int)(local / b.rows);
        t = (int)(local % b.rows);
        g = b.group_off + (int64_t)c * ((b.rows + P.gs - 1) / P.gs) + t / P.gs;
    } else {
        t = (int)(local / P.cols);
        c = (int)(local % P.cols);
        g = b.group_off + (int64_t)t * ((P.cols + P.gs - 1) / P.gs) + c / P.gs;
    }
    const uint32_t code = (P.words[idx / 16] >> (2 * (idx % 16))) & 3u;
    const float scale = P.params[2 * g], zero = P.params[2 * g + 1];
    P.out[(size_t)(b.row0 + t) * P.ld_out + c] = __fadd_rn(__fmul_rn((float)code, scale), zero);
}

}  // namespace

cudaError_t launch_attn_f32(const AttnF32Params& p, cudaStream_t s) {
    attn_rows_f32_kernel<<<p.lq, kRowThreads, 0, s>>>(p);
    if (cudaError_t e = cudaGetLastError()) return e;
    if (p.a_cumul) acumul_f32_kernel<<<(p.lk + 127) / 128, 128, 0, s>>>(p);
    return cudaGetLastError();
}
int attn_f32_max_dv() { return kRowThreads * kMaxDvPerThread; }

cudaError_t launch_decode_attn_f32(const DecodeF32Params& p, cudaStream_t s) {
    decode_attn_f32_kernel<<<1, kDecThreads, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_quantize_block(const QuantBlockParams& p, cudaStream_t s) {
    const int64_t ng = p.axis == 0 ? (int64_t)p.cols * ((p.rows + p.gs - 1) / p.gs)
                                   : (int64_t)p.rows * ((p.cols + p.gs - 1) / p.gs);
    if (ng == 0) return cudaSuccess;
    quantize_block_kernel<<<(unsigned)((ng + 127) / 128), 128, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_pack_codes(const uint8_t* codes, int64_t n, int64_t code_off, uint32_t init, uint32_t* words,
                              uint32_t* status, cudaStream_t s) {
    const int64_t nw = (code_off + n + 15) / 16 - code_off / 16;
    if (nw <= 0) return cudaSuccess;
    pack_codes_kernel<<<(unsigned)((nw + 127) / 128), 128, 0, s>>>(codes, n, code_off, init, words, status);
    return cudaGetLastError();
}

cudaError_t launch_dequantize(const DequantParams& p, cudaStream_t s) {
    if (p.total_codes == 0) return cudaSuccess;
    dequantize_kernel<<<(unsigned)((p.total_codes + 255) / 256), 256, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace mkv
