// h2o.cu -- the step-wise greedy H2O baseline (harness.cpp:83-150) on the device.
//
// The reference's comparison policy for MiniKV's persistence claim: running cumulative
// attention scores, one decode token at a time; after every step the lowest-scoring token
// outside the rw most recent positions is evicted until the budget holds (ties: lower index).
// One CTA per sequence.  Keys are never moved: the kept set is a compacted list of original
// positions (ascending, like the reference's erase-in-place vectors), keys are read from the
// prompt / decode arrays through it, and the scores live per original position.
//
// Arithmetic follows the reference's order exactly so the kept sets match it bit for bit:
// dot = sequential fp32 multiply-then-add over d (matrix.cpp:60-66, no contraction),
// attn = scale * dot, softmax_inplace (matrix.cpp:83-99): max, exp(x - max) rounded once
// from double (a correctly rounded expf), a sequential fp32 sum, IEEE division; scores
// accumulate in double.
#include <float.h>
#include <math.h>

#include "mkv_kernels.h"

namespace mkv {

namespace {
constexpr int kH2OThreads = 256;

struct ArgMin {
    double s;
    int i;
};

// victim = first index i < n_eval with the smallest score (strict <, like the reference's scan);
// -1 when no candidate compares below +inf
__device__ int block_argmin(const int* __restrict__ pos, const double* __restrict__ score, int n_eval,
                            ArgMin* red) {
    ArgMin best{INFINITY, 0x7fffffff};
    for (int i = threadIdx.x; i < n_eval; i += kH2OThreads) {
        const double s = score[pos[i]];
        if (s < best.s) best = ArgMin{s, i};  // i ascends per thread: first occurrence kept
    }
    red[threadIdx.x] = best;
    __syncthreads();
    for (int w = kH2OThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            const ArgMin o = red[threadIdx.x + w];
            const ArgMin m = red[threadIdx.x];
            if (o.s < m.s || (o.s == m.s && o.i < m.i)) red[threadIdx.x] = o;
        }
        __syncthreads();
    }
    const int v = red[0].i;
    __syncthreads();
    return v == 0x7fffffff ? -1 : v;
}

// drop pos[v], shifting the tail down one slot (chunked: read, barrier, write)
__device__ void erase_at(int* pos, int v, int n) {
    for (int base = v; base < n - 1; base += kH2OThreads) {
        const int i = base + threadIdx.x;
        const int x = (i < n - 1) ? pos[i + 1] : 0;
        __syncthreads();
        if (i < n - 1) pos[i] = x;
        __syncthreads();
    }
}

// evict_to_budget (harness.cpp:83-106)
__device__ int evict_to_budget(int* pos, const double* score, int n, int budget, int rw, ArgMin* red) {
    while (n > budget) {
        const int protect_from = n > rw ? n - rw : 0;
        const int v = block_argmin(pos, score, protect_from, red);
        if (v < 0) break;  // everything is inside the recent window
        erase_at(pos, v, n);
        --n;
    }
    return n;
}

__global__ void __launch_bounds__(kH2OThreads) h2o_kernel(const H2OParams P) {
    __shared__ ArgMin red[kH2OThreads];
    __shared__ float red_f[kH2OThreads];
    extern __shared__ float qs_sm[];  // one decode query
    const int L = P.l_prompt, d = P.d;
    int* pos = P.ws_pos;
    double* score = P.ws_score;
    float* attn = P.ws_attn;
    const int budget = P.hh_budget + P.rw_budget;
    for (int i = threadIdx.x; i < L; i += kH2OThreads) {
        pos[i] = i;
        score[i] = (double)P.prompt_scores[i];
    }
    __syncthreads();
    int n = evict_to_budget(pos, score, L, budget, P.rw_budget, red);
    for (int i = threadIdx.x; i < n; i += kH2OThreads) P.kept[i] = pos[i];
    if (threadIdx.x == 0) P.kept_count[0] = n;
    for (int s = 0; s < P.steps; ++s) {
        // append_row + index + zero score (harness.cpp:132-135)
        if (threadIdx.x == 0) {
            pos[n] = L + s;
            score[L + s] = 0.0;
        }
        for (int c = threadIdx.x; c < d; c += kH2OThreads) qs_sm[c] = P.qs[(size_t)s * d + c];
        __syncthreads();
        ++n;
        // attn[j] = scale * dot(q, key_j)
        float mloc = -INFINITY;
        for (int i = threadIdx.x; i < n; i += kH2OThreads) {
            const int p = pos[i];
            const float* key = p < L ? P.prompt_k + (size_t)p * P.ld_k : P.ks + (size_t)(p - L) * d;
            float acc = 0.0f;
            for (int c = 0; c < d; ++c) acc = __fadd_rn(acc, __fmul_rn(qs_sm[c], key[c]));
            const float a = __fmul_rn(P.scale, acc);
            attn[i] = a;
            mloc = fmaxf(mloc, a);
        }
        red_f[threadIdx.x] = mloc;
        __syncthreads();
        for (int w = kH2OThreads / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) red_f[threadIdx.x] = fmaxf(red_f[threadIdx.x], red_f[threadIdx.x + w]);
            __syncthreads();
        }
        const float m = red_f[0];
        for (int i = threadIdx.x; i < n; i += kH2OThreads) attn[i] = (float)exp((double)__fsub_rn(attn[i], m));
        __syncthreads();
        if (threadIdx.x == 0) {  // the reference's sequential fp32 sum
            float sum = 0.0f;
            for (int i = 0; i < n; ++i) sum = __fadd_rn(sum, attn[i]);
            red_f[0] = sum;
        }
        __syncthreads();
        const float sum = red_f[0];
        for (int i = threadIdx.x; i < n; i += kH2OThreads) {
            const int p = pos[i];
            score[p] = __dadd_rn(score[p], (double)__fdiv_rn(attn[i], sum));
        }
        __syncthreads();
        n = evict_to_budget(pos, score, n, budget, P.rw_budget, red);
        int* out = P.kept + (size_t)(s + 1) * P.kept_stride;
        for (int i = threadIdx.x; i < n; i += kH2OThreads) out[i] = pos[i];
        if (threadIdx.x == 0) P.kept_count[s + 1] = n;
        __syncthreads();
    }
}
}  // namespace

cudaError_t launch_h2o(const H2OParams& p, cudaStream_t s) {
    h2o_kernel<<<1, kH2OThreads, (size_t)p.d * sizeof(float), s>>>(p);
    return cudaGetLastError();
}

}  // namespace mkv
