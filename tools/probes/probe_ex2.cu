// Exponential throughput probe (B200): elements per SM-clock for
//   0: ex2.approx.ftz.f32                       (MUFU.EX2, one element per lane-op)
//   1: ex2.approx.f16x2                          (two elements per lane-op?)
//   2: the A_cumul inner sequence, fp32:  FFMA2 argument, 2 x ex2.f32, FADD2 into a pair sum
//   3: the same with f16x2 exponentials: FFMA2 argument, cvt.rn.f16x2.f32, ex2.f16x2, HADD2
//      into an f16x2 partial (widened every 8 elements)
// One CTA per SM, W warps, `iters` x 16 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pex2 probe_ex2.cu && /tmp/pex2
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) {
    uint32_t y;
    asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ uint32_t cvt_h2(float a, float b) {
    uint32_t y;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(b), "f"(a));
    return y;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned long long* cyc, float* sink) {
    float x[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = -0.001f * (threadIdx.x + j);
    float2 acc[4] = {};
    uint32_t hacc[4] = {};
    const float2 s2 = make_float2(0.99f, 0.99f);
    const float2 b2 = make_float2(-0.01f, -0.02f);
    __syncthreads();
    unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if constexpr (MODE == 0) {
#pragma unroll
            for (int j = 0; j < 16; ++j) x[j] = ex2f(x[j]);
        } else if constexpr (MODE == 1) {
#pragma unroll
            for (int j = 0; j < 16; j += 2) {
                uint32_t h = ex2h2(*reinterpret_cast<uint32_t*>(&x[j]));
                *reinterpret_cast<uint32_t*>(&x[j]) = h;
            }
        } else if constexpr (MODE == 2) {
#pragma unroll
            for (int j = 0; j < 16; j += 2) {
                float2 v = __ffma2_rn(make_float2(x[j], x[j + 1]), s2, b2);
                float2 e = make_float2(ex2f(v.x), ex2f(v.y));
                acc[(j >> 1) & 3] = __fadd2_rn(acc[(j >> 1) & 3], e);
                x[j] = v.y;  // keep the chain alive
                x[j + 1] = v.x;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; j += 2) {
                float2 v = __ffma2_rn(make_float2(x[j], x[j + 1]), s2, b2);
                uint32_t e = ex2h2(cvt_h2(v.x, v.y));
                uint32_t& h = hacc[(j >> 1) & 3];
                asm("add.rn.f16x2 %0, %0, %1;" : "+r"(h) : "r"(e));
                x[j] = v.y;
                x[j + 1] = v.x;
            }
        }
    }
    __syncthreads();
    unsigned long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    float s = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += x[j];
    for (int j = 0; j < 4; ++j) {
        s += acc[j].x + acc[j].y;
        __half2 hh = *reinterpret_cast<__half2*>(&hacc[j]);
        s += __low2float(hh) + __high2float(hh);
    }
    if (s == 12345.f) sink[threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, int threads) {
    unsigned long long* cyc;
    float* sink;
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&sink, 4096);
    const int iters = 4096;
    k<MODE><<<148, threads>>>(16, cyc, sink);
    k<MODE><<<148, threads>>>(iters, cyc, sink);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double elems = (double)threads * iters * 16;
    printf("%-40s threads %4d: %6.2f elements/clk/SM\n", name, threads, elems / avg);
    cudaFree(cyc);
    cudaFree(sink);
}

int main() {
    for (int t : {128, 256, 512}) {
        run<0>("ex2.approx.ftz.f32", t);
        run<1>("ex2.approx.f16x2 (elements)", t);
        run<2>("fp32 seq: FFMA2 + 2 MUFU + FADD2", t);
        run<3>("f16 seq: FFMA2 + cvt + ex2.f16x2 + HADD2", t);
    }
    return 0;
}
