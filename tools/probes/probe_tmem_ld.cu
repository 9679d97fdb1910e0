// TMEM read bandwidth probe (B200): W warps per CTA (W/4 per TMEM lane quarter) each issue
// `iters` x (4 x tcgen05.ld.32x32b.x32 + wait::ld), i.e. 512 B per warp per ld; one CTA per SM.
// Prints bytes per SM-clock.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ptm probe_tmem_ld.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int W>
__global__ void __launch_bounds__(W * 32, 1) k(int iters, unsigned long long* cyc, float* sink) {
    __shared__ uint32_t taddr;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = taddr + ((uint32_t)((warp & 3) * 32) << 16) + 128 * ((warp >> 2) & 3);
    float acc = 0.f;
    __syncthreads();
    unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t r[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
                "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                  "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                  "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(t + 32 * j));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
        }
    }
    __syncthreads();
    unsigned long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr));
}
template <int W>
void run(int sms) {
    unsigned long long* cyc; float* sink;
    cudaMalloc(&cyc, sms * 8); cudaMalloc(&sink, sms * W * 32 * 4);
    const int iters = 2000;
    k<W><<<sms, W * 32>>>(10, cyc, sink);
    k<W><<<sms, W * 32>>>(iters, cyc, sink);
    cudaDeviceSynchronize();
    unsigned long long h[256]; cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
    const double bytes = (double)W * iters * 4 * 32 * 32 * 4;  // per CTA
    printf("warps/SM %2d: %.1f bytes per SM clock (%.0f clk for %.0f KB)  err=%s\n", W, bytes / avg, avg, bytes / 1024,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(cyc); cudaFree(sink);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<4>(sms); run<8>(sms); run<12>(sms); run<16>(sms);
    return 0;
}
