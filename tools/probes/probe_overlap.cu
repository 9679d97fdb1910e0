// Probe: do legacy HMMA (mma.sync) and ALU/FMA-pipe instructions overlap on sm_100a?
// Per warp: N HMMA (8 independent chains) and/or M independent LOP3 / HMUL2 per iteration.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int kH, int kL, int kF>
__global__ void k(float* out, int iters, long long* cyc) {
    float acc[8][4];
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
    uint32_t b[2] = {threadIdx.x * 11u, threadIdx.x * 13u};
    uint32_t x[16], y[16];
    for (int i = 0; i < 16; ++i) { x[i] = threadIdx.x * (i + 1); y[i] = threadIdx.x ^ (i * 77); }
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < kH; ++c)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(acc[c & 7][0]), "+f"(acc[c & 7][1]), "+f"(acc[c & 7][2]), "+f"(acc[c & 7][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
#pragma unroll
        for (int c = 0; c < kL; ++c)
            asm volatile("lop3.b32 %0, %0, %1, 0x30003, 0xc0;" : "+r"(x[c & 15]) : "r"(y[c & 15]));
#pragma unroll
        for (int c = 0; c < kF; ++c)
            asm volatile("mul.rn.f16x2 %0, %0, %1;" : "+r"(y[c & 15]) : "r"(x[(c + 3) & 15]));
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
    for (int i = 0; i < 16; ++i) s += (float)(x[i] ^ y[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int H, int L, int F>
void run(int warps) {
    const int iters = 1000, blocks = 148;
    float* out; long long* cyc;
    cudaMalloc(&out, blocks * warps * 32 * sizeof(float));
    cudaMalloc(&cyc, blocks * sizeof(long long));
    k<H, L, F><<<blocks, warps * 32>>>(out, 10, cyc);
    k<H, L, F><<<blocks, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < blocks; ++i) c += h[i]; c /= blocks;
    printf("HMMA %2d LOP3 %2d HMUL2 %2d  warps/SMSP %d: %.1f cycles per iteration per SMSP\n", H, L, F, warps / 4,
           c / iters / (warps / 4));
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {8, 12, 16}) {
        run<8, 0, 0>(w);
        run<0, 32, 0>(w);
        run<0, 0, 16>(w);
        run<8, 32, 0>(w);
        run<8, 0, 16>(w);
        run<8, 32, 16>(w);
        run<0, 32, 16>(w);
    }
    return 0;
}
