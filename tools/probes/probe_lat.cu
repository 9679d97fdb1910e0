// Probe: legacy HMMA dependent-issue latency on sm_100a: kC independent accumulator chains
// per warp, one warp per SM sub-partition.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int kC>
__global__ void k(float* out, int iters, long long* cyc) {
    float acc[8][4];
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
    uint32_t b[2] = {threadIdx.x * 11u, threadIdx.x * 13u};
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < kC; ++c)
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                             : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int C> void run(int warps) {
    float* out; long long* cyc; const int iters = 500;
    cudaMalloc(&out, 148 * warps * 32 * 4); cudaMalloc(&cyc, 148 * 8);
    k<C><<<148, warps * 32>>>(out, 10, cyc); k<C><<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("chains/warp %d, warps/SMSP %d: %.1f cycles per dependent step (%.1f per HMMA per SMSP)\n", C, warps / 4,
           c / iters / 8, c / iters / 8 / C / (warps / 4));
}
int main() {
    for (int w : {4, 8}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); }
}
