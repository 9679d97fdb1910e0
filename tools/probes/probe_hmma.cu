// Throughput probe: legacy mma.sync on sm_100a (cycles per HMMA per SM sub-partition).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_hmma probe_hmma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int kVariant>
__global__ void k(float* out, int iters, long long* cyc) {
    float acc[8][4];
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
    uint32_t b[2] = {threadIdx.x * 11u, threadIdx.x * 13u};
    uint32_t acc16[8][2];
    for (int i = 0; i < 8; ++i) { acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f; acc16[i][0] = acc16[i][1] = 0; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (kVariant == 0) {
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                             : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            } else if (kVariant == 1) {
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};\n"
                             : "+r"(acc16[c][0]), "+r"(acc16[c][1])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            } else if (kVariant == 2) {
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                             : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                             : "r"(a[0]), "r"(a[1]), "r"(b[0]));
            } else if (kVariant == 3) {  // bf16
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                             : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            } else if (kVariant == 4) {  // int8 m16n8k32
                int* ai = reinterpret_cast<int*>(acc[c]);
                asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                             : "+r"(ai[0]), "+r"(ai[1]), "+r"(ai[2]), "+r"(ai[3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3] + (float)acc16[i][0] + (float)acc16[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, int warps) {
    const int iters = 2000, blocks = 148;
    float* out; long long* cyc;
    cudaMalloc(&out, blocks * warps * 32 * sizeof(float));
    cudaMalloc(&cyc, blocks * sizeof(long long));
    k<V><<<blocks, warps * 32>>>(out, 10, cyc);
    k<V><<<blocks, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < blocks; ++i) c += h[i]; c /= blocks;
    const double per_smsp = (double)iters * 8 * warps / 4;  // mma per SMSP
    printf("%-22s warps/SM %2d: %.2f cycles per mma per SMSP\n", name, warps, c / per_smsp);
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {4, 8, 16}) {
        run<0>("m16n8k16 f16->f32", w);
        run<1>("m16n8k16 f16->f16", w);
        run<2>("m16n8k8 f16->f32", w);
        run<3>("m16n8k16 bf16->f32", w);
        run<4>("m16n8k32 s8->s32", w);
    }
    return 0;
}
