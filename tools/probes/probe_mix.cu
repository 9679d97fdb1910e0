// Probe: marginal cost of an instruction class issued alongside a legacy-HMMA stream on
// sm_100a (cycles per loop iteration per SM sub-partition, 2 warps per sub-partition).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int kH, int kOp, int kN>
__global__ void k(float* out, int iters, long long* cyc) {
    __shared__ uint4 sm[1024];
    float acc[8][4];
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
    uint32_t b[2] = {threadIdx.x * 11u, threadIdx.x * 13u};
    uint32_t x[16], y[16];
    float f[16];
    for (int i = 0; i < 16; ++i) { x[i] = threadIdx.x * (i + 1); y[i] = threadIdx.x ^ (i * 77); f[i] = (float)i; }
    for (int i = 0; i < 1024; i += blockDim.x) sm[(i + threadIdx.x) & 1023] = make_uint4(i, 1, 2, 3);
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
        for (int c = 0; c < kN; ++c) {
            if (kOp == 0) asm volatile("lop3.b32 %0, %0, %1, 0x30003, 0x6a;" : "+r"(x[c & 15]) : "r"(y[c & 15]));
            if (kOp == 1) asm volatile("mul.rn.f16x2 %0, %0, %1;" : "+r"(y[c & 15]) : "r"(x[(c + 3) & 15]));
            if (kOp == 2) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c & 15]) : "f"(f[(c + 5) & 15]), "f"(f[(c + 7) & 15]));
            if (kOp == 3) asm volatile("mov.b32 %0, %1;" : "=r"(x[c & 15]) : "r"(x[(c + 1) & 15]));
            if (kOp == 4) { uint4 v; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"((unsigned)__cvta_generic_to_shared(&sm[(threadIdx.x + c * 32 + (x[0] & 1)) & 1023]))); x[c & 15] ^= v.x; }
            if (kOp == 5) asm volatile("shf.r.wrap.b32 %0, %0, %1, 10;" : "+r"(x[c & 15]) : "r"(y[c & 15]));
            if (kOp == 6) asm volatile("add.f32 %0, %0, %1;" : "+f"(f[c & 15]) : "f"(f[(c + 5) & 15]));
            if (kOp == 7) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[c & 15]));
            if (kOp == 8) asm volatile("shfl.sync.bfly.b32 %0, %0, 4, 0x1f, 0xffffffff;" : "+r"(x[c & 15]));
            if (kOp == 9) asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(x[c & 15]));
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
    for (int i = 0; i < 16; ++i) s += (float)(x[i] ^ y[i]) + f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

const char* kNames[] = {"LOP3", "HMUL2", "FFMA", "MOV", "LDS.128", "SHF", "FADD", "MUFU.EX2", "SHFL", "MOVM"};
template <int H, int Op, int N>
double run(int warps) {
    const int iters = 1000, blocks = 148;
    float* out; long long* cyc;
    cudaMalloc(&out, blocks * warps * 32 * sizeof(float));
    cudaMalloc(&cyc, blocks * sizeof(long long));
    k<H, Op, N><<<blocks, warps * 32>>>(out, 10, cyc);
    k<H, Op, N><<<blocks, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < blocks; ++i) c += h[i]; c /= blocks;
    cudaFree(out); cudaFree(cyc);
    return c / iters / (warps / 4);
}
template <int Op>
void row(int w) {
    const double t0 = run<8, Op, 0>(w), ta = run<0, Op, 32>(w), tb = run<8, Op, 32>(w);
    printf("%-9s x32 alone %6.1f | 8 HMMA alone %5.1f | together %6.1f | marginal per op with HMMA %.2f cyc\n",
           kNames[Op], ta, t0, tb, (tb - t0) / 32);
}
int main() {
    for (int w : {8, 12}) {
        printf("warps/SM %d\n", w);
        row<0>(w); row<1>(w); row<2>(w); row<3>(w); row<4>(w); row<5>(w); row<6>(w); row<7>(w); row<8>(w); row<9>(w);
    }
    return 0;
}
