// Microprobe: (1) does mma.sync.m16n8k16 f16->f32 honour fp16 subnormal inputs exactly?
// (2) legacy HMMA throughput on sm_100a; (3) streaming-load HBM bandwidth.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
    : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
    : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// A = all ones (1.0h); B = subnormal pattern codes*2^-24 (raw bits = code)
__global__ void subnormal_test(float* out, uint32_t braw) {
  uint32_t a[4]; uint32_t one2 = 0x3C003C00u;
  a[0]=a[1]=a[2]=a[3]=one2;
  uint32_t b[2] = {braw, braw};
  float d[4] = {0,0,0,0};
  mma16816(d, a, b);
  if (threadIdx.x == 0) { out[0]=d[0]; out[1]=d[1]; }
}

__global__ void mma_tput(float* out, int iters) {
  uint32_t a[4] = {0x3C003C00u, 0x3C003C00u, 0x3C003C00u, 0x3C003C00u};
  uint32_t b[2] = {0x00010001u ^ threadIdx.x, 0x3C00u};
  float d0[4]={0,0,0,0}, d1[4]={0,0,0,0}, d2[4]={0,0,0,0}, d3[4]={0,0,0,0};
  for (int i = 0; i < iters; ++i) {
    mma16816(d0, a, b); mma16816(d1, a, b); mma16816(d2, a, b); mma16816(d3, a, b);
  }
  if (d0[0]+d1[1]+d2[2]+d3[3] == 12345.f) out[0] = 1;
}

__global__ void stream_read(const int4* __restrict__ p, size_t n, int* out) {
  int acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"(p+i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  printf("device %s sms %d clock %d kHz l2 %d smemPerBlockOptin %zu\n", prop.name, prop.multiProcessorCount, prop.clockRate, prop.l2CacheSize, prop.sharedMemPerBlockOptin);
  float* d_out; cudaMalloc(&d_out, 64);
  float h[2];
  uint32_t pats[] = {0x00010001u, 0x00030002u, 0x03000100u, 0x00C00040u};
  for (uint32_t p : pats) {
    subnormal_test<<<1,32>>>(d_out, p);
    cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
    __half lo = __ushort_as_half((unsigned short)(p & 0xffff)), hi = __ushort_as_half((unsigned short)(p >> 16));
    double expect = 8.0 * ((double)__half2float(lo) + (double)__half2float(hi));
    printf("subnormal pattern %08x: mma=%.10e expect(8 k-pairs)=%.10e ratio=%.6f\n", p, h[0], expect, h[0]/expect);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int blocksPerSm : {4, 8, 16}) {
    int grid = prop.multiProcessorCount * blocksPerSm;
    mma_tput<<<grid, 128>>>(d_out, 16);
    cudaEventRecord(e0);
    mma_tput<<<grid, 128>>>(d_out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)grid * 4 /*warps*/ * iters * 4 * (16.0*8*16*2);
    printf("mma.sync m16n8k16 f16/f32: grid %d: %.3f ms  %.1f TFLOP/s\n", grid, ms, flops / ms / 1e9);
  }
  size_t bytes = (size_t)4 << 30;
  int4* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  int* dint; cudaMalloc(&dint, 4);
  for (int bps : {4, 8}) {
    int grid = prop.multiProcessorCount * bps;
    stream_read<<<grid, 512>>>(buf, bytes/16, dint);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) stream_read<<<grid, 512>>>(buf, bytes/16, dint);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("stream read grid %d: %.1f GB/s\n", grid, 5.0 * bytes / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
