// Probe: HBM bandwidth of the page kernel's memory pattern alone -- persistent CTAs,
// W warps each streaming a contiguous range through an S-stage ring of B-byte
// cp.async.bulk copies (mbarrier complete_tx), no compute.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int W, int S, int BYTES>
__global__ void __launch_bounds__(W * 32, 1) stream_kernel(const uint8_t* src, size_t total, size_t chunk, int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + (size_t)warp * S * BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)W * S * BYTES) + warp * S;
  const size_t wg = (size_t)blockIdx.x * W + warp;
  size_t beg = wg * chunk, end = beg + chunk < total ? beg + chunk : total;
  if (beg >= end) return;
  if (lane == 0) { for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bars[s]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  size_t pos = beg;
  auto issue = [&](int s) {
    if (pos >= end) return;
    uint32_t n = (uint32_t)((end - pos) < BYTES ? (end - pos) : BYTES);
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&bars[s])), "r"(n) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(su(ring + s * BYTES)), "l"(src + pos), "r"(n), "r"(su(&bars[s])) : "memory");
    }
    pos += n;
  };
  for (int s = 0; s < S; ++s) issue(s);
  int acc = 0; uint32_t phase = 0; int s = 0;
  for (size_t c = beg; c < end; c += BYTES) {
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra.uni D;\nbra.uni W;\nD:\n}" :: "r"(su(&bars[s])), "r"(phase) : "memory");
    acc ^= reinterpret_cast<const int*>(ring + s * BYTES)[lane];
    __syncwarp();
    issue(s);
    if (++s == S) { s = 0; phase ^= 1; }
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

template <int W, int S, int BYTES>
void run(const uint8_t* buf, size_t total, int* sink) {
  size_t smem = (size_t)W * S * BYTES + W * S * 8;
  cudaFuncSetAttribute(stream_kernel<W, S, BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int warps = 148 * W;
  size_t chunk = (total / warps + BYTES - 1) / BYTES * BYTES;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int r = 0; r < 3; ++r) stream_kernel<W, S, BYTES><<<148, W * 32, smem>>>(buf, total, chunk, sink);
  cudaEventRecord(a);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) stream_kernel<W, S, BYTES><<<148, W * 32, smem>>>(buf + (r % 4) * total, total, chunk, sink);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("W=%2d S=%d B=%6d  smem/CTA=%6zu KB  %.1f us/launch  %.0f GB/s  err=%s\n", W, S, BYTES, smem / 1024, 1e3 * ms / reps,
         total * reps / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  size_t total = 110u << 20;
  uint8_t* buf; cudaMalloc(&buf, total * 4); cudaMemset(buf, 1, total * 4);
  int* sink; cudaMalloc(&sink, 4);
  run<12, 2, 8192>(buf, total, sink);
  run<12, 2, 4096>(buf, total, sink);
  run<8, 3, 8192>(buf, total, sink);
  run<6, 4, 8192>(buf, total, sink);
  run<12, 1, 16384>(buf, total, sink);
  run<4, 4, 16384>(buf, total, sink);
  run<2, 6, 16384>(buf, total, sink);
  run<16, 2, 4096>(buf, total, sink);
  run<24, 2, 4096>(buf, total, sink);
  return 0;
}
