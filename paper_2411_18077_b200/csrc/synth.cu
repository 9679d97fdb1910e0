// synth.cu -- synthetic benchmark inputs generated on device.
//
// Bit-identical to mko_synth_fp16 / the uniform stand-in for A_cumul in
// oracle/minikv_oracle.c: integer splitmix mixing, an exact int sum, one IEEE
// fp32 multiply (__fmul_rn, no contraction) and one RN conversion to fp16, so
// host and device agree on every bit without sharing any libm call.
#include "mkv_kernels.h"

namespace mkv {

__device__ __forceinline__ uint64_t synth_mix(uint64_t seed, uint64_t stream, uint64_t index) {
    uint64_t z = seed + stream * 0xD1B54A32D192ED03ull + (index + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void synth_fp16_kernel(__half* out, int64_t n_rows, int64_t row_len, int64_t ld,
                                  uint64_t seed, uint64_t base, uint64_t step) {
    const int64_t total = n_rows * row_len;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / row_len, c = e - r * row_len;
        const uint64_t z = synth_mix(seed, base + (uint64_t)r * step, (uint64_t)c);
        const int32_t s = (int32_t)(z & 0xFFFFu) + (int32_t)((z >> 16) & 0xFFFFu) +
                          (int32_t)((z >> 32) & 0xFFFFu) + (int32_t)(z >> 48) - 131070;
        out[r * ld + c] = __float2half_rn(__fmul_rn(__int2float_rn(s), 2.6428997e-05f));
    }
}

__global__ void synth_uniform_kernel(float* out, int64_t n_rows, int64_t row_len, int64_t ld,
                                     uint64_t seed, uint64_t base, uint64_t step) {
    const int64_t total = n_rows * row_len;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / row_len, c = e - r * row_len;
        const uint64_t z = synth_mix(seed, base + (uint64_t)r * step, (uint64_t)c);
        out[r * ld + c] = __fmul_rn(__uint2float_rn((uint32_t)(z >> 40)), 1.0f / 16777216.0f);
    }
}

static int grid_for(int64_t total) {
    int64_t g = (total + 255) / 256;
    return (int)(g < 148 * 32 ? (g < 1 ? 1 : g) : 148 * 32);
}

cudaError_t launch_synth_fp16(__half* out, int64_t n_rows, int64_t row_len, int64_t ld,
                              uint64_t seed, uint64_t base, uint64_t step, cudaStream_t s) {
    if (n_rows * row_len == 0) return cudaSuccess;
    synth_fp16_kernel<<<grid_for(n_rows * row_len), 256, 0, s>>>(out, n_rows, row_len, ld, seed, base, step);
    return cudaGetLastError();
}

cudaError_t launch_synth_uniform(float* out, int64_t n_rows, int64_t row_len, int64_t ld,
                                 uint64_t seed, uint64_t base, uint64_t step, cudaStream_t s) {
    if (n_rows * row_len == 0) return cudaSuccess;
    synth_uniform_kernel<<<grid_for(n_rows * row_len), 256, 0, s>>>(out, n_rows, row_len, ld, seed, base, step);
    return cudaGetLastError();
}

}  // namespace mkv
