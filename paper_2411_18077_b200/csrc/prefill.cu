// prefill.cu -- K1: two-pass selective flash-attention prefill (placeholder
// until the tcgen05 kernel lands in the next commit).
#include "mkv_kernels.h"

namespace mkv {
cudaError_t launch_prefill_attn(const PrefillAttnParams&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace mkv
