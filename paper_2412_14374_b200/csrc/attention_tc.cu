// Tensor-core flash attention (bf16) -- placeholder until the mma kernels land;
// attention_tc_supported() routes every call to the exact SIMT path.
#include "common.cuh"

namespace pp200 {
bool attention_tc_supported(int, int64_t, int64_t) { return false; }
int attention_fwd_tc(int, int, int, int, const void*, int64_t, void*, int64_t, float*,
                     cudaStream_t) {
  set_error("attention_fwd_tc unavailable");
  return PC_ERR_UNSUPPORTED;
}
int attention_bwd_tc(int, int, int, int, const void*, int64_t, const void*, const void*, int64_t,
                     const float*, float*, void*, int64_t, cudaStream_t) {
  set_error("attention_bwd_tc unavailable");
  return PC_ERR_UNSUPPORTED;
}
}  // namespace pp200
