// placeholder: batched fp32 path (next)
#include "common.cuh"
namespace cpa {
cudaError_t launch_batched_f32(int64_t, int, int, const float*, float*, const cpa_svt_kernel&, int, int, double,
                               double, float*, int, cudaStream_t, int*) {
  return cudaErrorNotSupported;
}
}  // namespace cpa
