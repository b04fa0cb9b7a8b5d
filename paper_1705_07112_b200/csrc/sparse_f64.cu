// placeholder: sparse CSR path (next)
#include "common.cuh"
namespace cpa {
cudaError_t sparse_apply(int64_t, int64_t, int64_t, const int64_t*, const int32_t*, const double*, int64_t, int64_t,
                         double*, int64_t, const cpa_svt_kernel&, int, int, double, double, SeriesParams*, void*,
                         size_t, size_t* need, int, cudaStream_t, int*) {
  *need = 0;
  return cudaErrorNotSupported;
}
}  // namespace cpa
