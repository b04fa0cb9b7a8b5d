// Alg. 1 line 4 on the device: Lambda, tau and the Chebyshev-Gauss coefficients from
// lambda_hat (readings R6-R8).  Shared by the power kernels (power.cu)
// and the single-CTA small-problem kernel (small_f64.cu).
#pragma once
#include "common.cuh"

namespace cpa {

// Fill P from lambda_hat (block-wide; all threads of the calling block must enter).
__device__ __forceinline__ void compute_series(SeriesParams* P, const cpa_svt_kernel& kern, int K, double safety,
                               double lam_hat, const double* c_given) {
  __shared__ double s_hv[CPA_SVT_KMAX];
  __shared__ double s_hdr[4];
  if (threadIdx.x == 0) {
    const int degen = !(lam_hat > kDegenerateLambda);
    const double lam = safety * lam_hat;
    const double sig = sqrt(lam_hat > 0.0 ? lam_hat : 0.0);
    const double tau = resolve_tau(kern, sig);
    P->lambda_hat = lam_hat;
    P->lambda_max = lam;
    P->sigma_hat = sig;
    P->tau = tau;
    P->scale2 = degen ? 0.0 : 2.0 / lam;
    P->degenerate = degen;
    P->K = K;
    P->diverged = 0;
    s_hdr[0] = lam;
    s_hdr[1] = tau;
    s_hdr[2] = degen;
  }
  __syncthreads();
  const double lam = s_hdr[0], tau = s_hdr[1];
  const bool degen = s_hdr[2] != 0.0;
  if (c_given == nullptr) {
    for (int l = threadIdx.x; l < K; l += blockDim.x) {
      const double th = cheb_theta(l + 1, K);
      s_hv[l] = h_response(kern, lam / 2.0 * (cos(th) + 1.0), tau);  // h((L/2)(cos theta_l + 1))
    }
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      double acc = 0.0;
      for (int l = 0; l < K; ++l) acc += cos(k * cheb_theta(l + 1, K)) * s_hv[l];
      P->c[k] = degen ? 0.0 : 2.0 / K * acc;
    }
  } else {
    for (int k = threadIdx.x; k < K; k += blockDim.x) P->c[k] = degen ? 0.0 : c_given[k];
  }
  __syncthreads();
}

}  // namespace cpa
