// Lambda_max by power iteration (Alg. 1 line 3; reading R6) and
// the Chebyshev coefficients (Alg. 1 line 4, PAPER.md:363 / eq. 233), both on
// the device so the recurrence never waits for the host.
//
// k_power_dense: one cooperative persistent launch for all T products.  Each
// CTA owns a contiguous block of Gram rows (cached in shared memory when they
// fit), stages v_{t-1} in shared memory, computes its rows of u_t = G v_{t-1}
// with one warp per row, publishes u_t and its partial sum of squares, and
// meets the other CTAs at a grid barrier.  ||u_t|| is re-summed by every CTA
// in the same fixed order, so all CTAs agree bitwise.  The last barrier is
// followed by the coefficient computation in CTA 0.
#include "common.cuh"

namespace cpa {

// Fill P from lambda_hat (block-wide; all threads of the calling block must enter).
__device__ void compute_series(SeriesParams* P, const cpa_svt_kernel& kern, int K, double safety,
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

// lam_hat from *lam_src if non-null, else lam_override / safety.
__global__ void k_series(SeriesParams* P, cpa_svt_kernel kern, int K, double safety, double lam_override,
                         const double* lam_src, const double* c_given) {
  const double lh = lam_src ? *lam_src : lam_override / safety;
  compute_series(P, kern, K, safety, lh, c_given);
}

struct PowerArgs {
  const double* G;
  int64_t s;
  int T;
  double* ubuf;      // 2 * s
  double* part;      // 2 * gridDim.x
  unsigned int* bar; // [count, gen]
  SeriesParams* P;
  cpa_svt_kernel kern;
  int K;
  double safety;
  const double* c_given;
  int cache_rows;    // 1: this CTA's rows of G live in shared memory
  int rows_per_cta;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(256) k_power_dense(PowerArgs a) {
  extern __shared__ __align__(16) double psm[];
  __shared__ double s_warp[8];
  __shared__ double s_norm;
  const int64_t s = a.s;
  double* sv = psm;               // v (s doubles)
  double* sg = psm + s;           // cached rows (rows_per_cta * s) if cache_rows
  const int64_t r0 = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t r1 = min(s, r0 + a.rows_per_cta);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  if (a.cache_rows) {
    for (int64_t e = threadIdx.x; e < (r1 - r0) * s; e += blockDim.x) sg[e] = a.G[r0 * s + e];
  }
  const double v0 = 1.0 / sqrt((double)s);
  double inv = 0.0;
  double lam = 0.0;
  for (int t = 0; t < a.T; ++t) {
    // stage v_{t-1} = u_{t-1} / ||u_{t-1}|| (v_0 = 1/sqrt(s))
    const double* up = a.ubuf + ((t + 1) & 1) * s;
    for (int64_t j = threadIdx.x; j < s; j += blockDim.x) sv[j] = t == 0 ? v0 : __ldcg(up + j) * inv;
    __syncthreads();
    double mysq = 0.0;
    for (int64_t r = r0 + warp; r < r1; r += nwarps) {
      const double* grow = a.cache_rows ? sg + (r - r0) * s : a.G + r * s;
      double d = 0.0;
      for (int64_t j = lane; j < s; j += 32) d += grow[j] * sv[j];
      d = warp_sum(d);
      if (lane == 0) a.ubuf[(t & 1) * s + r] = d;
      mysq += d * d;  // identical in all lanes
    }
    if (lane == 0) s_warp[warp] = mysq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double p = 0.0;
      for (int w = 0; w < nwarps; ++w) p += s_warp[w];
      a.part[(t & 1) * gridDim.x + blockIdx.x] = p;
    }
    grid_barrier(a.bar, a.bar + 1, gridDim.x);
    if (threadIdx.x == 0) {
      double ss = 0.0;
      const double* pp = a.part + (t & 1) * gridDim.x;
      for (unsigned b = 0; b < gridDim.x; ++b) ss += __ldcg(pp + b);
      s_norm = sqrt(ss);
    }
    __syncthreads();
    lam = s_norm;
    if (!(lam > kDegenerateLambda)) { lam = 0.0; break; }
    inv = 1.0 / lam;
  }
  if (blockIdx.x == 0) compute_series(a.P, a.kern, a.K, a.safety, lam, a.c_given);
}

cudaError_t launch_series(SeriesParams* P, const cpa_svt_kernel& k, int K, double safety, double lam_override,
                          const double* lam_src, const double* c_given, cudaStream_t st) {
  k_series<<<1, 256, 0, st>>>(P, k, K, safety, lam_override, lam_src, c_given);
  return cudaGetLastError();
}

// Scratch needed by launch_power_dense (doubles): 2 s + 2 * 148 * 8, plus 2 uints.
size_t power_dense_scratch_doubles(int64_t s) { return (size_t)(2 * s + 2 * 2048); }

cudaError_t launch_power_dense(const double* G, int64_t s, int T, double* scratch, unsigned int* bar,
                               SeriesParams* P, const cpa_svt_kernel& k, int K, double safety,
                               const double* c_given, int num_sms, cudaStream_t st) {
  PowerArgs a{};
  a.G = G; a.s = s; a.T = T;
  a.ubuf = scratch; a.part = scratch + 2 * s;
  a.bar = bar; a.P = P; a.kern = k; a.K = K; a.safety = safety; a.c_given = c_given;
  int grid = (int)(s < num_sms ? s : num_sms);
  if (grid < 1) grid = 1;
  if (grid > 1024) grid = 1024;
  a.rows_per_cta = (int)((s + grid - 1) / grid);
  grid = (int)((s + a.rows_per_cta - 1) / a.rows_per_cta);
  const size_t budget = 200 * 1024;
  size_t smem = (size_t)s * sizeof(double);
  if (smem > budget) return cudaErrorInvalidValue;  // s > 25600 not supported by this kernel
  const size_t cached = smem + (size_t)a.rows_per_cta * s * sizeof(double);
  a.cache_rows = cached <= budget;
  if (a.cache_rows) smem = cached;
  cudaError_t e = cudaFuncSetAttribute(k_power_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((void*)k_power_dense, dim3(grid), dim3(256), args, smem, st);
}

}  // namespace cpa
