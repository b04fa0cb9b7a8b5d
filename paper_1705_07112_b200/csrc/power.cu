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

template <typename E>
struct PowerArgs {
  const E* G;
  const E* G4;       // c^4 G^4 (nullable): first q products use it
  int q;             // products by G4
  int64_t s;
  int64_t ld;        // row stride of G / G4 (elements)
  int T;
  double* ubuf;      // 2 * s
  double* part;      // 2 * gridDim.x
  unsigned int* bar; // monotonic arrival counter (zeroed before the launch)
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

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned int* p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

template <typename E>
__global__ void __launch_bounds__(256) k_power_dense(PowerArgs<E> a) {
  using T = E;
  extern __shared__ __align__(16) double psm[];
  __shared__ double s_warp[8];
  __shared__ double s_norm;
  const int64_t s = a.s;
  double* sv = psm;               // v_{t-1} (s doubles)
  T* sg = reinterpret_cast<T*>(psm + s);  // cached rows (rows_per_cta * s) if cache_rows
  const int64_t r0 = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t r1 = min(s, r0 + a.rows_per_cta);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const unsigned int nb = gridDim.x;
  // products: q by G4 (cached when present), then T - 4q by G; the last one gives lambda_hat
  const T* Gc = a.q > 0 ? a.G4 : a.G;  // the matrix whose rows are cached
  const int niter = a.T - 3 * a.q;
  if (a.cache_rows) {
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t j = threadIdx.x; j < s; j += blockDim.x) sg[(r - r0) * s + j] = Gc[r * a.ld + j];
  }
  const double v0 = 1.0 / sqrt((double)s);
  for (int64_t j = threadIdx.x; j < s; j += blockDim.x) sv[j] = v0;
  __syncthreads();
  double lam = 0.0;
  double inv = 1.0;  // 1/||u_{t-1}||, folded into this product (v_{t-1} = u_{t-1} * inv)
  for (int t = 0; t < niter; ++t) {
    const bool use4 = t < a.q;
    const T* Gt = use4 ? a.G4 : a.G;
    const bool cached = a.cache_rows && (use4 || a.q == 0);
    // u_t = G v_{t-1}: one warp per row, 8 independent partial sums per lane
    for (int64_t r = r0 + warp; r < r1; r += nwarps) {
      const T* grow = cached ? sg + (r - r0) * s : Gt + r * a.ld;
      double d[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int64_t j = lane;
      for (; j + 224 < s; j += 256) {
#pragma unroll
        for (int q = 0; q < 8; ++q) d[q] = fma((double)grow[j + 32 * q], sv[j + 32 * q], d[q]);
      }
      for (; j < s; j += 32) d[0] = fma((double)grow[j], sv[j], d[0]);
      const double dd = warp_sum(((d[0] + d[1]) + (d[2] + d[3])) + ((d[4] + d[5]) + (d[6] + d[7]))) * inv;
      if (lane == 0) a.ubuf[(t & 1) * s + r] = dd;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // arrive (release, cumulative over the bar.sync above): publishes this CTA's rows of u_t
      red_release_add(a.bar, 1u);
      const unsigned int target = nb * (unsigned)(t + 1);
      while (ld_relaxed_u32(a.bar) < target) {
      }
      __threadfence();  // acquire: the other CTAs' rows of u_t are visible below
    }
    __syncthreads();
    // stage u_t (all loads in flight before the first store) and ||u_t||^2 from the staged copy:
    // every CTA sums the same values in the same fixed order, so all agree bitwise.
    // v_t = u_t / ||u_t|| is applied inside the next product.
    const double* up = a.ubuf + (t & 1) * s;
    double sq = 0.0;
    for (int64_t j0 = 0; j0 < s; j0 += 8 * blockDim.x) {
      double uv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t j = j0 + threadIdx.x + (int64_t)i * blockDim.x;
        uv[i] = j < s ? __ldcg(up + j) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t j = j0 + threadIdx.x + (int64_t)i * blockDim.x;
        if (j < s) sv[j] = uv[i];
        sq = fma(uv[i], uv[i], sq);
      }
    }
    sq = warp_sum(sq);
    if (lane == 0) s_warp[warp] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double q = 0.0;
      for (int w = 0; w < nwarps; ++w) q += s_warp[w];
      s_norm = sqrt(q);
    }
    __syncthreads();
    lam = s_norm;
    if (!(lam > kDegenerateLambda) || !(lam < 1e300)) { lam = lam < 1e300 ? 0.0 : lam; break; }
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
size_t power_dense_scratch_doubles(int64_t s) { return (size_t)(2 * s + 4096 + 8); }

// c = 2^-e with e = ilogb(max_i G_ii): G_ii <= lambda_max <= s * max_i G_ii, so
// c^4 G^4 has its dominant eigenvalue in [1/16, 16 s^4]: no overflow/underflow.
__global__ void k_diag_scale(const double* G, int64_t s, double* scale) {
  __shared__ double red[256];
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < s; i += blockDim.x) mx = fmax(mx, G[i * s + i]);
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double m = red[0];
    const int e = (m > 0.0 && isfinite(m)) ? ilogb(m) : 0;
    scale[0] = ldexp(1.0, -2 * e);  // applied to G^2 (one factor c^2)
  }
}

cudaError_t launch_diag_scale(const double* G, int64_t s, double* scale, cudaStream_t st) {
  k_diag_scale<<<1, 256, 0, st>>>(G, s, scale);
  return cudaGetLastError();
}

// Squaring pays when two s^3 products cost less than the ~3T/4 products saved,
// each of which is latency-bound (~2.5 us) for small s.
bool power_use_squaring(int64_t s, int T) {
  if (T < 16) return false;
  const double gemm_us = 2.0 * (double)s * s * s / 25e12 * 1e6;
  const double iter_us = fmax(2.5, 8.0 * (double)s * s / 5e12 * 1e6);
  return gemm_us < 0.75 * T * iter_us;
}

template <typename E>
static cudaError_t launch_power_t(const E* G, const E* G4, int64_t s, int64_t ld, int T, double* scratch,
                                  unsigned int* bar, SeriesParams* P, const cpa_svt_kernel& k, int K, double safety,
                                  const double* c_given, int num_sms, cudaStream_t st) {
  PowerArgs<E> a{};
  a.ld = ld;
  a.G = G; a.s = s; a.T = T;
  a.G4 = G4;
  a.q = G4 ? (T - 1) / 4 : 0;
  a.ubuf = scratch; a.part = scratch + 2 * s;
  a.bar = bar; a.P = P; a.kern = k; a.K = K; a.safety = safety; a.c_given = c_given;
  // Fewest CTAs whose rows of G fit in shared memory (fewer arrivals per
  // barrier); otherwise one CTA per SM streaming its rows from L2/HBM.
  const size_t budget = 200 * 1024;
  size_t smem = (size_t)s * sizeof(double);
  if (smem > budget) return cudaErrorInvalidValue;  // s > 25600 not supported by this kernel
  // One CTA per SM (the product is latency-bound: fewer rows per CTA shortens
  // it); rows cached in shared memory when they fit.
  int64_t grid = s < num_sms ? s : num_sms;
  const int64_t rows_per = (s + grid - 1) / grid;
  a.cache_rows = smem + (size_t)rows_per * s * sizeof(E) <= budget;
  if (grid < 1) grid = 1;
  a.rows_per_cta = (int)((s + grid - 1) / grid);
  grid = (s + a.rows_per_cta - 1) / a.rows_per_cta;
  if (a.cache_rows) smem += (size_t)a.rows_per_cta * s * sizeof(E);
  cudaError_t e0 = cudaMemsetAsync(bar, 0, sizeof(unsigned int), st);
  if (e0 != cudaSuccess) return e0;
  cudaError_t e = cudaFuncSetAttribute(k_power_dense<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((void*)k_power_dense<E>, dim3((unsigned)grid), dim3(256), args, smem, st);
}

cudaError_t launch_power_dense(const double* G, const double* G4, int64_t s, int T, double* scratch,
                               unsigned int* bar, SeriesParams* P, const cpa_svt_kernel& k, int K, double safety,
                               const double* c_given, int num_sms, cudaStream_t st) {
  return launch_power_t<double>(G, G4, s, s, T, scratch, bar, P, k, K, safety, c_given, num_sms, st);
}
// fp32 Gram (TF32 path): the products are accumulated in fp64 all the same
cudaError_t launch_power_dense_f32(const float* G, int64_t s, int64_t ld, int T, double* scratch, unsigned int* bar,
                                   SeriesParams* P, const cpa_svt_kernel& k, int K, double safety,
                                   const double* c_given, int num_sms, cudaStream_t st) {
  return launch_power_t<float>(G, nullptr, s, ld, T, scratch, bar, P, k, K, safety, c_given, num_sms, st);
}

}  // namespace cpa
