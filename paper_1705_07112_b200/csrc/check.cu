// Divergence check of the recurrence (status CPA_SVT_E_DIVERGED of cpa_svt.h).
//
// The Chebyshev series is only bounded on [-1, 1] (eq.
// cheby_matrix_eigen_saiki3: |psi_k(x)| <= 1 there, cosh(k acosh x) outside), so a
// Lambda_max below the true top eigenvalue of the Gram (an override, or an unconverged
// power iteration) makes Psi_k grow geometrically.  After the output is written the
// library checks ||Y||_F <= 1e3 * sum_k |c_k| * ||X||_F; a NaN or Inf
// anywhere in Y fails the comparison too.  The sums of squares are block partials added
// in a fixed order (deterministic), and the verdict lands in SeriesParams::diverged,
// which the host reads when the call synchronises (fill_info in api.cu).
#include <type_traits>

#include "common.cuh"

namespace cpa {

constexpr int kCheckThreads = 256;
constexpr int kCheckBlocks = 148;   // per matrix (grid y: 0 = X, 1 = Y); one HBM pass over each

// Block partials of the sums of squares of X (blockIdx.y = 0) and Y (1), rows x cols row-major with
// leading dimensions; the last block to finish adds the partials in a fixed order (deterministic)
// and writes the verdict.  One launch.
template <class T>
__global__ void __launch_bounds__(kCheckThreads) k_divcheck(const T* __restrict__ X, int64_t xr, int64_t xc,
                                                            int64_t ldx, const T* __restrict__ Y, int64_t yr,
                                                            int64_t yc, int64_t ldy, double* __restrict__ part,
                                                            unsigned int* __restrict__ done, SeriesParams* P) {
  __shared__ double red[kCheckThreads / 32];
  __shared__ bool last;
  const bool isy = blockIdx.y == 1;
  const T* A = isy ? Y : X;
  const int64_t rows = isy ? yr : xr, cols = isy ? yc : xc, ld = isy ? ldy : ldx;
  double acc = 0.0;
  const int64_t n = rows * cols;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  constexpr int VW = 16 / sizeof(T);   // elements per 16-byte load
  if (ld == cols && (reinterpret_cast<uintptr_t>(A) & 15) == 0) {
    // 16-byte loads, four in flight per thread (c2: 10.7 -> ~3 us per check)
    using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    const V* A4 = reinterpret_cast<const V*>(A);
    const int64_t nv = n / VW;
    double a4[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; e + 3 * stride < nv; e += 4 * stride) {
      V v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(A4 + e + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const T* x = reinterpret_cast<const T*>(&v[u]);
#pragma unroll
        for (int i = 0; i < VW; ++i) a4[u] += (double)x[i] * (double)x[i];
      }
    }
    for (; e < nv; e += stride) {
      const V v = __ldcs(A4 + e);
      const T* x = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (int i = 0; i < VW; ++i) a4[0] += (double)x[i] * (double)x[i];
    }
    for (int64_t t = nv * VW + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += stride) {
      const double v = (double)A[t];
      a4[0] += v * v;
    }
    acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
  } else if (ld == cols) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += stride) {
      const double v = (double)A[e];
      acc += v * v;
    }
  } else {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += stride) {
      const double v = (double)A[(e / cols) * ld + e % cols];
      acc += v * v;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kCheckThreads / 32; ++w) s += red[w];
    part[blockIdx.y * kCheckBlocks + blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(done, 1u) == 2u * kCheckBlocks - 1u;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // warp 0 sums X's partials, warp 1 Y's, warp 2 sum |c_k|: lane-strided then a fixed butterfly
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v = 0.0;
  if (warp < 2) {
    for (int b = lane; b < kCheckBlocks; b += 32) v += __ldcg(part + warp * kCheckBlocks + b);
  } else if (warp == 2) {
    for (int k = lane; k < P->K; k += 32) v += fabs(P->c[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0 && warp < 3) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    const double bound = 1e3 * red[2] * sqrt(red[0]);
    const double ny = sqrt(red[1]);
    P->diverged = (P->degenerate || ny <= bound) ? 0 : 1;   // NaN / Inf in Y: not <=, so diverged
    *done = 0u;                                              // ready for the next call
  }
}

// Scratch: 2 * kCheckBlocks partials + the arrival counter (zeroed once by the caller).
size_t divergence_scratch_doubles() { return 2 * kCheckBlocks + 2; }

template <class T>
static cudaError_t check_impl(const T* X, int64_t xr, int64_t xc, int64_t ldx, const T* Y, int64_t yr, int64_t yc,
                              int64_t ldy, double* scratch, SeriesParams* P, cudaStream_t st) {
  k_divcheck<T><<<dim3(kCheckBlocks, 2), kCheckThreads, 0, st>>>(
      X, xr, xc, ldx, Y, yr, yc, ldy, scratch, (unsigned int*)(scratch + 2 * kCheckBlocks), P);
  return cudaGetLastError();
}

cudaError_t divergence_check_f64(const double* X, int64_t xr, int64_t xc, int64_t ldx, const double* Y, int64_t yr,
                                 int64_t yc, int64_t ldy, double* scratch, SeriesParams* P, cudaStream_t st) {
  return check_impl<double>(X, xr, xc, ldx, Y, yr, yc, ldy, scratch, P, st);
}

cudaError_t divergence_check_f32(const float* X, int64_t xr, int64_t xc, int64_t ldx, const float* Y, int64_t yr,
                                 int64_t yc, int64_t ldy, double* scratch, SeriesParams* P, cudaStream_t st) {
  return check_impl<float>(X, xr, xc, ldx, Y, yr, yc, ldy, scratch, P, st);
}

}  // namespace cpa
