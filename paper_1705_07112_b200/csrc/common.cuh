// Internal definitions shared by the CUDA translation units of libcpasvt.
// Product code only: nothing here is shared with oracle/ (which is Python).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <stdlib.h>
#include <stdio.h>

#include "cpa_svt.h"

namespace cpa {

constexpr double kDegenerateLambda = 1e-300;  // SPEC.md:287 / reading R17

// Series parameters produced on the device by the power-iteration tail and
// consumed by every recurrence kernel (no host round trip; reading R6/R7).
struct SeriesParams {
  double lambda_hat;   // power-iteration estimate (or override / safety)
  double lambda_max;   // safety * lambda_hat
  double sigma_hat;    // sqrt(lambda_hat)
  double tau;          // resolved absolute threshold
  double scale2;       // 2 / lambda_max  (0 when degenerate)
  int32_t degenerate;  // lambda_hat <= 1e-300
  int32_t K;
  int32_t diverged;    // set by the divergence check (check.cu) after the recurrence, reset by compute_series
  int32_t pad_;
  double c[CPA_SVT_KMAX];
};

// Profiling hook for multi-kernel phases: begin = 1 before, 0 after the launches.
typedef void (*SparsePhaseHook)(void* ctx, int phase, int begin);

// ---- the response h(x) of PAPER.md:496-519 (host and device) --------------
__host__ __device__ inline double h_response(const cpa_svt_kernel& k, double x, double tau) {
  const double r = sqrt(x);
  switch (k.kind) {
    case CPA_SVT_HARD:
      return r > tau ? 1.0 : 0.0;
    case CPA_SVT_SOFT:
      return r > tau ? (r - tau) / r : 0.0;
    default: {  // CPA_SVT_WSOFT
      const double xs = x - k.w_shift;
      const double w = k.w_c / (sqrt(xs > 0.0 ? xs : 0.0) + k.w_eps);
      return r > w ? (r - w) / r : 0.0;
    }
  }
}

__host__ __device__ inline double resolve_tau(const cpa_svt_kernel& k, double sigma_hat) {
  return k.tau_relative ? k.tau * sigma_hat : k.tau;
}

// Chebyshev-Gauss node l (1-based) of order K: theta_l = pi (l - 1/2) / K.
__host__ __device__ inline double cheb_theta(int l, int K) {
  return 3.141592653589793238462643383279502884 * ((double)l - 0.5) / (double)K;
}

// ---- checked builds (build.py --variant checked CPA_SVT_CHECKED=1): device-side bounds checks
// on the gathers / scatters whose indices come from data (CSR / CSC, tile decodes, all-gather
// slots); a failed check prints the site and traps.  compute-sanitizer is not available on the
// GPU pool, so this build plus the workspace guard bands (CPA_SVT_GUARD) stand in for memcheck.
#ifdef CPA_SVT_CHECKED
#define CPA_DCHECK(c)                                                                       \
  do {                                                                                      \
    if (!(c)) {                                                                             \
      printf("CPA_DCHECK failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__,  \
             (int)blockIdx.x, (int)threadIdx.x);                                            \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define CPA_DCHECK(c) \
  do {                \
  } while (0)
#endif

// Resident CTAs per SM of a kernel from its attributes and the device limits (registers in
// per-warp units of 8, shared memory with the 1 KB the system reserves per CTA, warps, CTA slots).
// cudaOccupancyMaxActiveBlocksPerMultiprocessor reports 1 for the tcgen05 batched kernel and the
// warp-specialized recurrence on this driver while 4 / 2 CTAs are measured resident (and run): the
// persistent launches size their grids with this instead.
inline int resident_ctas(const void* func, int threads, size_t dyn_smem, int device) {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, func) != cudaSuccess) return 1;
  int regs_sm = 65536, smem_sm = 233472, warps_sm = 64, blocks_sm = 32, reserved = 1024;
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, device);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  cudaDeviceGetAttribute(&blocks_sm, cudaDevAttrMaxBlocksPerMultiprocessor, device);
  cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, device);
  int tpm = 2048;
  cudaDeviceGetAttribute(&tpm, cudaDevAttrMaxThreadsPerMultiProcessor, device);
  warps_sm = tpm / 32;
  const int warps = (threads + 31) / 32;
  const int regs_warp = ((fa.numRegs + 7) / 8) * 8 * 32;
  int n = blocks_sm;
  if (regs_warp > 0) n = n < regs_sm / (regs_warp * warps) ? n : regs_sm / (regs_warp * warps);
  n = n < warps_sm / warps ? n : warps_sm / warps;
  const size_t per = fa.sharedSizeBytes + dyn_smem + (size_t)reserved;
  if (per > 0) n = n < (int)(smem_sm / per) ? n : (int)(smem_sm / per);
  return n > 0 ? n : 1;
}

// ---- small PTX helpers --------------------------------------------------------
// Experiment switches: true iff the environment variable is set to a non-empty value other than "0".
inline bool env_on(const char* name) {
  const char* v = getenv(name);
  return v != nullptr && v[0] != '\0' && !(v[0] == '0' && v[1] == '\0');
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8-byte async copy with zero fill when !pred (src-size 0).
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(pred ? 8 : 0));
}
// 16-byte async copy (L2 only) with zero fill when !pred.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D = A(8x4, row) * B(4x8, col) + C, fp64 tensor core (SASS DMMA.8x8x4).
// Lane l holds A[l/4][l%4], B[l%4][l/4], C[l/4][2(l%4)], C[l/4][2(l%4)+1].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Sense-free generation barrier for a cooperative (co-resident) grid.
// count: arrivals this generation (reset by the last arriver); gen: generation.
__device__ __forceinline__ void grid_barrier(unsigned int* count, volatile unsigned int* gen,
                                             unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd((unsigned int*)gen, 1u);
    } else {
      while (*gen == g) {
        __nanosleep(32);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

}  // namespace cpa
