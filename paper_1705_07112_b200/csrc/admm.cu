// NEXT-3: the paper's ADMM recovery with CPA shrinkage as the nuclear-norm prox
// (PAPER.md:657-692 ADMM, PAPER.md:1193-1214 eq. admm_algorithm_inp, synthetic experiment
// PAPER.md:1095-1100 without the average-term constraint).  Elementwise kernels of one
// iteration and the DCT-II matrix builder; the products (Psi = C_m . C_n^T) run on the DMMA
// GEMM of dense_f64.cu and the prox on the CPA path -- the driver is cpa_svt_admm_recover.
#include "common.cuh"

namespace cpa {

// C[k][j] = a_k cos(pi (2j + 1) k / (2n)), a_0 = sqrt(1/n), a_k = sqrt(2/n); CT = C^T
__global__ void k_dct2(double* C, double* CT, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / n, j = e % n;
    const double a = k == 0 ? sqrt(1.0 / (double)n) : sqrt(2.0 / (double)n);
    const double v = a * cos(3.141592653589793238462643383279502884 * (double)((2 * j + 1) * k) / (double)(2 * n));
    C[k * n + j] = v;
    CT[j * n + k] = v;
  }
}

// out = a - b
__global__ void k_sub(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out, int64_t N) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = a[e] - b[e];
}

// l = ((z1 - u1) + Psi^T(z2 - u2) + w (z3 - u3) + (z4 - u4)) / (3 + w),  z3 = w D;  t = l + u1
__global__ void k_admm_l(const double* __restrict__ z1, const double* __restrict__ u1, const double* __restrict__ pt,
                         const uint8_t* __restrict__ mask, const double* __restrict__ D, const double* __restrict__ u3,
                         const double* __restrict__ z4, const double* __restrict__ u4, double* __restrict__ l,
                         double* __restrict__ t, int64_t N) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
    const double w = mask[e] ? 1.0 : 0.0;
    const double v = ((z1[e] - u1[e]) + pt[e] + w * (w * D[e] - u3[e]) + (z4[e] - u4[e])) / (3.0 + w);
    l[e] = v;
    t[e] = v + u1[e];
  }
}

// z2 = soft(Psi l + u2, thr), z4 = clip(l + u4, 0, 1), u += K l - z; per-block partial sums of
// ||l - l_prev||^2 and ||l||^2 (fixed grid and order: deterministic)
__global__ void k_admm_tail(const double* __restrict__ l, const double* __restrict__ lprev,
                            const double* __restrict__ pl, const double* __restrict__ z1, const uint8_t* __restrict__ mask,
                            const double* __restrict__ D, double* __restrict__ z2, double* __restrict__ z4,
                            double* __restrict__ u1, double* __restrict__ u2, double* __restrict__ u3,
                            double* __restrict__ u4, double thr, int64_t N, double* __restrict__ part) {
  __shared__ double s_a[8], s_b[8];
  double sa = 0.0, sb = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
    const double le = l[e], pe = pl[e];
    const double v2 = pe + u2[e];
    const double a2 = fabs(v2) - thr;
    const double z2e = a2 > 0.0 ? copysign(a2, v2) : 0.0;
    const double v4 = le + u4[e];
    const double z4e = v4 < 0.0 ? 0.0 : (v4 > 1.0 ? 1.0 : v4);
    const double w = mask[e] ? 1.0 : 0.0;
    z2[e] = z2e;
    z4[e] = z4e;
    u1[e] += le - z1[e];
    u2[e] += pe - z2e;
    u3[e] += w * le - w * D[e];
    u4[e] += le - z4e;
    const double d = le - lprev[e];
    sa = fma(d, d, sa);
    sb = fma(le, le, sb);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_a[threadIdx.x >> 5] = sa;
    s_b[threadIdx.x >> 5] = sb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += s_a[w];
      b += s_b[w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

constexpr int kAdmmBlocks = 296, kAdmmThreads = 256;

cudaError_t admm_dct(double* C, double* CT, int64_t n, int num_sms, cudaStream_t st) {
  k_dct2<<<num_sms * 4, 256, 0, st>>>(C, CT, n);
  return cudaGetLastError();
}
cudaError_t admm_sub(const double* a, const double* b, double* out, int64_t N, cudaStream_t st) {
  k_sub<<<kAdmmBlocks * 2, kAdmmThreads, 0, st>>>(a, b, out, N);
  return cudaGetLastError();
}
cudaError_t admm_l(const double* z1, const double* u1, const double* pt, const uint8_t* mask, const double* D,
                   const double* u3, const double* z4, const double* u4, double* l, double* t, int64_t N,
                   cudaStream_t st) {
  k_admm_l<<<kAdmmBlocks * 2, kAdmmThreads, 0, st>>>(z1, u1, pt, mask, D, u3, z4, u4, l, t, N);
  return cudaGetLastError();
}
int admm_tail_blocks() { return kAdmmBlocks; }
cudaError_t admm_tail(const double* l, const double* lprev, const double* pl, const double* z1, const uint8_t* mask,
                      const double* D, double* z2, double* z4, double* u1, double* u2, double* u3, double* u4,
                      double thr, int64_t N, double* part, cudaStream_t st) {
  k_admm_tail<<<kAdmmBlocks, kAdmmThreads, 0, st>>>(l, lprev, pl, z1, mask, D, z2, z4, u1, u2, u3, u4, thr, N, part);
  return cudaGetLastError();
}

}  // namespace cpa
