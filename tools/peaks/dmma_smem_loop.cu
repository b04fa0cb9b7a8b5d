// Upper bound of the k_cheb_sym mainloop without its per-slab barriers and cp.async:
// every warp streams its 4 x 4 DMMA.8x8x4 fragments from a FIXED shared-memory slab with the
// exact addressing of mainloop() (LD = 68 doubles, A / B non-K-contiguous), 3 CTAs x 4 warps
// per SM.  Compare with the DMMA-only loop peak (37.16 TF/s) and the kernel's 82 % (c5).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <bool SYNC>
__global__ void __launch_bounds__(128, 3) k(double* out, int iters) {
  __shared__ double sA[16 * 68], sB[16 * 68];
  for (int i = threadIdx.x; i < 16 * 68; i += 128) { sA[i] = 1e-3 * i; sB[i] = 2e-3 * i; }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2] = {};
  for (int it = 0; it < iters; ++it) {
    if (SYNC) __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = sA[(kk + t) * 68 + wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = sB[(kk + t) * 68 + wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
  out[blockIdx.x * 128 + threadIdx.x] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 3 * 128 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  // resident CTAs per SM: 1, 2, 3 (the grid is 148 x cps; 3 fit by registers)
  for (int cps = 1; cps <= 3; ++cps)
    for (int sync = 0; sync < 2; ++sync)
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (sync) k<true><<<148 * cps, 128>>>(out, iters); else k<false><<<148 * cps, 128>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 2.0 * 64 * 64 * 16 * (double)iters * 148 * cps;
        if (rep) printf("smem-fed DMMA loop, %d CTA(s)/SM, %s: %.2f TFLOP/s\n", cps,
                        sync ? "__syncthreads per slab" : "no barrier", fl / ms / 1e9);
      }
  return 0;
}
