// Microbenchmark: cost of one iteration of the cooperative power-iteration
// structure (grid-wide counter barrier + all-gather of an s-vector) on B200.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void red_release(unsigned* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

// mode 0: barrier only; 1: barrier + stage s doubles; 2: + GEMV on 7 cached rows
__global__ void k(unsigned* bar, double* u, int s, int iters, int mode, long long* out) {
  extern __shared__ double sv[];
  const unsigned nb = gridDim.x;
  long long t0 = clock64();
  for (int t = 0; t < iters; ++t) {
    if (mode >= 2) {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      double d = 0;
      for (int j = lane; j < s; j += 32) d = fma(sv[j], sv[(j + warp) % s], d);
      if (lane == 0 && warp < 7) u[blockIdx.x * 7 + warp] = d;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      red_release(bar);
      const unsigned target = nb * (unsigned)(t + 1);
      while (ld_relaxed(bar) < target) {}
      __threadfence();
    }
    __syncthreads();
    if (mode >= 1) {
      for (int j = threadIdx.x; j < s; j += blockDim.x) sv[j] = __ldcg(u + j);
      __syncthreads();
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
  unsigned* bar; double* u; long long* out;
  cudaMalloc(&bar, 256); cudaMalloc(&u, 1 << 20); cudaMalloc(&out, 64);
  cudaMemset(u, 0, 1 << 20);
  int s = 1024, iters = 1000;
  for (int grid : {16, 64, 148}) for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(bar, 0, 256);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, s * 8);
    void* args[] = {&bar, &u, &s, &iters, &mode, &out};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k, dim3(grid), dim3(256), args, s * 8, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long cyc; cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    printf("grid %3d mode %d: %.3f us/iter (%lld cycles/iter) %s\n", grid, mode, ms * 1000 / iters, cyc / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
