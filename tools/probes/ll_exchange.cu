// Probe: per-iteration cost of the power iteration's LL all-gather on B200, without
// and with the per-product block reduction of k_power_reg (paper_1705_07112_b200/csrc/power.cu).
//   mode 0: publish ROWS values (LL words) + gather s values (P polling lanes) + barrier
//   mode 1: mode 0 + one block reduction of ROWS+1 values (2 barriers, warp butterflies)
//   mode 2: mode 1 + fp64 sqrt and reciprocal
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/ll_exchange tools/probes/ll_exchange.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_ll(unsigned long long* p, double v, unsigned flag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = ((unsigned long long)flag << 32) | (b >> 32);
  const unsigned long long w1 = ((unsigned long long)flag << 32) | (b & 0xffffffffull);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ void ld_ll(const unsigned long long* p, unsigned long long& w0, unsigned long long& w1) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int ROWS = 7;
__global__ void __launch_bounds__(256) k(unsigned long long* ll, int s, int iters, int mode, int np,
                                         long long* out) {
  __shared__ double sv[4096];
  __shared__ double s_part[8][ROWS + 1];
  __shared__ double s_res[ROWS + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blockIdx.x * ROWS;
  double x = 1.0 + threadIdx.x;
  long long t0 = clock64();
  for (int t = 0; t < iters; ++t) {
    double res = x;
    if (mode >= 1) {
      double p[ROWS + 1];
#pragma unroll
      for (int r = 0; r <= ROWS; ++r) p[r] = warp_sum(x * (r + 1));
      if (lane == 0)
#pragma unroll
        for (int r = 0; r <= ROWS; ++r) s_part[warp][r] = p[r];
      __syncthreads();
      if (threadIdx.x <= ROWS) {
        double acc = s_part[0][threadIdx.x];
        for (int w = 1; w < 8; ++w) acc += s_part[w][threadIdx.x];
        s_res[threadIdx.x] = acc;
      }
      __syncthreads();
      res = threadIdx.x < ROWS ? s_res[threadIdx.x] : 0.0;
      if (mode >= 2) res *= 1.0 / sqrt(s_res[ROWS] + 1.0);
    }
    const unsigned flag = (unsigned)t + 1u;
    unsigned long long* buf = ll + (size_t)(t & 1) * s * 2;
    if (threadIdx.x < ROWS && r0 + threadIdx.x < s) st_ll(buf + 2 * (r0 + threadIdx.x), res, flag);
    if (threadIdx.x < np) {
      for (int j0 = 0; j0 < s; j0 += np * 8) {
        unsigned long long w[8][2];
        unsigned pending = 0;
        for (int c = 0; c < 8; ++c)
          if (j0 + threadIdx.x + np * c < s) pending |= 1u << c;
        while (pending) {
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (pending & (1u << c)) ld_ll(buf + 2 * (j0 + threadIdx.x + np * c), w[c][0], w[c][1]);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if ((pending & (1u << c)) && (unsigned)(w[c][0] >> 32) == flag && (unsigned)(w[c][1] >> 32) == flag)
              pending &= ~(1u << c);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (j0 + threadIdx.x + np * c < s)
            sv[j0 + threadIdx.x + np * c] =
                __longlong_as_double((long long)(((w[c][0] & 0xffffffffull) << 32) | (w[c][1] & 0xffffffffull)));
      }
    }
    __syncthreads();
    x = sv[(threadIdx.x * 7 + t) % s] * 0.5 + 0.25;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  unsigned long long* ll;
  long long* out;
  cudaMalloc(&ll, 1 << 20);
  cudaMalloc(&out, 4096);
  const int iters = 2000;
  for (int s : {1024, 48})
    for (int np : {128, 256})
      for (int mode = 0; mode < 3; ++mode) {
        const int grid = (s + ROWS - 1) / ROWS;
        cudaMemset(ll, 0, 1 << 20);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        void* args[] = {&ll, (void*)&s, (void*)&iters, &mode, (void*)&np, &out};
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchCooperativeKernel((void*)k, dim3(grid), dim3(256), args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("s=%d grid=%d np=%d mode=%d: %.3f us/iter (%s)\n", s, grid, np, mode, ms * 1e3 / iters,
               cudaGetErrorString(e));
      }
  return 0;
}
