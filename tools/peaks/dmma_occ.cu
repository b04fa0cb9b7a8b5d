// DMMA throughput vs warps per SMSP (independent 8x8x4 f64 MMAs, 16 accumulators per warp)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wps : {1, 2, 3, 4, 8}) {  // warps per SMSP
    int thr = 128 * wps; int iters = 4000;
    k<<<148, thr>>>(d, 10);
    cudaEventRecord(e0); k<<<148, thr>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 16 * (double)iters * 148 * (thr / 32);
    printf("warps/SMSP %d: %.2f TFLOP/s\n", wps, fl / ms / 1e9);
  }
}
