// Microbenchmarks for the roofline denominators this path needs and that
// MEASURED_PEAKS.json does not carry: FP64 DFMA, FP64 DMMA (mma.sync f64),
// FP32 FFMA.  Each kernel runs a long dependent-free loop on every SM.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <int ILP>
__global__ void k_ffma(float* out, int iters, float a, float b) {
  float acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678f) out[0] = s;
}

template <int ILP>
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// FFMA with all three sources in (distinct, thread-varying) registers: the form a
// register-tiled outer-product GEMM issues.
template <int ILP>
__global__ void k_ffma3(float* out, int iters) {
  float acc[ILP], a[4], b[4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) { a[i] = 0.999f - threadIdx.x * 1e-6f * i; b[i] = 1e-3f * (i + 1) + threadIdx.x * 1e-7f; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fmaf(a[i & 3], b[(i >> 2) & 3], acc[i]);
#pragma unroll
    for (int i = 0; i < 4; ++i) { a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1) * 1.0000001f; }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678f) out[0] = s;
}

// packed dual FP32 FMA (fma.rn.f32x2 -> SASS FFMA2), register operands varying per thread
template <int ILP>
__global__ void k_ffma2(float* out, int iters) {
  unsigned long long acc[ILP], a[4], b[4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { float2 v = make_float2(threadIdx.x * 1e-3f + i, -i); acc[i] = *(unsigned long long*)&v; }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 va = make_float2(0.999f - threadIdx.x * 1e-6f * i, 0.998f), vb = make_float2(1e-3f * (i + 1), threadIdx.x * 1e-7f);
    a[i] = *(unsigned long long*)&va; b[i] = *(unsigned long long*)&vb;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i]) : "l"(a[i & 3]), "l"(b[(i >> 2) & 3]));
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] ^= (unsigned long long)(it & 1);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) { float2 v = *(float2*)&acc[i]; s += v.x + v.y; }
  if (s == 12345.678f) out[0] = s;
}

int main() {
  int dev = 0, nsm = 0, clk = 0, l2 = 0, smem = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  double* dout; CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int iters = 20000;
  printf("{\"sms\": %d, \"clock_khz\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %d", nsm, clk, l2, smem);
  for (int blocks_per_sm : {1, 2, 4}) {
    int grid = nsm * blocks_per_sm, thr = 512;
    k_dfma<8><<<grid, thr>>>(dout, 100, 0.999, 1e-3);
    cudaEventRecord(e0); k_dfma<8><<<grid, thr>>>(dout, iters, 0.999, 1e-3); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)grid * thr;
    printf(", \"dfma_tflops_b%d\": %.3f", blocks_per_sm, fl / ms / 1e9);
    k_dmma<8><<<grid, thr>>>(dout, 100);
    cudaEventRecord(e0); k_dmma<8><<<grid, thr>>>(dout, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 8 * iters * (double)grid * (thr / 32);
    printf(", \"dmma_tflops_b%d\": %.3f", blocks_per_sm, fl / ms / 1e9);
    k_ffma<8><<<grid, thr>>>((float*)dout, 100, 0.999f, 1e-3f);
    cudaEventRecord(e0); k_ffma<8><<<grid, thr>>>((float*)dout, iters, 0.999f, 1e-3f); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * iters * (double)grid * thr;
    printf(", \"ffma_tflops_b%d\": %.3f", blocks_per_sm, fl / ms / 1e9);
    k_ffma3<16><<<grid, thr>>>((float*)dout, 100);
    cudaEventRecord(e0); k_ffma3<16><<<grid, thr>>>((float*)dout, iters / 2); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * (iters / 2) * (double)grid * thr;
    printf(", \"ffma3reg_tflops_b%d\": %.3f", blocks_per_sm, fl / ms / 1e9);
    k_ffma2<16><<<grid, thr>>>((float*)dout, 100);
    cudaEventRecord(e0); k_ffma2<16><<<grid, thr>>>((float*)dout, iters / 2); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    fl = 4.0 * 16 * (iters / 2) * (double)grid * thr;
    printf(", \"ffma2_3reg_tflops_b%d\": %.3f", blocks_per_sm, fl / ms / 1e9);
  }
  printf("}\n");
  return 0;
}
