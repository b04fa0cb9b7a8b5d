// Legacy warp-level mma.sync throughput on sm_100a: m16n8k8 TF32 (fp32 accumulate) and
// m16n8k16 bf16, independent accumulator chains, registers only.  Is it worth a batched
// 3xTF32 kernel?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_sync_tf32.cu -o mma_sync_tf32
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void k_tf32(float* out, int iters) {
  float d[CHAINS][4] = {};
  unsigned a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
  unsigned b[2] = {threadIdx.x * 3, threadIdx.x * 5};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void k_bf16(float* out, int iters) {
  float d[CHAINS][4] = {};
  unsigned a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
  unsigned b[2] = {threadIdx.x * 3, threadIdx.x * 5};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_tf32<8><<<148 * 2, 32 * warps>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl = 2.0 * 16 * 8 * 8 * 8.0 * iters * 148 * 2 * warps;
      if (rep) printf("tf32 m16n8k8 mma.sync: %2d warps/CTA x 2 CTA/SM: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
      cudaEventRecord(e0);
      k_bf16<8><<<148 * 2, 32 * warps>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double fb = 2.0 * 16 * 8 * 16 * 8.0 * iters * 148 * 2 * warps;
      if (rep) printf("bf16 m16n8k16 mma.sync: %2d warps/CTA x 2 CTA/SM: %.1f TFLOP/s\n", warps, fb / ms / 1e9);
    }
  }
  return 0;
}
