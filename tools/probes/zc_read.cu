// Probe: host -> device bandwidth of pinned host memory read by a kernel (zero-copy, 16-byte loads,
// U loads in flight per thread) against cudaMemcpyAsync, 8 MiB (c2's X) and 64 MiB.  Also the
// reverse (kernel stores into pinned host memory) against the D2H copy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/zc_read tools/probes/zc_read.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void k_pull(const double2* __restrict__ src, double2* __restrict__ dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * stride < n ? src[i + u * stride] : make_double2(0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * stride < n) dst[i + u * stride] = v[u];
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (size_t bytes : {(size_t)8 << 20, (size_t)64 << 20}) {
    void *h, *hw, *d;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&hw, bytes, cudaHostAllocMapped | cudaHostAllocWriteCombined);
    cudaMalloc(&d, bytes);
    memset(h, 1, bytes);
    memset(hw, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    const int R = 10;
    for (int dir = 0; dir < 2; ++dir) {
      cudaMemcpy(d, h, bytes, dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice);
      cudaEventRecord(a);
      for (int r = 0; r < R; ++r)
        cudaMemcpyAsync(dir ? h : d, dir ? d : h, bytes, dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("%3zu MiB %s cudaMemcpyAsync          %6.1f GB/s\n", bytes >> 20, dir ? "D2H" : "H2D", bytes * R / ms / 1e6);
    }
    const int64_t n = bytes / 16;
    for (int hk = 0; hk < 2; ++hk)
      for (int dir = 0; dir < 2; ++dir)
        for (int bpsm : {1, 4, 8}) {
          for (int uu = 0; uu < 2; ++uu) {
            void* hp = hk ? hw : h;
            const double2* src = (const double2*)(dir ? d : hp);
            double2* dst = (double2*)(dir ? hp : d);
            auto go = [&]() {
              if (uu) k_pull<4><<<sms * bpsm, 256>>>(src, dst, n);
              else k_pull<1><<<sms * bpsm, 256>>>(src, dst, n);
            };
            go();
            cudaEventRecord(a);
            for (int r = 0; r < R; ++r) go();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("%3zu MiB %s kernel %s CTAs/SM %d U %d %6.1f GB/s\n", bytes >> 20, dir ? "D2H" : "H2D",
                   hk ? "wc    " : "mapped", bpsm, uu ? 4 : 1, bytes * R / ms / 1e6);
          }
        }
    cudaFreeHost(h);
    cudaFreeHost(hw);
    cudaFree(d);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
