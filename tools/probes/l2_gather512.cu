// Probe: random 512-byte gathers (32 lanes x 16 B: a 64-row interleaved block of the sparse path)
// against 256-byte ones (32 lanes x 8 B, the shipped 32-row blocks) at the same footprints: does a
// wider gather move more L2 bytes per second?  U independent gathers in flight per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/l2_gather512 tools/probes/l2_gather512.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U, bool WIDE>
__global__ void __launch_bounds__(256) k_g(const double* __restrict__ buf, const int32_t* __restrict__ idx,
                                           int64_t n_idx, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = 0.0;
  for (int64_t base = warp * U; base < n_idx; base += nwarps * U) {
    int32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = base + u < n_idx ? __ldg(idx + base + u) : 0;
    if (WIDE) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = reinterpret_cast<const double2*>(buf)[(int64_t)c[u] * 32 + lane];
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = fma(1.0000001, v[u].x + v[u].y, acc[u]);
    } else {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = buf[(int64_t)c[u] * 32 + lane];
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = fma(1.0000001, v[u], acc[u]);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) s += acc[u];
  if (s == 12345.678) out[0] = s;
}

template <int U, bool WIDE>
float run(const double* buf, const int32_t* idx, int64_t n_idx, double* out, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_g<U, WIDE><<<blocks, 256>>>(buf, idx, n_idx, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k_g<U, WIDE><<<blocks, 256>>>(buf, idx, n_idx, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n_idx = 1 << 23;
  int32_t* idx;
  double* buf;
  double* out;
  cudaMalloc(&idx, n_idx * 4);
  cudaMalloc(&buf, (size_t)512 << 20);
  cudaMalloc(&out, 8);
  cudaMemset(buf, 0, (size_t)512 << 20);
  int32_t* h = new int32_t[n_idx];
  for (double mb : {12.8, 25.6, 51.2}) {
    for (int wide = 0; wide < 2; ++wide) {
      const int64_t seg = wide ? 512 : 256;
      const int64_t nseg = (int64_t)(mb * 1e6) / seg;
      uint64_t x = 88172645463325252ull;
      for (int64_t i = 0; i < n_idx; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[i] = (int32_t)(x % nseg);
      }
      cudaMemcpy(idx, h, n_idx * 4, cudaMemcpyHostToDevice);
      const double bytes = (double)n_idx * seg;
      for (int bpsm : {4, 8}) {
        const int blocks = sms * bpsm;
        const float t1 = wide ? run<1, true>(buf, idx, n_idx, out, blocks) : run<1, false>(buf, idx, n_idx, out, blocks);
        const float t2 = wide ? run<2, true>(buf, idx, n_idx, out, blocks) : run<2, false>(buf, idx, n_idx, out, blocks);
        const float t4 = wide ? run<4, true>(buf, idx, n_idx, out, blocks) : run<4, false>(buf, idx, n_idx, out, blocks);
        printf("footprint %5.1f MB seg %3lld B blocks/SM %d: GB/s U=1 %6.0f U=2 %6.0f U=4 %6.0f\n", mb, (long long)seg,
               bpsm, bytes / t1 / 1e6, bytes / t2 / 1e6, bytes / t4 / 1e6);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
