// Probe: the L2 -> SM throughput ceiling of the sparse path's access pattern on B200.
// A warp gathers G-byte segments (G = 256: 32 lanes x 8 B, the 32-row interleaved blocks of
// sparse_f64.cu; G = 128: 16-row blocks) at uniformly random segment indices inside an
// F-byte buffer (L2-resident when F < ~100 MB), U independent loads in flight per warp, and
// reduces them into a register (the fma of the SpMM).  Reports bytes gathered per second.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/l2_gather tools/probes/l2_gather.cu
//   tools/probes/l2_gather
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U, int LANES>
__global__ void __launch_bounds__(256) k_gather(const double* __restrict__ buf, const int32_t* __restrict__ idx,
                                                int64_t n_idx, double* out) {
  // LANES lanes per segment (32: 256 B, 16: 128 B); 32 / LANES segments per warp instruction
  const int lane = threadIdx.x & 31;
  const int sub = lane / LANES, li = lane % LANES;
  constexpr int SEGS = 32 / LANES;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = 0.0;
  for (int64_t base = warp * U * SEGS; base < n_idx; base += nwarps * U * SEGS) {
    int32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + u * SEGS + sub;
      c[u] = e < n_idx ? __ldg(idx + e) : 0;
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = buf[(int64_t)c[u] * LANES + li];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = fma(1.0000001, v[u], acc[u]);
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) s += acc[u];
  if (s == 12345.678) out[0] = s;
}

template <int U, int LANES>
float run(const double* buf, const int32_t* idx, int64_t n_idx, double* out, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_gather<U, LANES><<<blocks, 256>>>(buf, idx, n_idx, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k_gather<U, LANES><<<blocks, 256>>>(buf, idx, n_idx, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n_idx = 1 << 24;   // 16 M gathers per launch
  int32_t* idx;
  double* buf;
  double* out;
  cudaMalloc(&idx, n_idx * 4);
  cudaMalloc(&buf, (size_t)512 << 20);
  cudaMalloc(&out, 8);
  cudaMemset(buf, 0, (size_t)512 << 20);
  int32_t* h = new int32_t[n_idx];
  for (double mb : {12.8, 25.6, 51.2, 80.0, 102.4, 400.0}) {
    for (int lanes : {32, 16}) {
      const int64_t seg = lanes * 8;
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
        float t1 = lanes == 32 ? run<1, 32>(buf, idx, n_idx, out, blocks) : run<1, 16>(buf, idx, n_idx, out, blocks);
        float t2 = lanes == 32 ? run<2, 32>(buf, idx, n_idx, out, blocks) : run<2, 16>(buf, idx, n_idx, out, blocks);
        float t4 = lanes == 32 ? run<4, 32>(buf, idx, n_idx, out, blocks) : run<4, 16>(buf, idx, n_idx, out, blocks);
        float t8 = lanes == 32 ? run<8, 32>(buf, idx, n_idx, out, blocks) : run<8, 16>(buf, idx, n_idx, out, blocks);
        float t16 = lanes == 32 ? run<16, 32>(buf, idx, n_idx, out, blocks) : run<16, 16>(buf, idx, n_idx, out, blocks);
        printf("footprint %6.1f MB seg %3lld B blocks/SM %d: GB/s U=1 %7.0f U=2 %7.0f U=4 %7.0f U=8 %7.0f U=16 %7.0f\n",
               mb, (long long)seg, bpsm, bytes / t1 / 1e6, bytes / t2 / 1e6, bytes / t4 / 1e6, bytes / t8 / 1e6,
               bytes / t16 / 1e6);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
