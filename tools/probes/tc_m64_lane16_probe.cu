// Probe: can the M=64 tcgen05.mma (kind::tf32, "ts" form) take its TMEM A operand and/or its
// D accumulator at lane offset 16 (the upper half of each warp's 32-lane quarter, which the
// M=64 layout leaves unused)?  If so, D + A_hi + A_lo fit 128 TMEM columns instead of 256.
// A[i][k] = (k==0)(i+1) + (k==1)(i+1)/2, B[j][k] = (k==0)(j+1)8 + (k==1)8
//   -> D(i,j) = (i+1)(j+1)8 + (i+1)4, expected at lane 32(i/16) + dlane + i%16.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(64 >> 4) << 24);
__device__ __forceinline__ uint32_t sw128(int r, int k) { return r * 128 + (((k >> 2) ^ (r & 7)) << 4) + (k & 3) * 4; }

__global__ void probe(float* out, int alane, int dlane) {
  __shared__ __align__(1024) uint8_t sB[64 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
    const int r = e / 32, k = e % 32;
    *(float*)(sB + sw128(r, k)) = k == 0 ? (float)((r + 1) * 8) : (k == 1 ? 8.f : 0.f);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tm = tslot, ta = tslot + 64;
  // zero everything, then A into columns [64, 96) at lanes alane..alane+15 of each quarter
  {
    const int l16 = lane - alane, row = warp * 16 + l16;
    const bool mine = l16 >= 0 && l16 < 16;
    uint32_t v[32];
    for (int k = 0; k < 32; ++k) {
      float x = 0.f;
      if (mine) x = k == 0 ? (float)(row + 1) : (k == 1 ? (float)(row + 1) * 0.5f : 0.f);
      v[k] = __float_as_uint(x);
    }
    uint32_t z[32];
    for (int k = 0; k < 32; ++k) z[k] = 0u;
#define ST32(addr, v)                                                                                                 \
  asm volatile(                                                                                                       \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"         \
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(addr),                              \
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),  \
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),   \
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),   \
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]))
    const uint32_t wl = (uint32_t)(warp * 32) << 16;
    ST32(tm + wl, z);
    ST32(tm + wl + 32, z);
    ST32(tm + wl + 96, z);
    ST32(ta + wl, v);
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t td = tm + ((uint32_t)dlane << 16), tA = ta + ((uint32_t)alane << 16);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t db = smem_desc(smem_u32(sB) + kk * 32);
      const uint32_t acc = kk > 0;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(td),
                   "r"(tA + kk * 8), "l"(db), "r"(IDESC), "r"(acc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
      smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c0 = 0; c0 < 64; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tm + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int q = 0; q < 8; ++q) out[(warp * 32 + lane) * 64 + c0 + q] = __uint_as_float(r[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tm));
}

int main(int argc, char** argv) {
  float* d;
  cudaMalloc(&d, 128 * 64 * sizeof(float));
  const int cases[4][2] = {{0, 0}, {16, 0}, {0, 16}, {16, 16}};
  for (int ci = 0; ci < 4; ++ci) {
    const int* c = cases[ci];
    if (argc > 1 && atoi(argv[1]) != ci) continue;
    cudaMemset(d, 0, 128 * 64 * sizeof(float));
    probe<<<1, 128>>>(d, c[0], c[1]);
    cudaError_t e = cudaDeviceSynchronize();
    static float h[128 * 64];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int good = 0, nonzero_other = 0;
    for (int w = 0; w < 4; ++w)
      for (int l = 0; l < 32; ++l)
        for (int j = 0; j < 64; ++j) {
          const int l16 = l - c[1];
          const float x = h[(w * 32 + l) * 64 + j];
          if (l16 >= 0 && l16 < 16) {
            const int i = w * 16 + l16;
            if (x == (float)((i + 1) * (j + 1) * 8) + (float)(i + 1) * 4.f) ++good;
          } else if (x != 0.f) {
            ++nonzero_other;
          }
        }
    printf("alane %2d dlane %2d: %s; D correct %d / 4096, nonzero elsewhere %d\n", c[0], c[1], cudaGetErrorString(e),
           good, nonzero_other);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
