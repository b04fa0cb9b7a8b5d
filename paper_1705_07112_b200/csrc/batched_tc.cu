// Batched fp32 path on the 5th-generation tensor cores (BASELINE configs[2]: 65536
// independent patch-group matrices, m, n <= 64): the whole of Alg. 1 (PAPER.md:354-373,
// T = I, eps = 0) per matrix inside one persistent CTA, every matrix product a
// tcgen05.mma (cta_group::1, kind::tf32, M = N = 64) in 3xTF32 (hi/lo operand split,
// round-to-nearest: acc = hi hi + hi lo + lo hi), accumulator in TMEM.
//
//   A = X (m <= n) or X^T, zero-padded to 64 x 64;  s = Gram side
//   line 1:    G = A A^T                          (tcgen05; both operands = rows of A)
//   line 3:    lambda_hat: T power steps on G      (fp32 CUDA cores, G rows in registers)
//   line 4:    c_k (fp64, K-node rule)
//   line 5-7:  Psi_1 = (2/L) G - I,  H = c_0/2 I + c_1 Psi_1
//   line 8-11: Psi_k = (4/L) G Psi_{k-1} - 2 Psi_{k-1} - Psi_{k-2},  H += c_k Psi_k   (tcgen05)
//   line 12:   Y = H A                             (tcgen05; B operand = rows of A^T)
//
// A step multiplies from the right, D = Psi_{k-1} G^T (A operand = rows of Psi_{k-1}, exactly
// as the epilogue thread that owns the row writes them; B operand = rows of the fixed G):
// G^T = G up to the Gram's rounding, a constant perturbation, and Psi_{k-1} G = G Psi_{k-1}
// (polynomials in G commute).  The other association, D = G Psi_{k-1}^T with the rows of
// Psi as B operand, assumes Psi symmetric: its antisymmetric rounding error then follows a
// recurrence with multiplier -2 - (4/L) sqrt(l_a l_b), outside [-2, 2] -- measured 1e-7 at
// K = 8 growing to 1e-4 at K = 20.
//
// Operands live in shared memory in the canonical K-major SWIZZLE_128B layout (128-byte
// rows of 32 fp32, 8-row atoms, 16-byte chunk c of row r at c ^ (r & 7)), two 8 KB
// k-blocks per 64 x 64 operand; descriptors as in tc_tf32.cu.  TMEM layout for M = 64
// (probed, tools/probes/tc_m64_probe.cu): row r of D lives in lane 32 (r / 16) + r % 16,
// column j in column j -- so lanes 0..15 of each lane quarter own the 64 rows (16 per quarter).
// TMEM columns [0, 64): D.  Eight warps: warp w reads rows 16 (w % 4) .. +15 (its quarter) and
// columns 32 (w / 4) .. +31 with tcgen05.ld.16x256b.x4 (all 32 threads: 2 rows x 8 columns
// each); Psi_{k-1}, Psi_{k-2} and H stay in registers in that layout.  Eight warps instead of
// four halve the epilogue between two MMAs, which is exposed (tensor pipe idle) whenever
// the other CTA on the SM is in its own epilogue.
#include <cstdlib>
#include <cstdio>

#include <algorithm>

#include "common.cuh"

namespace cpa {
namespace btc {

// Threads per CTA NT = 128 (default: 4 warps, warp w owns D rows 16 w .. +15, all 64 columns;
// 4 CTAs per SM) or 256 (CPA_SVT_BTC_NT=256: 8 warps, warp w owns rows 16 (w % 4) .. +15 and
// columns 32 (w / 4) .. +31 -- a TMEM lane quarter is warp w % 4's; 3 CTAs per SM, registers);
// FR = 4096 / NT fragment elements per thread.  More matrices in flight per SM beat a shorter
// epilogue per matrix: c3 8.05 ms (128) against 8.62 ms (256).
constexpr int OPB = 64 * 64 * 4;        // bytes of one 64 x 64 fp32 operand (two 8 KB k-blocks)
#ifndef BTC_LATE_H
#define BTC_LATE_H 1   // H += c_k Psi_k under the next step's MMA (0: in the epilogue, the round-2 order)
#endif

__device__ __forceinline__ uint32_t sw(int r, int k) {  // byte offset of (r, k) in a K-major SW128 operand
  return (uint32_t)((k >> 5) * 8192 + r * 128 + ((((k & 31) >> 2) ^ (r & 7)) << 4) + (k & 3) * 4);
}
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;        // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;      // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                // version 1
  d |= (uint64_t)2 << 61;                // SWIZZLE_128B
  return d;
}
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(64 >> 4) << 24);

__device__ __forceinline__ float rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// write fp32 x as TF32 hi / lo at (r, k) of the operand pair at (hi, hi + OPB)
__device__ __forceinline__ void put(uint8_t* hi, int r, int k, float x) {
  const float h = rna(x);
  const uint32_t o = sw(r, k);
  *reinterpret_cast<float*>(hi + o) = h;
  *reinterpret_cast<float*>(hi + OPB + o) = rna(x - h);
}
// 4 consecutive k (one 16-byte chunk) of row r
__device__ __forceinline__ void put4(uint8_t* hi, int r, int k, float x0, float x1, float x2, float x3) {
  const uint32_t o = sw(r, k);
  const float h0 = rna(x0), h1 = rna(x1), h2 = rna(x2), h3 = rna(x3);
  *reinterpret_cast<float4*>(hi + o) = make_float4(h0, h1, h2, h3);
  *reinterpret_cast<float4*>(hi + OPB + o) = make_float4(rna(x0 - h0), rna(x1 - h1), rna(x2 - h2), rna(x3 - h3));
}

// D0 + D1 = Aop * Bop^T over K = 64 in 3xTF32 (24 MMAs), A operand in TMEM ("ts" form, probed:
// A row r in the M = 64 D lane of row r, element k in column k; one UMMA_K = 8 columns), issued
// by one thread; completion on bar.  D0 (lane offset 0) accumulates hi*hi + hi*lo with A_hi at
// lane offset 0, D1 (lane offset 16) lo*hi with A_lo at lane offset 16: an M = 64 MMA runs on
// one 16-lane half of each lane quarter, A and D in the same half (probed,
// tools/probes/tc_m64_lane16_probe.cu), so D, A_hi and A_lo fit 128 TMEM columns instead of
// 192 (three CTAs per SM instead of two).  The epilogue adds D0 + D1.
// At M = 64 the smem-A form is limited by its shared-memory A reads (measured 61 cycles per
// M64 N64 K8 MMA against the 32-cycle floor), hence A in TMEM.
// ACC0: D0 accumulates onto its current contents from the first k-block (the step's
// -2 Psi_{k-1} - Psi_{k-2}, stored by the epilogue), D1 always starts from zero.
template <bool ACC0 = false>
__device__ __forceinline__ void mma64_ts(uint32_t tmem_d0, uint32_t tmem_d1, uint32_t ta_hi, uint32_t ta_lo,
                                         const uint8_t* b_hi, uint64_t* bar) {
  // opaque to the optimiser: the 16 descriptors are rebuilt per call by the issuing thread
  // instead of being hoisted out of the step loop into 32 registers of every thread
  uint32_t bh;
  asm volatile("mov.b32 %0, %1;\n" : "=r"(bh) : "r"(smem_u32(b_hi)));
  // the descriptor's start-address field is addr >> 4 in 14 bits (no carry below 256 KB), so a
  // k-block's descriptor is the base descriptor plus off >> 4
  const uint64_t dbh0 = desc(bh), dbl0 = desc(bh + OPB);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint32_t off = (kk >> 2) * 8192 + (kk & 3) * 32;
    const uint64_t dbh = dbh0 + (off >> 4), dbl = dbl0 + (off >> 4);
    asm volatile(
        "{\n.reg .pred p, p0;\nsetp.ne.b32 p, %4, 0;\nsetp.ne.b32 p0, %8, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%7], [%6], %2, %3, p;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %5, %3, 1;\n}\n" ::"r"(tmem_d0),
        "r"(ta_hi + kk * 8), "l"(dbh), "r"(IDESC), "r"(kk > 0 ? 1u : 0u), "l"(dbl), "r"(ta_lo + kk * 8),
        "r"(tmem_d1), "r"((ACC0 || kk > 0) ? 1u : 0u)
        : "memory");
  }
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}
// all generic-proxy smem writes and TMEM accesses of the CTA done before the next MMA issue
__device__ __forceinline__ void sync_for_mma() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

struct Args {
  int64_t batch;
  int m, n;
  const float* X;
  float* Y;
  cpa_svt_kernel kern;
  int K, T;
  double safety, lam_override;
  float* lambda_out;
  const double* costab;   // cos(k theta_l), K x K
  int psi2_sq;            // Psi_2 from the power iteration's first squaring (R29; CPA_SVT_NO_PSI2_SQ: off)
};

// smem: one B operand (hi, lo; 32 KB, 1 KB aligned): rows of A (line 1), of c^p G^p (squarings),
// of G (lines 8-11), of A^T (line 12); then H in the threads' fragment layout (16 KB, float4
// [FR / 4][NT]: conflict-free), which keeps the step's register state (Psi_{k-1}, Psi_{k-2}, D)
// within the 80 registers of three 256-thread CTAs per SM
constexpr int SMEM = 2 * OPB + 64 * 64 * 4 + 1024;

// tcgen05.ld.16x256b.x4: 16 rows x 32 columns of D in this warp's lane quarter, spread over
// all 32 threads (probed, tools/probes/tc_m64_probe.cu): thread t holds rows r0 = t/4 and
// r1 = t/4 + 8 (warp-local), columns 8c + 2(t%4) + {0, 1}, c = 0..3 (relative to the address), as
// v[4c + 0] = (r0, 8c+2q), v[4c + 1] = (r0, 8c+2q+1), v[4c + 2] = (r1, 8c+2q), v[4c + 3] = (r1, 8c+2q+1).
// D = D0 + D1 in the fragment layout above, in 16-column pieces of 8 registers each so that
// at most 16 loaded registers are live beside the recurrence state
template <int FR>
__device__ __forceinline__ void ld_frag2(uint32_t taddr0, uint32_t taddr1, float (&v)[FR]) {
#pragma unroll
  for (int hf = 0; hf < FR / 8; ++hf) {
    uint32_t r[8], u[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr0 + 16 * hf));
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
                 : "r"(taddr1 + 16 * hf));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[8 * hf + i] = __uint_as_float(r[i]) + __uint_as_float(u[i]);
  }
}
// store a fragment (layout of ld_frag2) as TF32 hi / lo A operands in TMEM (same layout)
#define BTC_ST16(addr, r)                                                                                          \
  asm volatile("tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" \
               ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),  \
               "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])          \
               : "memory")
template <int FR>
__device__ __forceinline__ void st_frag_hl(uint32_t t_hi, uint32_t t_lo, const float (&v)[FR]) {
#pragma unroll
  for (int c = 0; c < FR / 16; ++c) {   // 32 columns per x4 store; one piece's hi / lo live at a time
    uint32_t h[16], l[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float x = v[16 * c + i], hx = rna(x);
      h[i] = __float_as_uint(hx);
      l[i] = __float_as_uint(rna(x - hx));
    }
    BTC_ST16(t_hi + 32 * c, h);
    BTC_ST16(t_lo + 32 * c, l);
  }
}
// store a fragment (layout of ld_frag2) as fp32 into TMEM (the D0 accumulator)
template <int FR>
__device__ __forceinline__ void st_frag(uint32_t taddr, const float (&v)[FR]) {
#pragma unroll
  for (int c = 0; c < FR / 16; ++c) {
    uint32_t h[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) h[i] = __float_as_uint(v[16 * c + i]);
    BTC_ST16(taddr + 32 * c, h);
  }
}
#undef BTC_ST16
// TMEM stores done and visible to the next MMA issue (no shared-memory writes involved)
__device__ __forceinline__ void sync_tmem_for_mma() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// write a fragment (layout of ld_frag2) as TF32 hi / lo operand rows: element (row, col) at sw(row, col)
template <int FR>
__device__ __forceinline__ void put_frag(uint8_t* hi, int row0, int col0, const float (&v)[FR]) {
#pragma unroll
  for (int c = 0; c < FR / 4; ++c)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = row0 + 8 * h, k = col0 + 8 * c;
      const float x0 = v[4 * c + 2 * h], x1 = v[4 * c + 2 * h + 1];
      const float h0 = rna(x0), h1 = rna(x1);
      const uint32_t o = sw(r, k);
      *reinterpret_cast<float2*>(hi + o) = make_float2(h0, h1);
      *reinterpret_cast<float2*>(hi + OPB + o) = make_float2(rna(x0 - h0), rna(x1 - h1));
    }
}

template <int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 3 : 4) k_batched_tc(Args a) {
  constexpr int NW = NT / 32, FR = 4096 / NT, NCH = NW / 4;   // NCH column groups
  extern __shared__ uint8_t raw[];
  uint8_t* base = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);   // (stays in the shared window: STS, not ST)
  uint8_t* sB = base;                 // B operand
  float4* sH4 = reinterpret_cast<float4*>(base + 2 * OPB);   // H fragments
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ float sV2[2][64];
  __shared__ float sU2[2][NCH][64];   // per column group: partial row sums of a power product
  __shared__ float sRed2[2][2];
  __shared__ float sRed[NW];
  __shared__ double sNode[128];   // K <= 128 on the batched path (cpa_svt_apply_batched)
  __shared__ double sHn[128];
  __shared__ float sC[128];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = lane & 3, wq = warp & 3, ch = warp >> 2;
  const int row0 = wq * 16 + (lane >> 2), row1 = row0 + 8;      // this thread's two D rows
  const int col0 = 32 * ch + 2 * q;                              // and its first column
  // TMEM address of this warp's fragment: lane quarter wq, column half ch
  const uint32_t lane_off = ((uint32_t)(wq * 32) << 16) + 32u * ch;
  const bool left = a.m <= a.n;
  const int s = left ? a.m : a.n, L = left ? a.n : a.m;
  const int K = a.K;
  const int64_t mn = (int64_t)a.m * a.n;
  auto colof = [&](int e) { return col0 + 8 * (e >> 2) + (e & 1); };
  // 64 x 64 matrices at 8-byte aligned addresses take the float2 load path (A = X)
  const bool full64 = a.m == 64 && a.n == 64 && ((reinterpret_cast<uintptr_t>(a.X) & 7) == 0);
  auto rowof = [&](int e) { return (e & 2) ? row1 : row0; };
  // A (s x L, zero-padded to 64 x 64) in this thread's fragment layout: v[e] = A(rowof(e), colof(e))
  auto load_frag = [&](const float* X, float (&v)[FR]) {
    if (full64) {
#pragma unroll
      for (int e = 0; e < FR; e += 2) {
        const float2 x2 = __ldg(reinterpret_cast<const float2*>(X + rowof(e) * 64 + colof(e)));
        v[e] = x2.x;
        v[e + 1] = x2.y;
      }
    } else {
#pragma unroll
      for (int e = 0; e < FR; ++e) {
        const int i = rowof(e), j = colof(e);
        v[e] = (i < s && j < L) ? __ldg(left ? X + (int64_t)i * a.n + j : X + (int64_t)j * a.n + i) : 0.f;
      }
    }
  };

  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // lanes +0: D0 (columns 0-63), A_hi (64-127); lanes +16: D1, A_lo
  const uint32_t tD = tslot, tAh = tslot + 64, tD1 = tD + (16u << 16), tAl = tAh + (16u << 16);
  uint32_t phase = 0;
  // Chebyshev-Gauss nodes x_l / Lambda = (cos theta_l + 1) / 2, once per CTA
  for (int l = tid; l < K; l += NT) sNode[l] = 0.5 * (cos(cheb_theta(l + 1, K)) + 1.0);

  for (int64_t b = blockIdx.x; b < a.batch; b += gridDim.x) {
    const float* X = a.X + b * mn;
    // the CTA's next matrix into L2 while this one is processed (one bulk prefetch; 16-byte
    // granules only)
    if (tid == 0 && b + gridDim.x < a.batch) {
      const float* Xn = a.X + (b + gridDim.x) * mn;
      const uint32_t bytes = (uint32_t)(mn * 4);
      if (((reinterpret_cast<uintptr_t>(Xn) | bytes) & 15) == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(Xn), "r"(bytes) : "memory");
    }
    // ---- line 1: G = A A^T (A operand: A in TMEM; B operand: rows of A)
    {
      float av[FR];
      load_frag(X, av);
      put_frag(sB, row0, col0, av);
      st_frag_hl(tAh + lane_off, tAl + lane_off, av);
    }
    sync_for_mma();
    if (tid == 0) btc::mma64_ts(tD, tD1, tAh, tAl, sB, &bar);
    mbar_wait(&bar, phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    float g[FR];
    ld_frag2(tD + lane_off, tD1 + lane_off, g);
    // ---- line 3: Lambda_max by T power steps (fp32, fixed order).  Repeated squaring (as the
    //      dense path, reading R6): v_{T-1} ~ G^{T-1} v_0 through q = (T-1)/4 products by
    //      c^4 G^4 (c = 2^-ilogb(max G_ii), exact) then T - 4q by G; two extra tcgen05 products
    //      instead of 3q power steps.
    double lam_hat;
    // (reading R29: the first squaring's c^2 G^2, kept in the H buffer until the init forms Psi_2)
    bool have_g2 = false;
    float cs2v = 1.f;
    if (a.lam_override > 0.0) {
      lam_hat = a.lam_override / a.safety;
    } else {
      const int qsq = a.T >= 8 ? (a.T - 1) / 4 : 0;
      float g4[FR];
#pragma unroll
      for (int e = 0; e < FR; ++e) g4[e] = g[e];   // (only read when qsq > 0, then overwritten below)
      if (qsq > 0) {
        float dmax = 0.f;
#pragma unroll
        for (int e = 0; e < FR; ++e)
          if (rowof(e) == colof(e)) dmax = fmaxf(dmax, g[e]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        if (lane == 0) sRed[warp] = dmax;
        __syncthreads();
        dmax = sRed[0];
#pragma unroll
        for (int w = 1; w < NW; ++w) dmax = fmaxf(dmax, sRed[w]);
        const float cs = (dmax > 0.f && isfinite(dmax)) ? ldexpf(1.f, -ilogbf(dmax)) : 1.f;
#pragma unroll
        for (int e = 0; e < FR; ++e) g4[e] = cs * g[e];
        for (int sq = 0; sq < 2; ++sq) {               // (cG)^2, then (c^2 G^2)^2
          st_frag_hl(tAh + lane_off, tAl + lane_off, g4);
          put_frag(sB, row0, col0, g4);
          sync_for_mma();
          if (tid == 0) btc::mma64_ts(tD, tD1, tAh, tAl, sB, &bar);
          mbar_wait(&bar, phase);
          phase ^= 1;
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          ld_frag2(tD + lane_off, tD1 + lane_off, g4);
          if (sq == 0 && a.psi2_sq && K > 3) {        // c^2 G^2 into this thread's H slots (free until the init)
#pragma unroll
            for (int c = 0; c < FR / 4; ++c)
              sH4[c * NT + tid] = make_float4(g4[4 * c], g4[4 * c + 1], g4[4 * c + 2], g4[4 * c + 3]);
            have_g2 = true;
            cs2v = cs * cs;
          }
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          __syncthreads();                             // everyone has read D and the operands
        }
      }
      // u_t = G v_{t-1} with v_{t-1} = u_{t-1} / ||u_{t-1}|| folded in as a scale of the product:
      // each column half's partial row sums go to sU2, warps 0-1 add the halves (fixed order),
      // store u_t and reduce ||u_t||^2; ping-pong buffers, two CTA barriers per product
      if (tid < 64) sV2[0][tid] = tid < s ? rsqrtf((float)s) : 0.f;
      __syncthreads();
      float nrm = 0.f, inv = 1.f;
      const int niter = a.T - 3 * qsq;
      for (int t = 0; t < niter; ++t) {
        const bool use4 = t < qsq;
        const float* vin = sV2[t & 1];
        float u0a = 0.f, u0b = 0.f, u1a = 0.f, u1b = 0.f;   // row0 / row1 partial sums (2 chains each)
#pragma unroll
        for (int c = 0; c < FR / 4; ++c) {
          const float v0 = vin[col0 + 8 * c], v1 = vin[col0 + 8 * c + 1];
          u0a = fmaf(use4 ? g4[4 * c + 0] : g[4 * c + 0], v0, u0a);
          u0b = fmaf(use4 ? g4[4 * c + 1] : g[4 * c + 1], v1, u0b);
          u1a = fmaf(use4 ? g4[4 * c + 2] : g[4 * c + 2], v0, u1a);
          u1b = fmaf(use4 ? g4[4 * c + 3] : g[4 * c + 3], v1, u1b);
        }
        float u0 = u0a + u0b, u1 = u1a + u1b;
        u0 += __shfl_xor_sync(0xffffffffu, u0, 1);
        u1 += __shfl_xor_sync(0xffffffffu, u1, 1);
        u0 += __shfl_xor_sync(0xffffffffu, u0, 2);
        u1 += __shfl_xor_sync(0xffffffffu, u1, 2);
        if (q == 0) {
          sU2[t & 1][ch][row0] = u0;
          sU2[t & 1][ch][row1] = u1;
        }
        __syncthreads();
        if (tid < 64) {
          float u = sU2[t & 1][0][tid];
          if (NCH == 2) u += sU2[t & 1][NCH - 1][tid];
          u *= inv;
          sV2[(t + 1) & 1][tid] = u;
          float sq = u * u;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
          if (lane == 0) sRed2[t & 1][warp] = sq;
        }
        __syncthreads();
        nrm = sqrtf(sRed2[t & 1][0] + sRed2[t & 1][1]);
        if (!(nrm > 0.f)) break;
        inv = 1.f / nrm;
      }
      lam_hat = nrm > 0.f ? (double)nrm : 0.0;
    }
    // ---- line 4: coefficients (fp64) for this matrix's Lambda_max
    const bool degen = !(lam_hat > kDegenerateLambda);
    const double lam = a.safety * lam_hat;
    const double tau = resolve_tau(a.kern, sqrt(lam_hat));
    for (int l = tid; l < K; l += NT) sHn[l] = h_response(a.kern, lam * sNode[l], tau);
    __syncthreads();
    // c_k = (2/K) sum_l cos(k theta_l) h_l: 4 threads per k (residues of l mod 4), fixed-order reduction
    for (int k0 = 0; k0 < K; k0 += NT / 4) {
      const int k = k0 + (tid >> 2), r = tid & 3;
      double acc_c = 0.0;
      if (k < K) {
        const double* ct = a.costab + (int64_t)k * K;
        for (int l = r; l < K; l += 4) acc_c = fma(__ldg(ct + l), sHn[l], acc_c);
      }
      acc_c += __shfl_xor_sync(0xffffffffu, acc_c, 1);
      acc_c += __shfl_xor_sync(0xffffffffu, acc_c, 2);
      if (k < K && r == 0) sC[k] = degen ? 0.f : (float)(2.0 / K * acc_c);
    }
    __syncthreads();
    if (tid == 0 && a.lambda_out) a.lambda_out[b] = (float)lam;
    const float s2 = degen ? 0.f : (float)(2.0 / lam);
    const float s4 = 2.f * s2;

    // ---- lines 5-7: Psi_1 = s2 G - I, H = c0/2 I + c1 Psi_1 (all in this thread's fragment)
    // The steps run on the tensor core whole: B operand = rows of s4 G, and D0 is preloaded
    // with -2 Psi_{k-1} - Psi_{k-2}, so D0 + D1 = Psi_{k-1} (s4 G)^T - 2 Psi_{k-1} - Psi_{k-2}
    // = Psi_k (lines 8-9) and only Psi_{k-1} stays in registers.
    float wp[FR];
    int k_first = 2;
    if (have_g2) {
      // Psi_1 = s2 G - I and Psi_2 = 2 s2^2 G^2 - 2 s2 G ... = 2 B_hat^2 - I from the squaring's c^2 G^2
      // (reading R29): H = c0/2 I + c1 Psi_1 + c2 Psi_2, the steps start at k = 3 with A = Psi_2
      // and D0 = -2 Psi_2 - Psi_1
      const float h0 = 0.5f * sC[0], c1 = sC[1], c2 = sC[2];
      const float a2 = 2.f * s2 * s2 / cs2v, a4 = 2.f * s2;
      float hh[FR];
#pragma unroll
      for (int c = 0; c < FR / 4; ++c) {
        const float4 q4 = sH4[c * NT + tid];
        const float gq[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const int e = 4 * c + x;
          const float id = (rowof(e) == colof(e)) ? 1.f : 0.f;
          const float w = s2 * g[e] - id;                         // Psi_1
          const float p2 = a2 * gq[x] - 2.f * a4 * g[e] + id;     // Psi_2 = 2 s2^2 G^2 - 4 s2 G + I
          hh[e] = h0 * id + c1 * w + c2 * p2;
          wp[e] = p2;
          g[e] *= s4;
        }
      }
      k_first = 3;
#pragma unroll
      for (int c = 0; c < FR / 4; ++c) sH4[c * NT + tid] = make_float4(hh[4 * c], hh[4 * c + 1], hh[4 * c + 2], hh[4 * c + 3]);
      put_frag(sB, row0, col0, g);                      // B operand of the steps: rows of s4 G
      st_frag_hl(tAh + lane_off, tAl + lane_off, wp); // A operand (TMEM): rows of Psi_2
#pragma unroll
      for (int e = 0; e < FR; ++e) {                     // D0 = -2 Psi_2 - Psi_1 (Psi_1 recomputed from s4 G)
        const float id = (rowof(e) == colof(e)) ? 1.f : 0.f;
        hh[e] = -2.f * wp[e] - (0.5f * g[e] - id);
      }
      st_frag(tD + lane_off, hh);
    } else {
      const float h0 = 0.5f * sC[0], c1 = sC[1];
      float hh[FR];
#pragma unroll
      for (int e = 0; e < FR; ++e) {
        const float id = (rowof(e) == colof(e)) ? 1.f : 0.f;
        const float w = s2 * g[e] - id;
        wp[e] = w;
        hh[e] = h0 * id + c1 * w;
        g[e] *= s4;
      }
#pragma unroll
      for (int c = 0; c < FR / 4; ++c) sH4[c * NT + tid] = make_float4(hh[4 * c], hh[4 * c + 1], hh[4 * c + 2], hh[4 * c + 3]);
      put_frag(sB, row0, col0, g);                      // B operand of the steps: rows of s4 G
      st_frag_hl(tAh + lane_off, tAl + lane_off, wp); // A operand (TMEM): rows of Psi_1
#pragma unroll
      for (int e = 0; e < FR; ++e) hh[e] = -2.f * wp[e] - ((rowof(e) == colof(e)) ? 1.f : 0.f);   // Psi_0 = I
      st_frag(tD + lane_off, hh);
    }
    sync_for_mma();
    // ---- lines 8-11: Psi_k = D0 + D1, H += c_k Psi_k; next A = Psi_k, next D0 = -2 Psi_k - Psi_{k-1}
    // H += c_k Psi_k (this thread's fragment slots of H in shared memory)
    auto h_update = [&](float ck, const float (&v)[FR]) {
#pragma unroll
      for (int c = 0; c < FR / 4; ++c) {
        float4 h4 = sH4[c * NT + tid];
        h4.x = fmaf(ck, v[4 * c], h4.x);
        h4.y = fmaf(ck, v[4 * c + 1], h4.y);
        h4.z = fmaf(ck, v[4 * c + 2], h4.z);
        h4.w = fmaf(ck, v[4 * c + 3], h4.w);
        sH4[c * NT + tid] = h4;
      }
    };
    for (int k = k_first; k < K; ++k) {
      if (tid == 0) btc::mma64_ts<true>(tD, tD1, tAh, tAl, sB, &bar);
#if BTC_LATE_H
      // H += c_{k-1} Psi_{k-1} (wp) while the tensor core computes Psi_k: the update is not an
      // input of the MMA, so it leaves the epilogue's critical path (same sums, same order)
      if (k > k_first) h_update(sC[k - 1], wp);
#endif
      mbar_wait(&bar, phase);
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      float d[FR];
      ld_frag2(tD + lane_off, tD1 + lane_off, d);
#if BTC_LATE_H
      if (k + 1 == K) h_update(sC[k], d);
#else
      h_update(sC[k], d);
#endif
      if (k + 1 < K) {
        st_frag_hl(tAh + lane_off, tAl + lane_off, d);
#pragma unroll
        for (int e = 0; e < FR; ++e) {
          const float nx = -2.f * d[e] - wp[e];
          wp[e] = d[e];
          d[e] = nx;
        }
        st_frag(tD + lane_off, d);
      }
      sync_tmem_for_mma();
    }
    // ---- line 12: Y = H A  (A operand = rows of H, B operand = rows of A^T: A re-read, from L2)
    {
      float hh[FR];
#pragma unroll
      for (int c = 0; c < FR / 4; ++c) {
        const float4 h4 = sH4[c * NT + tid];
        hh[4 * c] = h4.x;
        hh[4 * c + 1] = h4.y;
        hh[4 * c + 2] = h4.z;
        hh[4 * c + 3] = h4.w;
      }
      st_frag_hl(tAh + lane_off, tAl + lane_off, hh);
    }
    {
      float av[FR];
      load_frag(X, av);
#pragma unroll
      for (int e = 0; e < FR; ++e) put(sB, colof(e), rowof(e), av[e]);
    }
    sync_for_mma();
    if (tid == 0) btc::mma64_ts(tD, tD1, tAh, tAl, sB, &bar);
    mbar_wait(&bar, phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    {
      float d[FR];
      ld_frag2(tD + lane_off, tD1 + lane_off, d);
      float* Yb = a.Y + b * mn;
#pragma unroll
      for (int e = 0; e < FR; ++e) {
        const int r = rowof(e), c = colof(e);
        if (r < s && c < L) {
          if (left) Yb[(int64_t)r * a.n + c] = d[e];
          else Yb[(int64_t)c * a.n + r] = d[e];
        }
      }
    }
    // TMEM D and the operands are rewritten by the next matrix only after this barrier
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tslot));
}

}  // namespace btc

__global__ void k_costab(double* tab, int K);

cudaError_t launch_batched_tc(int64_t batch, int m, int n, const float* X, float* Y, const cpa_svt_kernel& k, int K,
                              int T, double safety, double lam_override, float* lambda_out, int num_sms,
                              cudaStream_t st, int* launches, double* costab) {
  if (K > 128) return cudaErrorNotSupported;
  k_costab<<<(K * K + 255) / 256, 256, 0, st>>>(costab, K);
  if (launches) ++*launches;
  btc::Args a{batch, m, n, X, Y, k, K, T, safety, lam_override, lambda_out, costab, env_on("CPA_SVT_NO_PSI2_SQ") ? 0 : 1};
  const char* ntv = getenv("CPA_SVT_BTC_NT");
  const int nt = (ntv && atoi(ntv) == 256) ? 256 : 128;   // 128: measured c3 8.05 ms against 8.62 ms
  auto kern = nt == 128 ? btc::k_batched_tc<128> : btc::k_batched_tc<256>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, btc::SMEM);
  if (e != cudaSuccess) return e;
  // all of the unified L1 / shared storage as shared memory: without this preference the occupancy
  // query (and the launch) size residency for the default carveout -- one CTA per SM measured
  // (c3 7.6 -> 18.9 ms)
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, btc::SMEM);
  if (e != cudaSuccess) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  const int occ_api = per_sm;
  per_sm = resident_ctas((const void*)kern, nt, btc::SMEM, dev);
  if (env_on("CPA_SVT_DEBUG_OCC")) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)kern);
    fprintf(stderr, "k_batched_tc<%d>: occupancy API %d, resident %d CTAs/SM, regs %d, static smem %zu, dyn %d, max dyn %d, maxthreads %d\n",
            nt, occ_api, per_sm, fa.numRegs, fa.sharedSizeBytes, btc::SMEM, fa.maxDynamicSharedSizeBytes, fa.maxThreadsPerBlock);
  }
  // 3 x (49 KB smem, 256 thr x <= 80 regs, 128 TMEM columns) or 4 x (128 thr x <= 128 regs) fit one SM
  // (never more than `want`: each CTA holds its 128 TMEM columns for the whole persistent loop, so a
  // fifth CTA on an SM would block in tcgen05.alloc forever; fewer if registers / shared memory
  // limit residency -- the grid then stays one wave of what is actually resident)
  const int want = nt == 128 ? 4 : 3;
  if (per_sm > want) per_sm = want;
  if (const char* v = getenv("CPA_SVT_BTC_PER_SM")) per_sm = std::min(atoi(v), per_sm);
  int64_t grid = (int64_t)num_sms * (per_sm > 0 ? per_sm : 1);
  if (grid > batch) grid = batch;
  kern<<<(unsigned)grid, nt, btc::SMEM, st>>>(a);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace cpa
