// fp32 dense path on the 5th-generation tensor cores (tcgen05, kind::tf32):
// TMA -> shared memory (128-byte swizzle) -> tcgen05.mma (single elected thread,
// accumulator in TMEM, double-buffered) -> tcgen05.ld -> fused epilogue.
//
//   Gram (Alg. 1 l.1):   G = A A^T             (A = X, or X^T when m > n)
//   Init (l.5-7):    W_1 = (2/L) G A - A,  Y = c_0/2 A + c_1 W_1
//   Step (l.8-11):   W_k = (4/L) G W_{k-1} - 2 W_{k-1} - W_{k-2},  Y += c_k W_k
//
// Operand precision: the tensor core reads only the TF32
// bits of an fp32 word (truncation), which misses the 1e-4 bar.  Every operand
// is therefore written by the PRODUCING epilogue as a round-to-nearest TF32
// "hi" copy (cvt.rna.tf32) and, for 3xTF32, the residual "lo" = rna(x - hi):
//   TF32:    acc = hi(G) hi(W)
//   3xTF32:  acc = hi(G) hi(W) + hi(G) lo(W) + lo(G) hi(W)
// while the recurrence itself (2 W_{k-1} + W_{k-2}, Y) is carried in full fp32.
// The Gram is always 3xTF32 (its error moves every eigenvalue).
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator +
// MMA issuer, warps 2..5 = epilogue (TMEM lane quarter = warp % 4).  Persistent
// grid (one CTA per SM), static tile schedule in grouped-M raster order so the
// CTAs in flight share A and B panels through L2.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "tma.cuh"

namespace cpa {
namespace tc {

constexpr int BM = 128;         // UMMA M (cta_group::1): TMEM lane = tile row
constexpr int BK = 32;          // fp32 elements per 128-byte swizzled row = one k-slab
constexpr int UK = 8;           // UMMA K for kind::tf32
// Accumulation chunks: the tensor core's fp32 accumulation over a long K is biased
// (measured: 3xTF32 Gram diagonal -1e-5 relative at K = 1024, -5.5e-4 at K = 65536,
// i.e. not round-to-nearest).  Each TMEM accumulator therefore covers chunk_kb
// k-blocks only; four "drain" warps add every chunk into a TMEM sum buffer with
// fp32 round-to-nearest adds in a fixed order, and four epilogue warps consume a
// finished sum while the next tile is being drained (so the global write-out of
// one tile overlaps the MMAs and drains of the next).
// Warps: 0 TMA producer, 1 TMEM allocator + MMA issuer, 2..5 drain, 6..9 epilogue.
constexpr int NTHR = 320;
constexpr int CHUNK_KB_DEFAULT = 8;    // k-blocks (x BK = 32) per TMEM accumulation
// TMEM buffers: 128-column tiles use 2 chunk accumulators + 2 tile sums (512 columns); 256-column
// tiles (single-pass TF32: the whole K in one accumulator, 25% less operand traffic per flop on
// the L2-bound steps) use 1 + 1 -- the drain of a whole-K accumulator is a one-off copy.
template <int BN> struct Bufs {
  static constexpr int NACC = BN == 128 ? 2 : 1;
  static constexpr int NSUM = BN == 128 ? 2 : 1;
};

enum Mode { GRAM = 0, INIT = 1, STEP = 2 };

struct TcArgs {
  int M, N, Kd;                  // C (M x N) = A (M x Kd) B (Kd x N)
  int terms;                     // 1 (TF32) or 3 (3xTF32)
  int mode;
  float* out_f;                  // full fp32 result (G or W_k); nullable
  float* out_h;                  // rna-TF32 hi copy
  float* out_l;                  // rna-TF32 lo copy (terms_out == 3)
  int out_split;                 // 1: write hi only; 3: hi and lo
  int64_t ld_out;
  const float* wp;               // W_{k-1} (INIT: A = X copy), full fp32
  const float* wpp;              // W_{k-2} (full)
  int64_t ld_w;
  float* y;
  int64_t ld_y;
  const SeriesParams* P;
  int k;
  int tiles_m, tiles_n;
  int dbg_lbo, dbg_sbo;          // debugging overrides of the B (MN-major) descriptor strides
  // symmetric output (M == N, BN == BM): only tiles meeting the lower triangle run
  // (from tile_list), only elements r >= c are computed, and the TF32 operand copies
  // (and out_f when mirror_f) are mirrored to (c, r)
  int sym;
  int mirror_f;
  int chunk_kb;                  // k-blocks per TMEM accumulation chunk
  const int2* tile_list;
  int ntiles_list;
  // panel mode (multi-GPU symmetric steps): tile_list / ntiles_list are this rank's sub-range of the
  // lower-triangle list; W_k (or, when out_f is null -- the last step -- the updated H) of the tile at
  // local index t is written packed to gout + t * BM * BN (row-major BM x BN, elements r >= c) instead
  // of the out_* matrices; H accumulates in place on the own tiles
  float* gout;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// UMMA shared-memory descriptor (sm_100 "version 1").  layout 2 = SWIZZLE_128B
// (K-major operands), 1 = SWIZZLE_128B_BASE32B (the only MN-major layout for tf32).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;          // version = 1 (Blackwell)
  d |= (uint64_t)layout << 61;
  return d;
}
// Instruction descriptor, kind::tf32, fp32 accumulate.
__host__ __device__ constexpr uint32_t instr_desc(int M, int N, bool b_mn_major) {
  return (1u << 4)                      // c_format = F32
         | (2u << 7)                    // a_format = TF32
         | (2u << 10)                   // b_format = TF32
         | (0u << 15)                   // a K-major
         | ((b_mn_major ? 1u : 0u) << 16)
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
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
// 32 consecutive TMEM columns of this warp's 32 lanes -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
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
__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// grouped-M raster: tiles in groups of GROUP row-tiles, columns inside a group
__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& tm, int& tn) {
  constexpr int GROUP = 16;
  const int per_group = GROUP * tiles_n;
  const int g = t / per_group;
  const int first = g * GROUP;
  const int gsize = min(GROUP, tiles_m - first);
  const int r = t % per_group;
  tm = first + r % gsize;
  tn = r / gsize;
}

template <int BN, int TERMS, bool B_MN>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 4;                  // 16 KB per term
  static constexpr int B_BYTES = BN * BK * 4;                  // BN * 128 B per term
  static constexpr int STAGE = (TERMS == 3 ? 2 : 1) * (A_BYTES + B_BYTES);
  static constexpr int STAGES = (200 * 1024) / STAGE > 6 ? 6 : (200 * 1024) / STAGE;
  static constexpr int EPI = 4 * 32 * 33 * 4;                   // per-warp 32x33 transpose buffers
  static constexpr int BYTES = STAGES * STAGE + EPI + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN, int TERMS, bool B_MN>
__global__ void __launch_bounds__(NTHR, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA_h, const __grid_constant__ CUtensorMap tmA_l,
              const __grid_constant__ CUtensorMap tmB_h, const __grid_constant__ CUtensorMap tmB_l, TcArgs a) {
  using S = Smem<BN, TERMS, B_MN>;
  constexpr int ST = S::STAGES;
  constexpr int NACC = Bufs<BN>::NACC, NSUM = Bufs<BN>::NSUM;
  constexpr int NSPLIT = TERMS == 3 ? 2 : 1;
  extern __shared__ uint8_t raw_smem[];
  uint8_t* smem = raw_smem + ((1024u - (smem_u32(raw_smem) & 1023u)) & 1023u);   // (stays in the shared window)
  float* epi_buf = (float*)(smem + ST * S::STAGE);
  uint64_t* full = (uint64_t*)(smem + ST * S::STAGE + S::EPI);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + NACC;
  uint64_t* sfull = tempty + NACC;
  uint64_t* sempty = sfull + NSUM;
  uint32_t* tmem_slot = (uint32_t*)(sempty + NSUM);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = a.tile_list ? a.ntiles_list : a.tiles_m * a.tiles_n;
  const int nk = (a.Kd + BK - 1) / BK;
  auto coords = [&](int t, int& tm, int& tn) {
    if (a.tile_list) {
      const int2 v = a.tile_list[t];
      tm = v.x;
      tn = v.y;
    } else {
      tile_coords(t, a.tiles_m, a.tiles_n, tm, tn);
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < NACC; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, 4);
    }
    for (int b = 0; b < NSUM; ++b) {
      mbar_init(sfull + b, 4);
      mbar_init(sempty + b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {  // TMEM: NACC chunk accumulators + NSUM tile sums, BN fp32 columns each
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"((NACC + NSUM) * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA_h) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB_h) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int tm, tn;
        coords(t, tm, tn);
        const int m0 = tm * BM, n0 = tn * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* st = smem + stage * S::STAGE;
          mbar_expect_tx(full + stage, S::STAGE);
          const int k0 = kb * BK;
#pragma unroll
          for (int h = 0; h < NSPLIT; ++h) {
            uint8_t* sa = st + h * S::A_BYTES;
            uint8_t* sb = st + NSPLIT * S::A_BYTES + h * S::B_BYTES;
            tma_load_2d(sa, h ? &tmA_l : &tmA_h, k0, m0, full + stage);
            if (B_MN) {
#pragma unroll
              for (int c = 0; c < BN / 32; ++c) tma_load_2d(sb + c * 4096, h ? &tmB_l : &tmB_h, n0 + 32 * c, k0, full + stage);
            } else {
              tma_load_2d(sb, h ? &tmB_l : &tmB_h, k0, n0, full + stage);
            }
          }
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    constexpr uint32_t IDESC = instr_desc(BM, BN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kb0 = 0; kb0 < nk; kb0 += a.chunk_kb) {
        mbar_wait(tempty + acc, aphase ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem_base + (uint32_t)(acc * BN);
        const int kend = kb0 + a.chunk_kb < nk ? kb0 + a.chunk_kb : nk;
        for (int kb = kb0; kb < kend; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t st = smem_u32(smem + stage * S::STAGE);
            const uint32_t a_h = st, a_l = st + S::A_BYTES;
            const uint32_t b_h = st + NSPLIT * S::A_BYTES, b_l = b_h + S::B_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / UK; ++kk) {
              // A K-major: +32 B per UMMA_K inside the swizzled row; B MN-major: +1 KB (one 8-row group)
              const uint32_t aoff = kk * UK * 4;
              const uint32_t boff = B_MN ? kk * 1024 : kk * UK * 4;
              // MN-major B (tf32): SW128 with 32-byte atoms; 32-element MN chunks LBO = 4 KB
              // apart, 4-row K groups SBO = 512 B apart; one UMMA_K = 8 rows = +1 KB.
              const uint32_t blbo = B_MN ? (a.dbg_lbo ? a.dbg_lbo : 4096) : 16;
              const uint32_t bsbo = B_MN ? (a.dbg_sbo ? a.dbg_sbo : 512) : 1024;
              const uint32_t blay = B_MN ? 1u : 2u;
              const uint64_t dAh = smem_desc(a_h + aoff, 16, 1024);
              const uint64_t dBh = smem_desc(b_h + boff, blbo, bsbo, blay);
              const uint32_t accum = (kb > kb0 || kk > 0) ? 1u : 0u;
              mma_tf32(dtm, dAh, dBh, IDESC, accum);
              if (TERMS == 3) {
                const uint64_t dAl = smem_desc(a_l + aoff, 16, 1024);
                const uint64_t dBl = smem_desc(b_l + boff, blbo, bsbo, blay);
                mma_tf32(dtm, dAh, dBl, IDESC, 1u);
                mma_tf32(dtm, dAl, dBh, IDESC, 1u);
              }
            }
            mma_commit(empty + stage);  // frees the smem stage when these MMAs complete
          }
          __syncwarp();
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) mma_commit(tfull + acc);  // chunk accumulator ready for the epilogue
        __syncwarp();
        if (++acc == NACC) { acc = 0; aphase ^= 1; }
      }
    }
  } else if (warp < 6) {
    // ============================ drain (warps 2..5) ======================
    // sum_b = ((c_0 + c_1) + c_2) + ... over the tile's chunk accumulators (fp32 RN adds)
    const int quarter = warp & 3;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int acc = 0, sb = 0;
    uint32_t aphase = 0, sphase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(sempty + sb, sphase ^ 1);
      tc_fence_after();
      const uint32_t sum_col = (uint32_t)((NACC + sb) * BN);
      for (int kb0 = 0; kb0 < nk; kb0 += a.chunk_kb) {
        mbar_wait(tfull + acc, aphase);
        tc_fence_after();
#pragma unroll 1
        for (int cc = 0; cc < BN / 32; ++cc) {
          float v[32];
          tmem_ld32(tmem_base + lane_off + (uint32_t)(acc * BN + cc * 32), v);
          if (kb0 > 0) {
            float u[32];
            tmem_ld32(tmem_base + lane_off + sum_col + cc * 32, u);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = u[j] + v[j];
          }
          tmem_st32(tmem_base + lane_off + sum_col + cc * 32, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty + acc);
        if (++acc == NACC) { acc = 0; aphase ^= 1; }
      }
      if (lane == 0) mbar_arrive(sfull + sb);
      if (++sb == NSUM) { sb = 0; sphase ^= 1; }
    }
  } else {
    // ============================ epilogue (warps 6..9) ===================
    // Each warp owns TMEM lanes [32q, 32q+32) = 32 tile rows.  Per 32-column chunk:
    // tcgen05.ld of the tile sum (thread = row), transpose through a private 32x33 smem
    // buffer, then lane = column: every global load/store is one coalesced 128-byte row
    // segment.
    const int quarter = warp & 3;  // TMEM lane quarter accessible to this warp
    float* tb = epi_buf + (warp - 6) * (32 * 33);
    int sb = 0;
    uint32_t sphase = 0;
    const SeriesParams* P = a.P;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int tm, tn;
      coords(t, tm, tn);
      const int t_local = t;
      mbar_wait(sfull + sb, sphase);
      tc_fence_after();
      const uint32_t sum_col = (uint32_t)((NACC + sb) * BN);
      const int row0 = tm * BM + quarter * 32;
      float s2 = 0.f, h0 = 0.f, c1 = 0.f, ck = 0.f;
      if (a.mode != GRAM) {
        s2 = (float)P->scale2;
        h0 = (float)(0.5 * P->c[0]);
        c1 = (float)P->c[1];
        ck = (float)P->c[a.k];
      }
#pragma unroll 1
      for (int cc = 0; cc < BN / 32; ++cc) {
        {
          float v[32];
          tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + sum_col + cc * 32, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) tb[lane * 33 + j] = v[j];
        }
        __syncwarp();
        const int cbase = tn * BN + cc * 32;
        const int c = cbase + lane;
        if (c < a.N) {
#pragma unroll 4
          for (int i = 0; i < 32; ++i) {
            const int r = row0 + i;
            if (r >= a.M) break;
            if (a.sym && c > r) continue;                          // upper triangle: mirrored below
            const float accv = tb[i * 33 + lane];
            float w = accv;
            if (a.mode == INIT) {
              const float x = a.wp[(int64_t)r * a.ld_w + c];
              w = s2 * accv - x;                                   // W_1 = B_hat A
              a.y[(int64_t)r * a.ld_y + c] = h0 * x + c1 * w;      // Y = c0/2 A + c1 W_1
            } else if (a.mode == STEP) {
              const float wp = a.wp[(int64_t)r * a.ld_w + c];
              const float wpp = a.wpp[(int64_t)r * a.ld_w + c];
              w = 2.f * s2 * accv - 2.f * wp - wpp;                // W_k = 2 B_hat W_{k-1} - W_{k-2}
              float* yp = a.y + (int64_t)r * a.ld_y + c;
              const float yv = fmaf(ck, w, *yp);                   // Y += c_k W_k
              *yp = yv;
              if (a.gout) {   // panel mode: the all-gather slot (W_k, or H at the last step)
                a.gout[(int64_t)t_local * (BM * BN) + (int64_t)(r - tm * BM) * BN + (c - tn * BN)] =
                    a.out_f ? w : yv;
                continue;
              }
            }
            const int64_t o = (int64_t)r * a.ld_out + c;
            if (a.out_f) a.out_f[o] = w;
            if (a.out_h) {
              const float hi = rna_tf32(w);
              a.out_h[o] = hi;
              if (a.out_split == 3) a.out_l[o] = rna_tf32(w - hi);
            }
            if (a.sym) tb[i * 33 + lane] = w;
          }
        }
        __syncwarp();
        if (a.sym && !a.gout) {
          // mirror (r, c) -> (c, r) for r > c from the natural layout (lane = row): for a
          // fixed column j the warp writes one coalesced 128-byte segment of row c
          const int r = row0 + lane;
          if (r < a.M) {
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
              const int cm = cbase + j;
              if (cm >= a.N || cm >= r) break;
              const float w = tb[lane * 33 + j];
              const int64_t o = (int64_t)cm * a.ld_out + r;
              if (a.mirror_f && a.out_f) a.out_f[o] = w;
              if (a.out_h) {
                const float hi = rna_tf32(w);
                a.out_h[o] = hi;
                if (a.out_split == 3) a.out_l[o] = rna_tf32(w - hi);
              }
            }
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty + sb);
      if (++sb == NSUM) { sb = 0; sphase ^= 1; }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"((NACC + NSUM) * BN));
  }
}

// ------------------------------------------------------------------ host side
// 2-D fp32 tensor (rows x cols, row stride ld elements), box {32 cols, box_rows}, 128B swizzle
// (32-byte swizzle atoms for MN-major operands)
static cudaError_t make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld,
                            int box_rows, bool atom32 = false) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * sizeof(float))};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int BN, int TERMS, bool B_MN>
static cudaError_t launch_t(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
                            const CUtensorMap& bl, const TcArgs& a, int num_sms, cudaStream_t st) {
  using S = Smem<BN, TERMS, B_MN>;
  auto fn = k_tc_gemm<BN, TERMS, B_MN>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, S::BYTES);
  if (e != cudaSuccess) return e;
  const int ntiles = a.tile_list ? a.ntiles_list : a.tiles_m * a.tiles_n;
  const int grid = ntiles < num_sms ? ntiles : num_sms;
  fn<<<grid, NTHR, S::BYTES, st>>>(ah, al, bh, bl, a);
  return cudaGetLastError();
}

// Lower-triangle tile list (tm >= tn) of a T x T tile grid in the grouped-M raster
// order of tile_coords; built once per T and kept on the device.
// (one list per device: handles on several devices, or in several host threads, share the cache
// under a mutex)
static const int2* sym_tile_list(int tiles_m, int tiles_n, int bm, int bn, int* count) {
  static std::map<std::pair<int, long long>, std::pair<int2*, int>> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  const auto key = std::make_pair(dev, ((long long)tiles_m << 40) | ((long long)tiles_n << 16) | (bn << 1) | (bm == 128));
  auto it = cache.find(key);
  if (it != cache.end()) {
    *count = it->second.second;
    return it->second.first;
  }
  std::vector<int2> v;
  constexpr int GROUP = 16;
  for (int first = 0; first < tiles_m; first += GROUP) {
    const int gsize = std::min(GROUP, tiles_m - first);
    for (int tn = 0; tn < tiles_n; ++tn)
      for (int r = 0; r < gsize; ++r)
        if ((int64_t)(first + r) * bm + bm - 1 >= (int64_t)tn * bn) v.push_back(make_int2(first + r, tn));
  }
  int2* d = nullptr;
  if (cudaMalloc(&d, v.size() * sizeof(int2)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, v.data(), v.size() * sizeof(int2), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  cache[key] = {d, (int)v.size()};
  *count = (int)v.size();
  return d;
}

template <int BN>
static cudaError_t tc_gemm_bn(int mode, int terms, int M, int N, int Kd, const float* Ah, const float* Al,
                              int64_t lda, const float* Bh, const float* Bl, int64_t ldb, bool b_mn, float* out_f,
                              float* out_h, float* out_l, int out_split, int64_t ld_out, const float* wp,
                              const float* wpp, int64_t ld_w, float* y, int64_t ld_y, const SeriesParams* P, int k,
                              int num_sms, cudaStream_t st, int sym, int64_t p_tile0 = -1, int64_t p_ntile = 0,
                              float* gout = nullptr) {
  using namespace tc;
  CUtensorMap ah, al, bh, bl;
  cudaError_t e = make_map(&ah, Ah, M, Kd, lda, BM);
  if (e == cudaSuccess) e = make_map(&al, terms == 3 ? Al : Ah, M, Kd, lda, BM);
  if (b_mn) {
    if (e == cudaSuccess) e = make_map(&bh, Bh, Kd, N, ldb, BK, true);
    if (e == cudaSuccess) e = make_map(&bl, terms == 3 ? Bl : Bh, Kd, N, ldb, BK, true);
  } else {
    if (e == cudaSuccess) e = make_map(&bh, Bh, N, Kd, ldb, BN);
    if (e == cudaSuccess) e = make_map(&bl, terms == 3 ? Bl : Bh, N, Kd, ldb, BN);
  }
  if (e != cudaSuccess) return e;
  TcArgs a{};
  a.M = M; a.N = N; a.Kd = Kd; a.terms = terms; a.mode = mode;
  a.out_f = out_f; a.out_h = out_h; a.out_l = out_l; a.out_split = out_split; a.ld_out = ld_out;
  a.wp = wp; a.wpp = wpp; a.ld_w = ld_w; a.y = y; a.ld_y = ld_y; a.P = P; a.k = k;
  a.tiles_m = (M + BM - 1) / BM;
  a.tiles_n = (N + BN - 1) / BN;
  if (sym) {
    if (M != N) return cudaErrorInvalidValue;
    a.sym = 1;
    a.mirror_f = mode == GRAM;
    a.tile_list = sym_tile_list(a.tiles_m, a.tiles_n, BM, BN, &a.ntiles_list);
    if (!a.tile_list) return cudaErrorMemoryAllocation;
    if (p_tile0 >= 0) {   // panel mode: this rank's sub-range of the list, packed output
      if (mode != STEP || !gout || p_tile0 + p_ntile > a.ntiles_list) return cudaErrorInvalidValue;
      a.tile_list += p_tile0;
      a.ntiles_list = (int)p_ntile;
      a.gout = gout;
      if (p_ntile == 0) return cudaSuccess;
    }
  }
  // 256-wide tiles have one accumulator: the whole K for single-pass TF32, 16 k-blocks (K = 512)
  // for 3xTF32 (the MMA waits for each drain -- a short bubble against 3x the MMA work)
  a.chunk_kb = BN == 256 ? (terms == 1 ? (Kd + BK - 1) / BK : 16) : CHUNK_KB_DEFAULT;
  if (const char* v = getenv("CPA_SVT_TC_CHUNK")) a.chunk_kb = atoi(v) > 0 ? atoi(v) : a.chunk_kb;
  if (const char* v = getenv("CPA_SVT_DBG_LBO")) a.dbg_lbo = atoi(v);
  if (const char* v = getenv("CPA_SVT_DBG_SBO")) a.dbg_sbo = atoi(v);
  if (terms == 3) {
    return b_mn ? launch_t<BN, 3, true>(ah, al, bh, bl, a, num_sms, st)
                : launch_t<BN, 3, false>(ah, al, bh, bl, a, num_sms, st);
  }
  return b_mn ? launch_t<BN, 1, true>(ah, al, bh, bl, a, num_sms, st)
              : launch_t<BN, 1, false>(ah, al, bh, bl, a, num_sms, st);
}

}  // namespace tc

// One tcgen05 GEMM with the fused epilogue.
//   A: M x Kd, K-major (row stride lda), given as hi (and lo) fp32 copies
//   B: b_mn ? Kd x N (N contiguous, row stride ldb) : N x Kd (K contiguous)
// 128 x 128 tiles (BM = BN: the symmetric form needs square tiles).
cudaError_t tc_gemm(int mode, int terms, int M, int N, int Kd, const float* Ah, const float* Al, int64_t lda,
                    const float* Bh, const float* Bl, int64_t ldb, bool b_mn, float* out_f, float* out_h,
                    float* out_l, int out_split, int64_t ld_out, const float* wp, const float* wpp, int64_t ld_w,
                    float* y, int64_t ld_y, const SeriesParams* P, int k, int num_sms, cudaStream_t st, int sym) {
  // single-pass TF32 recurrence and line-12 products: 128 x 256 tiles (B MN-major); the
  // 3xTF32 products and the Gram keep 128 x 128 tiles with chunked accumulation
  int wide = terms == 1 && mode != 0 && b_mn;
  if (mode == 0 && terms == 1 && b_mn && !sym) wide = 1;
  // 3xTF32: the line-12 product gains from 256-wide tiles (213 -> 159 ms at c5), the steps do not
  // (950 -> 989 ms: one accumulator means the MMA waits for every chunk drain)
  if (terms == 3 && mode == 0 && !sym && b_mn) wide = 1;
  if (const char* v = getenv("CPA_SVT_TC_WIDE")) wide = wide && atoi(v) != 0;
  if (wide)
    return tc::tc_gemm_bn<256>(mode, terms, M, N, Kd, Ah, Al, lda, Bh, Bl, ldb, b_mn, out_f, out_h, out_l, out_split,
                               ld_out, wp, wpp, ld_w, y, ld_y, P, k, num_sms, st, sym);
  return tc::tc_gemm_bn<128>(mode, terms, M, N, Kd, Ah, Al, lda, Bh, Bl, ldb, b_mn, out_f, out_h, out_l, out_split,
                             ld_out, wp, wpp, ld_w, y, ld_y, P, k, num_sms, st, sym);
}

// ------------------------------------------------------------------ multi-GPU panels (symmetric steps)
// The step's tile geometry: 128 x 256 tiles for single-pass TF32 steps, 128 x 128 for 3xTF32 (the
// choice tc_gemm makes for mode STEP), and its lower-triangle tile list.
static int tf32_step_bn(int terms) { return terms == 1 ? 256 : 128; }

cudaError_t tf32_panel_list(int64_t s, int terms, const int2** list, int* count, int* bn) {
  const int BN = tf32_step_bn(terms);
  const int tm = (int)((s + tc::BM - 1) / tc::BM), tn = (int)((s + BN - 1) / BN);
  *list = tc::sym_tile_list(tm, tn, tc::BM, BN, count);
  *bn = BN;
  return *list ? cudaSuccess : cudaErrorMemoryAllocation;
}

// Step k of the symmetric TF32 recurrence on tiles [tile0, tile0 + ntile) of the list: W_k (or H
// at the last step, out_f == nullptr) packed into gout.  Arguments as tc_gemm mode STEP.
cudaError_t tc_gemm_panel(int terms, int s, const float* Ah, const float* Al, int64_t lda, const float* Bh,
                          const float* Bl, int64_t ldb, bool last, int64_t ld_out, const float* wp, const float* wpp,
                          int64_t ld_w, float* y, int64_t ld_y, const SeriesParams* P, int k, int64_t tile0,
                          int64_t ntile, float* gout, int num_sms, cudaStream_t st) {
  float* dummy = last ? nullptr : gout;   // non-null out_f marks "W_k" (the epilogue writes gout only)
  if (terms == 1)
    return tc::tc_gemm_bn<256>(2, 1, s, s, s, Ah, Al, lda, Bh, Bl, ldb, true, dummy, nullptr, nullptr, 1, ld_out, wp,
                               wpp, ld_w, y, ld_y, P, k, num_sms, st, 1, tile0, ntile, gout);
  return tc::tc_gemm_bn<128>(2, 3, s, s, s, Ah, Al, lda, Bh, Bl, ldb, true, dummy, nullptr, nullptr, 3, ld_out, wp,
                             wpp, ld_w, y, ld_y, P, k, num_sms, st, 1, tile0, ntile, gout);
}

// Gathered slots -> W_k: fp32 lower triangle into Wf, TF32 hi / lo copies of both triangles into
// Wh / Wl (the next step's B operand); at the last step (H != nullptr) the lower triangle into H.
// One CTA per tile of the list; owner p of list entry t: [ntiles p / P, ntiles (p+1) / P).
__global__ void __launch_bounds__(256) k_tf32_sym_unpack(const float* __restrict__ g, const int2* __restrict__ list,
                                                         int64_t ntiles, int P, int64_t slot_tiles, int BN, int64_t s,
                                                         int64_t ld, float* Wf, float* Wh, float* Wl, float* H) {
  __shared__ float tb[8][32][33];   // one 32 x 32 transpose buffer per warp
  const int64_t t = blockIdx.x;
  int p = (int)(t * P / ntiles);
  while (p + 1 < P && ntiles * (p + 1) / P <= t) ++p;
  while (p > 0 && ntiles * p / P > t) --p;
  const int64_t lt = t - ntiles * p / P;
  const float* src = g + ((int64_t)p * slot_tiles + lt) * (tc::BM * BN);
  const int2 tt = list[t];
  const int64_t r0 = (int64_t)tt.x * tc::BM, c0 = (int64_t)tt.y * BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nsub = (tc::BM / 32) * (BN / 32);
  // 32 x 32 sub-blocks: direct (r, c) stores along c, mirrored (c, r) stores along r via the buffer
  for (int sbk = warp; sbk < nsub; sbk += 8) {
    const int sr = (sbk / (BN / 32)) * 32, sc = (sbk % (BN / 32)) * 32;
    if (r0 + sr + 31 < c0 + sc) continue;   // entirely above the diagonal: nothing computed there
    for (int i = 0; i < 32; ++i) {
      const int64_t r = r0 + sr + i, c = c0 + sc + lane;
      const float v = __ldcs(src + (int64_t)(sr + i) * BN + sc + lane);
      tb[warp][i][lane] = v;
      if (r >= s || c >= s || c > r) continue;
      if (H) {
        H[r * ld + c] = v;
        continue;
      }
      Wf[r * ld + c] = v;
      const float hi = tc::rna_tf32(v);
      Wh[r * ld + c] = hi;
      if (Wl) Wl[r * ld + c] = tc::rna_tf32(v - hi);
    }
    __syncwarp();
    if (!H) {
      for (int j = 0; j < 32; ++j) {   // mirror: row c0 + sc + j of W, columns r0 + sr + lane
        const int64_t c = c0 + sc + j, r = r0 + sr + lane;
        if (r >= s || c >= s || c >= r) continue;
        const float v = tb[warp][lane][j];
        const float hi = tc::rna_tf32(v);
        Wh[c * ld + r] = hi;
        if (Wl) Wl[c * ld + r] = tc::rna_tf32(v - hi);
      }
    }
    __syncwarp();
  }
}

cudaError_t tf32_sym_unpack(const float* gbuf, int64_t s, int terms, int P, int64_t slot_tiles, int64_t ld, float* Wf,
                            float* Wh, float* Wl, float* H, cudaStream_t st) {
  const int2* list;
  int count, bn;
  cudaError_t e = tf32_panel_list(s, terms, &list, &count, &bn);
  if (e != cudaSuccess) return e;
  if (count == 0) return cudaSuccess;
  k_tf32_sym_unpack<<<count, 256, 0, st>>>(gbuf, list, count, P, slot_tiles, bn, s, ld, Wf, Wh, terms == 3 ? Wl : nullptr,
                                          H);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ prep / finish
// A (s x L, ld lda) <- X or X^T (m x n, ldx); writes full, hi, lo copies
__global__ void k_tf32_prep(const float* X, int64_t m, int64_t n, int64_t ldx, bool transpose, float* Af, float* Ah,
                            float* Al, int64_t lda) {
  const int64_t s = transpose ? n : m, L = transpose ? m : n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s * L; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i, j;
    if (transpose) {  // read X coalesced: e -> (X row j, X col i)
      j = e / s;
      i = e % s;
    } else {
      i = e / L;
      j = e % L;
    }
    const float x = transpose ? X[j * ldx + i] : X[i * ldx + j];
    const float hi = tc::rna_tf32(x);
    Af[i * lda + j] = x;
    Ah[i * lda + j] = hi;
    if (Al) Al[i * lda + j] = tc::rna_tf32(x - hi);
  }
}

// caller Y (m x n, ldy) <- Y_int (s x L) or its transpose
__global__ void k_tf32_finish(const float* Yi, int64_t ldi, int64_t m, int64_t n, bool transpose, float* Y,
                              int64_t ldy) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    Y[i * ldy + j] = transpose ? Yi[j * ldi + i] : Yi[i * ldi + j];
  }
}

__global__ void k_eye_f32(float* I, int64_t s, int64_t ld) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s * ld; e += (int64_t)gridDim.x * blockDim.x)
    I[e] = (e / ld == e % ld) ? 1.f : 0.f;
}
cudaError_t tf32_eye(float* I, int64_t s, int64_t ld, int num_sms, cudaStream_t st) {
  k_eye_f32<<<num_sms * 8, 256, 0, st>>>(I, s, ld);
  return cudaGetLastError();
}

// Symmetric s x s form, k = 1 (Alg. 1 l.5-7): W_1 = (2/L) G - I (full, hi, lo), H = c_0/2 I + c_1 W_1.
__global__ void k_sym_init_f32(const float* G, int64_t s, int64_t ld, float* Wf, float* Wh, float* Wl, float* H,
                               const SeriesParams* P) {
  const float s2 = (float)P->scale2, h0 = (float)(0.5 * P->c[0]), c1 = (float)P->c[1];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s * ld; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ld, j = e % ld;
    const float id = (i == j) ? 1.f : 0.f;
    const float w = j < s ? s2 * G[e] - id : 0.f;
    const float hi = tc::rna_tf32(w);
    Wf[e] = w;
    Wh[e] = hi;
    if (Wl) Wl[e] = tc::rna_tf32(w - hi);
    H[e] = j < s ? h0 * id + c1 * w : 0.f;
  }
}
cudaError_t tf32_sym_init(const float* G, int64_t s, int64_t ld, float* Wf, float* Wh, float* Wl, float* H,
                          const SeriesParams* P, int num_sms, cudaStream_t st) {
  k_sym_init_f32<<<num_sms * 8, 256, 0, st>>>(G, s, ld, Wf, Wh, Wl, H, P);
  return cudaGetLastError();
}

// H (lower triangle valid) -> hi / lo TF32 copies of the full symmetric matrix, through
// 32 x 32 shared-memory tiles (every global access coalesced).
__global__ void k_sym_prep_f32(const float* H, int64_t s, int64_t ld, float* Hh, float* Hl) {
  __shared__ float t[32][33];
  const int T = (int)((s + 31) / 32);
  for (int64_t b = blockIdx.x; b < (int64_t)T * T; b += gridDim.x) {
    const int bi = (int)(b / T), bj = (int)(b % T);
    if (bi < bj) continue;
    const int64_t r0 = (int64_t)bi * 32, c0 = (int64_t)bj * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int64_t r = r0 + i, c = c0 + threadIdx.x;
      t[i][threadIdx.x] = (r < s && c < s && (bi != bj || c <= r)) ? H[r * ld + c] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int64_t r = r0 + i, c = c0 + threadIdx.x;   // lower block (bi, bj)
      // diagonal block: element (r, c) above its diagonal comes from (c, r)
      const float v = (bi == bj && threadIdx.x > i) ? t[threadIdx.x][i] : t[i][threadIdx.x];
      if (r < s && c < s) {
        const float hi = tc::rna_tf32(v);
        Hh[r * ld + c] = hi;
        Hl[r * ld + c] = tc::rna_tf32(v - hi);
      }
      const int64_t rm = c0 + i, cm = r0 + threadIdx.x;  // mirror block (bj, bi): element (rm, cm) = H(cm, rm)
      if (bi != bj && rm < s && cm < s) {
        const float w = t[threadIdx.x][i];
        const float hi = tc::rna_tf32(w);
        Hh[rm * ld + cm] = hi;
        Hl[rm * ld + cm] = tc::rna_tf32(w - hi);
      }
    }
    __syncthreads();
  }
}
cudaError_t tf32_sym_prep(const float* H, int64_t s, int64_t ld, float* Hh, float* Hl, int num_sms, cudaStream_t st) {
  k_sym_prep_f32<<<num_sms * 8, dim3(32, 8), 0, st>>>(H, s, ld, Hh, Hl);
  return cudaGetLastError();
}

cudaError_t tf32_prep(const float* X, int64_t m, int64_t n, int64_t ldx, bool transpose, float* Af, float* Ah,
                      float* Al, int64_t lda, int num_sms, cudaStream_t st) {
  k_tf32_prep<<<num_sms * 8, 256, 0, st>>>(X, m, n, ldx, transpose, Af, Ah, Al, lda);
  return cudaGetLastError();
}
cudaError_t tf32_finish(const float* Yi, int64_t ldi, int64_t m, int64_t n, bool transpose, float* Y, int64_t ldy,
                        int num_sms, cudaStream_t st) {
  k_tf32_finish<<<num_sms * 8, 256, 0, st>>>(Yi, ldi, m, n, transpose, Y, ldy);
  return cudaGetLastError();
}

}  // namespace cpa
