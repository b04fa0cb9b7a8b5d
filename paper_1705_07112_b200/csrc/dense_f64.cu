// fp64 dense path on sm_100a: Gram product and the fused Chebyshev recurrence
// step, both on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4;
// sm_100a has no tcgen05 kind::f64).
//
//   Gram  (Alg. 1 line 1):      G = X X^T (left) / X^T X (right),
//          lower-triangle tiles only, mirrored -> G exactly symmetric.
//   Init  (Alg. 1 lines 5-7): W_1 = (2/L) G X - X,
//          Y = c_0/2 X + c_1 W_1.
//   Step  (Alg. 1 lines 8-11): W_k = (4/L) G W_{k-1} - 2 W_{k-1} - W_{k-2},
//          Y += c_k W_k   -- GEMM + update + accumulation in ONE kernel.
//
// CTA tile 64x64, k-slab 16, 4 warps of 32x32 (4x4 DMMA tiles), 4-stage
// cp.async pipeline (16-byte copies when the leading dimension allows).
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "tma.cuh"

namespace cpa {

#ifndef CPA_DMMA_BK
#define CPA_DMMA_BK 16
#endif
#ifndef CPA_DMMA_STAGES
#define CPA_DMMA_STAGES 4
#endif
constexpr int BM = 64, BN = 64, BKS = CPA_DMMA_BK, STAGES = CPA_DMMA_STAGES, NTHREADS = 128;
constexpr int PAD = 4;

enum EpiMode { EPI_GRAM = 0, EPI_INIT = 1, EPI_STEP = 2, EPI_STORE = 3 };

struct GemmArgs {
  int64_t M, N, Kd;             // C (M x N) = A (M x Kd) * B (Kd x N)
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* Wout;                 // W_k (nullable)
  int64_t ldwo;
  const double* Wp;             // W_{k-1} (INIT: X)
  int64_t ldwp;
  const double* Wpp;            // W_{k-2} (STEP)
  int64_t ldwpp;
  double* Y;
  int64_t ldy;
  const SeriesParams* P;
  int k;                        // coefficient index (STEP)
  int vec_a, vec_b;             // 16-byte loads allowed
  const double* gscale;         // GRAM: optional device scalar multiplying the output (exact power of 2)
  double* partial;              // GRAM split-K: tiles * split * 64 * 64 partial sums (gridDim.y = split)
  int* tcount;                  // GRAM split-K: per-tile arrival counters (zeroed before the launch)
  int sS, sq0;                  // split-K across launches: S units per tile, this launch is unit sq0
                                // (sS = 0: one launch, gridDim.y units)
};

// Elements per stage of an operand whose global slab is OUTER x INNER (INNER contiguous).
template <bool KCONTIG, int MN>
struct OpLayout {
  static constexpr int OUTER = KCONTIG ? MN : BKS;
  static constexpr int INNER = KCONTIG ? BKS : MN;
  static constexpr int LD = INNER + PAD;
  static constexpr int SIZE = OUTER * LD;
  // smem index of element (mn, k)
  __device__ static __forceinline__ int idx(int mn, int k) { return KCONTIG ? mn * LD + k : k * LD + mn; }
};

// Copy one OUTER x INNER slab starting at global (o0, i0); elements outside
// [0, olim) x [0, ilim) are zero-filled.  16-byte chunks go through
// cp.async.cg (L2 only); ragged or unaligned elements are loaded with ld.global.cg
// and stored directly -- never through L1, because the recurrence rewrites
// W in place while a persistent CTA may still hold old lines in its L1.
template <class L>
__device__ __forceinline__ void load_slab(double* s, const double* g, int64_t ld, int64_t o0, int64_t i0,
                                          int64_t olim, int64_t ilim, bool vec) {
  constexpr int CH = L::INNER / 2;                // 16-byte chunks per row
  constexpr int TOTAL = L::OUTER * CH;
#pragma unroll
  for (int c = threadIdx.x; c < TOTAL; c += NTHREADS) {
    const int o = c / CH, i = (c % CH) * 2;
    const int64_t go = o0 + o, gi = i0 + i;
    double* dst = s + o * L::LD + i;
    const bool orow = go < olim;
    const double* src = g + (orow ? go : 0) * ld + gi;
    if (vec && orow && gi + 1 < ilim) {
      cp_async16(dst, src, true);
    } else {
      dst[0] = orow && gi < ilim ? __ldcg(src) : 0.0;
      dst[1] = orow && gi + 1 < ilim ? __ldcg(src + 1) : 0.0;
    }
  }
}

// acc = A[m0:m0+64, :] * B[:, n0:n0+64] over the full Kd, 4-stage cp.async pipeline.
// Ends with all stages drained and a CTA barrier (smem reusable on return).
template <bool A_KC, bool B_KC>
__device__ __forceinline__ void mainloop(const double* Ag, int64_t lda, const double* Bg, int64_t ldb, int64_t M,
                                         int64_t N, int64_t Kd, int64_t m0, int64_t n0, bool vec_a, bool vec_b,
                                         double* smem, double (&acc)[4][4][2], int kbeg = 0, int kend = -1) {
  using LA = OpLayout<A_KC, BM>;
  using LB = OpLayout<B_KC, BN>;
  double* sA = smem;
  double* sB = smem + STAGES * LA::SIZE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  if (kend < 0) kend = (int)((Kd + BKS - 1) / BKS);
  const int nk = kend - kbeg;
  auto load_stage = [&](int kt, int st) {
    const int64_t k0 = (int64_t)(kbeg + kt) * BKS;
    if (A_KC) load_slab<LA>(sA + st * LA::SIZE, Ag, lda, m0, k0, M, Kd, vec_a);
    else      load_slab<LA>(sA + st * LA::SIZE, Ag, lda, k0, m0, Kd, M, vec_a);
    if (B_KC) load_slab<LB>(sB + st * LB::SIZE, Bg, ldb, n0, k0, N, Kd, vec_b);
    else      load_slab<LB>(sB + st * LB::SIZE, Bg, ldb, k0, n0, Kd, N, vec_b);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) load_stage(nxt, nxt % STAGES);
      cp_async_commit();
    }
    const double* cA = sA + (kt % STAGES) * LA::SIZE;
    const double* cB = sB + (kt % STAGES) * LB::SIZE;
#pragma unroll
    for (int kk = 0; kk < BKS; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = cA[LA::idx(wm + i * 8 + g, kk + t)];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = cB[LB::idx(wn + j * 8 + g, kk + t)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// Fused recurrence epilogue on one 64x64 accumulator tile (Alg. 1 lines 5-11).
//   init:  W_1 = (2/L) acc - X,                   Y  = c_0/2 X + c_1 W_1
//   step:  W_k = (4/L) acc - 2 W_{k-1} - W_{k-2}, Y += c_k W_k
// Wp = W_{k-1} (init: X), Wpp = W_{k-2}; Wout may alias Wpp (in place).  Loads
// bypass L1 (ld.global.cg): other CTAs of a persistent launch rewrite W and Y.
__device__ __forceinline__ void cheb_epilogue(const double (&acc)[4][4][2], int64_t m0, int64_t n0, int64_t M,
                                              int64_t N, bool init, const double* Wp, int64_t ldwp,
                                              const double* Wpp, int64_t ldwpp, double* Wout, int64_t ldwo,
                                              double* Y, int64_t ldy, const SeriesParams* P, int k) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const double s2 = P->scale2;
  const double h0 = 0.5 * P->c[0], c1 = P->c[1];
  const double s4 = 2.0 * s2, ck = init ? 0.0 : P->c[k];
  // Wout may alias Wpp (W_k overwrites W_{k-2} in place), so the compiler cannot hoist
  // loads past stores: load one 8-element row group into registers first, then store.
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + wm + i * 8 + g;
    const bool rok = r < M;
    double vp[8], vpp[8], vy[8];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + wn + j * 8 + 2 * t + e;
        const bool ok = rok && c < N;
        vp[j * 2 + e] = ok ? __ldcg(Wp + r * ldwp + c) : 0.0;
        vpp[j * 2 + e] = (ok && !init) ? __ldcg(Wpp + r * ldwpp + c) : 0.0;
        vy[j * 2 + e] = (ok && !init) ? __ldcg(Y + r * ldy + c) : 0.0;
      }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + wn + j * 8 + 2 * t + e;
        if (!(rok && c < N)) continue;
        const int q = j * 2 + e;
        double w, y;
        if (init) {
          w = s2 * acc[i][j][e] - vp[q];                 // W_1 = B_hat X
          y = h0 * vp[q] + c1 * w;                       // Y = c0/2 W_0 + c1 W_1
        } else {
          w = s4 * acc[i][j][e] - 2.0 * vp[q] - vpp[q];  // W_k = 2 B_hat W_{k-1} - W_{k-2}
          y = vy[q] + ck * w;                            // Y += c_k W_k
        }
        if (Wout) Wout[r * ldwo + c] = w;
        Y[r * ldy + c] = y;
      }
  }
}

// ---------------------------------------------------------------------------
// Persistent dataflow kernel: the init and all K-2 steps in ONE launch.
// Tiles are claimed in ticket order (step k, panel p, tile q); a tile of step
// k waits only until its panel of step k-1 is complete (left: column panel of
// W_{k-1} feeding the B operand; right: row panel feeding A), so SMs that
// finish a step early start the next one and the 28-launch tail effect and
// launch gaps disappear.  In-place W_k -> W_{k-2} is safe because every
// reader of W_{k-2}'s panel belongs to step k-1, which is complete.
// ---------------------------------------------------------------------------
struct FlowArgs {
  int64_t M, N, s;      // output M x N (shape of X); s = Gram side
  const double* G;
  const double* X;
  int64_t ldx;
  double* Wa;
  double* Wb;
  int64_t ldw;
  double* Y;
  int64_t ldy;
  const SeriesParams* P;
  int K;
  int tiles_m, tiles_n;
  int split;            // k-splits per tile (units per tile)
  int* sync;            // [0] ticket | K * npanels panel counters | ntiles split counters
  double* partial;      // ntiles * (split - 1) * 64 * 64 (split > 1)
  int vec_x, vec_w, vec_g;
};

__device__ __forceinline__ void red_release_add_i32(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin (relaxed loads: no L1 invalidation per poll) until *p >= target, then one
// acquire fence: the fence-based form of the release/acquire pattern.
__device__ __forceinline__ void wait_geq(const int* p, int target) {
  while (ld_relaxed(p) < target) __nanosleep(32);
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
}

// Unit = (step k, panel, tile-in-panel, k-split q); claimed in that order.
// Splits q < split-1 publish partial sums; split split-1 waits for them, adds
// all partials in the fixed order q = 0..split-1 (deterministic) and runs the
// fused epilogue.  A unit of step k >= 2 first waits until its panel of
// step k-1 is complete.
#ifndef CPA_FLOW_MINB
#define CPA_FLOW_MINB 3
#endif
template <bool LEFT>
__global__ void __launch_bounds__(NTHREADS, CPA_FLOW_MINB) k_cheb_flow(FlowArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_ticket;
  const int npanels = LEFT ? a.tiles_n : a.tiles_m;
  const int ninner = LEFT ? a.tiles_m : a.tiles_n;
  const int ntiles = a.tiles_m * a.tiles_n;
  const int S = a.split;
  const int per_step = ntiles * S;
  const int total = (a.K - 1) * per_step;
  int* panel_cnt = a.sync + 1;
  int* split_cnt = a.sync + 1 + a.K * npanels;
  const int nk = (int)((a.s + BKS - 1) / BKS);
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.sync, 1);
    __syncthreads();
    const int tk = s_ticket;
    if (tk >= total) break;
    const int k = 1 + tk / per_step;
    const int r = tk % per_step;
    const int q = r % S;
    const int tile = r / S;                 // panel-major tile id
    const int panel = tile / ninner, inner = tile % ninner;
    const int tm = LEFT ? inner : panel, tn = LEFT ? panel : inner;
    if (threadIdx.x == 0 && k >= 2) {
      const int* cnt = panel_cnt + (k - 1) * npanels + panel;
      while (ld_acquire(cnt) < ninner) __nanosleep(64);
    }
    __syncthreads();
    // W_{k-1}: k=1 -> X; else (k-1 odd ? Wa : Wb).  W_k -> (k odd ? Wa : Wb); W_{k-2} aliases W_k (k >= 3).
    const double* src = k == 1 ? a.X : (((k - 1) & 1) ? a.Wa : a.Wb);
    const int64_t ldsrc = k == 1 ? a.ldx : a.ldw;
    const bool vsrc = k == 1 ? a.vec_x : a.vec_w;
    const int64_t m0 = (int64_t)tm * BM, n0 = (int64_t)tn * BN;
    const int kb = (int)((int64_t)nk * q / S), ke = (int)((int64_t)nk * (q + 1) / S);
    double acc[4][4][2];
    if (LEFT) mainloop<false, false>(a.G, a.s, src, ldsrc, a.M, a.N, a.s, m0, n0, a.vec_g, vsrc, smem, acc, kb, ke);
    else      mainloop<true, false>(src, ldsrc, a.G, a.s, a.M, a.N, a.s, m0, n0, vsrc, a.vec_g, smem, acc, kb, ke);
    if (S > 1) {
      // splits q < S-1 publish partial sums; split S-1 (the last ticket of the tile,
      // so it never waits on a later one) adds them in the fixed order q = 0..S-1.
      double* slot = a.partial + (int64_t)tile * (S - 1) * (BM * BN);
      if (q < S - 1) {
        double* mine = slot + (int64_t)q * (BM * BN);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) __stcg(mine + ((i * 4 + j) * 2 + e) * NTHREADS + threadIdx.x, acc[i][j][e]);
        __syncthreads();
        if (threadIdx.x == 0) red_release_add_i32(split_cnt + tile, 1);  // release, cumulative over bar.sync
        continue;
      }
      if (threadIdx.x == 0) {
        while (ld_acquire(split_cnt + tile) < (S - 1) * k) __nanosleep(32);
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // the 8 accumulators of row group i x (S-1) partials in flight, then a fixed-order sum
        double part[8][3];
#pragma unroll
        for (int q8 = 0; q8 < 8; ++q8)
#pragma unroll
          for (int p = 0; p < 3; ++p)
            part[q8][p] = p < S - 1 ? __ldcg(slot + (int64_t)p * (BM * BN) + (i * 8 + q8) * NTHREADS + threadIdx.x)
                                    : 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int q8 = j * 2 + e;
            double sum = part[q8][0];
#pragma unroll
            for (int p = 1; p < 3; ++p)
              if (p < S - 1) sum += part[q8][p];
            acc[i][j][e] = sum + acc[i][j][e];
          }
      }
    }
    double* out = (k & 1) ? a.Wa : a.Wb;
    const double* pp = k == 2 ? a.X : out;
    const int64_t ldpp = k == 2 ? a.ldx : a.ldw;
    if (k == a.K - 1) out = nullptr;
    cheb_epilogue(acc, m0, n0, a.M, a.N, k == 1, src, ldsrc, pp, ldpp, out, a.ldw, a.Y, a.ldy, a.P, k);
    __syncthreads();
    if (threadIdx.x == 0) red_release_add_i32(panel_cnt + k * npanels + panel, 1);
  }
}

// ---------------------------------------------------------------------------
// Alg. 1 literally on the s x s Gram, symmetric storage.
// Every Psi_k(B_hat) is a polynomial in the symmetric G, so it is symmetric and
// G Psi_{k-1} = Psi_{k-1} G: each step computes only the LOWER-triangle tiles
// (a >= b) -- s^3 instead of 2 s^3 flops -- and mirrors W_k into the upper
// triangle so the next step reads full column panels.  Only elements r >= c are
// computed (the diagonal tiles' upper halves are mirror images), so every W_k
// and H_hat is exactly symmetric.
//   init (k_sym_init):  W_1 = (2/L) G - I,  H = c_0/2 I + c_1 W_1
//   step k = 2..K-1:    W_k = (4/L) G W_{k-1} - 2 W_{k-1} - W_{k-2}   (W_0 = I)
//                       H += c_k W_k   (lower triangle; mirrored at k = K-1)
// Dependencies: tile (a,b) of step k reads column panel b of W_{k-1} (lower
// tiles of row b and column b: "cross" b) and overwrites W_{k-2} at (a,b) and
// (b,a), which step k-1 reads through column panels b and a.  So it waits for
// crosses a and b of step k-1.  Cross j has exactly T tiles (T tiles per dim):
// tile (a,b) increments the counters of a and of b (once when a == b).
// ---------------------------------------------------------------------------
struct SymArgs {
  int64_t s;
  const double* G;
  double* W[3];         // W_k lives in W[k % 3]; W[1] = W_1 from k_sym_init
  double* H;            // H_hat (s x s, ld s)
  const SeriesParams* P;
  int K;
  int T;                // tiles per dimension
  int split;            // k-splits per tile
  int* sync;            // [0] ticket | K * T cross counters | ntri split counters
  double* partial;      // ntri * (split - 1) * 64 * 64
  int vec;
  // panel mode (multi-GPU row panels of the lower triangle): this launch computes ONE step
  // (kstep) on the ntile tiles [tile0, tile0 + ntile) of the column-major lower-triangle order,
  // with W_{k-1} / W_{k-2} complete on entry (no dependency waits), and writes W_k (or, at the
  // last step, H) of those tiles PACKED to gout: tile t at gout + (t - tile0) * 4096, row-major
  // 64 x 64 -- the slot the all-gather exchanges.  H accumulates in place on the own tiles.
  int panel, kstep, tile0, ntile;
  double* gout;
  // m-chain mode (chain = m = 2 or 3, see chain_buf): the products of step k = 2 .. K-1 are
  //   k = 2 .. m:  Psi_k = 2 B_hat Psi_{k-1} - Psi_{k-2}                 (A = G: the one-chain step)
  //   k > m:       Psi_k = 2 Psi_m Psi_{k-m} - Psi_{|k-2m|}              (A = Psi_m = T_m(B_hat))
  // i.e. T_k = 2 T_m T_{k-m} - T_{|k-2m|}: the Psi_k of each residue k mod m form an independent
  // chain of the same K-2 products, so consecutive steps no longer depend on each other.  Buffers
  // C[4m]: [j-1] Psi_j for j = 1..m (Psi_1 from k_sym_init), then three rotation buffers per chain;
  // the terms of residue (k-2) mod m = j accumulate in H (j = 0, with the init's c_0/2 I + c_1 Psi_1)
  // or HX[j-1] (from zero), summed by the last product's epilogue.
  int chain;
  double* C[12];
  double* HX[2];
  int red_bias;         // chains: the reducing split's k-range is (100 + red_bias)% of the others'
  int k0;               // first step of the launch: 2, or 3 when Psi_2 is given (k_sym_init from G^2)
  // m chains, left side: Alg. 1 line 12 (Y = H_hat X, X: s x L) appended to the launch as units
  // (row panel r, column tile c, k-split q) after the last product's; a unit waits for cross r of
  // step K-1 (H_hat's row panel r final)
  int l12;              // 0: line 12 runs as its own launch
  double* Y;
  int64_t ldy, L;
  int l12_tn, l12_split;   // column tiles of Y, k-splits per line-12 tile
  double* l12_partial;     // tiles * (l12_split - 1) * 64 * 64
  const double* X;         // (host side: the map of line 12's B operand)
  int64_t ldx;
};

// Buffer of Psi_k in m-chain mode (k >= 1): Psi_k overwrites Psi_{k-3m} of its own chain.
__host__ __device__ __forceinline__ int chain_buf(int k, int m) {
  if (k <= m) return k - 1;
  const int r = (k - m - 1) % m, idx = (k - m - 1) / m;
  return m + 3 * r + idx % 3;
}
// sync layout of the symmetric kernels: [0] ticket | K * T cross counters | ntri split-K counters
// (m chains: m ntri, per tile and chain) | K * ntri tile-done flags | product-m tile count
__host__ __device__ __forceinline__ int sym_split_off(int K, int T) { return 1 + K * T; }
__host__ __device__ __forceinline__ int sym_tdone_off(int K, int T, int m) {
  return 1 + K * T + (m > 1 ? m : 1) * (T * (T + 1) / 2);
}
__host__ __device__ __forceinline__ int sym_pm_off(int K, int T, int m) {
  return sym_tdone_off(K, T, m) + K * (T * (T + 1) / 2);
}
// (line 12 in the launch: its split-K counters, one per Y tile, after the Psi_m count)
__host__ __device__ __forceinline__ int sym_l12_off(int K, int T, int m) { return sym_pm_off(K, T, m) + 1; }

// Psi_2 from the power iteration's squaring (m-chain mode): G2 holds c^2 G^2 (c^2 = *c2, an exact
// power of 2, k_diag_scale); Psi_2 = 2 B_hat^2 - I = 2 a^2 G^2 - 4 a G + I with a = 2/L (Alg. 1
// line 9 at k = 2 with the product G G the squaring already formed), written over G2; and
// H = c_0/2 I + c_1 Psi_1 + c_2 Psi_2.
__global__ void k_sym_init2(const double* __restrict__ G, int64_t s, double* __restrict__ W1, double* G2,
                            const double* __restrict__ c2, double* __restrict__ H, const SeriesParams* __restrict__ P) {
  const double a = P->scale2, h0 = 0.5 * P->c[0], c1 = P->c[1], cc2 = P->c[2];
  const double a2 = 2.0 * a * a / *c2, a4 = 4.0 * a;
  const int64_t n = s * s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double id = (e / s == e % s) ? 1.0 : 0.0;
    const double g = G[e];
    const double w = a * g - id;                      // Psi_1 = B_hat = (2/L) G - I
    const double p2 = a2 * G2[e] - a4 * g + id;       // Psi_2 = 2 B_hat^2 - I
    W1[e] = w;
    G2[e] = p2;
    H[e] = h0 * id + c1 * w + cc2 * p2;
  }
}
// the state of the sync array after step 2 (tile-done flags, the chain-0 split counters, the
// Psi_2 count) when Psi_2 comes from k_sym_init2
__global__ void k_sym_mark_step2(int* sync, int K, int T, int m, int split_arrivals) {
  const int ntri = T * (T + 1) / 2;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntri; t += gridDim.x * blockDim.x) {
    sync[sym_tdone_off(K, T, m) + 2 * ntri + t] = 1;
    sync[sym_split_off(K, T) + m * t] = split_arrivals;
    if (t == 0 && m == 2) sync[sym_pm_off(K, T, m)] = ntri;
  }
}

__global__ void k_sym_init(const double* __restrict__ G, int64_t s, double* __restrict__ W1, double* __restrict__ H,
                           const SeriesParams* __restrict__ P) {
  const double s2 = P->scale2, h0 = 0.5 * P->c[0], c1 = P->c[1];
  const int64_t n = s * s;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double id = (e / s == e % s) ? 1.0 : 0.0;
    const double w = s2 * G[e] - id;                  // W_1 = B_hat = (2/L) G - I   (Alg. 1 line 5-6)
    if (W1) W1[e] = w;
    H[e] = h0 * id + c1 * w;                          // H = c_0/2 Psi_0 + c_1 Psi_1 (line 7)
  }
}

__device__ __forceinline__ void tri_decode(int b, int& row, int& col) {
  int r = (int)((sqrt(8.0 * b + 1.0) - 1.0) * 0.5);
  while ((r + 1) * (r + 2) / 2 <= b) ++r;
  while (r * (r + 1) / 2 > b) --r;
  row = r;
  col = b - r * (r + 1) / 2;
}

// mainloop for the symmetric kernel: the A slabs (rows of the static G) of the
// pipeline prologue are issued BEFORE the dependency wait, the B slabs (W_{k-1},
// produced by the previous step) after it.  cp.async groups: group 0 = {A0..A2, B0},
// group j = {Bj}: wait_group semantics of the main loop are unchanged.
template <class Wait>
__device__ __forceinline__ void mainloop_dep(const double* Ag, const double* Bg, int64_t s, int64_t m0, int64_t n0,
                                             bool vec, double* smem, double (&acc)[4][4][2], int kbeg, int kend,
                                             Wait&& wait) {
  using LA = OpLayout<false, BM>;
  using LB = OpLayout<false, BN>;
  double* sA = smem;
  double* sB = smem + STAGES * LA::SIZE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nk = kend - kbeg;
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st)
    if (st < nk) load_slab<LA>(sA + st * LA::SIZE, Ag, s, (int64_t)(kbeg + st) * BKS, m0, s, s, vec);
  wait();
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nk) load_slab<LB>(sB + st * LB::SIZE, Bg, s, (int64_t)(kbeg + st) * BKS, n0, s, s, vec);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) {
        const int64_t k0 = (int64_t)(kbeg + nxt) * BKS;
        load_slab<LA>(sA + (nxt % STAGES) * LA::SIZE, Ag, s, k0, m0, s, s, vec);
        load_slab<LB>(sB + (nxt % STAGES) * LB::SIZE, Bg, s, k0, n0, s, s, vec);
      }
      cp_async_commit();
    }
    const double* cA = sA + (kt % STAGES) * LA::SIZE;
    const double* cB = sB + (kt % STAGES) * LB::SIZE;
#pragma unroll
    for (int kk = 0; kk < BKS; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = cA[LA::idx(wm + i * 8 + g, kk + t)];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = cB[LB::idx(wn + j * 8 + g, kk + t)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// Column-major lower-triangle tile index -> (row i, column j), i >= j.
// Column j holds T - j tiles; C(j) = j (2T - j + 1) / 2 tiles precede it.
__device__ __forceinline__ void tri_decode_colmajor(int idx, int T, int& row, int& col) {
  const double b = 2.0 * T + 1.0;
  int j = (int)((b - sqrt(b * b - 8.0 * idx)) * 0.5);
  auto C = [&](int jj) { return jj * (2 * T - jj + 1) / 2; };
  while (j > 0 && C(j) > idx) --j;
  while (C(j + 1) <= idx) ++j;
  col = j;
  row = j + (idx - C(j));
}

// Dataflow schedule with three W buffers (W_k overwrites W_{k-3}).  Units
// (step k, tile in column-major lower-triangle order, k-split q) are claimed by
// ticket.  Tile (i, j) of step k reads column panel j of W_{k-1} = cross j of
// step k-1 (tiles (l, j), l >= j, and (j, l), l < j) -- in column-major order
// that cross is complete as soon as column j of step k-1 is, so consecutive
// steps overlap as a wavefront instead of meeting at a barrier.  Its writes
// (i, j) and (j, i) land on W_{k-3}, read by step k-2 through column panels j
// and i (crosses j and i of step k-2; j is implied by cross j of step k-1) and
// by the step k-1 epilogue of tile (i, j) (in cross j of step k-1): so it also
// waits for cross i of step k-2.
// After the mainloop of unit (step k, tile (ti, tj), k-split q): split-K publish (q < S-1)
// or reduce (q = S-1, all partials summed in the fixed order q = 0..S-1), then the fused
// epilogue on the tile's r >= c elements and the release of its crosses.
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// WS: run by the 128 epilogue threads (warps 4-7) of k_cheb_sym_ws, thread u = threadIdx.x - 128
// playing the role of MMA thread u (same fragment positions), synchronised on named barrier 2.
template <bool tma, bool WS, bool PANEL, int NW, int CH, class Acc>
__device__ __forceinline__ void sym_finish_impl(const SymArgs& a, int k, int tile, int q, int ti, int tj, Acc&& acc) {
  const int T = a.T;
  const int S = a.split;
  int* cross = a.sync + 1;
  int* split_cnt = a.sync + sym_split_off(a.K, T);
  const int64_t s = a.s;
  constexpr bool CHAIN = CH > 1;          // m-chain instance (CH = m; one chain: CH = 0)
  constexpr bool chain = CHAIN;
  // NW = 4: warps own 32 x 32 sub-tiles (WJ = 4 column fragments); NW = 8: 32 x 16 (WJ = 2)
  constexpr int NT = 32 * NW, WJ = NW == 4 ? 4 : 2, NV = 4 * WJ * 2;
  const int u = WS ? (int)threadIdx.x - NTHREADS : (int)threadIdx.x;
  auto group_sync = [] {
    if (WS) named_bar(2, NTHREADS);
    else __syncthreads();
  };
  const int warp = u >> 5, lane = u & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = NW == 4 ? (warp >> 1) * 32 : (warp >> 2) * 32;
  const int wn = NW == 4 ? (warp & 1) * 32 : (warp & 3) * 16;
  auto buf = [&](int i) { return i == 0 ? a.W[0] : (i == 1 ? a.W[1] : a.W[2]); };
  // one chain: W_k = s4 (G W_{k-1}) - 2 W_{k-1} - W_{k-2}, over W_{k-3}
  // m chains, k > m: Psi_k = 2 (Psi_m Psi_{k-m}) - Psi_{|k-2m|}, over Psi_{k-3m}; k <= m as one chain
  constexpr int mc = CHAIN ? CH : 1;
  const bool cstep = chain && k > mc;   // a chain product (A = Psi_m)
  const double* src = chain ? a.C[chain_buf(cstep ? k - mc : k - 1, mc)] : buf((k - 1) % 3);
  const double* wpp;                    // (nullptr: the identity Psi_0, implicit)
  if (!chain) wpp = buf((k - 2) % 3);
  else if (!cstep) wpp = k == 2 ? nullptr : a.C[chain_buf(k - 2, mc)];
  else wpp = k == 2 * mc ? nullptr : a.C[chain_buf(k > 2 * mc ? k - 2 * mc : 2 * mc - k, mc)];
  double* out = chain ? a.C[chain_buf(k, mc)] : buf(k % 3);
  const int hj = chain ? (k - 2) % mc : 0;            // accumulator of this product's chain
  double* hmine = hj == 0 ? a.H : a.HX[hj - 1];
  const bool hzero = chain && hj > 0 && k == 2 + hj;  // first term of an HX accumulator
  const int64_t m0 = (int64_t)ti * BM, n0 = (int64_t)tj * BN;
  // split counters: per launch in panel mode (zeroed before it); per tile and chain with m chains
  // (consecutive products of one tile may be in flight together); kc - 1 = the product's ordinal
  // among those of its tile and chain
  const int kc = PANEL ? 2 : chain ? (k - 2 - hj) / mc + 2 : k;
  const int sidx = chain ? mc * tile + hj : tile;
  if (S > 1) {
    double* slot = a.partial + (int64_t)(sidx - (PANEL ? a.tile0 : 0)) * (S - 1) * (BM * BN);
    CPA_DCHECK(tile - (PANEL ? a.tile0 : 0) >= 0 && tile < a.T * (a.T + 1) / 2);
    if (q < S - 1) {
      double* mine = slot + (int64_t)q * (BM * BN);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) __stcg(mine + ((i * WJ + j) * 2 + e) * NT + u, acc(i, j, e));
      group_sync();
      if (u == 0) red_release_add_i32(split_cnt + sidx, 1);
      return;
    }
    if (u == 0) wait_geq(split_cnt + sidx, (S - 1) * (kc - 1));
    group_sync();
    if (!WS) {
      double sum[NV];
#pragma unroll
      for (int rr = 0; rr < NV; ++rr) sum[rr] = __ldcg(slot + rr * NT + u);
      for (int p = 1; p < S - 1; ++p) {
        double v[NV];
#pragma unroll
        for (int rr = 0; rr < NV; ++rr) v[rr] = __ldcg(slot + (int64_t)p * (BM * BN) + rr * NT + u);
#pragma unroll
        for (int rr = 0; rr < NV; ++rr) sum[rr] += v[rr];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) acc(i, j, e) = sum[(i * WJ + j) * 2 + e] + acc(i, j, e);
    } else {
      // the same sums in the same order, eight elements at a time (register budget of the 2-CTA kernel)
#pragma unroll
      for (int c8 = 0; c8 < 4; ++c8) {
        double sum[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) sum[x] = __ldcg(slot + (c8 * 8 + x) * NT + u);
        for (int p = 1; p < S - 1; ++p) {
          double v[8];
#pragma unroll
          for (int x = 0; x < 8; ++x) v[x] = __ldcg(slot + (int64_t)p * (BM * BN) + (c8 * 8 + x) * NT + u);
#pragma unroll
          for (int x = 0; x < 8; ++x) sum[x] += v[x];
        }
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const int rr = c8 * 8 + x;
          acc(rr >> 3, (rr >> 1) & 3, rr & 1) = sum[x] + acc(rr >> 3, (rr >> 1) & 3, rr & 1);   // (NW = 4 only)
        }
      }
    }
  }
  // fused epilogue on the elements r >= c of the tile
  const double s4 = 2.0 * a.P->scale2, ck = a.P->c[k];
  const bool last = k == a.K - 1;
  if (CHAIN && chain) {
    // chain product (k > m): Psi_k = 2 (Psi_m Psi_{k-m}) - Psi_{|k-2m|} (Psi_0 = I); a G step
    // (k <= m): the one-chain update.  H_j += c_k Psi_k for the product's chain j (HX from zero at
    // its first term); the last product adds the other chains' sums (their last tiles are complete:
    // dependencies of this unit) and writes H mirrored.  Psi_k is stored only while a later
    // product reads it (k + m <= K - 1).
    const bool store_w = k + mc <= a.K - 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t rr = m0 + wm + i * 8 + g;
      double vp[2 * WJ], vpp[2 * WJ], vy[2 * WJ];
#pragma unroll
      for (int j = 0; j < WJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = n0 + wn + j * 8 + 2 * t + e;
          const bool ok = rr < s && c <= rr;
          const int64_t o = rr * s + c;
          vp[j * 2 + e] = (!cstep && ok) ? __ldcg(src + o) : 0.0;
          vpp[j * 2 + e] = wpp == nullptr ? (rr == c ? 1.0 : 0.0) : (ok ? __ldcg(wpp + o) : 0.0);
          double y0 = (hzero || !ok) ? 0.0 : __ldcg(hmine + o);
          if (last && ok)
            for (int jj = 0; jj < mc; ++jj)
              if (jj != hj) y0 += __ldcg((jj == 0 ? a.H : a.HX[jj - 1]) + o);
          vy[j * 2 + e] = y0;
        }
#pragma unroll
      for (int j = 0; j < WJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = n0 + wn + j * 8 + 2 * t + e;
          if (!(rr < s && c <= rr)) continue;
          const int qq = j * 2 + e;
          const double wv = cstep ? 2.0 * acc(i, j, e) - vpp[qq] : s4 * acc(i, j, e) - 2.0 * vp[qq] - vpp[qq];
          const double y = vy[qq] + ck * wv;
          if (store_w) {
            out[rr * s + c] = wv;
            out[c * s + rr] = wv;
          }
          if (last) {
            a.H[rr * s + c] = y;
            a.H[c * s + rr] = y;
          } else {
            hmine[rr * s + c] = y;
          }
        }
    }
  } else {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t rr = m0 + wm + i * 8 + g;
    double vp[2 * WJ], vpp[2 * WJ], vy[2 * WJ];
#pragma unroll
    for (int j = 0; j < WJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + wn + j * 8 + 2 * t + e;
        const bool ok = rr < s && c <= rr;
        const int64_t o = rr * s + c;
        vp[j * 2 + e] = ok ? __ldcg(src + o) : 0.0;
        vpp[j * 2 + e] = k == 2 ? (rr == c ? 1.0 : 0.0) : (ok ? __ldcg(wpp + o) : 0.0);
        vy[j * 2 + e] = ok ? __ldcg(a.H + o) : 0.0;
      }
#pragma unroll
    for (int j = 0; j < WJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + wn + j * 8 + 2 * t + e;
        if (!(rr < s && c <= rr)) continue;
        const int qq = j * 2 + e;
        const double wv = s4 * acc(i, j, e) - 2.0 * vp[qq] - vpp[qq];  // W_k = 2 B_hat W_{k-1} - W_{k-2}
        const double y = vy[qq] + ck * wv;                               // H += c_k W_k
        if (PANEL) {   // packed slot of the all-gather: W_k, or H at the last step
          CPA_DCHECK(tile >= a.tile0 && tile < a.tile0 + a.ntile);
          a.gout[(int64_t)(tile - a.tile0) * (BM * BN) + (rr - m0) * BN + (c - n0)] = last ? y : wv;
          if (!last) a.H[rr * s + c] = y;
          continue;
        }
        if (!last) {
          out[rr * s + c] = wv;
          out[c * s + rr] = wv;
        }
        a.H[rr * s + c] = y;
        if (last) a.H[c * s + rr] = y;
      }
  }
  }
  if (PANEL) {   // (the launch boundary orders the stores; no crosses to release)
    group_sync();
    return;
  }
  if (tma) fence_proxy_async_global();   // W_k / H stores -> later TMA (async-proxy) reads
  group_sync();
  if (u == 0) {
    red_release_add_i32(cross + k * T + ti, 1);
    if (ti != tj) red_release_add_i32(cross + k * T + tj, 1);
    red_release_add_i32(a.sync + sym_tdone_off(a.K, T, mc) + k * (T * (T + 1) / 2) + tile, 1);   // tile done
    if (CHAIN && chain && k == mc) red_release_add_i32(a.sync + sym_pm_off(a.K, T, mc), 1);   // Psi_m progress
  }
}

// k_cheb_sym / k_cheb_sym_tma: the accumulators in registers
template <bool tma, bool PANEL, int NW = 4, int CH = 0>
__device__ __forceinline__ void sym_finish(const SymArgs& a, int k, int tile, int q, int ti, int tj,
                                           double (&acc)[4][NW == 4 ? 4 : 2][2]) {
  sym_finish_impl<tma, false, PANEL, NW, CH>(a, k, tile, q, ti, tj,
                                         [&](int i, int j, int e) -> double& { return acc[i][j][e]; });
}

template <bool PANEL>
__global__ void __launch_bounds__(NTHREADS, CPA_FLOW_MINB) k_cheb_sym(SymArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_ticket;
  const int T = a.T;
  const int ntri = T * (T + 1) / 2;
  const int S = a.split;
  const int per_step = (PANEL ? a.ntile : ntri) * S;
  const int total = PANEL ? per_step : (a.K - 2) * per_step;
  int* cross = a.sync + 1;
  const int64_t s = a.s;
  const int nk = (int)((s + BKS - 1) / BKS);
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.sync, 1);
    __syncthreads();
    const int tk = s_ticket;
    if (tk >= total) break;
    const int k = PANEL ? a.kstep : 2 + tk / per_step;
    const int r = tk % per_step;
    const int q = r % S;
    const int tile = r / S + (PANEL ? a.tile0 : 0);
    int ti, tj;
    tri_decode_colmajor(tile, T, ti, tj);
    CPA_DCHECK(ti >= 0 && ti < T && tj >= 0 && tj <= ti);
    auto buf = [&](int i) { return i == 0 ? a.W[0] : (i == 1 ? a.W[1] : a.W[2]); };
    const double* src = buf((k - 1) % 3);   // W_{k-1}
    const int64_t m0 = (int64_t)ti * BM, n0 = (int64_t)tj * BN;
    const int kb = (int)((int64_t)nk * q / S), ke = (int)((int64_t)nk * (q + 1) / S);
    double acc[4][4][2];
    mainloop_dep(a.G, src, s, m0, n0, a.vec, smem, acc, kb, ke, [&] {
#ifndef CPA_SYM_NOWAIT  // (timing experiment only: wrong results without the waits)
      if (threadIdx.x == 0 && !PANEL) {
        if (k >= 3) wait_geq(cross + (k - 1) * T + tj, T);
        if (k >= 4) wait_geq(cross + (k - 2) * T + ti, T);
      }
#endif
      __syncthreads();
    });
    sym_finish<false, PANEL>(a, k, tile, q, ti, tj, acc);
  }
}

// TMA-fed variant of k_cheb_sym (same units, dependencies and epilogue).  The k-slabs of
// G and W_{k-1} arrive by cp.async.bulk.tensor (16-column x 16-row boxes, 128-byte swizzle)
// into a 4-stage ring guarded by mbarriers: thread 0 is the producer (it refills the stage
// of slab kt-1 at the top of slab kt, after the empty barrier says all four warps are done
// with it); the warps wait only on the full barrier of the slab they consume -- no CTA
// barrier per slab and no per-thread copy instructions.  Fragment loads: DMMA step kk
// consumes the k rows {8(kk/2) + 2t + kk%2 : t = 0..3} (a fixed permutation of the slab's
// 16 rows, the same for A and B), so the four rows a half-warp reads carry the XOR
// patterns {0,2,4,6} or {1,3,5,7} of the swizzle and hit 32 distinct banks.
#ifndef CPA_TMA_STAGES
#define CPA_TMA_STAGES 4
#endif
constexpr int TBK = 16, TSTAGES = CPA_TMA_STAGES;
constexpr int BOX_BYTES = 16 * TBK * 8;          // 16 doubles x TBK rows
constexpr int TSTAGE_BYTES = 8 * BOX_BYTES;      // A: 4 boxes (64 m), B: 4 boxes (64 n)

struct SymMaps {
  CUtensorMap g;
  CUtensorMap w[3];
};
struct SymMapsChain {   // m-chain mode: plus the maps of SymArgs::C (and line 12's H_hat, X)
  CUtensorMap g;
  CUtensorMap w[3];
  CUtensorMap c[12];
  CUtensorMap h, x;
};
template <int CH>
using SymMapsT = typename std::conditional<(CH > 1), SymMapsChain, SymMaps>::type;
// SBK-deep slabs in an SSTAGES ring: <16, 4> (64 KB) for short units (c2: ~11 slabs each),
// <32, 2> (64 KB, half the mbarrier round trips) for long ones (s >= 4096: c5 shape 608 ->
// 586 ms; at c2 it costs 1.27 -> 1.39 ms).
// NW = 8 (CPA_SVT_SYM_NW=8): eight warps of 32 x 16 sub-tiles per 64 x 64 tile -- half the
// accumulator registers per thread, so three 256-thread CTAs (24 warps, six per SMSP) fit an SM
// where the 4-warp kernel keeps twelve; the same per-element DMMA order (bitwise-equal results).
#ifdef CPA_SYM_TRACE
// Trace build (build.py --variant trace CPA_SYM_TRACE=1): per unit (ticket) the globaltimer at the
// claim, after the claim broadcast, after the dependency wait, at the mainloop end and at the
// epilogue end, and the SM / CTA; read with cpa_svt_debug_sym_trace (tools/sym_trace.py).
constexpr int kTraceUnits = 1 << 16;
__device__ uint64_t g_trace[kTraceUnits * 6];
__device__ __forceinline__ uint64_t trace_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t smid_now() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
#endif

// Line 12 unit's epilogue (m-chain launch): split-K publish / fixed-order reduce (the reducer q =
// S-1 waits for the others), then Y = the tile's sum (row r0.., column c0.. of the caller's Y).
__device__ __forceinline__ void l12_finish(const SymArgs& a, int t12, int q, int64_t r0, int64_t c0,
                                           double (&acc)[4][4][2]) {
  constexpr int NT = NTHREADS, NV = 32;
  const int u = threadIdx.x;
  const int warp = u >> 5, lane = u & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int S = a.l12_split;
  if (S > 1) {
    double* slot = a.l12_partial + (int64_t)t12 * (S - 1) * (BM * BN);
    int* cnt = a.sync + sym_l12_off(a.K, a.T, a.chain) + t12;
    if (q < S - 1) {
      double* mine = slot + (int64_t)q * (BM * BN);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) __stcg(mine + ((i * 4 + j) * 2 + e) * NT + u, acc[i][j][e]);
      __syncthreads();
      if (u == 0) red_release_add_i32(cnt, 1);
      return;
    }
    if (u == 0) wait_geq(cnt, S - 1);
    __syncthreads();
#pragma unroll
    for (int c8 = 0; c8 < NV / 8; ++c8) {
      double sum[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) sum[x] = __ldcg(slot + (c8 * 8 + x) * NT + u);
      for (int p = 1; p < S - 1; ++p) {
        double v[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) v[x] = __ldcg(slot + (int64_t)p * (BM * BN) + (c8 * 8 + x) * NT + u);
#pragma unroll
        for (int x = 0; x < 8; ++x) sum[x] += v[x];
      }
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const int rr = c8 * 8 + x;
        acc[rr >> 3][(rr >> 1) & 3][rr & 1] = sum[x] + acc[rr >> 3][(rr >> 1) & 3][rr & 1];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t rr = r0 + wm + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = c0 + wn + j * 8 + 2 * t + e;
        if (rr < a.s && c < a.L) a.Y[rr * a.ldy + c] = acc[i][j][e];
      }
  }
}

template <int SBK, int SSTAGES, bool PANEL, int NW = 4, int CH = 0>
__global__ void __launch_bounds__(32 * NW, CPA_FLOW_MINB)
    k_cheb_sym_tma(const __grid_constant__ SymMapsT<CH> mp, SymArgs a) {
  constexpr bool CHAIN = CH > 1;
  constexpr int SBOX_BYTES = 16 * SBK * 8;
  constexpr int SSTAGE_BYTES = 8 * SBOX_BYTES;
  extern __shared__ unsigned char tsm_raw[];
  __shared__ __align__(8) uint64_t full[SSTAGES], empty[SSTAGES];
  __shared__ int s_ticket;
  // 1024-byte aligned ring (the 128-byte swizzle pattern repeats every 1024 bytes); pointer
  // arithmetic on the __shared__ array keeps the fragment loads in the shared window (LDS)
  unsigned char* base = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
  const int T = a.T;
  const int ntri = T * (T + 1) / 2;
  const int S = a.split;
  const int per_step = (PANEL ? a.ntile : ntri) * S;
  const int rec_total = PANEL ? per_step : (a.K - (CH > 1 ? a.k0 : 2)) * per_step;
  // (m chains: line 12's units after the recurrence's)
  const int total = rec_total + ((CH > 1 && a.l12) ? T * a.l12_tn * a.l12_split : 0);
  int* cross = a.sync + 1;
  const int nk = (int)((a.s + SBK - 1) / SBK);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  constexpr int WJ = NW == 4 ? 4 : 2;
  const int wm = NW == 4 ? (warp >> 1) * 32 : (warp >> 2) * 32;
  const int wn = NW == 4 ? (warp & 1) * 32 : (warp & 3) * 16;
  if (threadIdx.x == 0) {
    for (int st = 0; st < SSTAGES; ++st) {
      mbar_init(full + st, 1);
      mbar_init(empty + st, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // byte offset of element (row r, column c) of a box: r*128 + (((c/2) ^ (r%8)) * 16) + (c%2)*8
  uint32_t coff[2][2];
#pragma unroll
  for (int par = 0; par < 2; ++par)
#pragma unroll
    for (int h = 0; h < 2; ++h) coff[par][h] = ((((h * 8 + g) >> 1) ^ (2 * t + par)) << 4) | ((g & 1) * 8);
  const uint32_t roff = 256 * t;
  const uint32_t boxa = (wm >> 4) * SBOX_BYTES, boxb = (4 + (wn >> 4)) * SBOX_BYTES;
  uint32_t it = 0;  // slabs consumed by this CTA so far (stage = it % SSTAGES, phase = it / SSTAGES)
  for (;;) {
#ifdef CPA_SYM_TRACE
    uint64_t t_claim0 = 0;
    if (threadIdx.x == 0) t_claim0 = trace_now();
#endif
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.sync, 1);
    __syncthreads();
    const int tk = s_ticket;
#ifdef CPA_SYM_TRACE
    if (threadIdx.x == 0 && tk < total && tk < kTraceUnits) {
      g_trace[tk * 6 + 0] = t_claim0;
      g_trace[tk * 6 + 1] = trace_now();
      g_trace[tk * 6 + 5] = smid_now() | ((uint64_t)blockIdx.x << 16);
    }
#endif
    if (tk >= total) break;
    const bool is12 = CHAIN && tk >= rec_total;   // a line-12 unit (Y tile (ti, tj), k-split q)
    int k, q, tile, ti, tj;
    if (is12) {
      const int u12 = tk - rec_total;
      q = u12 % a.l12_split;
      tile = u12 / a.l12_split;
      ti = tile / a.l12_tn;
      tj = tile % a.l12_tn;
      k = a.K;
    } else {
      k = PANEL ? a.kstep : (CH > 1 ? a.k0 : 2) + tk / per_step;
      const int r = tk % per_step;
      q = r % S;
      tile = r / S + (PANEL ? a.tile0 : 0);
      tri_decode_colmajor(tile, T, ti, tj);
      CPA_DCHECK(ti >= 0 && ti < T && tj >= 0 && tj <= ti);
    }
    // B operand: W_{k-1} (one chain; a G step of the m-chain mode: Psi_{k-1}) / Psi_{k-m} (a chain
    // product, k > m) / X (line 12); A operand: the static G, Psi_m for the chain products, or H_hat
    constexpr int mc = CHAIN ? CH : 1;
    const bool cstep = CHAIN && k > mc && !is12;
    const CUtensorMap* wmap;
    const CUtensorMap* amap;
    if constexpr (CHAIN) {
      wmap = is12 ? &mp.x : &mp.c[chain_buf(cstep ? k - mc : k - 1, mc)];
      amap = is12 ? &mp.h : cstep ? &mp.c[mc - 1] : &mp.g;
    } else {
      wmap = &mp.w[(k - 1) % 3];
      amap = &mp.g;
    }
    const int m0 = ti * BM, n0 = tj * BN;
    int kb = (int)((int64_t)nk * q / S), ke = (int)((int64_t)nk * (q + 1) / S);
    if (CHAIN) {   // the reducer (q = S - 1) starts last and sums the others: a longer k-range
      const int SS = is12 ? a.l12_split : S;
      const int64_t wt = 100 * SS + (is12 ? 0 : a.red_bias);
      kb = (int)((int64_t)nk * q * 100 / wt);
      ke = q == SS - 1 ? nk : (int)((int64_t)nk * (q + 1) * 100 / wt);
    }
    const int nku = ke - kb;
    if (warp == 0) {
      // prologue: lane 0 issues the A slabs when they are static (G; Psi_m once complete) while the
      // lanes poll the unit's dependency flags in parallel (each satisfied wait costs one L2 round
      // trip, not one per flag); after the warp barrier lane 0 issues the B slabs (and late A slabs)
      const int P = nku < SSTAGES - 1 ? nku : SSTAGES - 1;
      bool a_early = !is12;   // (line 12: H_hat's rows are final only after the dependency)
      if (cstep) {
        const int v = lane == 0 ? ld_acquire(a.sync + sym_pm_off(a.K, T, mc)) : 0;
        a_early = __shfl_sync(0xffffffffu, v, 0) >= ntri;
      }
      auto issue_a = [&] {
        for (int p = 0; p < P; ++p) {
          const uint32_t sl = it + p, st = sl % SSTAGES;
          mbar_wait(empty + st, ((sl / SSTAGES) & 1) ^ 1);
          mbar_expect_tx(full + st, SSTAGE_BYTES);
          for (int b = 0; b < 4; ++b)
            tma_load_2d(base + st * SSTAGE_BYTES + b * SBOX_BYTES, amap, m0 + 16 * b, (kb + p) * SBK, full + st);
        }
      };
      if (lane == 0 && a_early) issue_a();
#ifdef CPA_EXP_NODEP
      if (false) {
#else
      if (!PANEL) {
#endif
        // Fine-grained dependencies: this split reads rows [kb SBK, ke SBK) of column panel tj of
        // its B operand, i.e. only the tiles (l, tj) / (tj, l) of the tile rows l it covers (not the
        // whole cross tj), plus the unit's own tile of the previous step of its chain (the
        // epilogue's W / H reads).  The in-place write over W_{k-3} (m chains: Psi_{k-3m}) at
        // (ti, tj) and (tj, ti) still waits for crosses ti and tj of step k-2 (k-2m): every reader
        // of those panels.  m chains add, for the chain products k <= 2m: the own tile of step m
        // (it implies the G steps' own tiles: the epilogue's Psi_{2m-k}) and, unless Psi_m is
        // complete, the A rows of Psi_m (tiles (ti, l) of step m) -- both implied for k > 2m by the
        // own tile of step k-m; for the last product, the own tiles of steps K-2 .. K-m (the other
        // chains' H).  Flags are polled lane-strided, any count.
        const int* tdone = a.sync + sym_tdone_off(a.K, T, mc);
        const int l0 = (kb * SBK) / BM, l1e = (ke * SBK - 1) / BM, l1 = l1e < T - 1 ? l1e : T - 1;
        const int nl = l1 - l0 + 1;
        auto tri_idx = [&](int r, int c) { return c * (2 * T - c + 1) / 2 + (r - c); };   // r >= c
        const int kprev = cstep ? k - mc : k - 1;   // the step whose tiles are B (and own tile)
        const int khaz = cstep ? (k >= 4 * mc + 1 ? k - 2 * mc : 0) : 0;
        const bool need_b = kprev >= 2;
        const bool need_m = cstep && k <= 2 * mc;
        const bool need_a = need_m && !a_early;
        const bool need_h = CHAIN && k == a.K - 1;
        // flag list: [0, 1] crosses ti, tj of khaz | [2] own tile of kprev | [3] own tile of step m |
        // [4, 5] own tiles of steps K-2, K-3 (last product) | B tiles l0..l1 | A tiles l0..l1
        if (is12) {
          if (lane == 0) wait_geq(cross + (a.K - 1) * T + ti, T);   // H_hat's row panel ti is final
        } else if (!CHAIN) {
          // one chain (the round-1/2 lane layout, kept instruction for instruction: this kernel's
          // claim-to-start path is measurably sensitive to code changes): lanes 0, 1 crosses ti, tj
          // of step k-2, lane 2 the own tile of step k-1, lanes 3.. the B tiles (29 per pass)
          const int* flag = nullptr;
          int target = 0;
          if (lane == 0 && k >= 4) { flag = cross + (k - 2) * T + ti; target = T; }
          if (lane == 1 && k >= 4) { flag = cross + (k - 2) * T + tj; target = T; }
          if (lane == 2 && k >= 3) { flag = tdone + (k - 1) * ntri + tile; target = 1; }
          if (lane >= 3 && k >= 3 && l0 + lane - 3 <= l1) {
            const int l = l0 + lane - 3;
            flag = tdone + (k - 1) * ntri + (l >= tj ? tri_idx(l, tj) : tri_idx(tj, l));
            target = 1;
            if (l1 - l0 > 28) {   // (more B tile rows than lanes: the whole cross tj instead)
              flag = cross + (k - 1) * T + tj;
              target = T;
            }
          }
          if (flag) wait_geq(flag, target);
        } else {
          const int nflags = 6 + nl + (need_a ? nl : 0);
          for (int f = lane; f < nflags; f += 32) {
            const int* flag = nullptr;
            int target = 1;
            if (f < 2) {
              if (khaz) { flag = cross + khaz * T + (f == 0 ? ti : tj); target = T; }
            } else if (f == 2) {
              if (need_b) flag = tdone + kprev * ntri + tile;
            } else if (f == 3) {
              if (need_m) flag = tdone + mc * ntri + tile;
            } else if (f < 6) {
              if (need_h && f - 3 < mc) flag = tdone + (a.K - 1 - (f - 3)) * ntri + tile;
            } else if (f < 6 + nl) {
              const int l = l0 + f - 6;
              if (need_b) flag = tdone + kprev * ntri + (l >= tj ? tri_idx(l, tj) : tri_idx(tj, l));
            } else {
              const int l = l0 + f - 6 - nl;
              flag = tdone + mc * ntri + (l >= ti ? tri_idx(l, ti) : tri_idx(ti, l));
            }
            if (flag) wait_geq(flag, target);
          }
        }
        __syncwarp();
      }
#ifdef CPA_SYM_TRACE
      if (lane == 0 && tk < kTraceUnits) g_trace[tk * 6 + 2] = trace_now();
#endif
      if (lane == 0) {
        fence_proxy_async_global();   // generic-proxy W stores of other CTAs -> TMA reads
        if (!a_early) issue_a();
        for (int p = 0; p < P; ++p) {
          const uint32_t st = (it + p) % SSTAGES;
          for (int b = 0; b < 4; ++b)
            tma_load_2d(base + st * SSTAGE_BYTES + (4 + b) * SBOX_BYTES, wmap, n0 + 16 * b, (kb + p) * SBK,
                        full + st);
        }
      }
    }
    // The epilogue's generic loads of W_{k-1}, W_{k-2} and H must be ordered after thread 0's
    // acquire of the dependency: every warp waits on the full barrier of a refilled slab, whose
    // expect_tx arrive thread 0 made after that acquire (release -> acquire at CTA scope); a
    // unit too short to refill (nku < SSTAGES) takes a CTA barrier instead.
    if (nku < SSTAGES) __syncthreads();
    else __syncwarp();
    double acc[4][WJ][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < WJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < nku; ++kt) {
      if (threadIdx.x == 0 && kt + SSTAGES - 1 < nku) {   // refill the stage of slab kt-1
        const int kn = kt + SSTAGES - 1;
        const uint32_t sl = it + kn, st = sl % SSTAGES;
        mbar_wait(empty + st, ((sl / SSTAGES) & 1) ^ 1);
        mbar_expect_tx(full + st, SSTAGE_BYTES);
        unsigned char* d = base + st * SSTAGE_BYTES;
        for (int b = 0; b < 4; ++b) tma_load_2d(d + b * SBOX_BYTES, amap, m0 + 16 * b, (kb + kn) * SBK, full + st);
        for (int b = 0; b < 4; ++b)
          tma_load_2d(d + (4 + b) * SBOX_BYTES, wmap, n0 + 16 * b, (kb + kn) * SBK, full + st);
      }
      __syncwarp();
      const uint32_t sl = it + kt, st = sl % SSTAGES;
      mbar_wait(full + st, (sl / SSTAGES) & 1);
      const unsigned char* sa = base + st * SSTAGE_BYTES + boxa;
      const unsigned char* sb = base + st * SSTAGE_BYTES + boxb;
#pragma unroll
      for (int kk = 0; kk < SBK / 4; ++kk) {
        const int par = kk & 1;
        const uint32_t ro = 1024 * (kk >> 1) + 128 * par + roff;
        double fa[4], fb[WJ];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          fa[i] = *reinterpret_cast<const double*>(sa + (i >> 1) * SBOX_BYTES + ro + coff[par][i & 1]);
#pragma unroll
        for (int j = 0; j < WJ; ++j)
          fb[j] = *reinterpret_cast<const double*>(sb + (j >> 1) * SBOX_BYTES + ro + coff[par][j & 1]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < WJ; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
      }
      // the stage is rewritten by the async proxy (TMA) once all four warps have arrived:
      // order this warp's generic-proxy fragment loads before that (without the fence ptxas
      // may issue the arrive before the loads have completed -- a measured data race)
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
    }
    it += nku;
#ifdef CPA_SYM_TRACE
    if (threadIdx.x == 0 && tk < kTraceUnits) g_trace[tk * 6 + 3] = trace_now();
#endif
#ifdef CPA_EXP_NOEPI
    if (CH > 1) {   // (timing experiment: no reduction / epilogue; one store keeps the mainloop live)
      double sacc = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < WJ; ++j) sacc += acc[i][j][0] + acc[i][j][1];
      if (sacc == 1.2345e-300) a.H[threadIdx.x] = sacc;
      __syncthreads();
      continue;
    }
#endif
    if constexpr (CH > 1 && NW == 4) {
      if (is12) {
        l12_finish(a, tile, q, (int64_t)m0, (int64_t)n0, acc);
        continue;
      }
    }
    sym_finish<true, PANEL, NW, CH>(a, k, tile, q, ti, tj, acc);
#ifdef CPA_SYM_TRACE
    if (threadIdx.x == 0 && tk < kTraceUnits) g_trace[tk * 6 + 4] = trace_now();
#endif
  }
}

// Warp-specialized variant of k_cheb_sym_tma (CPA_SVT_SYM_WS): the same units,
// dependencies, ring and fragment loads, but the four MMA warps (warp 0 lane 0: tickets + TMA) hand
// each unit's accumulators to four EPILOGUE warps through a double-buffered 32 KB shared-memory
// staging area (fragment layout, the layout of the split-K slots) and go straight on to the next
// unit; the epilogue warps run the split-K publish / fixed-order reduction and the fused update
// (sym_finish<.., WS>) concurrently.  So the DMMA pipe does not idle through the reducer's L2 round
// trips and the epilogue.  mbarriers: sfull[b] (4 MMA-warp arrivals: unit in staging b),
// sempty[b] (4 epilogue-warp arrivals: staging b read); meta[b] carries the unit; k < 0 ends.
struct WsMeta {
  int k, tile, q, ti, tj;
};

template <int SBK, int SSTAGES>
__global__ void __launch_bounds__(2 * NTHREADS, 2)
    k_cheb_sym_ws(const __grid_constant__ SymMaps mp, SymArgs a) {
  constexpr int SBOX_BYTES = 16 * SBK * 8;
  constexpr int SSTAGE_BYTES = 8 * SBOX_BYTES;
  // all shared state in the dynamic allocation (no static shared memory: two CTAs fill the SM's
  // 228 KB exactly): mbarriers / ticket / unit records in the first 128 bytes, then the 1024-byte
  // aligned ring (128-byte swizzle) and the two staging buffers
  extern __shared__ __align__(16) unsigned char tsm_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm_raw);
  uint64_t* empty = full + SSTAGES;
  uint64_t* sfull = empty + SSTAGES;
  uint64_t* sempty = sfull + 2;
  int& s_ticket = *reinterpret_cast<int*>(sempty + 2);
  WsMeta* meta = reinterpret_cast<WsMeta*>(sempty + 4);
  const uint32_t raw = smem_u32(tsm_raw);
  unsigned char* base = tsm_raw + (((raw + 128u + 1023u) & ~1023u) - raw);
  double* stage = reinterpret_cast<double*>(base + SSTAGES * SSTAGE_BYTES);   // 2 x 64 x 64 doubles
  {
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;\n" : "=r"(dyn));
    if ((uint32_t)(base - tsm_raw) + SSTAGES * SSTAGE_BYTES + 2 * BM * BN * 8 > dyn) __trap();   // layout check
  }
  const int T = a.T;
  const int ntri = T * (T + 1) / 2;
  const int S = a.split;
  const int per_step = (false ? a.ntile : ntri) * S;
  const int total = false ? per_step : (a.K - 2) * per_step;
  int* cross = a.sync + 1;
  const int nk = (int)((a.s + SBK - 1) / SBK);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < SSTAGES; ++st) {
      mbar_init(full + st, 1);
      mbar_init(empty + st, 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(sfull + b, 4);
      mbar_init(sempty + b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp >= 4) {
    // ---------------- epilogue warps ----------------
    const int u = threadIdx.x - NTHREADS;
    for (int n = 0;; ++n) {
      const int b = n & 1;
      mbar_wait(sfull + b, (n >> 1) & 1);
      const WsMeta mt = meta[b];
      if (mt.k < 0) break;
      // the accumulators stay in the staging buffer (read where used: the register budget of the
      // 2-CTA kernel); the buffer is released after the unit
      double* stg = stage + b * (BM * BN);
      sym_finish_impl<true, true, false, 4, 0>(a, mt.k, mt.tile, mt.q, mt.ti, mt.tj, [&](int i, int j, int e) -> double& {
        return stg[((i * 4 + j) * 2 + e) * NTHREADS + u];
      });
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty + b);   // staging b may be refilled
    }
    return;
  }
  // ---------------- MMA warps (thread 0: tickets and TMA producer) ----------------
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  uint32_t coff[2][2];
#pragma unroll
  for (int par = 0; par < 2; ++par)
#pragma unroll
    for (int h = 0; h < 2; ++h) coff[par][h] = ((((h * 8 + g) >> 1) ^ (2 * t + par)) << 4) | ((g & 1) * 8);
  const uint32_t roff = 256 * t;
  const uint32_t boxa = (wm >> 4) * SBOX_BYTES, boxb = (4 + (wn >> 4)) * SBOX_BYTES;
  uint32_t it = 0;    // slabs consumed by this CTA so far
  int nunit = 0;      // units handed to the epilogue so far
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.sync, 1);
    named_bar(1, NTHREADS);
    const int tk = s_ticket;
    named_bar(1, NTHREADS);   // (s_ticket is rewritten by the next claim)
    const int b = nunit & 1;
    if (tk >= total) {
      mbar_wait(sempty + b, ((nunit >> 1) & 1) ^ 1);
      if (threadIdx.x == 0) meta[b].k = -1;
      __syncwarp();
      if (lane == 0) mbar_arrive(sfull + b);
      break;
    }
    const int k = false ? a.kstep : 2 + tk / per_step;
    const int r = tk % per_step;
    const int q = r % S;
    const int tile = r / S + (false ? a.tile0 : 0);
    int ti, tj;
    tri_decode_colmajor(tile, T, ti, tj);
    CPA_DCHECK(ti >= 0 && ti < T && tj >= 0 && tj <= ti);
    const CUtensorMap* wmap = &mp.w[(k - 1) % 3];   // W_{k-1}
    const int m0 = ti * BM, n0 = tj * BN;
    const int kb = (int)((int64_t)nk * q / S), ke = (int)((int64_t)nk * (q + 1) / S);
    const int nku = ke - kb;
    if (threadIdx.x == 0) {
      const int P = nku < SSTAGES - 1 ? nku : SSTAGES - 1;
      for (int p = 0; p < P; ++p) {
        const uint32_t sl = it + p, st = sl % SSTAGES;
        mbar_wait(empty + st, ((sl / SSTAGES) & 1) ^ 1);
        mbar_expect_tx(full + st, SSTAGE_BYTES);
        for (int bb = 0; bb < 4; ++bb)
          tma_load_2d(base + st * SSTAGE_BYTES + bb * SBOX_BYTES, &mp.g, m0 + 16 * bb, (kb + p) * SBK, full + st);
      }
      if (!false) {
        if (k >= 3) wait_geq(cross + (k - 1) * T + tj, T);
        if (k >= 4) wait_geq(cross + (k - 2) * T + ti, T);
      }
      fence_proxy_async_global();
      for (int p = 0; p < P; ++p) {
        const uint32_t st = (it + p) % SSTAGES;
        for (int bb = 0; bb < 4; ++bb)
          tma_load_2d(base + st * SSTAGE_BYTES + (4 + bb) * SBOX_BYTES, wmap, n0 + 16 * bb, (kb + p) * SBK,
                      full + st);
      }
    }
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < nku; ++kt) {
      if (threadIdx.x == 0 && kt + SSTAGES - 1 < nku) {
        const int kn = kt + SSTAGES - 1;
        const uint32_t sl = it + kn, st = sl % SSTAGES;
        mbar_wait(empty + st, ((sl / SSTAGES) & 1) ^ 1);
        mbar_expect_tx(full + st, SSTAGE_BYTES);
        unsigned char* d = base + st * SSTAGE_BYTES;
        for (int bb = 0; bb < 4; ++bb) tma_load_2d(d + bb * SBOX_BYTES, &mp.g, m0 + 16 * bb, (kb + kn) * SBK, full + st);
        for (int bb = 0; bb < 4; ++bb)
          tma_load_2d(d + (4 + bb) * SBOX_BYTES, wmap, n0 + 16 * bb, (kb + kn) * SBK, full + st);
      }
      __syncwarp();
      const uint32_t sl = it + kt, st = sl % SSTAGES;
      mbar_wait(full + st, (sl / SSTAGES) & 1);
      const unsigned char* sa = base + st * SSTAGE_BYTES + boxa;
      const unsigned char* sb = base + st * SSTAGE_BYTES + boxb;
#pragma unroll
      for (int kk = 0; kk < SBK / 4; ++kk) {
        const int par = kk & 1;
        const uint32_t ro = 1024 * (kk >> 1) + 128 * par + roff;
        double fa[4], fb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          fa[i] = *reinterpret_cast<const double*>(sa + (i >> 1) * SBOX_BYTES + ro + coff[par][i & 1]);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          fb[j] = *reinterpret_cast<const double*>(sb + (j >> 1) * SBOX_BYTES + ro + coff[par][j & 1]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
    }
    it += nku;
    // hand the accumulators to the epilogue warps
    mbar_wait(sempty + b, ((nunit >> 1) & 1) ^ 1);
    double* stg = stage + b * (BM * BN);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) stg[((i * 4 + j) * 2 + e) * NTHREADS + threadIdx.x] = acc[i][j][e];
    if (threadIdx.x == 0) meta[b] = WsMeta{k, tile, q, ti, tj};
    __syncwarp();
    if (lane == 0) mbar_arrive(sfull + b);
    ++nunit;
  }
}

// Ping-pong m-chain recurrence (k_cheb_sym_pp, opt-in CPA_SVT_SYM_PP=1, measured slower): ONE
// persistent 384-thread CTA per SM with two MMA warp groups and one epilogue warp group.  Each MMA
// group (warps 0-3 / 4-7) claims its own units, polls their dependencies, runs its own 4-stage TMA
// ring and DMMA mainloop, and hands the accumulators to the epilogue group (warps 8-11) through its
// own 32 KB staging buffer; so while one MMA group claims / waits / refills its ring, the other
// keeps the DMMA pipe fed (two MMA warps per SMSP sustain 36.8 of the 37.2 TF/s: tools/peaks/
// dmma_smem_loop), and no MMA warp runs an epilogue.  Split-K by LAST ARRIVAL: every split
// publishes its partial, the last one to count itself in (acq_rel atomic, ordinal per tile and
// chain) sums the S partials in the fixed order q = 0 .. S-1 -- the order of k_cheb_sym_tma's
// reducer, so the results are bitwise equal to it -- and runs the fused chain epilogue; nothing
// on the epilogue group ever waits for another CTA.
constexpr int PP_HDR = 256;   // mbarriers, tickets, unit records
struct PpMeta {
  int k, tile, q, ti, tj;
};

template <int CH>
__device__ __forceinline__ void pp_finish(const SymArgs& a, int k, int tile, int q, int ti, int tj, const double* stg,
                                          int u, int* s_last) {
  constexpr int mc = CH, NT = NTHREADS, NV = 32;
  const int T = a.T;
  const int S = a.split;
  const int ntri = T * (T + 1) / 2;
  int* cross = a.sync + 1;
  const int64_t s = a.s;
  const int warp = u >> 5, lane = u & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const bool cstep = k > mc;
  const int hj = (k - 2) % mc;
  const int sidx = mc * tile + hj;
  const int ord = (k - 2 - hj) / mc + 1;          // products of this tile and chain so far
  double v[NV];
#pragma unroll
  for (int rr = 0; rr < NV; ++rr) v[rr] = stg[rr * NT + u];
  if (S > 1) {
    double* slots = a.partial + (int64_t)sidx * S * (BM * BN);
    CPA_DCHECK(tile >= 0 && tile < ntri && q >= 0 && q < S);
#pragma unroll
    for (int rr = 0; rr < NV; ++rr) __stcg(slots + (int64_t)q * (BM * BN) + rr * NT + u, v[rr]);
    named_bar(3, NTHREADS);
    if (u == 0) {
      int old;
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;\n"
                   : "=r"(old)
                   : "l"(a.sync + sym_split_off(a.K, T) + sidx)
                   : "memory");
      *s_last = old + 1 == S * ord;
    }
    named_bar(3, NTHREADS);
    if (!*s_last) return;
    // the last arrival: the S partials in the fixed order q = 0 .. S-1 (its own from registers),
    // eight values at a time (register budget)
#pragma unroll
    for (int c8 = 0; c8 < NV / 8; ++c8) {
      double sum[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) sum[x] = q == 0 ? v[c8 * 8 + x] : __ldcg(slots + (c8 * 8 + x) * NT + u);
      for (int p = 1; p < S; ++p) {
        double w[8];
#pragma unroll
        for (int x = 0; x < 8; ++x)
          w[x] = p == q ? v[c8 * 8 + x] : __ldcg(slots + (int64_t)p * (BM * BN) + (c8 * 8 + x) * NT + u);
#pragma unroll
        for (int x = 0; x < 8; ++x) sum[x] += w[x];
      }
#pragma unroll
      for (int x = 0; x < 8; ++x) v[c8 * 8 + x] = sum[x];
    }
  }
  // the fused chain epilogue (as sym_finish_impl's m-chain branch)
  const double* src = a.C[chain_buf(cstep ? k - mc : k - 1, mc)];
  const double* wpp = !cstep ? (k == 2 ? nullptr : a.C[chain_buf(k - 2, mc)])
                             : (k == 2 * mc ? nullptr : a.C[chain_buf(k > 2 * mc ? k - 2 * mc : 2 * mc - k, mc)]);
  double* out = a.C[chain_buf(k, mc)];
  double* hmine = hj == 0 ? a.H : a.HX[hj - 1];
  const bool hzero = hj > 0 && k == 2 + hj;
  const int64_t m0 = (int64_t)ti * BM, n0 = (int64_t)tj * BN;
  const double s4 = 2.0 * a.P->scale2, ck = a.P->c[k];
  const bool last = k == a.K - 1;
  const bool store_w = k + mc <= a.K - 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t rr = m0 + wm + i * 8 + g;
    double vp[8], vpp[8], vy[8];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + wn + j * 8 + 2 * t + e;
        const bool ok = rr < s && c <= rr;
        const int64_t o = rr * s + c;
        vp[j * 2 + e] = (!cstep && ok) ? __ldcg(src + o) : 0.0;
        vpp[j * 2 + e] = wpp == nullptr ? (rr == c ? 1.0 : 0.0) : (ok ? __ldcg(wpp + o) : 0.0);
        double y0 = (hzero || !ok) ? 0.0 : __ldcg(hmine + o);
        if (last && ok)
          for (int jj = 0; jj < mc; ++jj)
            if (jj != hj) y0 += __ldcg((jj == 0 ? a.H : a.HX[jj - 1]) + o);
        vy[j * 2 + e] = y0;
      }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + wn + j * 8 + 2 * t + e;
        if (!(rr < s && c <= rr)) continue;
        const int qq = j * 2 + e;
        const double acc = v[(i * 4 + j) * 2 + e];
        const double wv = cstep ? 2.0 * acc - vpp[qq] : s4 * acc - 2.0 * vp[qq] - vpp[qq];
        const double y = vy[qq] + ck * wv;
        if (store_w) {
          out[rr * s + c] = wv;
          out[c * s + rr] = wv;
        }
        if (last) {
          a.H[rr * s + c] = y;
          a.H[c * s + rr] = y;
        } else {
          hmine[rr * s + c] = y;
        }
      }
  }
  fence_proxy_async_global();   // Psi_k / H stores -> later TMA (async-proxy) reads
  named_bar(3, NTHREADS);
  if (u == 0) {
    red_release_add_i32(cross + k * T + ti, 1);
    if (ti != tj) red_release_add_i32(cross + k * T + tj, 1);
    red_release_add_i32(a.sync + sym_tdone_off(a.K, T, mc) + k * ntri + tile, 1);   // tile done
    if (k == mc) red_release_add_i32(a.sync + sym_pm_off(a.K, T, mc), 1);          // Psi_m progress
  }
}

template <int SBK, int SSTAGES, int CH>
__global__ void __launch_bounds__(3 * NTHREADS, 1) k_cheb_sym_pp(const __grid_constant__ SymMapsChain mp, SymArgs a) {
  constexpr int SBOX_BYTES = 16 * SBK * 8;
  constexpr int SSTAGE_BYTES = 8 * SBOX_BYTES;
  constexpr int RING_BYTES = SSTAGES * SSTAGE_BYTES;
  constexpr int mc = CH;
  extern __shared__ __align__(16) unsigned char tsm_raw[];
  uint64_t* fullb = reinterpret_cast<uint64_t*>(tsm_raw);   // [2][SSTAGES]
  uint64_t* emptyb = fullb + 2 * SSTAGES;                    // [2][SSTAGES]
  uint64_t* sfull = emptyb + 2 * SSTAGES;                    // [2]
  uint64_t* sempty = sfull + 2;                              // [2]
  int* s_ticket = reinterpret_cast<int*>(sempty + 2);        // [2][2]
  int* s_ctl = s_ticket + 4;                                 // [0] selected group, [1] last arrival
  PpMeta* meta = reinterpret_cast<PpMeta*>(s_ctl + 2);       // [2]
  static_assert(8 * (4 * SSTAGES + 4) + 4 * 6 + 2 * sizeof(PpMeta) <= PP_HDR, "header");
  const uint32_t raw = smem_u32(tsm_raw);
  unsigned char* base = tsm_raw + (((raw + PP_HDR + 1023u) & ~1023u) - raw);
  double* stage = reinterpret_cast<double*>(base + 2 * RING_BYTES);   // [2][64 x 64]
  {
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;\n" : "=r"(dyn));
    if ((uint32_t)(base - tsm_raw) + 2 * RING_BYTES + 2 * BM * BN * 8 > dyn) __trap();   // layout check
  }
  const int T = a.T;
  const int ntri = T * (T + 1) / 2;
  const int S = a.split;
  const int per_step = ntri * S;
  const int total = (a.K - a.k0) * per_step;
  int* cross = a.sync + 1;
  const int nk = (int)((a.s + SBK - 1) / SBK);
  const int wg = threadIdx.x / NTHREADS;
  const int tid = threadIdx.x % NTHREADS;
  const int warp = tid >> 5, lane = tid & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < 2 * SSTAGES; ++st) {
      mbar_init(fullb + st, 1);
      mbar_init(emptyb + st, 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(sfull + b, 4);
      mbar_init(sempty + b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (wg == 2) {
    // ---------------- epilogue warp group: serves the two MMA groups in arrival order ----------------
    uint32_t n0 = 0, n1 = 0;
    bool done0 = false, done1 = false;
    for (;;) {
      if (tid == 0) {
        int sel = -1;
        while (sel < 0) {
          uint32_t ok = 0;
          if (!done0) {
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok) : "r"(smem_u32(sfull)), "r"(n0 & 1) : "memory");
            if (ok) sel = 0;
          }
          if (sel < 0 && !done1) {
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok) : "r"(smem_u32(sfull + 1)), "r"(n1 & 1) : "memory");
            if (ok) sel = 1;
          }
        }
        s_ctl[0] = sel;
      }
      named_bar(3, NTHREADS);
      const int gsel = s_ctl[0];
      named_bar(3, NTHREADS);   // (s_ctl[0] is rewritten by the next selection)
      const uint32_t n = gsel ? n1 : n0;
      mbar_wait(sfull + gsel, n & 1);   // (complete: orders this thread's staging reads after it)
      const PpMeta mt = meta[gsel];
      if (mt.k >= 0) {
        pp_finish<CH>(a, mt.k, mt.tile, mt.q, mt.ti, mt.tj, stage + gsel * (BM * BN), tid, s_ctl + 1);
        __syncwarp();
      }
      if (lane == 0) mbar_arrive(sempty + gsel);   // staging gsel may be refilled
      if (gsel) { ++n1; done1 = mt.k < 0; } else { ++n0; done0 = mt.k < 0; }
      if (done0 && done1) break;
    }
    return;
  }
  // ---------------- MMA warp groups (thread 0 of each: tickets and TMA producer) ----------------
  unsigned char* ring = base + wg * RING_BYTES;
  uint64_t* full = fullb + wg * SSTAGES;
  uint64_t* empty = emptyb + wg * SSTAGES;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  uint32_t coff[2][2];
#pragma unroll
  for (int par = 0; par < 2; ++par)
#pragma unroll
    for (int h = 0; h < 2; ++h) coff[par][h] = ((((h * 8 + g) >> 1) ^ (2 * t + par)) << 4) | ((g & 1) * 8);
  const uint32_t roff = 256 * t;
  const uint32_t boxa = (wm >> 4) * SBOX_BYTES, boxb = (4 + (wn >> 4)) * SBOX_BYTES;
  const int bar_id = 1 + wg;
  uint32_t it = 0;   // slabs consumed by this group so far
  uint32_t nunit = 0;
  for (;;) {
    int* my_ticket = s_ticket + 2 * wg + (nunit & 1);
    if (tid == 0) *my_ticket = atomicAdd(a.sync, 1);
    named_bar(bar_id, NTHREADS);
    const int tk = *my_ticket;
    if (tk >= total) {
      mbar_wait(sempty + wg, (nunit & 1) ^ 1);
      if (tid == 0) meta[wg].k = -1;
      __syncwarp();
      if (lane == 0) mbar_arrive(sfull + wg);
      break;
    }
    const int k = a.k0 + tk / per_step;
    const int r = tk % per_step;
    const int q = r % S;
    const int tile = r / S;
    int ti, tj;
    tri_decode_colmajor(tile, T, ti, tj);
    CPA_DCHECK(ti >= 0 && ti < T && tj >= 0 && tj <= ti);
    const bool cstep = k > mc;
    const CUtensorMap* wmap = &mp.c[chain_buf(cstep ? k - mc : k - 1, mc)];
    const CUtensorMap* amap = cstep ? &mp.c[mc - 1] : &mp.g;
    const int m0 = ti * BM, n0 = tj * BN;
    int kb, ke;
    {   // the last split takes a (100 + red_bias)% k-range (as k_cheb_sym_tma's m-chain instance)
      const int64_t wt = 100 * S + a.red_bias;
      kb = (int)((int64_t)nk * q * 100 / wt);
      ke = q == S - 1 ? nk : (int)((int64_t)nk * (q + 1) * 100 / wt);
    }
    const int nku = ke - kb;
    if (warp == 0) {
      const int P = nku < SSTAGES - 1 ? nku : SSTAGES - 1;
      bool a_early = true;
      if (cstep) {
        const int v = lane == 0 ? ld_acquire(a.sync + sym_pm_off(a.K, T, mc)) : 0;
        a_early = __shfl_sync(0xffffffffu, v, 0) >= ntri;
      }
      auto issue_a = [&] {
        for (int p = 0; p < P; ++p) {
          const uint32_t sl = it + p, st = sl % SSTAGES;
          mbar_wait(empty + st, ((sl / SSTAGES) & 1) ^ 1);
          mbar_expect_tx(full + st, SSTAGE_BYTES);
          for (int b = 0; b < 4; ++b)
            tma_load_2d(ring + st * SSTAGE_BYTES + b * SBOX_BYTES, amap, m0 + 16 * b, (kb + p) * SBK, full + st);
        }
      };
      if (lane == 0 && a_early) issue_a();
      {   // dependencies: the rules of k_cheb_sym_tma's m-chain instance (see there)
        const int* tdone = a.sync + sym_tdone_off(a.K, T, mc);
        const int l0 = (kb * SBK) / BM, l1e = (ke * SBK - 1) / BM, l1 = l1e < T - 1 ? l1e : T - 1;
        const int nl = l1 - l0 + 1;
        auto tri_idx = [&](int rr, int cc) { return cc * (2 * T - cc + 1) / 2 + (rr - cc); };   // rr >= cc
        const int kprev = cstep ? k - mc : k - 1;
        const int khaz = cstep ? (k >= 4 * mc + 1 ? k - 2 * mc : 0) : 0;
        const bool need_b = kprev >= 2;
        const bool need_m = cstep && k <= 2 * mc;
        const bool need_a = need_m && !a_early;
        const bool need_h = k == a.K - 1;
        const int nflags = 6 + nl + (need_a ? nl : 0);
        for (int f = lane; f < nflags; f += 32) {
          const int* flag = nullptr;
          int target = 1;
          if (f < 2) {
            if (khaz) { flag = cross + khaz * T + (f == 0 ? ti : tj); target = T; }
          } else if (f == 2) {
            if (need_b) flag = tdone + kprev * ntri + tile;
          } else if (f == 3) {
            if (need_m) flag = tdone + mc * ntri + tile;
          } else if (f < 6) {
            if (need_h && f - 3 < mc) flag = tdone + (a.K - 1 - (f - 3)) * ntri + tile;
          } else if (f < 6 + nl) {
            const int l = l0 + f - 6;
            if (need_b) flag = tdone + kprev * ntri + (l >= tj ? tri_idx(l, tj) : tri_idx(tj, l));
          } else {
            const int l = l0 + f - 6 - nl;
            flag = tdone + mc * ntri + (l >= ti ? tri_idx(l, ti) : tri_idx(ti, l));
          }
          if (flag) wait_geq(flag, target);
        }
        __syncwarp();
      }
      if (lane == 0) {
        fence_proxy_async_global();   // generic-proxy stores of other CTAs -> TMA reads
        if (!a_early) issue_a();
        for (int p = 0; p < P; ++p) {
          const uint32_t st = (it + p) % SSTAGES;
          for (int b = 0; b < 4; ++b)
            tma_load_2d(ring + st * SSTAGE_BYTES + (4 + b) * SBOX_BYTES, wmap, n0 + 16 * b, (kb + p) * SBK,
                        full + st);
        }
      }
    }
    // (the epilogue group's generic loads are ordered after warp 0's acquire through the full
    // barriers of refilled slabs and the staging handover; a unit too short to refill takes a
    // group barrier, as in k_cheb_sym_tma)
    if (nku < SSTAGES) named_bar(bar_id, NTHREADS);
    else __syncwarp();
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < nku; ++kt) {
      if (tid == 0 && kt + SSTAGES - 1 < nku) {   // refill the stage of slab kt-1
        const int kn = kt + SSTAGES - 1;
        const uint32_t sl = it + kn, st = sl % SSTAGES;
        mbar_wait(empty + st, ((sl / SSTAGES) & 1) ^ 1);
        mbar_expect_tx(full + st, SSTAGE_BYTES);
        unsigned char* d = ring + st * SSTAGE_BYTES;
        for (int b = 0; b < 4; ++b) tma_load_2d(d + b * SBOX_BYTES, amap, m0 + 16 * b, (kb + kn) * SBK, full + st);
        for (int b = 0; b < 4; ++b)
          tma_load_2d(d + (4 + b) * SBOX_BYTES, wmap, n0 + 16 * b, (kb + kn) * SBK, full + st);
      }
      __syncwarp();
      const uint32_t sl = it + kt, st = sl % SSTAGES;
      mbar_wait(full + st, (sl / SSTAGES) & 1);
      const unsigned char* sa = ring + st * SSTAGE_BYTES + boxa;
      const unsigned char* sb = ring + st * SSTAGE_BYTES + boxb;
#pragma unroll
      for (int kk = 0; kk < SBK / 4; ++kk) {
        const int par = kk & 1;
        const uint32_t ro = 1024 * (kk >> 1) + 128 * par + roff;
        double fa[4], fb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          fa[i] = *reinterpret_cast<const double*>(sa + (i >> 1) * SBOX_BYTES + ro + coff[par][i & 1]);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          fb[j] = *reinterpret_cast<const double*>(sb + (j >> 1) * SBOX_BYTES + ro + coff[par][j & 1]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
    }
    it += nku;
    // hand the accumulators to the epilogue group (layout [reg][thread], the split-K slot layout)
    mbar_wait(sempty + wg, (nunit & 1) ^ 1);
    double* stg = stage + wg * (BM * BN);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) stg[((i * 4 + j) * 2 + e) * NTHREADS + tid] = acc[i][j][e];
    if (tid == 0) meta[wg] = PpMeta{k, tile, q, ti, tj};
    __syncwarp();
    if (lane == 0) mbar_arrive(sfull + wg);
    ++nunit;
  }
}

// Cluster variant of k_cheb_sym for small s (c2): the CS k-splits of a tile run as one
// thread-block cluster and reduce through distributed shared memory instead of L2 partial
// buffers and a single reducer.  Each CTA stores its partial accumulators in its own shared
// memory; after a cluster barrier CTA q sums warp-tile q (32 x 32) of all CS partials in the
// fixed order r = 0..CS-1 and runs the fused epilogue for that quarter of the tile -- every CTA
// of the cluster shares the epilogue, so the tile's reduction latency on the dataflow's
// critical path is one DSMEM round trip.  Tickets are per tile (claimed by the leader CTA);
// the dependency rule and the three-buffer rotation are those of k_cheb_sym.
template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(NTHREADS, CPA_FLOW_MINB) k_cheb_sym_cl(SymArgs a) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_ticket;
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const int T = a.T;
  const int ntri = T * (T + 1) / 2;
  const int total = (a.K - 2) * ntri;
  int* cross = a.sync + 1;
  const int64_t s = a.s;
  const int nk = (int)((s + BKS - 1) / BKS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = (int)((int64_t)nk * q / CS), ke = (int)((int64_t)nk * (q + 1) / CS);
  for (;;) {
    // the leader claims the tile's ticket and writes it into every CTA's own shared memory
    // (no CTA reads a peer's shared memory after the last barrier: safe exit)
    if (q == 0 && threadIdx.x == 0) {
      const int t0 = atomicAdd(a.sync, 1);
#pragma unroll
      for (int r = 0; r < CS; ++r) *cl.map_shared_rank(&s_ticket, r) = t0;
    }
    cl.sync();
    const int tk = s_ticket;
    if (tk >= total) break;
    const int k = 2 + tk / ntri;
    const int tile = tk % ntri;
    int ti, tj;
    tri_decode_colmajor(tile, T, ti, tj);
    CPA_DCHECK(ti >= 0 && ti < T && tj >= 0 && tj <= ti);
    auto buf = [&](int i) { return i == 0 ? a.W[0] : (i == 1 ? a.W[1] : a.W[2]); };
    const double* src = buf((k - 1) % 3);   // W_{k-1}
    const double* wpp = buf((k - 2) % 3);   // W_{k-2} (k = 2: identity, implicit)
    double* out = buf(k % 3);               // W_k over W_{k-3}
    const int64_t m0 = (int64_t)ti * BM, n0 = (int64_t)tj * BN;
    double acc[4][4][2];
    mainloop_dep(a.G, src, s, m0, n0, a.vec, smem, acc, kb, ke, [&] {
      if (threadIdx.x == 0) {
        if (k >= 3) wait_geq(cross + (k - 1) * T + tj, T);
        if (k >= 4) wait_geq(cross + (k - 2) * T + ti, T);
      }
      __syncthreads();
    });
    // partial accumulators into own shared memory: [warp][reg][lane] (32 x 32 doubles per warp)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) smem[(warp * 32 + (i * 4 + j) * 2 + e) * 32 + lane] = acc[i][j][e];
    cl.sync();                                               // every partial written
    // reduce-scatter: this CTA owns the values [q 4096/CS, (q+1) 4096/CS) of the tile's partial
    // layout [warp][reg][lane]
    const double s4 = 2.0 * a.P->scale2, ck = a.P->c[k];
    const bool last = k == a.K - 1;
    constexpr int PER = 4096 / CS;
    double* peer[CS];
#pragma unroll
    for (int r = 0; r < CS; ++r) peer[r] = cl.map_shared_rank(smem, r) + q * PER;
#pragma unroll
    for (int it = 0; it < PER / NTHREADS; ++it) {
      const int el = it * NTHREADS + threadIdx.x;
      double v = peer[0][el];
#pragma unroll
      for (int r = 1; r < CS; ++r) v += peer[r][el];
      const int e = q * PER + el;
      const int wsrc = e >> 10, reg = (e >> 5) & 31, ln = e & 31;
      const int ii = reg >> 3, jj = (reg >> 1) & 3, ee = reg & 1;
      const int64_t rr = m0 + (wsrc >> 1) * 32 + ii * 8 + (ln >> 2);
      const int64_t c = n0 + (wsrc & 1) * 32 + jj * 8 + 2 * (ln & 3) + ee;
      if (rr < s && c <= rr) {
        const int64_t o = rr * s + c;
        const double vp = __ldcg(src + o);
        const double vpp = k == 2 ? (rr == c ? 1.0 : 0.0) : __ldcg(wpp + o);
        const double wv = s4 * v - 2.0 * vp - vpp;             // W_k = 2 B_hat W_{k-1} - W_{k-2}
        const double y = __ldcg(a.H + o) + ck * wv;            // H += c_k W_k
        if (!last) {
          out[o] = wv;
          out[c * s + rr] = wv;
        }
        a.H[o] = y;
        if (last) a.H[c * s + rr] = y;
      }
    }
    __threadfence();
    cl.sync();                                               // tile complete; shared memory reusable
    if (q == 0 && threadIdx.x == 0) {
      red_release_add_i32(cross + k * T + ti, 1);
      if (ti != tj) red_release_add_i32(cross + k * T + tj, 1);
    }
  }
}

// Lower-triangle tile (tm >= tn) of linear index b (GRAM); row-major tile order (STORE).
template <int MODE>
__device__ __forceinline__ void gemm_tile(const GemmArgs& a, int& tm, int& tn) {
  if (MODE == EPI_GRAM) {
    const int b = blockIdx.x;
    int r = (int)((sqrt(8.0 * b + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= b) ++r;
    while (r * (r + 1) / 2 > b) --r;
    tm = r;
    tn = b - r * (r + 1) / 2;
  } else if (MODE == EPI_STORE) {
    const int tiles_n = (int)((a.N + BN - 1) / BN);
    tm = blockIdx.x / tiles_n;
    tn = blockIdx.x % tiles_n;
  } else {
    tm = blockIdx.x;
    tn = blockIdx.y;
  }
}

// split-K over gridDim.y units per tile (the triangle alone has too few tiles to give
// every SMSP more than one warp): every unit publishes its partial; the last to arrive
// sums them in the fixed order q = 0..S-1 (deterministic) into acc and returns true.
__device__ __forceinline__ bool gemm_split_reduce(const GemmArgs& a, double (&acc)[4][4][2]) {
  __shared__ int s_last;
  const int S = a.sS ? a.sS : gridDim.y, q = a.sq0 + blockIdx.y;
  double* slot = a.partial + (int64_t)blockIdx.x * S * (BM * BN);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        __stcg(slot + (int64_t)q * (BM * BN) + ((i * 4 + j) * 2 + e) * NTHREADS + threadIdx.x, acc[i][j][e]);
  __syncthreads();
  if (threadIdx.x == 0) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;\n" : "=r"(old) : "l"(a.tcount + blockIdx.x) : "memory");
    s_last = old == S - 1;
  }
  __syncthreads();
  if (!s_last) return false;
  // the 8 accumulators of row group i, summed over the splits in the fixed order p = 0..S-1,
  // four splits' loads in flight at a time (the register budget of three CTAs per SM)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double sum[8];
#pragma unroll
    for (int p0 = 0; p0 < 8; p0 += 4) {
      if (p0 >= S) break;
      double pv[4][8];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q8 = 0; q8 < 8; ++q8)
          pv[p][q8] = p0 + p < S ? __ldcg(slot + (int64_t)(p0 + p) * (BM * BN) + (i * 8 + q8) * NTHREADS + threadIdx.x)
                                 : 0.0;
#pragma unroll
      for (int q8 = 0; q8 < 8; ++q8) {
        double v = p0 == 0 ? pv[0][q8] : sum[q8] + pv[0][q8];
#pragma unroll
        for (int p = 1; p < 4; ++p)
          if (p0 + p < S) v += pv[p][q8];
        sum[q8] = v;
      }
    }
#pragma unroll
    for (int q8 = 0; q8 < 8; ++q8) acc[i][q8 >> 1][q8 & 1] = sum[q8];
  }
  return true;
}

// GRAM: the r >= c elements of the tile, mirrored (times the optional exact scale);
// STORE: plain product (Alg. 1 line 12: Y = H_hat X or X H_hat).
template <int MODE>
__device__ __forceinline__ void gemm_store_tile(const GemmArgs& a, const double (&acc)[4][4][2], int64_t m0,
                                                int64_t n0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  if (MODE == EPI_GRAM) {
    double* G = a.Wout;
    const int64_t ld = a.ldwo;
    const double sc = a.gscale ? *a.gscale : 1.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t r = m0 + wm + i * 8 + g, c = n0 + wn + j * 8 + 2 * t + e;
          if (r < a.M && c < a.N && r >= c) {
            const double v = acc[i][j][e] * sc;
            G[r * ld + c] = v;
            G[c * ld + r] = v;
          }
        }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t r = m0 + wm + i * 8 + g, c = n0 + wn + j * 8 + 2 * t + e;
          if (r < a.M && c < a.N) a.Y[r * a.ldy + c] = acc[i][j][e];
        }
  }
}

template <bool A_KC, bool B_KC, int MODE>
__global__ void __launch_bounds__(NTHREADS) k_dmma_gemm(GemmArgs a) {
  extern __shared__ __align__(16) double smem[];
  int tm, tn;
  gemm_tile<MODE>(a, tm, tn);
  const int64_t m0 = (int64_t)tm * BM, n0 = (int64_t)tn * BN;
  double acc[4][4][2];
  if ((MODE == EPI_GRAM || MODE == EPI_STORE) && (a.sS ? a.sS : (int)gridDim.y) > 1) {
    const int S = a.sS ? a.sS : gridDim.y, q = a.sq0 + blockIdx.y;
    const int nk = (int)((a.Kd + BKS - 1) / BKS);
    mainloop<A_KC, B_KC>(a.A, a.lda, a.B, a.ldb, a.M, a.N, a.Kd, m0, n0, a.vec_a, a.vec_b, smem, acc,
                         (int)((int64_t)nk * q / S), (int)((int64_t)nk * (q + 1) / S));
    if (!gemm_split_reduce(a, acc)) return;
  } else {
    mainloop<A_KC, B_KC>(a.A, a.lda, a.B, a.ldb, a.M, a.N, a.Kd, m0, n0, a.vec_a, a.vec_b, smem, acc);
  }
  if (MODE == EPI_GRAM || MODE == EPI_STORE) {
    gemm_store_tile<MODE>(a, acc, m0, n0);
    return;
  }
  cheb_epilogue(acc, m0, n0, a.M, a.N, MODE == EPI_INIT, a.Wp, a.ldwp, a.Wpp, a.ldwpp, a.Wout, a.ldwo, a.Y, a.ldy,
                a.P, a.k);
}

// TMA-fed GEMM for the GRAM and STORE modes (Gram, the squarings of the power iteration,
// Alg. 1 line 12).  Operand layouts in shared memory, both 128-byte swizzled, 16 KB per stage:
//   ROWK  (the operand's k index runs down global rows: right Gram, B of STORE):
//         4 boxes of 16 (m or n) columns x 16 k rows;
//   ROWMN (k runs along global rows, "K-major": left Gram, A of STORE):
//         1 box of 16 k columns x 64 (m or n) rows.
// DMMA step kk consumes the k indices {0, 10, 5, 15}[t] ^ kk of the slab: for either layout
// the 16 (row, column) pairs a half-warp reads then fall in 32 distinct banks.  Pipeline as
// in k_cheb_sym_tma (thread 0 produces; one CTA per unit, so the ring starts fresh).
struct GemmMaps {
  CUtensorMap a, b;
};
template <bool ROWK>
__device__ __forceinline__ double frag_ld(const unsigned char* st, int mn, int k) {
  uint32_t off;
  if (ROWK) {  // box mn/16, row k, column mn%16
    const int c = mn & 15;
    off = (mn >> 4) * BOX_BYTES + k * 128 + ((((c >> 1) ^ (k & 7)) << 4) | ((c & 1) << 3));
  } else {     // row mn, column k
    off = mn * 128 + ((((k >> 1) ^ (mn & 7)) << 4) | ((k & 1) << 3));
  }
  return *reinterpret_cast<const double*>(st + off);
}
template <bool ROWK>
__device__ __forceinline__ void tma_operand(unsigned char* dst, const CUtensorMap* map, int mn0, int k0,
                                            uint64_t* bar) {
  if (ROWK) {
    for (int b = 0; b < 4; ++b) tma_load_2d(dst + b * BOX_BYTES, map, mn0 + 16 * b, k0, bar);
  } else {
    tma_load_2d(dst, map, k0, mn0, bar);
  }
}
template <bool A_ROWK, bool B_ROWK, int MODE>
__global__ void __launch_bounds__(NTHREADS, 3) k_dmma_gemm_tma(const __grid_constant__ GemmMaps mp, GemmArgs a) {
  extern __shared__ unsigned char gsm_raw[];
  __shared__ __align__(8) uint64_t full[TSTAGES], empty[TSTAGES];
  unsigned char* base = gsm_raw + ((1024u - (smem_u32(gsm_raw) & 1023u)) & 1023u);
  int tm, tn;
  gemm_tile<MODE>(a, tm, tn);
  const int m0 = tm * BM, n0 = tn * BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int nk = (int)((a.Kd + TBK - 1) / TBK);
  const int S = a.sS ? a.sS : gridDim.y, q = a.sq0 + blockIdx.y;
  const int kb = (int)((int64_t)nk * q / S), ke = (int)((int64_t)nk * (q + 1) / S);
  const int nku = ke - kb;
  if (threadIdx.x == 0) {
    for (int st = 0; st < TSTAGES; ++st) {
      mbar_init(full + st, 1);
      mbar_init(empty + st, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int sl) {   // slab sl of this unit into stage sl % TSTAGES
    const int st = sl % TSTAGES;
    mbar_wait(empty + st, ((sl / TSTAGES) & 1) ^ 1);
    mbar_expect_tx(full + st, TSTAGE_BYTES);
    unsigned char* d = base + st * TSTAGE_BYTES;
    tma_operand<A_ROWK>(d, &mp.a, m0, (kb + sl) * TBK, full + st);
    tma_operand<B_ROWK>(d + 4 * BOX_BYTES, &mp.b, n0, (kb + sl) * TBK, full + st);
  };
  if (threadIdx.x == 0)
    for (int p = 0; p < TSTAGES - 1 && p < nku; ++p) issue(p);
  __syncwarp();
  const int kbase = (t == 0 ? 0 : t == 1 ? 10 : t == 2 ? 5 : 15);
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kt = 0; kt < nku; ++kt) {
    if (threadIdx.x == 0 && kt + TSTAGES - 1 < nku) issue(kt + TSTAGES - 1);
    __syncwarp();
    const int st = kt % TSTAGES;
    mbar_wait(full + st, (kt / TSTAGES) & 1);
    const unsigned char* sa = base + st * TSTAGE_BYTES;
    const unsigned char* sb = sa + 4 * BOX_BYTES;
#pragma unroll
    for (int kk = 0; kk < TBK / 4; ++kk) {
      const int kx = kbase ^ kk;
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = frag_ld<A_ROWK>(sa, wm + i * 8 + g, kx);
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = frag_ld<B_ROWK>(sb, wn + j * 8 + g, kx);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // loads done before the TMA refill
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }
  if (S > 1 && !gemm_split_reduce(a, acc)) return;
  gemm_store_tile<MODE>(a, acc, m0, n0);
}

// 2-D fp64 tensor map (rows x cols, row stride ld elements), box {16, box_rows}, 128B swizzle
static bool make_map_f64(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15) || (ld % 2) || rows < 1 || cols < 1) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * sizeof(double))};
  cuuint32_t box[2] = {16u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// k-splits (1..8, >= 4 k-slabs each) whose units fill whole waves of the resident
// slots best; ties (within 3%) go to fewer splits.  Only when the tiles alone
// leave slots idle (fewer than 3 waves).
static int best_split(int64_t tiles, int64_t nk, int64_t slots) {
  if (tiles >= 3 * slots) return 1;
  int best = 1;
  double best_eff = 0.0;
  for (int S = 1; S <= 8; ++S) {
    if (S > 1 && nk / S < 4) break;
    const int64_t u = tiles * S, waves = (u + slots - 1) / slots;
    const double eff = (double)u / (double)(waves * slots);
    if (eff > best_eff + 0.03) { best_eff = eff; best = S; }
  }
  return best;
}

template <bool A_KC, bool B_KC, int MODE>
static cudaError_t launch(const GemmArgs& a, cudaStream_t st) {
  using LA = OpLayout<A_KC, BM>;
  using LB = OpLayout<B_KC, BN>;
  const size_t smem = (size_t)STAGES * (LA::SIZE + LB::SIZE) * sizeof(double);
  auto fn = k_dmma_gemm<A_KC, B_KC, MODE>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t tm = (a.M + BM - 1) / BM, tn = (a.N + BN - 1) / BN;
  dim3 grid;
  if (MODE == EPI_GRAM || MODE == EPI_STORE) {
    const int64_t tiles = MODE == EPI_GRAM ? tm * (tm + 1) / 2 : tm * tn, nk = (a.Kd + BKS - 1) / BKS;
    int split = 1;
    if (a.sS > 0) {               // one unit of an across-launch split (dense_gram_f64_chunk)
      if (a.sq0 == 0) {
        cudaError_t ez = cudaMemsetAsync(a.tcount, 0, tiles * sizeof(int), st);
        if (ez != cudaSuccess) return ez;
      }
    } else if (a.partial && a.tcount) {  // split-K needs scratch (sized by dense_split_partial_doubles)
      int dev = 0, sms = 148, per_sm = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NTHREADS, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
      split = best_split(tiles, nk, (int64_t)sms * per_sm);
      if (const char* v = getenv(MODE == EPI_STORE ? "CPA_SVT_STORE_SPLIT" : "CPA_SVT_GRAM_SPLIT");
          v && atoi(v) >= 1 && atoi(v) <= 8)
        split = atoi(v);   // (experiments)
      if (split > 1) {
        cudaError_t ez = cudaMemsetAsync(a.tcount, 0, tiles * sizeof(int), st);
        if (ez != cudaSuccess) return ez;
      }
    }
    grid = dim3((unsigned)tiles, (unsigned)split);
    // TMA-fed kernel when both operands admit a tensor map (16-byte aligned rows)
    if constexpr (MODE == EPI_GRAM || MODE == EPI_STORE) {
    GemmMaps mp;
    if (!env_on("CPA_SVT_GEMM_NOTMA") && a.M <= INT32_MAX / 2 && a.N <= INT32_MAX / 2 && a.Kd <= INT32_MAX / 2 &&
        (A_KC ? make_map_f64(&mp.a, a.A, a.M, a.Kd, a.lda, 64) : make_map_f64(&mp.a, a.A, a.Kd, a.M, a.lda, 16)) &&
        (B_KC ? make_map_f64(&mp.b, a.B, a.N, a.Kd, a.ldb, 64) : make_map_f64(&mp.b, a.B, a.Kd, a.N, a.ldb, 16))) {
      auto tf = k_dmma_gemm_tma<!A_KC, !B_KC, MODE>;
      const size_t tsmem = (size_t)TSTAGES * TSTAGE_BYTES + 1024;
      e = cudaFuncSetAttribute(tf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
      if (e != cudaSuccess) return e;
      tf<<<grid, NTHREADS, tsmem, st>>>(mp, a);
      return cudaGetLastError();
    }
    }
  } else {
    grid = dim3((unsigned)tm, (unsigned)tn);
  }
  fn<<<grid, NTHREADS, smem, st>>>(a);
  return cudaGetLastError();
}

static inline bool aligned16(const void* p, int64_t ld) {
  return ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && (ld % 2 == 0);
}

// G (s x s, ld s) = X X^T (left, s = m) or X^T X (right, s = n); X m x n row-major.
// partial / tcount: optional scratch (dense_gram_partial_doubles(s) doubles, tiles ints) enabling split-K
cudaError_t dense_gram_f64(const double* X, int64_t m, int64_t n, int64_t ldx, bool left, double* G,
                           cudaStream_t st, const double* gscale, double* partial, int* tcount) {
  GemmArgs a{};
  a.gscale = gscale;
  a.partial = partial;
  a.tcount = tcount;
  if (left) {  // G(i,j) = sum_l X[i][l] X[j][l]: A(m,k)=X[m][k] (k contig), B(k,n)=X[n][k] (k contig)
    a.M = m; a.N = m; a.Kd = n;
    a.A = X; a.lda = ldx; a.B = X; a.ldb = ldx;
  } else {     // G(i,j) = sum_l X[l][i] X[l][j]: A(m,k)=X[k][m] (m contig), B(k,n)=X[k][n] (n contig)
    a.M = n; a.N = n; a.Kd = m;
    a.A = X; a.lda = ldx; a.B = X; a.ldb = ldx;
  }
  a.Wout = G; a.ldwo = a.M;
  a.vec_a = a.vec_b = aligned16(X, ldx);
  if (a.M == 0) return cudaSuccess;
  return left ? launch<true, true, EPI_GRAM>(a, st) : launch<false, false, EPI_GRAM>(a, st);
}

// Unit q of an S-way split-K Gram as its own launch (see dense_gram_chunk_range); the launch
// of the last-arriving unit stores G.  S <= 8, dense_gram_partial_doubles(s) > 0.
cudaError_t dense_gram_f64_chunk(const double* X, int64_t m, int64_t n, int64_t ldx, bool left, double* G,
                                 cudaStream_t st, double* partial, int* tcount, int q, int S) {
  GemmArgs a{};
  a.partial = partial;
  a.tcount = tcount;
  a.sS = S;
  a.sq0 = q;
  if (left) {
    a.M = m; a.N = m; a.Kd = n;
    a.A = X; a.lda = ldx; a.B = X; a.ldb = ldx;
  } else {
    a.M = n; a.N = n; a.Kd = m;
    a.A = X; a.lda = ldx; a.B = X; a.ldb = ldx;
  }
  a.Wout = G; a.ldwo = a.M;
  a.vec_a = a.vec_b = aligned16(X, ldx);
  if (a.M == 0 || S < 1 || S > 8 || !partial || !tcount) return cudaErrorInvalidValue;
  return left ? launch<true, true, EPI_GRAM>(a, st) : launch<false, false, EPI_GRAM>(a, st);
}

// One recurrence launch.  left: out(s x L) = G (s x s) * Wsrc (s x L);
// right: out (L x s) = Wsrc (L x s) * G.  mode INIT uses Wsrc = X; STEP uses
// Wsrc = W_{k-1}, Wpp = W_{k-2}.  Shapes: rows x cols of the output = (m, n) of X.
cudaError_t dense_cheb_launch(bool left, bool init, int64_t m, int64_t n, const double* G,
                              const double* Wsrc, int64_t ldsrc, const double* Wpp, int64_t ldpp,
                              double* Wout, int64_t ldout, double* Y, int64_t ldy, const SeriesParams* P,
                              int k, cudaStream_t st) {
  GemmArgs a{};
  a.M = m; a.N = n;
  if (left) {  // A = G (symmetric, read as G[k][m], m contiguous), B = Wsrc[k][n]
    a.Kd = m;
    a.A = G; a.lda = m; a.B = Wsrc; a.ldb = ldsrc;
    a.vec_a = aligned16(G, m); a.vec_b = aligned16(Wsrc, ldsrc);
  } else {     // A = Wsrc[m][k] (k contiguous), B = G[k][n]
    a.Kd = n;
    a.A = Wsrc; a.lda = ldsrc; a.B = G; a.ldb = n;
    a.vec_a = aligned16(Wsrc, ldsrc); a.vec_b = aligned16(G, n);
  }
  a.Wout = Wout; a.ldwo = ldout;
  a.Wp = Wsrc; a.ldwp = ldsrc;
  a.Wpp = Wpp; a.ldwpp = ldpp;
  a.Y = Y; a.ldy = ldy;
  a.P = P; a.k = k;
  if (m == 0 || n == 0) return cudaSuccess;
  if (left) return init ? launch<false, false, EPI_INIT>(a, st) : launch<false, false, EPI_STEP>(a, st);
  return init ? launch<true, false, EPI_INIT>(a, st) : launch<true, false, EPI_STEP>(a, st);
}

size_t dense_store_partial_doubles(int64_t M, int64_t N);

// C (M x N, ldc) = A (M x Kd, row-major, k contiguous) * B (Kd x N, row-major, n contiguous).
// Used for Alg. 1 line 12 in the s x s polynomial form: Y = H_hat X (left) or X H_hat (right).
cudaError_t dense_gemm_store(int64_t M, int64_t N, int64_t Kd, const double* A, int64_t lda, const double* B,
                             int64_t ldb, double* C, int64_t ldc, cudaStream_t st, double* partial, int* tcount) {
  GemmArgs a{};
  a.partial = dense_store_partial_doubles(M, N) ? partial : nullptr;
  a.tcount = tcount;
  a.M = M; a.N = N; a.Kd = Kd;
  a.A = A; a.lda = lda; a.B = B; a.ldb = ldb;
  a.vec_a = aligned16(A, lda); a.vec_b = aligned16(B, ldb);
  a.Y = C; a.ldy = ldc;
  if (M == 0 || N == 0) return cudaSuccess;
  return launch<true, false, EPI_STORE>(a, st);
}

__global__ void k_eye(double* I, int64_t s) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s * s; e += (int64_t)gridDim.x * blockDim.x)
    I[e] = (e / s == e % s) ? 1.0 : 0.0;
}
cudaError_t dense_eye(double* I, int64_t s, cudaStream_t st) {
  k_eye<<<1184, 256, 0, st>>>(I, s);
  return cudaGetLastError();
}

// Whole recurrence (init + K-2 steps) in one persistent launch.
// k-split per tile: enough units per step to spread over every SM slot
// (c2: 256 tiles x 4 = 1024 units), at least 4 k-slabs per unit.
static int flow_split(int64_t m, int64_t n, int64_t s, int num_sms) {
  const int64_t tiles = ((m + BM - 1) / BM) * ((n + BN - 1) / BN);
  const int64_t nk = (s + BKS - 1) / BKS;
  int split = 1;
  while (split < 4 && tiles * split < 6 * num_sms && nk / (2 * split) >= 4) split *= 2;  // <= 4 (reducer registers)
  if (const char* v = getenv("CPA_SVT_FLOW_SPLIT")) split = (atoi(v) > 0 && atoi(v) <= 4) ? atoi(v) : split;
  return split;
}

size_t dense_flow_sync_ints(int64_t m, int64_t n, int K) {
  const int64_t tm = (m + BM - 1) / BM, tn = (n + BN - 1) / BN;
  return (size_t)(1 + (int64_t)K * (tm > tn ? tm : tn) + tm * tn);
}

size_t dense_gram_partial_doubles(int64_t s) {
  const int64_t t = (s + BM - 1) / BM, tiles = t * (t + 1) / 2;
  return tiles < 1332 ? (size_t)tiles * 8 * BM * BN : 0;   // (no split-K beyond 3 waves of 3 x 148)
}

// Unit q of S of the split-K Gram in its own launch (the host pipeline of cpa_svt_apply_host
// launches unit q as soon as the q-th k-range of X has arrived): k-range of unit q in
// elements, and the launch.  partial / tcount as for dense_gram_f64 (S <= 8, tiles < 1332).
void dense_gram_chunk_range(int64_t kd, int q, int S, int64_t* k0, int64_t* k1) {
  const int64_t nk = (kd + BKS - 1) / BKS;
  *k0 = std::min(kd, nk * q / S * BKS);
  *k1 = std::min(kd, nk * (q + 1) / S * BKS);
}

// split-K scratch of dense_gemm_store (M x N output): used only when the tiles
// leave slots idle (< 3 waves of 3 x 148), so bounded by 1332 tiles x 8 splits.
size_t dense_store_partial_doubles(int64_t M, int64_t N) {
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  return tiles < 1332 ? (size_t)tiles * 8 * BM * BN : 0;
}

size_t dense_flow_partial_doubles(int64_t m, int64_t n, int num_sms) {
  const int64_t s = m <= n ? m : n;
  const int split = flow_split(m, n, s, num_sms);
  const int64_t tiles = ((m + BM - 1) / BM) * ((n + BN - 1) / BN);
  return split > 1 ? (size_t)(tiles * (split - 1) * BM * BN) : 0;
}

cudaError_t dense_cheb_flow(bool left, int64_t m, int64_t n, const double* G, const double* X, int64_t ldx,
                            double* Wa, double* Wb, double* Y, int64_t ldy, const SeriesParams* P, int K, int* sync,
                            double* partial, int num_sms, cudaStream_t st) {
  if (m == 0 || n == 0) return cudaSuccess;
  FlowArgs a{};
  a.M = m; a.N = n; a.s = left ? m : n;
  a.G = G; a.X = X; a.ldx = ldx; a.Wa = Wa; a.Wb = Wb; a.ldw = n; a.Y = Y; a.ldy = ldy; a.P = P; a.K = K;
  a.tiles_m = (int)((m + BM - 1) / BM);
  a.tiles_n = (int)((n + BN - 1) / BN);
  a.split = flow_split(m, n, a.s, num_sms);
  a.sync = sync;
  a.partial = partial;
  a.vec_x = aligned16(X, ldx); a.vec_w = aligned16(Wa, n) && aligned16(Wb, n); a.vec_g = aligned16(G, a.s);
  cudaError_t e = cudaMemsetAsync(sync, 0, dense_flow_sync_ints(m, n, K) * sizeof(int), st);
  if (e != cudaSuccess) return e;
  using LA = OpLayout<false, BM>;
  using LB = OpLayout<false, BN>;
  using LA2 = OpLayout<true, BM>;
  const size_t smem = (size_t)STAGES * ((left ? LA::SIZE : LA2::SIZE) + LB::SIZE) * sizeof(double);
  auto fn = left ? k_cheb_flow<true> : k_cheb_flow<false>;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NTHREADS, smem);
  if (e != cudaSuccess) return e;
  int64_t total = (int64_t)(K - 1) * a.tiles_m * a.tiles_n * a.split;
  int64_t grid = (int64_t)num_sms * (per_sm > 0 ? per_sm : 1);
  if (grid > total) grid = total;
  fn<<<(unsigned)grid, NTHREADS, smem, st>>>(a);
  return cudaGetLastError();
}

// ---- symmetric s x s form -------------------------------------------------------
static size_t sym_smem() { return (size_t)STAGES * (OpLayout<false, BM>::SIZE + OpLayout<false, BN>::SIZE) * sizeof(double); }

static int sym_slots(int num_sms) {
  int per_sm = 0;
  cudaFuncSetAttribute(k_cheb_sym<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sym_smem());
  cudaFuncSetAttribute(k_cheb_sym<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sym_smem());
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cheb_sym<false>, NTHREADS, sym_smem()) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  return num_sms * per_sm;
}

// k-splits per tile: about two units per resident slot per step (shorter units
// make the wavefront finer; c2 measured: S = 4 / 6 / 8 -> 1.46 / 1.31 / 1.39 ms),
// at least 4 k-slabs per unit, at most 8.
static int sym_split(int64_t s, int slots, int64_t ntiles = -1) {
  const int64_t T = (s + BM - 1) / BM, ntri = ntiles >= 0 ? ntiles : T * (T + 1) / 2;
  const int64_t nk = (s + BKS - 1) / BKS;
  int S = 1;
  while (S < 8 && ntri * S * 10 < 18 * (int64_t)slots && nk / (S + 1) >= 4) ++S;
  if (const char* v = getenv("CPA_SVT_FLOW_SPLIT")) S = (atoi(v) > 0 && atoi(v) <= 16) ? atoi(v) : S;
  return S;
}

size_t dense_sym_sync_ints(int64_t s, int K, int num_sms, int64_t L) {
  (void)num_sms;
  const int64_t T = (s + BM - 1) / BM;
  if (L > 0)   // (+ line 12 in the m-chain launch: one split-K counter per Y tile)
    return dense_sym_sync_ints(s, K, num_sms, 0) + (size_t)(T * ((L + BN - 1) / BN));
  // [0] ticket | K * T cross counters | up to 3 ntri split counters (m chains) | K * ntri tile-done
  // flags | Psi_m count
  return (size_t)(1 + (int64_t)K * T + 3 * (T * (T + 1) / 2) + (int64_t)K * (T * (T + 1) / 2) + 1);
}

// m-chain mode (SymArgs::chain = m) for the one-launch recurrence: on by default (m = 2) while
// the lower tiles of one step leave the resident slots short of work (the latency-bound regime,
// c2); CPA_SVT_SYM_CHAIN=0|1 (off) / 2 / 3 forces it.  Needs K >= 2m + 2.  Returns m, 0 = off.
int dense_sym_use_chain(int64_t s, int K, int num_sms) {
  if (s % 2 != 0 || s > INT32_MAX / 2 || env_on("CPA_SVT_SYM_NOTMA")) return 0;
  const int64_t T = (s + BM - 1) / BM;
  int m = T * (T + 1) / 2 < 4 * (int64_t)sym_slots(num_sms) ? 2 : 0;
  if (const char* v = getenv("CPA_SVT_SYM_CHAIN"); v && *v) m = atoi(v) >= 2 && atoi(v) <= 3 ? atoi(v) : 0;
  return K >= 2 * m + 2 ? m : 0;
}

static int sym_split_mode(int64_t s, int slots, int m) {
  const int64_t T = (s + BM - 1) / BM;
  int S = sym_split(s, slots, m > 1 ? m * (T * (T + 1) / 2) : -1);
  if (m > 1) {
    if (const char* v = getenv("CPA_SVT_CHAIN_SPLIT")) S = (atoi(v) > 0 && atoi(v) <= 16) ? atoi(v) : S;
  }
  return S;
}

// Ping-pong kernel for the m-chain mode (k_cheb_sym_pp: one CTA per SM, two MMA groups, last-
// arrival split-K), opt-in with CPA_SVT_SYM_PP=1: measured slower than the 3-CTA k_cheb_sym_tma
// instance at c2.
static bool sym_use_pp(int m) { return m > 1 && getenv("CPA_SVT_SYM_PP") && atoi(getenv("CPA_SVT_SYM_PP")) == 1; }

static int sym_split_pp(int64_t s, int num_sms, int m) {
  const int64_t T = (s + BM - 1) / BM;
  int S = sym_split(s, 2 * num_sms, m * (T * (T + 1) / 2));
  if (const char* v = getenv("CPA_SVT_CHAIN_SPLIT")) S = (atoi(v) > 0 && atoi(v) <= 16) ? atoi(v) : S;
  return S;
}

size_t dense_sym_partial_doubles(int64_t s, int num_sms, int m) {
  const int64_t T = (s + BM - 1) / BM;
  const int S = sym_use_pp(m) ? sym_split_pp(s, num_sms, m) : sym_split_mode(s, sym_slots(num_sms), m);
  // (m chains: S slots per tile and chain -- the ping-pong kernel publishes every split)
  return S > 1 ? (size_t)(T * (T + 1) / 2 * (m > 1 ? m * S : S - 1) * BM * BN) : 0;
}

// W_1 = B_hat (into W1 when K > 2) and H = c_0/2 I + c_1 W_1; with G2 (c^2 G^2 from the power
// iteration's first squaring, c^2 = *c2; K > 2): also Psi_2 over G2 and c_2 Psi_2 in H.
cudaError_t dense_sym_init(int64_t s, const double* G, double* W1, double* H, const SeriesParams* P, int K,
                           int num_sms, cudaStream_t st, double* G2, const double* c2) {
  if (s == 0) return cudaSuccess;
  if (G2 && K > 2) k_sym_init2<<<num_sms * 4, 256, 0, st>>>(G, s, W1, G2, c2, H, P);
  else k_sym_init<<<num_sms * 4, 256, 0, st>>>(G, s, K > 2 ? W1 : nullptr, H, P);
  return cudaGetLastError();
}

static cudaError_t sym_launch(SymArgs& a, int64_t total, int slots, int num_sms, cudaStream_t st);

// H_hat += sum_{k=2}^{K-1} c_k Psi_k(B_hat) on the s x s Gram: one persistent launch
// for all K-2 steps.  W0, W1, W2: s x s buffers, W1 = W_1 from dense_sym_init.  m-chain mode
// (m > 1: 4m s x s buffers in chain, chain[0] = W1 = Psi_1, plus m - 1 accumulators HX).
static int sym_l12_split(int64_t s, int64_t L, int num_sms) {
  const int64_t T = (s + BM - 1) / BM, tn = (L + BN - 1) / BN;
  int S = sym_split(s, sym_slots(num_sms), T * tn);
  if (const char* v = getenv("CPA_SVT_L12_SPLIT")) S = (atoi(v) > 0 && atoi(v) <= 16) ? atoi(v) : S;
  return S;
}
size_t dense_sym_l12_partial_doubles(int64_t s, int64_t L, int num_sms) {
  const int64_t T = (s + BM - 1) / BM, tn = (L + BN - 1) / BN;
  const int S = sym_l12_split(s, L, num_sms);
  return S > 1 ? (size_t)(T * tn * (S - 1) * BM * BN) : 0;
}

cudaError_t dense_cheb_sym(int64_t s, const double* G, double* W0, double* W1, double* W2, double* H,
                           const SeriesParams* P, int K, int* sync, double* partial, int num_sms, cudaStream_t st,
                           int m, double* const* chain, double* const* HX, bool psi2_given, const double* X,
                           int64_t ldx, double* Y, int64_t ldy, int64_t L, double* l12_partial) {
  if (s == 0 || K <= 2) return cudaSuccess;
  SymArgs a{};
  a.s = s; a.G = G; a.W[0] = W0; a.W[1] = W1; a.W[2] = W2; a.H = H; a.P = P; a.K = K;
  a.T = (int)((s + BM - 1) / BM);
  a.chain = (m == 2 || m == 3) && chain != nullptr && HX != nullptr ? m : 0;
  if (a.chain) {
    for (int i = 0; i < 4 * m; ++i) a.C[i] = chain[i];
    for (int i = 0; i < m - 1; ++i) a.HX[i] = HX[i];
    a.red_bias = 20;   // (c2 sweep: 0 / 10 / 20 / 35 / 50 -> 1.167 / 1.163 / 1.160 / 1.166 / 1.176 ms)
    if (const char* v = getenv("CPA_SVT_RED_BIAS")) a.red_bias = atoi(v);
  }
  const size_t smem = sym_smem();
  const int slots = sym_slots(num_sms);
  const bool pp = sym_use_pp(a.chain);
  a.split = pp ? sym_split_pp(s, num_sms, a.chain) : sym_split_mode(s, slots, a.chain);
  a.sync = sync;
  a.partial = partial;
  a.vec = aligned16(G, s) && aligned16(W0, s) && aligned16(W1, s) && aligned16(W2, s);
  // line 12 (Y = H_hat X, left side) folded into the m-chain launch (X rows 16-byte aligned for TMA)
  if (a.chain && X && Y && L > 0 && ldx % 2 == 0 && ((uintptr_t)X & 15) == 0 && !sym_use_pp(a.chain)) {
    a.l12 = 1;
    a.Y = Y;
    a.ldy = ldy;
    a.L = L;
    a.l12_tn = (int)((L + BN - 1) / BN);
    a.l12_split = sym_l12_split(s, L, num_sms);
    a.l12_partial = l12_partial;
    a.X = X;
    a.ldx = ldx;
  }
  cudaError_t e = cudaMemsetAsync(sync, 0, dense_sym_sync_ints(s, K, num_sms, a.l12 ? L : 0) * sizeof(int), st);
  if (e != cudaSuccess) return e;
  a.k0 = 2;
  if (a.chain && psi2_given) {   // Psi_2 formed by the init from the squaring's G^2: start at k = 3
    a.k0 = 3;
    k_sym_mark_step2<<<(a.T * (a.T + 1) / 2 + 255) / 256, 256, 0, st>>>(sync, K, a.T, a.chain,
                                                                          pp ? a.split : a.split - 1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  int cs = 0;
  if (const char* v = getenv("CPA_SVT_SYM_CLUSTER")) cs = atoi(v);
  if (a.split > 1 && (cs == 2 || cs == 4 || cs == 8) && !a.chain) {
    // small s: CS-CTA clusters, k-splits reduced through distributed shared memory
    auto go = [&](auto kern, int CS) -> cudaError_t {
      cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e2 != cudaSuccess) return e2;
      int64_t grid = (slots / CS) * CS;
      const int64_t tiles_total = (int64_t)(K - 2) * a.T * (a.T + 1) / 2 * CS;
      if (grid > tiles_total) grid = tiles_total;
      if (grid < CS) grid = CS;
      kern<<<(unsigned)grid, NTHREADS, smem, st>>>(a);
      return cudaGetLastError();
    };
    if (cs == 2) return go(k_cheb_sym_cl<2>, 2);
    if (cs == 4) return go(k_cheb_sym_cl<4>, 4);
    return go(k_cheb_sym_cl<8>, 8);
  }
  const int64_t total = (int64_t)(K - a.k0) * a.T * (a.T + 1) / 2 * a.split +
                        (a.l12 ? (int64_t)a.T * a.l12_tn * a.l12_split : 0);
  return sym_launch(a, total, slots, num_sms, st);
}

// The persistent symmetric-step kernel over `total` units: TMA-fed for even s (the cp.async
// kernel for odd s, whose rows are not 16-byte aligned).
static cudaError_t sym_launch(SymArgs& a, int64_t total, int slots, int num_sms, cudaStream_t st) {
  const int64_t s = a.s;
  const size_t smem = sym_smem();
  const int64_t grid = slots < total ? slots : total;
  cudaError_t e;
  if (!env_on("CPA_SVT_SYM_NOTMA") && s % 2 == 0 && s <= INT32_MAX / 2) {
    // one fp64 tensor map per operand (16 x 16 boxes, 128-byte swizzle)
    EncodeTiledFn fn = encode_fn();
    SymMapsChain mpc;
    SymMaps mp;
    bool ok = fn != nullptr;
    const int sbk = s >= 4096 ? 32 : 16;   // slab depth of the k_cheb_sym_tma instance (see there)
    const double* ops[16] = {a.G, a.W[0], a.W[1], a.W[2]};
    CUtensorMap* maps[16] = {&mpc.g, &mpc.w[0], &mpc.w[1], &mpc.w[2]};
    const int nmaps = 4 + 4 * a.chain;
    for (int i = 0; i < 4 * a.chain; ++i) {
      ops[4 + i] = a.C[i];
      maps[4 + i] = &mpc.c[i];
    }
    if (a.l12 && ok) {   // line 12 in the m-chain launch: H_hat (symmetric, as G) and X (s x L, ld)
      cuuint64_t hd[2] = {(cuuint64_t)s, (cuuint64_t)s}, hs[1] = {(cuuint64_t)(s * sizeof(double))};
      cuuint64_t xd[2] = {(cuuint64_t)a.L, (cuuint64_t)s}, xs[1] = {(cuuint64_t)(a.ldx * sizeof(double))};
      cuuint32_t box[2] = {16u, (cuuint32_t)sbk}, estr[2] = {1u, 1u};
      ok = fn(&mpc.h, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)a.H, hd, hs, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
               CUDA_SUCCESS &&
           fn(&mpc.x, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)a.X, xd, xs, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
               CUDA_SUCCESS;
      if (!ok) return cudaErrorInvalidValue;
    }
    for (int i = 0; i < nmaps && ok; ++i) {
      cuuint64_t dims[2] = {(cuuint64_t)s, (cuuint64_t)s};
      cuuint64_t strides[1] = {(cuuint64_t)(s * sizeof(double))};
      cuuint32_t box[2] = {16u, (cuuint32_t)sbk};
      cuuint32_t estr[2] = {1u, 1u};
      ok = fn(maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)ops[i], dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    mp.g = mpc.g;
    for (int i = 0; i < 3; ++i) mp.w[i] = mpc.w[i];
    if (ok && env_on("CPA_SVT_SYM_WS") && !a.panel && !a.chain) {
      // warp-specialized kernel: 3 x 16-deep (48 KB) or 2 x 32-deep (64 KB) ring + 64 KB staging, 2 CTAs per SM
      const size_t wsmem = (sbk == 32 ? (size_t)2 * 8 * (16 * 32 * 8) : (size_t)3 * 8 * (16 * 16 * 8)) +
                           (size_t)2 * BM * BN * 8 + 1024;   // (+ header and alignment: see k_cheb_sym_ws)
      auto kf = sbk == 32 ? k_cheb_sym_ws<32, 2> : k_cheb_sym_ws<16, 3>;
      e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
      if (e != cudaSuccess) return e;
      int dev = 0;
      cudaGetDevice(&dev);
      int per_sm = resident_ctas((const void*)kf, 2 * NTHREADS, wsmem, dev);
      if (env_on("CPA_SVT_DEBUG_OCC")) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, (const void*)kf);
        fprintf(stderr, "k_cheb_sym_ws: occupancy %d CTAs/SM, regs %d, static smem %zu, dyn %zu\n", per_sm, fa.numRegs,
                fa.sharedSizeBytes, wsmem);
      }
      int64_t tgrid = (int64_t)num_sms * per_sm;
      if (tgrid > total) tgrid = total;
      void* targs[] = {&mp, &a};
      return cudaLaunchCooperativeKernel((void*)kf, dim3((unsigned)tgrid), dim3(2 * NTHREADS), targs, wsmem, st);
    }
    if (ok) {
      // both instances use a 64 KB ring: 4 x 16-deep or 2 x 32-deep stages
      const size_t tsmem = (size_t)4 * 8 * (16 * 16 * 8) + 1024;
      const int nw = (getenv("CPA_SVT_SYM_NW") && atoi(getenv("CPA_SVT_SYM_NW")) == 8) ? 8 : 4;
      const void* kf =
          a.chain == 3 ? (sbk == 32 ? (const void*)k_cheb_sym_tma<32, 2, false, 4, 3>
                                    : (const void*)k_cheb_sym_tma<16, 4, false, 4, 3>)
          : a.chain == 2 ? (sbk == 32 ? (const void*)k_cheb_sym_tma<32, 2, false, 4, 2>
                                      : (const void*)k_cheb_sym_tma<16, 4, false, 4, 2>)
                  : (const void*)(nw == 8 ? (a.panel ? (sbk == 32 ? k_cheb_sym_tma<32, 2, true, 8> : k_cheb_sym_tma<16, 4, true, 8>)
                                     : (sbk == 32 ? k_cheb_sym_tma<32, 2, false, 8> : k_cheb_sym_tma<16, 4, false, 8>))
                          : (a.panel ? (sbk == 32 ? k_cheb_sym_tma<32, 2, true> : k_cheb_sym_tma<16, 4, true>)
                                     : (sbk == 32 ? k_cheb_sym_tma<32, 2, false> : k_cheb_sym_tma<16, 4, false>)));
      e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
      if (e != cudaSuccess) return e;
      int dev = 0;
      cudaGetDevice(&dev);
      const int per_sm = resident_ctas((const void*)kf, 32 * nw, tsmem, dev);
      if (env_on("CPA_SVT_DEBUG_OCC")) fprintf(stderr, "k_cheb_sym_tma<%d,NW=%d>: %d CTAs/SM\n", sbk, nw, per_sm);
      int64_t tgrid = (int64_t)num_sms * per_sm;
      if (tgrid > total) tgrid = total;
      void* targs[] = {a.chain ? (void*)&mpc : (void*)&mp, &a};
      if (a.chain && sym_use_pp(a.chain)) {
        // ping-pong: one 384-thread CTA per SM, two 64 KB rings + two 32 KB staging buffers
        // (16-deep slabs: 5 stages per ring by default -- two 80 KB rings and the staging fill the
        // 227 KB; CPA_SVT_PP_STAGES=4 for 64 KB rings; 32-deep slabs: 2 stages)
        const int pst = sbk == 32 ? 2 : (getenv("CPA_SVT_PP_STAGES") && atoi(getenv("CPA_SVT_PP_STAGES")) == 4 ? 4 : 5);
        const size_t psmem = PP_HDR + 1024 + 2 * (size_t)pst * 8 * (16 * sbk * 8) + 2 * BM * BN * 8;
        const void* pk =
            a.chain == 3 ? (sbk == 32 ? (const void*)k_cheb_sym_pp<32, 2, 3>
                                      : pst == 4 ? (const void*)k_cheb_sym_pp<16, 4, 3> : (const void*)k_cheb_sym_pp<16, 5, 3>)
                         : (sbk == 32 ? (const void*)k_cheb_sym_pp<32, 2, 2>
                                      : pst == 4 ? (const void*)k_cheb_sym_pp<16, 4, 2> : (const void*)k_cheb_sym_pp<16, 5, 2>);
        e = cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
        if (e != cudaSuccess) return e;
        int64_t pgrid = num_sms;
        if (env_on("CPA_SVT_DEBUG_OCC")) fprintf(stderr, "k_cheb_sym_pp<%d>: %d CTAs, smem %zu\n", sbk, (int)pgrid, psmem);
        return cudaLaunchCooperativeKernel((void*)pk, dim3((unsigned)pgrid), dim3(3 * NTHREADS), targs, psmem, st);
      }
      return cudaLaunchCooperativeKernel((void*)kf, dim3((unsigned)tgrid), dim3(32 * nw), targs, tsmem, st);
    }
  }
  if (a.chain) return cudaErrorInvalidValue;   // (two chains: TMA kernel only; dense_sym_use_chain)
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel(a.panel ? (void*)k_cheb_sym<true> : (void*)k_cheb_sym<false>, dim3((unsigned)grid),
                                     dim3(NTHREADS), args, smem, st);
}

// ---- panel mode (multi-GPU): one step on a contiguous range of lower tiles ------------
// Tiles of the column-major lower-triangle order are split in P contiguous, balanced ranges;
// rank p owns [panel_tile0(p), panel_tile0(p + 1)).
int64_t dense_sym_ntri(int64_t s) {
  const int64_t T = (s + BM - 1) / BM;
  return T * (T + 1) / 2;
}
int64_t dense_sym_panel_tile0(int64_t s, int p, int P) { return dense_sym_ntri(s) * p / P; }
int64_t dense_sym_panel_slot(int64_t s, int P) {   // tiles per all-gather slot (the largest range)
  const int64_t n = dense_sym_ntri(s);
  return (n + P - 1) / P;
}
size_t dense_sym_panel_partial_doubles(int64_t s, int P, int num_sms) {
  const int64_t nt = dense_sym_panel_slot(s, P);
  const int S = sym_split(s, sym_slots(num_sms), nt);
  return S > 1 ? (size_t)(nt * (S - 1) * BM * BN) : 0;
}

// Step kstep of the symmetric recurrence on tiles [tile0, tile0 + ntile): W_k (or, at the last
// step, H) of those tiles packed into gout (ntile x 64 x 64, row-major tiles).  W0..W2 / H as in
// dense_cheb_sym, with W_{kstep-1} and W_{kstep-2} complete (unpacked) on entry.
cudaError_t dense_cheb_sym_panel(int64_t s, const double* G, double* W0, double* W1, double* W2, double* H,
                                 const SeriesParams* P, int K, int kstep, int64_t tile0, int64_t ntile,
                                 double* gout, int* sync, double* partial, int num_sms, cudaStream_t st) {
  if (s == 0 || K <= 2 || ntile <= 0) return cudaSuccess;
  SymArgs a{};
  a.s = s; a.G = G; a.W[0] = W0; a.W[1] = W1; a.W[2] = W2; a.H = H; a.P = P; a.K = K;
  a.T = (int)((s + BM - 1) / BM);
  const int slots = sym_slots(num_sms);
  a.split = sym_split(s, slots, ntile);
  a.sync = sync;
  a.partial = partial;
  a.vec = aligned16(G, s) && aligned16(W0, s) && aligned16(W1, s) && aligned16(W2, s);
  a.panel = 1;
  a.kstep = kstep;
  a.tile0 = (int)tile0;
  a.ntile = (int)ntile;
  a.gout = gout;
  cudaError_t e = cudaMemsetAsync(sync, 0, dense_sym_sync_ints(s, K, num_sms, 0) * sizeof(int), st);
  if (e != cudaSuccess) return e;
  return sym_launch(a, ntile * a.split, slots, num_sms, st);
}

// Gathered slots -> full symmetric matrix: tile t (global column-major lower order) of owner p
// sits at g + (p * slot + t - tile0(p)) * 4096; element (r, c), r >= c, lands at (r, c) and
// (c, r).  One CTA per tile, the mirror written through a shared-memory transpose (coalesced).
__global__ void __launch_bounds__(256) k_sym_unpack(const double* __restrict__ g, int64_t s, int T, int P,
                                                    int64_t ntri, int64_t slot, double* __restrict__ out) {
  __shared__ double tile_s[BM][BN + 1];
  const int64_t t = blockIdx.x;
  int p = (int)(t * P / ntri);
  while (p + 1 < P && (ntri * (p + 1)) / P <= t) ++p;
  while (p > 0 && (ntri * p) / P > t) --p;
  const int64_t lt = t - (ntri * p) / P;
  CPA_DCHECK(p >= 0 && p < P && lt >= 0 && lt < slot && (ntri * p) / P <= t && t < (ntri * (p + 1)) / P);
  const double* src = g + ((int64_t)p * slot + lt) * (BM * BN);
  int ti, tj;
  tri_decode_colmajor((int)t, T, ti, tj);
  const int64_t m0 = (int64_t)ti * BM, n0 = (int64_t)tj * BN;
  for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
    const int r = e / BN, c = e % BN;
    const double v = __ldcs(src + e);
    tile_s[r][c] = v;
    const int64_t rr = m0 + r, cc = n0 + c;
    if (rr < s && cc < s && (ti != tj || r >= c)) out[rr * s + cc] = v;
  }
  __syncthreads();
  // mirror: out[(n0 + c) * s + m0 + r] = tile(r, c), rows of the transposed tile contiguous
  for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
    const int c = e / BM, r = e % BM;
    const int64_t rr = m0 + r, cc = n0 + c;
    if (rr < s && cc < s && (ti != tj || r > c)) out[cc * s + rr] = tile_s[r][c];
  }
}

cudaError_t dense_sym_unpack(const double* gbuf, int64_t s, int P, double* out, cudaStream_t st) {
  const int64_t ntri = dense_sym_ntri(s);
  if (ntri == 0) return cudaSuccess;
  k_sym_unpack<<<(unsigned)ntri, 256, 0, st>>>(gbuf, s, (int)((s + BM - 1) / BM), P, ntri,
                                              dense_sym_panel_slot(s, P), out);
  return cudaGetLastError();
}

// ---- NEXT-2: one-level Haar DWT of the Gram index (reading R22)
// A = X (left, Gram index = rows) or X^T (right, Gram index = columns); s = Gram side,
// nh = s / 2 pairs, nl = s - nh low-pass coefficients (odd s: the last sample is its own).
//   split:   A_L[i] = (A[2i] + A[2i+1]) / sqrt 2,  A_H[i] = (A[2i] - A[2i+1]) / sqrt 2
//   combine: Y[2i] = (Y_L[i] + h0 A_H[i]) / sqrt 2,  Y[2i+1] = (Y_L[i] - h0 A_H[i]) / sqrt 2,
//            h0 = h_hat(0) = c_0/2 + sum_k c_k (-1)^k  (the series on the zeroed high band)
// Layout: left: A_L nl x n, A_H nh x n (ld n); right: A_L m x nl (ld nl), A_H m x nh (ld nh).
constexpr double kRsqrt2 = 0.70710678118654752440;

__global__ void k_haar_split(const double* __restrict__ X, int64_t m, int64_t n, int64_t ldx, int left,
                             double* __restrict__ AL, double* __restrict__ AH) {
  const int64_t s = left ? m : n, nh = s / 2, nl = s - nh, L = left ? n : m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nl * L; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i, l;  // i: low-pass index, l: position along the long side
    if (left) { i = e / L; l = e % L; } else { l = e / nl; i = e % nl; }
    auto x = [&](int64_t g) { return left ? X[g * ldx + l] : X[l * ldx + g]; };
    double lo, hi = 0.0;
    if (i < nh) {
      const double a = x(2 * i), b = x(2 * i + 1);
      lo = (a + b) * kRsqrt2;
      hi = (a - b) * kRsqrt2;
    } else {
      lo = x(s - 1);
    }
    if (left) {
      AL[i * L + l] = lo;
      if (i < nh) AH[i * L + l] = hi;
    } else {
      AL[l * nl + i] = lo;
      if (i < nh) AH[l * nh + i] = hi;
    }
  }
}

__global__ void k_haar_combine(const double* __restrict__ YL, const double* __restrict__ AH,
                               const SeriesParams* __restrict__ P, int64_t m, int64_t n, int left,
                               double* __restrict__ Y, int64_t ldy) {
  __shared__ double s_h0;
  if (threadIdx.x == 0) {
    double h0 = 0.5 * P->c[0];
    for (int k = 1; k < P->K; ++k) h0 += (k & 1) ? -P->c[k] : P->c[k];
    s_h0 = h0;
  }
  __syncthreads();
  const double h0 = s_h0;
  const int64_t s = left ? m : n, nh = s / 2, nl = s - nh, L = left ? n : m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s * L; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t g, l;  // g: Gram index, l: long-side position
    if (left) { g = e / L; l = e % L; } else { l = e / s; g = e % s; }
    const int64_t i = g / 2;
    double v;
    if (i >= nh) {
      v = left ? YL[(nl - 1) * L + l] : YL[l * nl + (nl - 1)];
    } else {
      const double lo = left ? YL[i * L + l] : YL[l * nl + i];
      const double hi = h0 * (left ? AH[i * L + l] : AH[l * nh + i]);
      v = ((g & 1) ? lo - hi : lo + hi) * kRsqrt2;
    }
    if (left) Y[g * ldy + l] = v; else Y[l * ldy + g] = v;
  }
}

cudaError_t dense_haar_split(const double* X, int64_t m, int64_t n, int64_t ldx, bool left, double* AL, double* AH,
                             int num_sms, cudaStream_t st) {
  k_haar_split<<<num_sms * 8, 256, 0, st>>>(X, m, n, ldx, left ? 1 : 0, AL, AH);
  return cudaGetLastError();
}
cudaError_t dense_haar_combine(const double* YL, const double* AH, const SeriesParams* P, int64_t m, int64_t n,
                               bool left, double* Y, int64_t ldy, int num_sms, cudaStream_t st) {
  k_haar_combine<<<num_sms * 8, 256, 0, st>>>(YL, AH, P, m, n, left ? 1 : 0, Y, ldy);
  return cudaGetLastError();
}

}  // namespace cpa

#ifdef CPA_SYM_TRACE
extern "C" int cpa_svt_debug_sym_trace(void* host_out, int64_t units) {
  if (units > cpa::kTraceUnits) units = cpa::kTraceUnits;
  return (int)cudaMemcpyFromSymbol(host_out, cpa::g_trace, (size_t)units * 6 * sizeof(uint64_t));
}
#endif
