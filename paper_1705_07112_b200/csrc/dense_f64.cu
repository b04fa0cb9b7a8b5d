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
#include "common.cuh"

namespace cpa {

constexpr int BM = 64, BN = 64, BKS = 16, STAGES = 4, NTHREADS = 128;
constexpr int PAD = 4;

enum EpiMode { EPI_GRAM = 0, EPI_INIT = 1, EPI_STEP = 2 };

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
// [0, olim) x [0, ilim) are zero-filled.
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
      cp_async8(dst, orow && gi < ilim ? src : g, orow && gi < ilim);
      cp_async8(dst + 1, orow && gi + 1 < ilim ? src + 1 : g, orow && gi + 1 < ilim);
    }
  }
}

template <bool A_KC, bool B_KC, int MODE>
__global__ void __launch_bounds__(NTHREADS) k_dmma_gemm(GemmArgs a) {
  using LA = OpLayout<A_KC, BM>;
  using LB = OpLayout<B_KC, BN>;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * LA::SIZE;

  int tm, tn;
  if (MODE == EPI_GRAM) {
    // lower-triangular tile (tm >= tn) from the linear block index
    const int b = blockIdx.x;
    int r = (int)((sqrt(8.0 * b + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= b) ++r;
    while (r * (r + 1) / 2 > b) --r;
    tm = r;
    tn = b - r * (r + 1) / 2;
  } else {
    tm = blockIdx.x;
    tn = blockIdx.y;
  }
  const int64_t m0 = (int64_t)tm * BM, n0 = (int64_t)tn * BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (int)((a.Kd + BKS - 1) / BKS);
  auto load_stage = [&](int kt, int st) {
    const int64_t k0 = (int64_t)kt * BKS;
    if (A_KC) load_slab<LA>(sA + st * LA::SIZE, a.A, a.lda, m0, k0, a.M, a.Kd, a.vec_a);
    else      load_slab<LA>(sA + st * LA::SIZE, a.A, a.lda, k0, m0, a.Kd, a.M, a.vec_a);
    if (B_KC) load_slab<LB>(sB + st * LB::SIZE, a.B, a.ldb, n0, k0, a.N, a.Kd, a.vec_b);
    else      load_slab<LB>(sB + st * LB::SIZE, a.B, a.ldb, k0, n0, a.Kd, a.N, a.vec_b);
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

  // ---------------- epilogue -------------------------------------------------
  if (MODE == EPI_GRAM) {
    double* G = a.Wout;
    const int64_t ld = a.ldwo;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t r = m0 + wm + i * 8 + g, c = n0 + wn + j * 8 + 2 * t + e;
          if (r < a.M && c < a.N && r >= c) {
            G[r * ld + c] = acc[i][j][e];
            G[c * ld + r] = acc[i][j][e];
          }
        }
    return;
  }
  const SeriesParams* P = a.P;
  const double s2 = P->scale2;
  if (MODE == EPI_INIT) {
    const double h0 = 0.5 * P->c[0], c1 = P->c[1];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t r = m0 + wm + i * 8 + g, c = n0 + wn + j * 8 + 2 * t + e;
          if (r < a.M && c < a.N) {
            const double x = a.Wp[r * a.ldwp + c];
            const double w = s2 * acc[i][j][e] - x;          // W_1 = B_hat X
            if (a.Wout) a.Wout[r * a.ldwo + c] = w;
            a.Y[r * a.ldy + c] = h0 * x + c1 * w;           // Y = c0/2 W_0 + c1 W_1
          }
        }
  } else {
    const double s4 = 2.0 * s2, ck = P->c[a.k];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t r = m0 + wm + i * 8 + g, c = n0 + wn + j * 8 + 2 * t + e;
          if (r < a.M && c < a.N) {
            const double wp = a.Wp[r * a.ldwp + c];
            const double wpp = a.Wpp[r * a.ldwpp + c];
            const double w = s4 * acc[i][j][e] - 2.0 * wp - wpp;  // W_k = 2 B_hat W_{k-1} - W_{k-2}
            if (a.Wout) a.Wout[r * a.ldwo + c] = w;
            a.Y[r * a.ldy + c] += ck * w;                      // Y += c_k W_k
          }
        }
  }
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
  if (MODE == EPI_GRAM) grid = dim3((unsigned)(tm * (tm + 1) / 2));
  else grid = dim3((unsigned)tm, (unsigned)tn);
  fn<<<grid, NTHREADS, smem, st>>>(a);
  return cudaGetLastError();
}

static inline bool aligned16(const void* p, int64_t ld) {
  return ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && (ld % 2 == 0);
}

// G (s x s, ld s) = X X^T (left, s = m) or X^T X (right, s = n); X m x n row-major.
cudaError_t dense_gram_f64(const double* X, int64_t m, int64_t n, int64_t ldx, bool left, double* G,
                           cudaStream_t st) {
  GemmArgs a{};
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

}  // namespace cpa
