// Small fp64 problems (s <= 64, L <= 128; BASELINE configs[0] is 64 x 48): the whole of
// Algorithm 1 in ONE thread block of 4 warps, every operand in shared
// memory (64 x 64 padded, leading dimension 68: conflict-free DMMA fragments).  The grid
// path spends ~10 us per recurrence step on one 64 x 64 tile (ticket, dependency wait, TMA
// prologue and epilogue of a grid-wide dataflow); here a step is one DMMA.8x8x4 product of
// the block (each warp a 32 x 32 quarter) and a barrier.
//
//   line 1   G = A A^T from At = A^T (left: A = X, right: A = X^T)
//   line 3   power iteration, T products (reading R6), squared as on the grid path:
//            q products by c^p G^p (p = 2^j, c = 2^-ilogb(max G_ii)), the rest by G;
//            lambda_hat = ||G v_{T-1}||
//   line 4   compute_series (series.cuh)
//   5 - 11   W_1 = (2/L) G - I, H = c_0/2 I + c_1 W_1;  W_k = 2 (2/L) G W_{k-1} - 2 W_{k-1} - W_{k-2},
//            H += c_k W_k  (the s x s form, reading R19)
//   line 12  P = H A: left Y = P, right Y = P^T
// Sums run in fixed orders (deterministic).
#include <algorithm>

#include "common.cuh"
#include "series.cuh"

namespace cpa {

struct SmallArgs {
  const double* X;
  int64_t ldx;
  double* Y;
  int64_t ldy;
  int m, n;
  SeriesParams* P;
  cpa_svt_kernel kern;
  int K, T;
  double safety;
  double lam_override;   // > 0: Lambda given, no power iteration
  const double* c_given; // device, nullable
  int nsq;               // squarings before the power iteration
  int check;             // SPEC.md:215 divergence check folded in (check.cu's rule): ||Y|| vs 1e3 sum|c_k| ||X||
  int chain;             // two Chebyshev chains (R28) with Psi_2 from the first squaring (R29): one more buffer
};

constexpr int SM_THREADS = 128;   // 4 warps: one 32 x 32 quarter of a 64 x 64 DMMA tile each
constexpr int LDP = 68;           // padded leading dimension of the s x s operands (conflict-free fragments)

__device__ __forceinline__ double warp_sum_s(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// The block's output tile is (16h x 16h) for h = ceil(ceil(s / 8) / 2) <= 4 8 x 8 DMMA tiles per
// warp and dimension: warp w covers rows wm = 8h (w / 2) and columns wn = 8h (w % 2) of it, so
// the four warps split the s x s products evenly (s = 48: 3 x 3 tiles each, no padding work).
// acc = A * B over k < kd on DMMA.8x8x4: A stored k-major (element (m, k) at A[k * lda + m]),
// B stored k-major (element (k, n) at B[k * ldb + n]); rows / columns / k beyond the operands'
// extent are zero in shared memory.  acc[i][j][e] (i, j < h) holds
// C(wm + 8i + g, n0 + wn + 8j + 2t + e).
template <int h>
__device__ __forceinline__ void dmma_tile(const double* A, int lda, const double* B, int ldb, int kd, int n0,
                                          double (&acc)[4][4][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 8 * h, wn = (warp & 1) * 8 * h;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < kd; kk += 4) {
    double fa[4], fb[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) fa[i] = i < h ? A[(kk + t) * lda + wm + i * 8 + g] : 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) fb[j] = j < h ? B[(kk + t) * ldb + n0 + wn + j * 8 + g] : 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i < h && j < h) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
  }
}

// C (padded, ld LDP) = scale * A B for symmetric s x s operands (stored row-major, which is the
// k-major form of a symmetric matrix).  C aliases neither A nor B.
template <int h>
__device__ __forceinline__ void sq_product(const double* A, const double* B, double* C, int s, double scale) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 8 * h, wn = (warp & 1) * 8 * h;
  double acc[4][4][2];
  dmma_tile<h>(A, LDP, B, LDP, (s + 3) & ~3, 0, acc);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (i < h && j < h)
#pragma unroll
        for (int e = 0; e < 2; ++e) C[(wm + i * 8 + g) * LDP + wn + j * 8 + 2 * t + e] = acc[i][j][e] * scale;
  __syncthreads();
}

template <int h>   // 8 x 8 DMMA tiles per warp and dimension: ceil(ceil(s / 8) / 2)
__global__ void __launch_bounds__(SM_THREADS, 1) k_small_f64(SmallArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double s_red[SM_THREADS / 32];
  __shared__ double s_v[64], s_u[64];
  __shared__ double s_scal[2];
  const bool left = a.m <= a.n;
  const int s = left ? a.m : a.n, L = left ? a.n : a.m;
  const int kL = (L + 3) & ~3, ldt = LDP, lda = ((L + 3) & ~3) + 4;
  double* G = sm;                  // 64 x LDP each, zero outside s x s
  double* Gp = G + 64 * LDP;       // c^p G^p, then H
  double* Wa = Gp + 64 * LDP;
  double* Wb = Wa + 64 * LDP;
  double* Op = Wb + 64 * LDP;      // At (kL x LDP: k-major A^T) for line 1, A (64 x lda) for line 12
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3, wm = (warp >> 1) * 8 * h, wn = (warp & 1) * 8 * h;
#ifdef CPA_SMALL_TRACE
  long long stamp[8];
  int ns = 0;
  stamp[ns++] = clock64();
#define STAMP() stamp[ns++] = clock64()
#else
#define STAMP()
#endif
  for (int e = tid; e < 4 * 64 * LDP; e += SM_THREADS) sm[e] = 0.0;
  // ---- At(l, i) = A(i, l): right A = X^T so At = X (L = m rows); left A = X so At = X^T
  for (int e = tid; e < kL * ldt; e += SM_THREADS) {
    const int r = e / ldt, c = e % ldt;
    double v = 0.0;
    if (r < L && c < s) v = left ? a.X[(int64_t)c * a.ldx + r] : a.X[(int64_t)r * a.ldx + c];
    Op[e] = v;
  }
  __syncthreads();
  // ---- line 1: G = A A^T: G(i, j) = sum_l At(l, i) At(l, j)
  {
    double acc[4][4][2];
    dmma_tile<h>(Op, ldt, Op, ldt, kL, 0, acc);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i < h && j < h)
#pragma unroll
          for (int e = 0; e < 2; ++e) G[(wm + i * 8 + g) * LDP + wn + j * 8 + 2 * t + e] = acc[i][j][e];
  }
  __syncthreads();
  STAMP();
  // ---- line 3: power iteration
  double lam = 0.0;
  if (a.lam_override > 0.0) {
    lam = a.lam_override / a.safety;
  } else {
    int p = 1, q = 0;
    if (a.nsq > 0) {
      if (tid == 0) {
        double mx = 0.0;
        for (int i = 0; i < s; ++i) mx = fmax(mx, G[i * LDP + i]);
        const int e = (mx > 0.0 && isfinite(mx)) ? ilogb(mx) : 0;
        s_scal[0] = ldexp(1.0, -2 * e);   // c^2, exact
      }
      __syncthreads();
      sq_product<h>(G, G, Gp, s, s_scal[0]);          // c^2 G^2
      if (a.chain) {                                  // (kept for Psi_2: Wb is free until the recurrence)
        for (int e = tid; e < 64 * LDP; e += SM_THREADS) Wb[e] = Gp[e];
        __syncthreads();
      }
      p = 2;
      for (int j = 1; j < a.nsq && 2 * p <= a.T - 1; ++j) {
        sq_product<h>(Gp, Gp, Wa, s, 1.0);            // c^{2p} G^{2p}
        for (int e = tid; e < 64 * LDP; e += SM_THREADS) Gp[e] = Wa[e];
        __syncthreads();
        p *= 2;
      }
      q = (a.T - 1) / p;
    }
    const int niter = a.T - (p - 1) * q;
    for (int i = tid; i < 64; i += SM_THREADS) s_v[i] = i < s ? 1.0 / sqrt((double)s) : 0.0;
    __syncthreads();
    bool degenerate = false;
    for (int it = 0; it < niter; ++it) {
      const double* M = it < q ? Gp : G;
      double u = 0.0;
      if (tid < s)
        for (int l = 0; l < s; ++l) u = fma(M[tid * LDP + l], s_v[l], u);
      if (tid < 64) s_u[tid] = u;
      const double sq = warp_sum_s(u * u);
      if (lane == 0) s_red[warp] = sq;
      __syncthreads();
      if (tid == 0) {
        double tot = 0.0;
        for (int w = 0; w < SM_THREADS / 32; ++w) tot += s_red[w];
        s_scal[1] = sqrt(tot);
      }
      __syncthreads();
      lam = s_scal[1];
      if (!(lam > kDegenerateLambda) || !(lam < 1e300)) { degenerate = true; break; }
      if (tid < s) s_v[tid] = s_u[tid] / lam;
      __syncthreads();
    }
    if (degenerate) lam = lam < 1e300 ? 0.0 : lam;
  }
  STAMP();
  // ---- line 4
  compute_series(a.P, a.kern, a.K, a.safety, lam, a.c_given);
  __syncthreads();
  STAMP();
  const double s2 = a.P->scale2, s4 = 2.0 * s2;
  double* H = Gp;
  const int ks = (s + 3) & ~3;
  if (a.chain && a.K >= 4 && a.lam_override <= 0.0 && a.nsq > 0) {
    // ---- two chains (R28): Psi_1 (Wa), Psi_2 = 2 s2^2 G^2 - 4 s2 G + I from the squaring's c^2 G^2
    //      (R29, over G), H = c0/2 I + c1 Psi_1 + c2 Psi_2; then the products in pairs
    //      Psi_k = 2 Psi_2 Psi_{k-2} - Psi_{|k-4|} (k odd, k + 1 even) sharing the A fragments of
    //      Psi_2: twice the independent DMMAs per barrier.  Odd chain in Wa / Wb, even in E1 / E2
    //      (E2 = the operand buffer, free until line 12); Psi_k over Psi_{k-4}, own elements.
    const double c2inv = 1.0 / s_scal[0];
    double* P2 = G;
    const int opn = max(max(kL * LDP, 64 * (((L + 63) & ~63) + 4)), 64 * LDP);   // small_f64_smem's op
    double* E1 = Op + opn + 64;       // the extra buffer (small_f64_smem with chains)
    double* E2 = Op;
    for (int e = tid; e < 64 * LDP; e += SM_THREADS) {
      const int r = e / LDP, c = e % LDP;
      const bool in = r < s && c < s;
      const double id = (r == c && r < s) ? 1.0 : 0.0;
      const double gg = G[e];
      const double w1 = in ? s2 * gg - id : 0.0;
      const double p2 = in ? 2.0 * s2 * s2 * (Wb[e] * c2inv) - 2.0 * s4 * gg + id : 0.0;
      Wa[e] = w1;
      P2[e] = p2;
      H[e] = 0.5 * a.P->c[0] * id + a.P->c[1] * w1 + a.P->c[2] * p2;
      E1[e] = 0.0;
      E2[e] = 0.0;
    }
    __syncthreads();
    auto ebuf = [&](int k) { return k == 2 ? P2 : (((k - 4) >> 1) & 1) ? E2 : E1; };   // even k >= 2
    auto obuf = [&](int k) { return (((k - 1) >> 1) & 1) ? Wb : Wa; };                // odd k >= 1
    for (int k = 3; k < a.K; k += 2) {
      const bool two = k + 1 < a.K;   // the pair (k odd, k + 1 even); the last may be single
      const double* Bo = obuf(k - 2);
      const double* Be = ebuf(k - 1);   // (k + 1) - 2
      double acc_o[4][4][2], acc_e[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc_o[i][j][0] = acc_o[i][j][1] = acc_e[i][j][0] = acc_e[i][j][1] = 0.0;
#pragma unroll 2
      for (int kk = 0; kk < ks; kk += 4) {
        double fa[4], fo[4], fe[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) fa[i] = i < h ? P2[(kk + t) * LDP + wm + i * 8 + g] : 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          fo[j] = j < h ? Bo[(kk + t) * LDP + wn + j * 8 + g] : 0.0;
          fe[j] = (j < h && two) ? Be[(kk + t) * LDP + wn + j * 8 + g] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (i < h && j < h) {
              dmma_8x8x4(acc_o[i][j][0], acc_o[i][j][1], fa[i], fo[j]);
              if (two) dmma_8x8x4(acc_e[i][j][0], acc_e[i][j][1], fa[i], fe[j]);
            }
      }
      const double cko = a.P->c[k], cke = two ? a.P->c[k + 1] : 0.0;
      double* Oo = obuf(k);                       // Psi_k over Psi_{k-4} (k = 3: a fresh buffer)
      const double* Qo = obuf(k == 3 ? 1 : k - 4);
      double* Oe = ebuf(k + 1);
      const double* Qe = (k + 1) == 4 ? nullptr : ebuf(k - 3);   // Psi_{k+1-4} (Psi_0 = I at k + 1 = 4)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (i < h && j < h)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int r = wm + i * 8 + g, c = wn + j * 8 + 2 * t + e, o = r * LDP + c;
              const double wo = 2.0 * acc_o[i][j][e] - Qo[o];
              double hv = H[o] + cko * wo;
              Oo[o] = wo;                                                // (read only by this thread)
              if (two) {
                const double q = Qe ? Qe[o] : ((r == c && r < s) ? 1.0 : 0.0);
                const double we = 2.0 * acc_e[i][j][e] - q;
                Oe[o] = we;
                hv += cke * we;
              }
              H[o] = hv;
            }
      __syncthreads();
    }
  } else {
  // ---- lines 5-7: W_1 (Wa), H (Gp), zero outside s x s
  for (int e = tid; e < 64 * LDP; e += SM_THREADS) {
    const int r = e / LDP, c = e % LDP;
    const double id = (r == c && r < s) ? 1.0 : 0.0;
    const double w = (r < s && c < s) ? s2 * G[e] - id : 0.0;
    Wa[e] = w;
    H[e] = 0.5 * a.P->c[0] * id + a.P->c[1] * w;
  }
  __syncthreads();
  // ---- lines 8-11: W_k = s4 G W_{k-1} - 2 W_{k-1} - W_{k-2} over W_{k-2}, H += c_k W_k
  double* Wp = Wa;   // W_{k-1}
  double* Wq = Wb;   // W_{k-2} (k = 2: the identity, implicit)
  for (int k = 2; k < a.K; ++k) {
    double acc[4][4][2];
    dmma_tile<h>(G, LDP, Wp, LDP, ks, 0, acc);
    const double ck = a.P->c[k];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i < h && j < h)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = wm + i * 8 + g, c = wn + j * 8 + 2 * t + e, o = r * LDP + c;
          const double wpp = k == 2 ? ((r == c && r < s) ? 1.0 : 0.0) : Wq[o];
          const double w = s4 * acc[i][j][e] - 2.0 * Wp[o] - wpp;   // W_k = 2 B_hat W_{k-1} - W_{k-2}
          Wq[o] = w;                                                   // (read only by this thread)
          H[o] += ck * w;                                              // H += c_k W_k
        }
    __syncthreads();
    double* tmp = Wp;
    Wp = Wq;
    Wq = tmp;
  }
  }
  STAMP();
  // ---- line 12: P = H A (s x L; A(k, n) k-major = row-major A), right Y = P^T, left Y = P
  double xsq = 0.0, ysq = 0.0;   // divergence check: this thread's sums of squares of X and Y
  for (int e = tid; e < 64 * lda; e += SM_THREADS) {
    const int r = e / lda, c = e % lda;
    double v = 0.0;
    if (r < s && c < L) v = left ? a.X[(int64_t)r * a.ldx + c] : a.X[(int64_t)c * a.ldx + r];
    Op[e] = v;
    xsq = fma(v, v, xsq);
  }
  __syncthreads();
  for (int n0 = 0; n0 < L; n0 += 16 * h) {
    double acc[4][4][2];
    dmma_tile<h>(H, LDP, Op, lda, ks, n0, acc);   // H symmetric: k-major H = row-major H
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i < h && j < h)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = wm + i * 8 + g, c = n0 + wn + j * 8 + 2 * t + e;
          if (r < s && c < L) {
            if (left) a.Y[(int64_t)r * a.ldy + c] = acc[i][j][e];
            else      a.Y[(int64_t)c * a.ldy + r] = acc[i][j][e];
            ysq = fma(acc[i][j][e], acc[i][j][e], ysq);
          }
        }
  }
  if (a.check) {   // fixed-order block sums (warp butterflies, then warps in order): deterministic
    __shared__ double s_chk[2][SM_THREADS / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      xsq += __shfl_xor_sync(0xffffffffu, xsq, o);
      ysq += __shfl_xor_sync(0xffffffffu, ysq, o);
    }
    if ((tid & 31) == 0) {
      s_chk[0][tid >> 5] = xsq;
      s_chk[1][tid >> 5] = ysq;
    }
    __syncthreads();
    if (tid == 0) {
      double sx = 0.0, sy = 0.0, cs = 0.0;
      for (int w = 0; w < SM_THREADS / 32; ++w) {
        sx += s_chk[0][w];
        sy += s_chk[1][w];
      }
      for (int k = 0; k < a.P->K; ++k) cs += fabs(a.P->c[k]);
      a.P->diverged = (a.P->degenerate || sqrt(sy) <= 1e3 * cs * sqrt(sx)) ? 0 : 1;
    }
  }
#ifdef CPA_SMALL_TRACE
  __syncthreads();
  STAMP();
  if (tid == 0)
    for (int i = 0; i < ns; ++i) a.Y[i] = (double)(stamp[i] - stamp[0]);
#endif
#undef STAMP
}

size_t small_f64_smem(int64_t m, int64_t n, bool chain) {
  const int64_t s = m < n ? m : n, L = m < n ? n : m;
  const int64_t kL = (L + 3) / 4 * 4, ncol = (L + 63) / 64 * 64;
  const int64_t op = std::max(std::max(kL * LDP, 64 * (ncol + 4)), chain ? (int64_t)64 * LDP : (int64_t)0);   // At for line 1 / A for line 12 (/ E2)
  (void)s;
  // (+64: line-12 fragment reads past the last row; chains: one more s x s buffer after Op)
  return (size_t)((4 + (chain ? 1 : 0)) * 64 * LDP + op + 64) * sizeof(double);
}
bool small_f64_fits(int64_t m, int64_t n) {
  const int64_t s = m < n ? m : n, L = m < n ? n : m;
  return s >= 1 && s <= 64 && L <= 128 && small_f64_smem(m, n, false) <= 220 * 1024;
}

// two chains when the extra buffer fits (CPA_SVT_SMALL_CHAIN=0: the one-chain recurrence)
static bool small_f64_chain_buf(int64_t m, int64_t n) {
  const char* e = getenv("CPA_SVT_SMALL_CHAIN");
  return small_f64_smem(m, n, true) <= 220 * 1024 && !(e && atoi(e) == 0);
}

// recurrence products the kernel performs: K - 3 with the chains (Psi_2 from the squaring), else K - 2
int small_f64_products(int64_t m, int64_t n, int K, int nsq, double lam_override) {
  const bool ch = small_f64_chain_buf(m, n) && K >= 4 && !(lam_override > 0.0) && nsq > 0;
  return K < 2 ? 0 : ch ? K - 3 : K - 2;
}

cudaError_t launch_small_f64(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t m, int64_t n,
                             SeriesParams* P, const cpa_svt_kernel& k, int K, int T, double safety,
                             double lam_override, const double* c_given, int nsq, cudaStream_t st, int check) {
  SmallArgs a{};
  a.check = check;
  a.X = X; a.ldx = ldx; a.Y = Y; a.ldy = ldy; a.m = (int)m; a.n = (int)n;
  a.P = P; a.kern = k; a.K = K; a.T = T; a.safety = safety; a.lam_override = lam_override;
  a.c_given = c_given; a.nsq = nsq;
  a.chain = small_f64_chain_buf(m, n);
  const size_t smem = small_f64_smem(m, n, a.chain != 0);
  const int64_t s = m < n ? m : n;
  const int h = (int)(((s + 7) / 8 + 1) / 2);
  auto kf = h == 1 ? k_small_f64<1> : h == 2 ? k_small_f64<2> : h == 3 ? k_small_f64<3> : k_small_f64<4>;
  cudaError_t e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kf<<<1, SM_THREADS, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cpa
