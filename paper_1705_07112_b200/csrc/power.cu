// Lambda_max by power iteration (Alg. 1 line 3; reading R6) and
// the Chebyshev coefficients (Alg. 1 line 4, PAPER.md:363 / eq. 233), both on
// the device so the recurrence never waits for the host.
//
// k_power_dense: one cooperative persistent launch for all T products.  Each
// CTA owns a contiguous block of Gram rows (cached in shared memory when they
// fit), stages v_{t-1} in shared memory, computes its rows of u_t = G v_{t-1}
// with one warp per row and publishes them as flag-carrying LL words; every CTA
// gathers the whole u_t by spinning on those words (no grid barrier).  ||u_t||
// is re-summed by every CTA in the same fixed order, so all CTAs agree bitwise.
// After the last product CTA 0 computes the coefficients.
#include <cstdlib>

#ifndef CPA_POLL_WARPS
#define CPA_POLL_WARPS 4
#endif

#include "common.cuh"
#include "series.cuh"

namespace cpa {

// lam_hat from *lam_src if non-null, else lam_override / safety.
__global__ void k_series(SeriesParams* P, cpa_svt_kernel kern, int K, double safety, double lam_override,
                         const double* lam_src, const double* c_given) {
  const double lh = lam_src ? *lam_src : lam_override / safety;
  compute_series(P, kern, K, safety, lh, c_given);
}

template <typename E>
struct PowerArgs {
  const E* G;
  const E* G4;       // c^p G^p (nullable): first q products use it
  int q;             // products by G4
  int pw;            // p = 2^j, the power G4 holds
  int poll;          // polling lanes of the LL gather
  int64_t s;
  int64_t ld;        // row stride of G / G4 (elements)
  int T;
  unsigned long long* ll;  // 2 (parity) * s * 2 LL words, zeroed before the launch
  SeriesParams* P;
  cpa_svt_kernel kern;
  int K;
  double safety;
  const double* c_given;
  int cache_rows;    // 1: this CTA's rows of G live in shared memory
  int rows_per_cta;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// LL ("low-latency") exchange words: an 8-byte store is single-copy atomic, so a
// word carrying 32 data bits next to a 32-bit epoch flag is valid exactly when the
// reader sees the flag of the epoch it waits for.  A double travels as two words.
__device__ __forceinline__ void st_ll(unsigned long long* p, double v, unsigned flag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = ((unsigned long long)flag << 32) | (b >> 32);
  const unsigned long long w1 = ((unsigned long long)flag << 32) | (b & 0xffffffffull);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ void ld_ll(const unsigned long long* p, unsigned long long& w0, unsigned long long& w1) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}

// Gather the s LL-encoded doubles of epoch `flag` into shared memory dst.  Only
// the first CPA_POLL_WARPS warps poll (every thread of every CTA spinning on the
// same lines stalls the whole exchange for ~10 us -- measured); each polling lane
// keeps 8 words in flight and re-issues only the late ones.  Ends with a CTA barrier.
__device__ __forceinline__ void ll_gather(const unsigned long long* buf, int64_t s, unsigned flag, double* dst,
                                          int np = 32 * CPA_POLL_WARPS) {
  const int NP = np;
  if (threadIdx.x < NP) {
    const int pl = threadIdx.x;
    for (int64_t j0 = 0; j0 < s; j0 += NP * 8) {
      unsigned long long w[8][2];
      unsigned pending = 0;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (j0 + pl + NP * c < s) pending |= 1u << c;
      while (pending) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (pending & (1u << c)) ld_ll(buf + 2 * (j0 + pl + NP * c), w[c][0], w[c][1]);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if ((pending & (1u << c)) && (unsigned)(w[c][0] >> 32) == flag && (unsigned)(w[c][1] >> 32) == flag)
            pending &= ~(1u << c);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (j0 + pl + NP * c < s)
          dst[j0 + pl + NP * c] =
              __longlong_as_double((long long)(((w[c][0] & 0xffffffffull) << 32) | (w[c][1] & 0xffffffffull)));
    }
  }
  __syncthreads();
}

// One persistent (cooperative) launch for all T products.  Product t: every CTA
// computes its rows of u_t = G v_{t-1} (one warp per row) and publishes them as LL
// words with flag t+1 in buffer t&1; every CTA then reads the whole u_t, spinning
// per word until its flag arrives -- the data and its readiness travel together,
// so there is no grid barrier and no separate flag round trip.  Buffer t&1 is
// rewritten at t+2 only by a CTA that has read all of u_{t+1}, which every CTA
// publishes after reading all of u_t.  ||u_t|| is re-summed by every CTA in the
// same fixed order from the staged copy, so all CTAs agree bitwise.
template <typename E>
__global__ void __launch_bounds__(256) k_power_dense(PowerArgs<E> a) {
  using T = E;
  extern __shared__ __align__(16) double psm[];
  __shared__ double s_warp[8];
  __shared__ double s_norm;
  const int64_t s = a.s;
  double* sv = psm;               // v_{t-1} (s doubles)
  T* sg = reinterpret_cast<T*>(psm + s);  // cached rows (rows_per_cta * s) if cache_rows
  const int64_t r0 = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t r1 = min(s, r0 + a.rows_per_cta);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  // products: q by G4 (cached when present), then T - 1 - pq by G; the last one gives lambda_hat
  const T* Gc = a.q > 0 ? a.G4 : a.G;  // the matrix whose rows are cached
  const int niter = a.T - (a.pw - 1) * a.q;
  if (a.cache_rows) {
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t j = threadIdx.x; j < s; j += blockDim.x) sg[(r - r0) * s + j] = Gc[r * a.ld + j];
  }
  const double v0 = 1.0 / sqrt((double)s);
  for (int64_t j = threadIdx.x; j < s; j += blockDim.x) sv[j] = v0;
  __syncthreads();
  double lam = 0.0;
  double inv = 1.0;  // 1/||u_{t-1}||, folded into this product (v_{t-1} = u_{t-1} * inv)
  for (int t = 0; t < niter; ++t) {
    const bool use4 = t < a.q;
    const T* Gt = use4 ? a.G4 : a.G;
    const bool cached = a.cache_rows && (use4 || a.q == 0);
    const unsigned flag = (unsigned)t + 1u;
    unsigned long long* buf = a.ll + (int64_t)(t & 1) * s * 2;
    // u_t = G v_{t-1}: one warp per row, 8 independent partial sums per lane
    for (int64_t r = r0 + warp; r < r1; r += nwarps) {
      const T* grow = cached ? sg + (r - r0) * s : Gt + r * a.ld;
      double d[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int64_t j = lane;
      for (; j + 224 < s; j += 256) {
#pragma unroll
        for (int q = 0; q < 8; ++q) d[q] = fma((double)grow[j + 32 * q], sv[j + 32 * q], d[q]);
      }
      for (; j < s; j += 32) d[0] = fma((double)grow[j], sv[j], d[0]);
      const double dd = warp_sum(((d[0] + d[1]) + (d[2] + d[3])) + ((d[4] + d[5]) + (d[6] + d[7]))) * inv;
      if (lane == 0) st_ll(buf + 2 * r, dd, flag);
    }
    __syncthreads();  // every warp is done reading sv before it is overwritten below
    // gather u_t into sv, then ||u_t||^2 from the staged copy in a fixed order
    ll_gather(buf, s, flag, sv);
    double sq = 0.0;
    for (int64_t j = threadIdx.x; j < s; j += blockDim.x) sq = fma(sv[j], sv[j], sq);
    sq = warp_sum(sq);
    if (lane == 0) s_warp[warp] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double q = 0.0;
      for (int w = 0; w < nwarps; ++w) q += s_warp[w];
      s_norm = sqrt(q);
    }
    __syncthreads();
    lam = s_norm;
    if (!(lam > kDegenerateLambda) || !(lam < 1e300)) { lam = lam < 1e300 ? 0.0 : lam; break; }
    inv = 1.0 / lam;
  }
  if (blockIdx.x == 0) compute_series(a.P, a.kern, a.K, a.safety, lam, a.c_given);
}

// Small s, one warp per row (s <= 32 C): lane x of warp w holds columns j = x + 32 c of
// Gram row r0 + w in registers; v_{t-1} is staged in shared memory by the gather.  Each
// warp computes its row of u_t = G v_{t-1} AND ||v_{t-1}||^2 over the whole staged vector
// itself (the same loads, the same fixed butterfly order in every warp of every CTA, so
// all of them hold the same norm bitwise) -- a product needs no block reduction, only
// the gather's barrier.  Measured at c2 (s = 1024, 128 CTAs): 2.1 us per product against
// 3.1 us for the previous layout (8 rows per CTA, thread-owned columns, one block
// reduction per product: tools/probes/ll_exchange.cu puts that reduction at ~0.5 us and
// the bare 147-CTA exchange at 1.3 us).  Splitting the gather across an 8-CTA cluster
// (one L2 poller per cluster, DSMEM broadcast, cluster barrier) measured no faster.
template <int C>
__global__ void __launch_bounds__(256) k_power_warp(PowerArgs<double> a) {
  __shared__ __align__(16) double s_v[32 * C];
  const int64_t s = a.s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + warp;
  const bool has_row = row < s;
  double g[C];
  auto load_row = [&](const double* M) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int64_t j = lane + 32 * c;
      g[c] = (has_row && j < s) ? M[row * a.ld + j] : 0.0;
    }
  };
  load_row(a.q > 0 ? a.G4 : a.G);
  {
    const double v0 = 1.0 / sqrt((double)s);
    for (int j = threadIdx.x; j < 32 * C; j += blockDim.x) s_v[j] = j < s ? v0 : 0.0;
  }
  __syncthreads();
  const int niter = a.T - (a.pw - 1) * a.q;
  double lam = 0.0, inv = 1.0;
  bool degenerate = false;
  for (int t = 0; t <= niter; ++t) {
    if (a.q > 0 && t == a.q) load_row(a.G);   // remaining products by G itself
    double d0 = 0.0, d1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
    for (int c = 0; c < C; c += 2) {
      const double x0 = s_v[lane + 32 * c];
      d0 = fma(g[c], x0, d0);
      q0 = fma(x0, x0, q0);
      if (c + 1 < C) {
        const double x1 = s_v[lane + 32 * (c + 1)];
        d1 = fma(g[c + 1], x1, d1);
        q1 = fma(x1, x1, q1);
      }
    }
    const double d = warp_sum(d0 + d1), sq = warp_sum(q0 + q1);
    if (t > 0) {  // ||u_{t-1}||: v_{t-1} = u_{t-1} / ||u_{t-1}|| is folded into this product
      lam = sqrt(sq);
      if (!(lam > kDegenerateLambda) || !(lam < 1e300)) { degenerate = true; break; }
      inv = 1.0 / lam;
    }
    if (t == niter) break;     // lambda_hat = ||u_{niter-1}||
    const unsigned flag = (unsigned)t + 1u;
    unsigned long long* buf = a.ll + (int64_t)(t & 1) * s * 2;
    if (lane == 0 && has_row) st_ll(buf + 2 * row, d * inv, flag);
    __syncthreads();  // every warp is done reading s_v before the gather overwrites it
    ll_gather(buf, s, flag, s_v, a.poll);
  }
  if (degenerate) lam = lam < 1e300 ? 0.0 : lam;
  if (blockIdx.x == 0) compute_series(a.P, a.kern, a.K, a.safety, lam, a.c_given);
}

// Large s: the Gram does not fit on chip, so every product streams G from HBM
// once.  One CTA (512 threads) per SM owns a contiguous block of rows; a warp
// reads a row with 16-byte vector loads, 8 in flight per lane (4 KB per warp,
// 64 KB per SM: enough memory-level parallelism for the HBM roofline); v_{t-1}
// (fp64) lives in shared memory.  Exchange and norm as in k_power_dense, with
// enough polling lanes that a gather takes a few rounds.
template <typename E>
__global__ void __launch_bounds__(512) k_power_stream(PowerArgs<E> a) {
  extern __shared__ __align__(16) double psm[];
  __shared__ double s_warp[16];
  __shared__ double s_norm;
  constexpr int VEC = 16 / sizeof(E);  // elements per 16-byte load
  const int64_t s = a.s;
  double* sv = psm;
  const int64_t r0 = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t r1 = min(s, r0 + a.rows_per_cta);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const bool vec = (a.ld % VEC) == 0 && ((reinterpret_cast<uintptr_t>(a.G) & 15) == 0) &&
                   (a.G4 == nullptr || (reinterpret_cast<uintptr_t>(a.G4) & 15) == 0);
  const double v0 = 1.0 / sqrt((double)s);
  for (int64_t j = threadIdx.x; j < s; j += blockDim.x) sv[j] = v0;
  __syncthreads();
  const int np = (int)min((int64_t)blockDim.x, max((int64_t)128, (s + 7) / 8 / 32 * 32));
  double lam = 0.0, inv = 1.0;
  const int niter = a.T - (a.pw - 1) * a.q;   // q products by c^p G^p, then the rest by G
  for (int t = 0; t < niter; ++t) {
    const unsigned flag = (unsigned)t + 1u;
    unsigned long long* buf = a.ll + (int64_t)(t & 1) * s * 2;
    const E* Gt = t < a.q ? a.G4 : a.G;
    for (int64_t r = r0 + warp; r < r1; r += nwarps) {
      const E* row = Gt + r * a.ld;
      double d[4] = {0, 0, 0, 0};
      int64_t j = 0;
      if (vec) {
        constexpr int STEP = 32 * VEC * 8;   // elements per warp iteration (8 loads per lane)
        for (; j + STEP <= s; j += STEP) {
          E x[8][VEC];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const E* p = row + j + (int64_t)(u * 32 + lane) * VEC;
            if constexpr (VEC == 4) {
              const float4 q = __ldcs(reinterpret_cast<const float4*>(p));
              x[u][0] = q.x; x[u][1] = q.y; x[u][2] = q.z; x[u][3] = q.w;
            } else {
              const double2 q = __ldcs(reinterpret_cast<const double2*>(p));
              x[u][0] = q.x; x[u][1] = q.y;
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              const int64_t jj = j + (int64_t)(u * 32 + lane) * VEC + e;
              d[(u * VEC + e) & 3] = fma((double)x[u][e], sv[jj], d[(u * VEC + e) & 3]);
            }
        }
      }
      for (int64_t jj = j + lane; jj < s; jj += 32) d[0] = fma((double)row[jj], sv[jj], d[0]);
      const double dd = warp_sum((d[0] + d[1]) + (d[2] + d[3])) * inv;
      if (lane == 0) st_ll(buf + 2 * r, dd, flag);
    }
    __syncthreads();  // every warp is done reading sv
    ll_gather(buf, s, flag, sv, np);
    double sq = 0.0;
    for (int64_t j = threadIdx.x; j < s; j += blockDim.x) sq = fma(sv[j], sv[j], sq);
    sq = warp_sum(sq);
    if (lane == 0) s_warp[warp] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double q = 0.0;
      for (int w = 0; w < nwarps; ++w) q += s_warp[w];
      s_norm = sqrt(q);
    }
    __syncthreads();
    lam = s_norm;
    if (!(lam > kDegenerateLambda) || !(lam < 1e300)) { lam = lam < 1e300 ? 0.0 : lam; break; }
    inv = 1.0 / lam;
  }
  if (blockIdx.x == 0) compute_series(a.P, a.kern, a.K, a.safety, lam, a.c_given);
}

cudaError_t launch_series(SeriesParams* P, const cpa_svt_kernel& k, int K, double safety, double lam_override,
                          const double* lam_src, const double* c_given, cudaStream_t st) {
  k_series<<<1, 256, 0, st>>>(P, k, K, safety, lam_override, lam_src, c_given);
  return cudaGetLastError();
}

// Scratch needed by launch_power_dense (doubles): the LL exchange (4 s words) and
// the squaring scale slot at power_scale_offset(s).
size_t power_dense_scratch_doubles(int64_t s) { return (size_t)(4 * s + 16); }
size_t power_scale_offset(int64_t s) { return (size_t)(4 * s + 8); }

// c = 2^-e with e = ilogb(max_i G_ii): G_ii <= lambda_max <= s * max_i G_ii, so
// c^p G^p has its dominant eigenvalue in [2^-p, (2s)^p]: no overflow for p <= 32.
__global__ void k_diag_scale(const double* G, int64_t s, double* scale) {
  __shared__ double red[256];
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < s; i += blockDim.x) mx = fmax(mx, G[i * s + i]);
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double m = red[0];
    const int e = (m > 0.0 && isfinite(m)) ? ilogb(m) : 0;
    scale[0] = ldexp(1.0, -2 * e);  // applied to G^2 (one factor c^2)
  }
}

cudaError_t launch_diag_scale(const double* G, int64_t s, double* scale, cudaStream_t st) {
  k_diag_scale<<<1, 256, 0, st>>>(G, s, scale);
  return cudaGetLastError();
}

// Number j of squarings (G -> c^2 G^2 -> ... -> c^p G^p, p = 2^j) for the power iteration:
// the q = (T-1)/p products by c^p G^p plus the T - 1 - pq remaining ones by G and the norm
// replace T products.  A squaring is one symmetric s x s DMMA product (measured 54 us at
// s = 1024, ~20 TF/s; ~30 TF/s for large s); a product costs ~1.2 + 0.9 s/1024 us
// (k_power_warp, latency-bound: 2.1 us measured at s = 1024), ~3 us with the rows in
// shared memory, or one HBM pass over G when streamed.  j = 3 at c2 (measured: j = 2 / 3 / 4
// give 0.292 / 0.269 / ~0.29 ms for the whole phase).  j <= 5 keeps (c lambda)^p finite.
int power_squarings(int64_t s, int T) {
  if (T < 4) return 0;
  const double sd = (double)s;
  const double gemm_us = fmax(6.0, sd * sd * sd / (s <= 2048 ? 20e12 : 30e12) * 1e6);
  double iter_us;
  if (s <= 1024) iter_us = 1.2 + 0.9 * sd / 1024.0;
  else if (sd * 8.0 * 2.0 <= 200.0 * 1024.0) iter_us = 3.0;
  else iter_us = 8.0 * sd * sd / 6.5e12 * 1e6 + 2.0;
  int best = 0;
  double best_cost = (double)T * iter_us;
  for (int j = 1; j <= 5 && (1 << j) <= T - 1; ++j) {
    const int p = 1 << j, q = (T - 1) / p;
    const double cost = j * gemm_us + (double)(T - (p - 1) * q) * iter_us;
    if (cost < best_cost) { best_cost = cost; best = j; }
  }
  return best;
}

template <typename E>
static cudaError_t launch_power_t(const E* G, const E* G4, int pw, int64_t s, int64_t ld, int T, double* scratch,
                                  unsigned int* bar, SeriesParams* P, const cpa_svt_kernel& k, int K, double safety,
                                  const double* c_given, int num_sms, cudaStream_t st) {
  PowerArgs<E> a{};
  a.ld = ld;
  a.G = G; a.s = s; a.T = T;
  a.G4 = G4;
  a.pw = G4 ? pw : 1;
  a.q = G4 ? (T - 1) / pw : 0;
  a.poll = 32 * CPA_POLL_WARPS;
  a.ll = reinterpret_cast<unsigned long long*>(scratch);
  (void)bar;
  a.P = P; a.kern = k; a.K = K; a.safety = safety; a.c_given = c_given;
  // Fewest CTAs whose rows of G fit in shared memory (fewer arrivals per
  // barrier); otherwise one CTA per SM streaming its rows from L2/HBM.
  const size_t budget = 200 * 1024;
  size_t smem = (size_t)s * sizeof(double);
  if (smem > budget) return cudaErrorInvalidValue;  // s > 25600 not supported by this kernel
  // One CTA per SM (the product is latency-bound: fewer rows per CTA shortens
  // it); rows cached in shared memory when they fit.
  int64_t grid = s < num_sms ? s : num_sms;
  const int64_t rows_per = (s + grid - 1) / grid;
  a.cache_rows = smem + (size_t)rows_per * s * sizeof(E) <= budget;
  if (grid < 1) grid = 1;
  a.rows_per_cta = (int)((s + grid - 1) / grid);
  grid = (s + a.rows_per_cta - 1) / a.rows_per_cta;
  if (a.cache_rows) smem += (size_t)a.rows_per_cta * s * sizeof(E);
  cudaError_t e0 = cudaMemsetAsync(scratch, 0, (size_t)4 * s * sizeof(double), st);
  if (e0 != cudaSuccess) return e0;
  if (!a.cache_rows) {
    // rows do not fit on chip: stream G (or c^4 G^4) from HBM / L2 every product
    a.rows_per_cta = (int)((s + num_sms - 1) / num_sms);
    const int64_t g2 = (s + a.rows_per_cta - 1) / a.rows_per_cta;
    const size_t sm2 = (size_t)s * sizeof(double);
    cudaError_t e2 = cudaFuncSetAttribute(k_power_stream<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    if (e2 != cudaSuccess) return e2;
    void* args[] = {&a};
    return cudaLaunchCooperativeKernel((void*)k_power_stream<E>, dim3((unsigned)g2), dim3(512), args, sm2, st);
  }
  if constexpr (sizeof(E) == sizeof(double)) {
    // s <= 1024 (c1, c2): one warp per Gram row, the row in registers
    if (s <= 1024 && !env_on("CPA_SVT_POWER_SMEM")) {
      a.rows_per_cta = 8;
      a.poll = 256;
      const int64_t gw = (s + 7) / 8;
      void* args[] = {&a};
      void* kf = s <= 64 ? (void*)k_power_warp<2> : s <= 256 ? (void*)k_power_warp<8> : (void*)k_power_warp<32>;
      return cudaLaunchCooperativeKernel(kf, dim3((unsigned)gw), dim3(256), args, 0, st);
    }
  }
  cudaError_t e = cudaFuncSetAttribute(k_power_dense<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((void*)k_power_dense<E>, dim3((unsigned)grid), dim3(256), args, smem, st);
}

cudaError_t launch_power_dense(const double* G, const double* G4, int pw, int64_t s, int T, double* scratch,
                               unsigned int* bar, SeriesParams* P, const cpa_svt_kernel& k, int K, double safety,
                               const double* c_given, int num_sms, cudaStream_t st) {
  return launch_power_t<double>(G, G4, pw, s, s, T, scratch, bar, P, k, K, safety, c_given, num_sms, st);
}
// fp32 Gram (TF32 path): the products are accumulated in fp64 all the same
cudaError_t launch_power_dense_f32(const float* G, int64_t s, int64_t ld, int T, double* scratch, unsigned int* bar,
                                   SeriesParams* P, const cpa_svt_kernel& k, int K, double safety,
                                   const double* c_given, int num_sms, cudaStream_t st) {
  return launch_power_t<float>(G, nullptr, 1, s, ld, T, scratch, bar, P, k, K, safety, c_given, num_sms, st);
}

}  // namespace cpa

namespace cpa {
// ---------------------------------------------------------------------------------------------
// Row-sharded power iteration (multi-GPU s x s path, Alg. 1 line 3; reading R6).
// Rank p owns rows [s p / P, s (p+1) / P) of G.  Product t computes its rows of
// u_t = G u_{t-1} / ||u_{t-1}|| (u_0 := sqrt(s) v_0, i.e. v_0 = 1/sqrt(s) (1, ..., 1)), writes them and
// the sum of their squares (last entry) into its slot of an all-gather buffer; after the
// all-gather every rank holds all of u_t and ||u_t||^2 = the slots' sums added in rank order.
// lambda_hat = ||u_T|| (= ||G v_{T-1}||).  Two gather buffers alternate (a product reads the
// previous one).  Deterministic for a fixed P: every sum runs in a fixed order.
constexpr int kPRThreads = 1024;

__device__ __forceinline__ double pr_norm2(const double* g, int P, int64_t slot) {
  double n2 = 0.0;
  for (int p = 0; p < P; ++p) n2 += __ldcg(g + (int64_t)p * slot + slot - 1);
  return n2;
}

template <typename E>
__global__ void __launch_bounds__(kPRThreads, 1) k_power_rows(const E* __restrict__ G, int64_t s, int64_t ld, int P,
                                                              int64_t slot, const double* __restrict__ gin,
                                                              int64_t r0, int64_t r1, double* __restrict__ gout,
                                                              double* __restrict__ bpart, unsigned int* counter) {
  extern __shared__ double u_s[];   // u_{t-1} (s doubles)
  __shared__ double red[kPRThreads / 32];
  __shared__ double s_inv;
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    if (gin) {
      const double n = sqrt(pr_norm2(gin, P, slot));
      s_inv = n > kDegenerateLambda ? 1.0 / n : 0.0;   // a zero Gram stays zero: lambda_hat = 0 (R17)
    } else {
      s_inv = 1.0;
    }
  }
  if (gin) {
    for (int p = 0; p < P; ++p) {   // slot p holds rows [s p / P, s (p+1) / P): one coalesced copy each
      const int64_t b = s * p / P, e = s * (p + 1) / P;
      const double* src = gin + (int64_t)p * slot - b;
      for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) u_s[i] = __ldcg(src + i);
    }
  } else {
    const double v0 = 1.0 / sqrt((double)s);
    for (int64_t i = threadIdx.x; i < s; i += blockDim.x) u_s[i] = v0;
  }
  __syncthreads();
  const double inv = s_inv;
  double sq = 0.0;   // lane 0: squares of this warp's rows, in row order
  // rows interleaved over the CTAs first (row = r0 + warp * grid + block), so a short panel still
  // spreads over every SM
  for (int64_t row = r0 + (int64_t)warp * gridDim.x + blockIdx.x; row < r1;
       row += (int64_t)gridDim.x * (kPRThreads / 32)) {
    const E* g = G + row * ld;
    double a0 = 0.0, a1 = 0.0;
    int64_t c = 2 * lane;
    if (sizeof(E) == 8 && ((uintptr_t)g & 15) == 0) {
      for (; c + 1 < s; c += 64) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(g + c));
        a0 = fma(v.x, u_s[c], a0);
        a1 = fma(v.y, u_s[c + 1], a1);
      }
      if (c < s) a0 = fma((double)__ldcs(g + c), u_s[c], a0);
    } else {
      for (c = lane; c < s; c += 32) a0 = fma((double)__ldcs(g + c), u_s[c], a0);
    }
    double d = a0 + a1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    const double val = d * inv;
    if (lane == 0) {
      gout[row - r0] = val;
      sq = fma(val, val, sq);
    }
  }
  if (lane == 0) red[warp] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < kPRThreads / 32; ++w) b += red[w];
    bpart[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double tot = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) tot += __ldcg(bpart + b);
    gout[slot - 1] = tot;   // this slot's sum of squares
    *counter = 0u;
  }
}

__global__ void k_power_rows_final(const double* g, int P, int64_t slot, double* lam_hat) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *lam_hat = sqrt(pr_norm2(g, P, slot));
}

int64_t power_rows_slot(int64_t s, int P) { return (s + P - 1) / P + 1; }
size_t power_rows_scratch_doubles(int64_t s, int P, int num_sms) {
  return (size_t)(2 * P * power_rows_slot(s, P) + num_sms + 8);
}

// Product t (1-based) of the row-sharded power iteration for virtual rank v of P: reads the
// gathered buffer of product t-1 (none at t = 1), writes rank v's slot of the buffer of product t.
// scratch: [2 * P * slot gather buffers | num_sms block partials | counter | lambda_hat].
template <typename E>
static cudaError_t launch_power_rows_t(const E* G, int64_t s, int64_t ld, int t, int v, int P, double* scratch,
                                       int num_sms, cudaStream_t st) {
  const int64_t slot = power_rows_slot(s, P);
  double* gb[2] = {scratch, scratch + P * slot};
  double* bpart = scratch + 2 * P * slot;
  unsigned int* counter = reinterpret_cast<unsigned int*>(bpart + num_sms);
  const double* gin = t == 1 ? nullptr : gb[(t - 1) & 1];
  double* gout = gb[t & 1] + (int64_t)v * slot;
  const int64_t r0 = s * v / P, r1 = s * (v + 1) / P;
  const size_t smem = (size_t)s * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_power_rows<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int grid = num_sms;
  if (grid > r1 - r0) grid = (int)(r1 - r0 > 0 ? r1 - r0 : 1);
  k_power_rows<E><<<grid, kPRThreads, smem, st>>>(G, s, ld, P, slot, gin, r0, r1, gout, bpart, counter);
  return cudaGetLastError();
}
cudaError_t launch_power_rows(const double* G, int64_t s, int t, int v, int P, double* scratch, int num_sms,
                              cudaStream_t st) {
  return launch_power_rows_t<double>(G, s, s, t, v, P, scratch, num_sms, st);
}
// fp32 Gram (the TF32 path), row stride ld; the products still accumulate in fp64
cudaError_t launch_power_rows_f32(const float* G, int64_t s, int64_t ld, int t, int v, int P, double* scratch,
                                  int num_sms, cudaStream_t st) {
  return launch_power_rows_t<float>(G, s, ld, t, v, P, scratch, num_sms, st);
}
// The buffer product t writes (for the all-gather) and the final lambda_hat slot.
double* power_rows_buffer(double* scratch, int64_t s, int t, int P) {
  return scratch + (int64_t)(t & 1) * P * power_rows_slot(s, P);
}
cudaError_t launch_power_rows_final(double* scratch, int64_t s, int T, int P, int num_sms, double** lam_hat,
                                    cudaStream_t st) {
  const int64_t slot = power_rows_slot(s, P);
  double* lam = scratch + 2 * P * slot + num_sms + 2;
  k_power_rows_final<<<1, 32, 0, st>>>(scratch + (int64_t)(T & 1) * P * slot, P, slot, lam);
  *lam_hat = lam;
  return cudaGetLastError();
}
}  // namespace cpa
