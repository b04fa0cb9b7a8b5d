// Sparse path (BASELINE configs[3]): X is m x n CSR fp64; Y = X H_hat(X^T X)
// with the n x n Gram never formed (PAPER.md:278-307 identity, sparsity
// motivation PAPER.md:316-334).  Right-apply recurrence, one SpMM pair per step:
//
//   Z       = W_{k-1} X^T                                   (rows x m, dense)
//   W_k     = (4/L) Z X - 2 W_{k-1} - W_{k-2},  Y += c_k W_k   (fused epilogue)
//   init:   W_1 = (2/L) (X X^T)|rows X - X,  Y = c_0/2 X + c_1 W_1
//
// Layout: this rank's rows [row_begin, row_end) are cut into blocks of RB = 64
// rows; every dense operand (W, Y, Z) is stored block-interleaved --
// element (i, c) of block b at ((b * C + c) * RB + i%RB) -- so one warp owns a
// block row and each gathered column c is one coalesced 512-byte load, and
// rows of a block never interact (the recurrence is row-independent).  Kernels
// launch block-major, so the gathered W (or Z) block stays L2-resident.
// Sums run in a fixed order (CSR row order / sorted CSC column order): the
// result is deterministic.
//
// Lambda_max: power iteration on the m-side, v -> X (X^T v) (reading R4), two
// SpMVs and a deterministic two-level norm per step.
#include <algorithm>

#include <cub/cub.cuh>

#include "common.cuh"

namespace cpa {

// Rows per interleaved block RB = 32 VW: lane l owns rows VW l .. VW l + VW - 1 of its block, so a
// gathered column is one coalesced 32 VW x 8-byte warp load.  VW = 2 (512-byte gathers) moves
// 19-20 TB/s of random L2 gathers where 256-byte ones (VW = 1) move 12.6 (tools/probes/
// l2_gather512.cu); CPA_SP_VW=1 builds the 32-row layout.
#ifndef CPA_SP_VW
#define CPA_SP_VW 2
#endif
constexpr int VW = CPA_SP_VW;
constexpr int RB = 32 * VW;     // rows per interleaved block
constexpr int SP_WARPS = 8;     // warps per CTA in the SpMM kernels

// VW consecutive doubles of a lane (one 8- or 16-byte access)
struct Vw {
  double v[VW];
};
__device__ __forceinline__ Vw ldv(const double* p) {
  Vw r;
  if constexpr (VW >= 2) {
#pragma unroll
    for (int h = 0; h < VW / 2; ++h) {
      const double2 q = reinterpret_cast<const double2*>(p)[h];
      r.v[2 * h] = q.x;
      r.v[2 * h + 1] = q.y;
    }
  } else {
    r.v[0] = *p;
  }
  return r;
}
__device__ __forceinline__ void stv(double* p, const Vw& a) {
  if constexpr (VW >= 2) {
#pragma unroll
    for (int h = 0; h < VW / 2; ++h) reinterpret_cast<double2*>(p)[h] = make_double2(a.v[2 * h], a.v[2 * h + 1]);
  } else {
    *p = a.v[0];
  }
}

__device__ __forceinline__ double warp_sum_sp(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- CSC build
__global__ void k_col_count(const int32_t* col, int64_t nnz, int* cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + col[e], 1);
}
__global__ void k_col_fill(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t m,
                           const int64_t* cptr, int* cursor, int32_t* crow, double* cval, int64_t n_cols) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      const int c = col[e];
      CPA_DCHECK(c >= 0 && c < n_cols);
      const int64_t p = cptr[c] + atomicAdd(cursor + c, 1);
      CPA_DCHECK(p < cptr[c + 1]);
      crow[p] = (int32_t)i;
      cval[p] = val[e];
    }
  }
}
// sort each column's (row, val) pairs by row (insertion sort, ~nnz/n entries): fixed summation order
__global__ void k_col_sort(const int64_t* cptr, int64_t n, int32_t* crow, double* cval) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = cptr[c], e = cptr[c + 1];
    for (int64_t p = b + 1; p < e; ++p) {
      const int32_t r = crow[p];
      const double v = cval[p];
      int64_t q = p - 1;
      while (q >= b && crow[q] > r) {
        crow[q + 1] = crow[q];
        cval[q + 1] = cval[q];
        --q;
      }
      crow[q + 1] = r;
      cval[q + 1] = v;
    }
  }
}
__global__ void k_widen(const int* cnt, int64_t n, int64_t* out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    out[c] = cnt[c];
}

// ---------------------------------------------------------------- power iteration
// u = X^T v (n-vector) via the sorted CSC; one thread per column
__global__ void k_spmv_t(const int64_t* cptr, const int32_t* crow, const double* cval, int64_t n, const double* v,
                         const double* scale, double* u) {
  const double sc = scale ? *scale : 1.0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t e = cptr[c]; e < cptr[c + 1]; ++e) s = fma(cval[e], v[crow[e]], s);
    u[c] = s * sc;
  }
}
// y = X t (m-vector) via CSR; one warp per row; per-block partial sums of y^2
__global__ void k_spmv(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t m, const double* t,
                       double* y, double* part) {
  __shared__ double ws[SP_WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double sq = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)SP_WARPS + warp; i < m; i += (int64_t)gridDim.x * SP_WARPS) {
    double s = 0.0;
    for (int64_t e = row_ptr[i] + lane; e < row_ptr[i + 1]; e += 32) s = fma(val[e], t[col[e]], s);
    s = warp_sum_sp(s);
    if (lane == 0) y[i] = s;
    sq = fma(s, s, sq);
  }
  if (lane == 0) ws[warp] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double p = 0.0;
    for (int w = 0; w < SP_WARPS; ++w) p += ws[w];
    part[blockIdx.x] = p;
  }
}
// norm from per-block partials (fixed order); writes lambda_hat and 1/||y||
__global__ void k_norm(const double* part, int nparts, double* nrm, double* inv) {
  __shared__ double red[256];
  double s = 0.0;
  for (int b = threadIdx.x; b < nparts; b += blockDim.x) s += part[b];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double q = sqrt(red[0]);
    *nrm = q;
    *inv = q > kDegenerateLambda ? 1.0 / q : 0.0;
  }
}
__global__ void k_fill(double* v, int64_t n, double x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = x;
}

// ---------------------------------------------------------------- recurrence
// W0 (interleaved) <- rows [r0, r0+rows) of X (densify)
__global__ void k_densify(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t r0, int64_t rows,
                          int64_t n, double* W) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t i = blockIdx.x * (int64_t)SP_WARPS + warp; i < rows; i += (int64_t)gridDim.x * SP_WARPS) {
    const int64_t b = i / RB, li = i % RB;
    for (int64_t e = row_ptr[r0 + i] + lane; e < row_ptr[r0 + i + 1]; e += 32)
      W[(b * n + col[e]) * RB + li] = val[e];
  }
}

// Row split points of the CSR for the column passes of k_spmm_wxt: rs[j * (NP + 1) + h] = first
// entry of row j with column >= n h / NP (columns are sorted within a row).
__global__ void k_row_split(const int64_t* row_ptr, const int32_t* col, int64_t m, int64_t n, int NP, int64_t* rs) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = row_ptr[j], e1 = row_ptr[j + 1];
    rs[j * (NP + 1)] = e0;
    for (int h = 1; h < NP; ++h) {
      const int64_t cb = n * h / NP;
      int64_t lo = e0, hi = e1;   // first e in [e0, e1) with col[e] >= cb
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (col[mid] < cb) lo = mid + 1; else hi = mid;
      }
      rs[j * (NP + 1) + h] = lo;
    }
    rs[j * (NP + 1) + NP] = e1;
  }
}

// Z[b][j][:] (+)= sum_{l in row j of X, l in column pass h} x_jl W[b][l][:]   (one warp per (b, j)).
// The NP column passes run as NP launches in order (pass 0 writes, the others add: a fixed order),
// so the L2 footprint of a block is its W slice (32 x n / NP doubles) plus the matching CSR slice
// instead of the whole 51 MB block row (DRAM re-reads of W measured 3.5x with one pass).
// sum_{e in [e0, e1)} x[e] V[idx[e]][lane] with U gathers in flight (U accumulators, the tail in
// accumulator 0, summed in a fixed tree: a fixed order)
template <int U>
__device__ __forceinline__ Vw gather_sum(const int32_t* __restrict__ idx, const double* __restrict__ x, int64_t e0,
                                         int64_t e1, const double* __restrict__ Vb, int64_t nidx) {
  (void)nidx;
  Vw acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int q = 0; q < VW; ++q) acc[u].v[q] = 0.0;
  int64_t e = e0;
  for (; e + U <= e1; e += U) {
    int32_t c[U];
    double xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = __ldg(idx + e + u);
      xv[u] = __ldg(x + e + u);
      CPA_DCHECK(c[u] >= 0 && c[u] < nidx);
    }
    Vw g[U];
#pragma unroll
    for (int u = 0; u < U; ++u) g[u] = ldv(Vb + (int64_t)c[u] * RB);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < VW; ++q) acc[u].v[q] = fma(xv[u], g[u].v[q], acc[u].v[q]);
  }
  for (; e < e1; ++e) {
    const Vw g = ldv(Vb + (int64_t)__ldg(idx + e) * RB);
    const double xe = __ldg(x + e);
#pragma unroll
    for (int q = 0; q < VW; ++q) acc[0].v[q] = fma(xe, g.v[q], acc[0].v[q]);
  }
#pragma unroll
  for (int w = 1; w < U; w *= 2)
#pragma unroll
    for (int u = 0; u + w < U; u += 2 * w)
#pragma unroll
      for (int q = 0; q < VW; ++q) acc[u].v[q] += acc[u + w].v[q];
  return acc[0];
}

template <int U>
__global__ void __launch_bounds__(SP_WARPS * 32) k_spmm_wxt(const int64_t* row_ptr, const int32_t* col,
                                                            const double* val, int64_t m, int64_t n, int64_t nblk,
                                                            const double* __restrict__ W, double* __restrict__ Z,
                                                            const int64_t* __restrict__ rs, int NP, int h) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = blockIdx.x * (int64_t)SP_WARPS + warp;  // block-major: item = b * m + j
  if (item >= nblk * m) return;
  const int64_t b = item / m, j = item % m;
  const double* Wb = W + b * n * RB + VW * lane;
  const int64_t e0 = NP > 1 ? rs[j * (NP + 1) + h] : row_ptr[j];
  const int64_t e1 = NP > 1 ? rs[j * (NP + 1) + h + 1] : row_ptr[j + 1];
  Vw sum = gather_sum<U>(col, val, e0, e1, Wb, n);
  double* zp = Z + (b * m + j) * RB + VW * lane;
  if (h != 0) {
    const Vw z = ldv(zp);
#pragma unroll
    for (int q = 0; q < VW; ++q) sum.v[q] = z.v[q] + sum.v[q];
  }
  stv(zp, sum);
}

// W_k[b][l][:] = s * sum_{j in col l} x_jl Z[b][j][:] - ... (fused epilogue), one warp per (b, l)
// W_k[b][l][:] = 2 s (sum_{j in col l} x_jl Z[b][j][:]) - 2 W_{k-1} - W_{k-2}, Y += c_k W_k (fused
// epilogue), one warp per (b, l).  (Evict-first / streaming hints on the epilogue's streamed
// operands, loaded ahead of the gathers, measured slower: 74.5 -> 77.5 ms per c4 step.)
template <int U, bool INIT>
__global__ void __launch_bounds__(SP_WARPS * 32) k_spmm_zx(const int64_t* cptr, const int32_t* crow,
                                                           const double* cval, int64_t m, int64_t n, int64_t nblk,
                                                           const double* __restrict__ Z, const double* Wp,
                                                           const double* Wpp, double* Wout, double* Yb,
                                                           const SeriesParams* P, int k, int yterms) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = blockIdx.x * (int64_t)SP_WARPS + warp;  // item = b * n + l
  if (item >= nblk * n) return;
  const int64_t b = item / n, l = item % n;
  const Vw acc = gather_sum<U>(crow, cval, cptr[l], cptr[l + 1], Z + b * m * RB + VW * lane, m);
  const int64_t o = item * RB + VW * lane;
  const double s2 = P->scale2;
  if (INIT) {
    const Vw x = ldv(Wp + o);
    Vw w, y;
#pragma unroll
    for (int q = 0; q < VW; ++q) {
      w.v[q] = s2 * acc.v[q] - x.v[q];                       // W_1 = B_hat X
      y.v[q] = 0.5 * P->c[0] * x.v[q] + P->c[1] * w.v[q];    // Y = c0/2 W_0 + c1 W_1
    }
    if (Wout) stv(Wout + o, w);
    stv(Yb + o, y);
  } else {
    const Vw wp = ldv(Wp + o), wpp = ldv(Wpp + o);
    Vw w;
#pragma unroll
    for (int q = 0; q < VW; ++q) w.v[q] = 2.0 * s2 * acc.v[q] - 2.0 * wp.v[q] - wpp.v[q];   // W_k = 2 B_hat W_{k-1} - W_{k-2}
    if (Wout) stv(Wout + o, w);
    // Y += c_j W_j for the yterms latest j (1 to 3: W_{k-2}, W_{k-1} are in registers already), so Y
    // is read and written once every third step (sparse_apply)
    if (yterms > 0) {
      Vw y = ldv(Yb + o);
#pragma unroll
      for (int q = 0; q < VW; ++q) {
        double t = P->c[k] * w.v[q];
        if (yterms >= 2) t = P->c[k - 1] * wp.v[q] + t;
        if (yterms >= 3) t = P->c[k - 2] * wpp.v[q] + t;
        y.v[q] += t;
      }
      stv(Yb + o, y);
    }
  }
}

// caller Y (row-major, ld) <- interleaved Yb, via 64 x 64 shared-memory transposes (blockIdx.z: the
// 64-row piece of the RB-row block)
constexpr int UT = 64;
__global__ void k_unblock(const double* Yb, int64_t rows, int64_t n, double* Y, int64_t ldy) {
  __shared__ double t[UT][UT + 1];
  const int64_t b = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * UT;
  const int i0 = blockIdx.z * UT;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const int ni = RB - i0 < UT ? RB - i0 : UT;     // rows of this piece (RB = 32: 32)
  for (int r = ty; r < UT; r += 8) {   // r: column within the tile, i: row within the piece
    const int64_t c = c0 + r;
    for (int i = tx; i < ni; i += 32) t[r][i] = c < n ? Yb[(b * n + c) * RB + i0 + i] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < ni; r += 8) {   // r: row within the piece
    const int64_t i = b * RB + i0 + r;
    for (int cc = tx; cc < UT; cc += 32) {
      const int64_t c = c0 + cc;
      if (i < rows && c < n) Y[i * ldy + c] = t[cc][r];
    }
  }
}

static inline size_t al(size_t b) { return (b + 255) / 256 * 256; }

cudaError_t launch_series(SeriesParams* P, const cpa_svt_kernel& k, int K, double safety, double lam_override,
                          const double* lam_src, const double* c_given, cudaStream_t st);

cudaError_t sparse_apply(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                         const double* val, int64_t row_begin, int64_t row_end, double* Y, int64_t ldy,
                         const cpa_svt_kernel& kern, int K, int T, double safety, double lam_override,
                         SeriesParams* P, void* ws, size_t ws_bytes, size_t* ws_needed, int num_sms,
                         cudaStream_t st, int* launches, SparsePhaseHook hook, void* hook_ctx, const double* c_given) {
  const int64_t rows = row_end - row_begin;
  const int64_t nblk = (rows + RB - 1) / RB;
  // workspace layout
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n + 1));
  const int npart = 4 * num_sms;
  size_t off = 0;
  const size_t o_cptr = off; off += al((n + 1) * sizeof(int64_t));
  const size_t o_cnt = off;  off += al((n + 1) * sizeof(int64_t));  // int counts, then int64 widened
  const size_t o_crow = off; off += al(nnz * sizeof(int32_t));
  const size_t o_cval = off; off += al(nnz * sizeof(double));
  const size_t o_scan = off; off += al(scan_bytes);
  const size_t o_v = off;    off += al(m * sizeof(double));
  const size_t o_t = off;    off += al(n * sizeof(double));
  const size_t o_part = off; off += al(npart * sizeof(double));
  const size_t o_nrm = off;  off += al(4 * sizeof(double));
  const size_t blkW = (size_t)nblk * n * RB, blkZ = (size_t)nblk * m * RB;
  const size_t o_Wa = off;   off += al(blkW * sizeof(double));
  const size_t o_Wb = off;   off += al(blkW * sizeof(double));
  const size_t o_Y = off;    off += al(blkW * sizeof(double));
  const size_t o_Z = off;    off += al(blkZ * sizeof(double));
  // column passes of Z = W X^T: W slices of <= ~52 MB per block (CPA_SVT_SP_PASSES overrides)
  // (a pass's W slice <= ~52 MB: c4 with 64-row blocks takes 2 passes -- Z kernel per step 44.6 ms
  // against 45.2 / 46.7 / 49.0 ms for 3 / 4 / 6 passes)
  int NP = (int)std::max<int64_t>(1, (n * RB * 8 + (52 << 20) - 1) / (52 << 20));
  if (const char* v = getenv("CPA_SVT_SP_PASSES")) NP = std::max(1, atoi(v));
  const size_t o_rs = off;   off += al((size_t)m * (NP + 1) * sizeof(int64_t));
  *ws_needed = off;
  if (!ws || ws_bytes < off) return cudaSuccess;  // size query
  char* base = (char*)ws;
  int64_t* cptr = (int64_t*)(base + o_cptr);
  int* cnt = (int*)(base + o_cnt);
  int64_t* cnt64 = (int64_t*)(base + o_cnt);
  int32_t* crow = (int32_t*)(base + o_crow);
  double* cval = (double*)(base + o_cval);
  double* v = (double*)(base + o_v);
  double* tv = (double*)(base + o_t);
  double* part = (double*)(base + o_part);
  double* nrm = (double*)(base + o_nrm);
  double* Wa = (double*)(base + o_Wa);
  double* Wb = (double*)(base + o_Wb);
  double* Yb = (double*)(base + o_Y);
  double* Z = (double*)(base + o_Z);
  int64_t* rs = (int64_t*)(base + o_rs);
  int L = 0;
  cudaError_t e;
  const int g = 4 * num_sms;
#define SPCK(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
  // ---- CSC of X (= CSR of X^T), rows sorted within each column
  if (hook) hook(hook_ctx, CPA_SVT_PH_GRAM, 1);  // structure pass (CSC of X) in the Gram slot
  SPCK(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int), st));
  k_col_count<<<g, 256, 0, st>>>(col, nnz, cnt); ++L;
  // widen int counts to int64 in place is unsafe; use cptr as scratch for the widened counts
  k_widen<<<g, 256, 0, st>>>(cnt, n, cptr); ++L;
  SPCK(cudaMemsetAsync(cptr + n, 0, sizeof(int64_t), st));
  SPCK(cub::DeviceScan::ExclusiveSum(base + o_scan, scan_bytes, cptr, cnt64, (int)(n + 1), st)); ++L;
  SPCK(cudaMemcpyAsync(cptr, cnt64, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  SPCK(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int), st));
  k_col_fill<<<g, 256, 0, st>>>(row_ptr, col, val, m, cptr, cnt, crow, cval, n); ++L;
  k_col_sort<<<g, 256, 0, st>>>(cptr, n, crow, cval); ++L;
  if (hook) hook(hook_ctx, CPA_SVT_PH_GRAM, 0);
  // ---- Lambda_max (m-side power iteration) and coefficients
  if (hook) hook(hook_ctx, CPA_SVT_PH_POWER, 1);
  if (lam_override > 0.0) {
    SPCK(launch_series(P, kern, K, safety, lam_override, nullptr, c_given, st)); ++L;
  } else {
    k_fill<<<g, 256, 0, st>>>(v, m, 1.0 / sqrt((double)m)); ++L;
    const int spg = (int)std::min<int64_t>((m + SP_WARPS - 1) / SP_WARPS, npart);
    for (int t = 0; t < T; ++t) {
      // t = X^T v_{t-1} (v_{t-1} = y_{t-1} / ||y_{t-1}||, scale folded in), y_t = X t
      k_spmv_t<<<g, 256, 0, st>>>(cptr, crow, cval, n, v, t == 0 ? nullptr : nrm + 1, tv); ++L;
      k_spmv<<<spg, SP_WARPS * 32, 0, st>>>(row_ptr, col, val, m, tv, v, part); ++L;
      k_norm<<<1, 256, 0, st>>>(part, spg, nrm, nrm + 1); ++L;
    }
    SPCK(launch_series(P, kern, K, safety, 0.0, nrm, c_given, st)); ++L;
  }
  if (hook) hook(hook_ctx, CPA_SVT_PH_POWER, 0);
  // ---- recurrence on this rank's rows
  if (rows > 0) {
    SPCK(cudaMemsetAsync(Wa, 0, blkW * sizeof(double), st));  // W_0 = X rows (Wa), densified
    k_densify<<<g, SP_WARPS * 32, 0, st>>>(row_ptr, col, val, row_begin, rows, n, Wa); ++L;
    // W_0 = X rows in Wa, W_1 -> Wb, then W_k overwrites W_{k-2} in place
    // (the epilogue reads W_{k-2}[o] and writes W_k[o] in the same thread).
    double* W0 = Wa;
    double* W1 = Wb;
    const int64_t itemsZ = nblk * m, itemsW = nblk * n;
    // gathers in flight per warp in the SpMM pair (CPA_SVT_SP_UNROLL = 2 | 4 | 8; c4 per step, Z / W
    // kernels: 55.0 / 77.6, 55.6 / 91.6, 78.2 / 109.7 ms -- more loads in flight only add L2
    // contention; the index loads of a pair ahead of the two gathers: Z 65 -> 55 ms)
    // (64-row blocks: the Z kernel best at 2, the W kernel at 1 -- c4 per step 44.4 / 52.4 ms against
    // 45.7 / 56.4 the other way round)
    int U = 2, UW = 1;
    if (const char* v = getenv("CPA_SVT_SP_UNROLL")) UW = U = atoi(v) == 8 ? 8 : atoi(v) == 4 ? 4 : atoi(v) == 1 ? 1 : 2;
    const bool yevery = env_on("CPA_SVT_SP_YEVERY");
    const unsigned gz = (unsigned)((itemsZ + SP_WARPS - 1) / SP_WARPS);
    const unsigned gw = (unsigned)((itemsW + SP_WARPS - 1) / SP_WARPS);
    const double* prev = W0;   // W_{k-1}
    const double* prev2 = nullptr;
    if (NP > 1) {
      k_row_split<<<g, 256, 0, st>>>(row_ptr, col, m, n, NP, rs);
      ++L;
    }
    for (int k = 1; k < K; ++k) {
      if (hook) hook(hook_ctx, CPA_SVT_PH_SPARSE_Z, 1);
      for (int hp = 0; hp < NP; ++hp) {
        auto kz = U == 8 ? k_spmm_wxt<8> : U == 4 ? k_spmm_wxt<4> : U == 1 ? k_spmm_wxt<1> : k_spmm_wxt<2>;
        kz<<<gz, SP_WARPS * 32, 0, st>>>(row_ptr, col, val, m, n, nblk, prev, Z, rs, NP, hp);
        ++L;
      }
      if (hook) hook(hook_ctx, CPA_SVT_PH_SPARSE_Z, 0);
      if (hook) hook(hook_ctx, CPA_SVT_PH_SPARSE_W, 1);
      double* out;
      if (k == 1) out = W1;                  // W_1 -> Wb
      else out = (k & 1) ? Wb : Wa;          // W_k overwrites W_{k-2} in place
      if (k == K - 1) out = nullptr;
      {
        auto kw = k == 1 ? (UW == 8 ? k_spmm_zx<8, true> : UW == 4 ? k_spmm_zx<4, true> : UW == 1 ? k_spmm_zx<1, true> : k_spmm_zx<2, true>)
                         : (UW == 8 ? k_spmm_zx<8, false> : UW == 4 ? k_spmm_zx<4, false> : UW == 1 ? k_spmm_zx<1, false> : k_spmm_zx<2, false>);
        // Y += c_j W_j in groups of three steps (k = 4, 7, 10, ...: the terms since the last group),
        // the last step flushing the rest (CPA_SVT_SP_YEVERY=1: every step, Alg. 1's order)
        int yt = 1;
        if (!yevery && k >= 2) {
          const int last = k - ((k - 1) % 3 == 0 ? 3 : (k - 1) % 3);   // the latest group step < k (1 = init)
          yt = ((k - 1) % 3 == 0 || k == K - 1) ? k - last : 0;
        }
        kw<<<gw, SP_WARPS * 32, 0, st>>>(cptr, crow, cval, m, n, nblk, Z, prev, k == 1 ? nullptr : prev2, out, Yb, P, k,
                                         yt);
      }
      ++L;
      if (hook) hook(hook_ctx, CPA_SVT_PH_SPARSE_W, 0);
      prev2 = prev;
      prev = (k & 1) ? (const double*)Wb : (const double*)Wa;
    }
    dim3 ub((unsigned)((n + UT - 1) / UT), (unsigned)nblk, (unsigned)((RB + UT - 1) / UT));
    k_unblock<<<ub, dim3(32, 8), 0, st>>>(Yb, rows, n, Y, ldy); ++L;
  }
#undef SPCK
  if (launches) *launches += L;
  return cudaGetLastError();
}

}  // namespace cpa
