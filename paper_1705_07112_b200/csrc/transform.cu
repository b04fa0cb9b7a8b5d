// NEXT-2, DCT variant: Phi = T G T^T with T the orthonormal
// DCT-II of the Gram index, line 2 thresholds its components (eq. threshold_components,
// keep |Phi_ij| >= epsilon; epsilon absolute or the k-th largest |Phi_ij|,
// PAPER.md:968-975), and lines 5-11 run on the sparse Phi_ (CSR) against dense Psi_k:
//   Psi_k(i, :) = (4/L) sum_p Phi_(i, col_p) Psi_{k-1}(col_p, :) - 2 Psi_{k-1}(i, :) - Psi_{k-2}(i, :)
//   H(i, :)    += c_k Psi_k(i, :)
// one CTA per row, threads across the row (every gathered Psi_{k-1} row is a coalesced read),
// the nonzeros of a row summed in column order: deterministic.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace cpa {

// keys = bit patterns of |Phi| (monotone in the value for non-negative doubles)
__global__ void k_abs_keys(const double* __restrict__ A, int64_t N, unsigned long long* __restrict__ keys) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
    keys[e] = (unsigned long long)__double_as_longlong(fabs(A[e]));
}
// epsilon: absolute (mode 1) or the k-th largest |Phi| from the descending sort (mode 2)
__global__ void k_set_eps(const unsigned long long* __restrict__ sorted, int64_t k, double eps_abs, int mode,
                          double* __restrict__ eps) {
  *eps = mode == 2 ? __longlong_as_double((long long)sorted[k - 1]) : eps_abs;
}
// Phi_ in place (|x| < eps -> 0) and the kept count of each row (one warp per row)
__global__ void k_thresh_rows(double* __restrict__ A, int64_t s, const double* __restrict__ eps_p,
                              int64_t* __restrict__ cnt) {
  const double eps = *eps_p;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < s; r += nw) {
    int64_t c_row = 0;
    for (int64_t j0 = 0; j0 < s; j0 += 32) {
      const int64_t j = j0 + lane;
      bool keep = false;
      if (j < s) {
        const double x = A[r * s + j];
        keep = fabs(x) >= eps;
        if (!keep) A[r * s + j] = 0.0;
      }
      c_row += __popc(__ballot_sync(0xffffffffu, keep));
    }
    if (lane == 0) cnt[r] = c_row;
  }
}
// exclusive scan of the s row counts into row_ptr[0..s] (one CTA, fixed order)
__global__ void k_scan_rows(const int64_t* __restrict__ cnt, int64_t s, int64_t* __restrict__ rp) {
  __shared__ int64_t part[1024];
  const int64_t per = (s + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * per, e = min(s, b + per);
  int64_t acc = 0;
  for (int64_t i = b; i < e; ++i) acc += cnt[i];
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      const int64_t v = part[t];
      part[t] = run;
      run += v;
    }
    rp[s] = run;
  }
  __syncthreads();
  int64_t run = part[threadIdx.x];
  for (int64_t i = b; i < e; ++i) {
    rp[i] = run;
    run += cnt[i];
  }
}
// CSR of Phi_, columns ascending within each row (one warp per row, ballot prefix)
__global__ void k_csr_fill(const double* __restrict__ A, int64_t s, const double* __restrict__ eps_p,
                           const int64_t* __restrict__ rp, int32_t* __restrict__ col, double* __restrict__ val) {
  const double eps = *eps_p;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < s; r += nw) {
    int64_t pos = rp[r];
    for (int64_t j0 = 0; j0 < s; j0 += 32) {
      const int64_t j = j0 + lane;
      double x = 0.0;
      bool keep = false;
      if (j < s) {
        x = A[r * s + j];
        keep = fabs(x) >= eps;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int64_t o = pos + __popc(m & ((1u << lane) - 1u));
        col[o] = (int32_t)j;
        val[o] = x;
      }
      pos += __popc(m);
    }
  }
}
// one recurrence step on the sparse Phi_ (see the file comment); k = 2 uses Psi_0 = I
__global__ void __launch_bounds__(256) k_sparse_sym_step(int64_t s, const int64_t* __restrict__ rp,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ Wp, double* __restrict__ Wo,
                                                         double* __restrict__ H, const SeriesParams* __restrict__ P,
                                                         int k, int last) {
  const double s4 = 2.0 * P->scale2, ck = P->c[k];
  for (int64_t r = blockIdx.x; r < s; r += gridDim.x) {
    const int64_t p0 = rp[r], p1 = rp[r + 1];
    for (int64_t j = threadIdx.x; j < s; j += blockDim.x) {
      double acc = 0.0;
      for (int64_t p = p0; p < p1; ++p) acc = fma(val[p], Wp[(int64_t)col[p] * s + j], acc);
      const double wpp = k == 2 ? (r == j ? 1.0 : 0.0) : Wo[r * s + j];
      const double w = s4 * acc - 2.0 * Wp[r * s + j] - wpp;   // Psi_k = 2 B_hat Psi_{k-1} - Psi_{k-2}
      H[r * s + j] += ck * w;                                    // H += c_k Psi_k
      if (!last) Wo[r * s + j] = w;
    }
  }
}

// NEXT-2 block DCT (reading R24): C = blockdiag(C_8, ..., C_8, C_r), C_w the
// orthonormal DCT-II of size w (C_w[k][j] = a_k cos(pi (2j + 1) k / (2w)), a_0 = sqrt(1/w),
// a_k = sqrt(2/w)), r = s mod 8 for a ragged last block.  out = C A C^T (inverse = 0) or
// C^T A C (inverse = 1) for an s x s A: one 64-thread CTA per 8 x 8 block pair,
// out_IJ = C_wI A_IJ C_wJ^T (or the transposed factors) -- 16 FMAs per element instead of
// two dense s^3 products.  Fixed summation order.
__global__ void __launch_bounds__(64) k_block_dct_sandwich(const double* __restrict__ A, double* __restrict__ out,
                                                           int64_t s, int inverse) {
  __shared__ double sA[8][8], sT[8][8], sCi[8][8], sCj[8][8];
  const int64_t nb = (s + 7) / 8;
  const int64_t bi = blockIdx.x / nb, bj = blockIdx.x % nb;
  const int64_t i0 = bi * 8, j0 = bj * 8;
  const int wi = (int)min((int64_t)8, s - i0), wj = (int)min((int64_t)8, s - j0);
  const int r = threadIdx.x >> 3, c = threadIdx.x & 7;
  auto dctc = [](int w, int k, int j) {   // C_w[k][j]
    if (k >= w || j >= w) return 0.0;
    const double a = k == 0 ? sqrt(1.0 / w) : sqrt(2.0 / w);
    return a * cos(3.141592653589793238462643383279502884 * (double)((2 * j + 1) * k) / (double)(2 * w));
  };
  sCi[r][c] = dctc(wi, r, c);
  sCj[r][c] = dctc(wj, r, c);
  sA[r][c] = (r < wi && c < wj) ? A[(i0 + r) * s + j0 + c] : 0.0;
  __syncthreads();
  // T = F_I A_IJ, F_I = C_wI (forward) or C_wI^T (inverse)
  double t = 0.0;
  for (int p = 0; p < 8; ++p) t = fma(inverse ? sCi[p][r] : sCi[r][p], sA[p][c], t);
  sT[r][c] = t;
  __syncthreads();
  // out_IJ = T F_J^T
  double o = 0.0;
  for (int q = 0; q < 8; ++q) o = fma(sT[r][q], inverse ? sCj[q][c] : sCj[c][q], o);
  if (r < wi && c < wj) out[(i0 + r) * s + j0 + c] = o;
}

cudaError_t block_dct_sandwich(const double* A, double* out, int64_t s, int inverse, cudaStream_t st) {
  const int64_t nb = (s + 7) / 8;
  if (nb * nb > INT32_MAX) return cudaErrorInvalidValue;
  k_block_dct_sandwich<<<(unsigned)(nb * nb), 64, 0, st>>>(A, out, s, inverse);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------- host
size_t dct_eps_scratch_bytes(int64_t s) {
  const size_t N = (size_t)s * s;
  size_t temp = 0;
  cub::DeviceRadixSort::SortKeysDescending(nullptr, temp, (const unsigned long long*)nullptr,
                                           (unsigned long long*)nullptr, (int)N);
  // keys in / out | temp | row counts | row_ptr | eps | col | val
  return 2 * N * 8 + temp + 256 + (size_t)(s + 1) * 8 * 2 + 64 + N * 4 + N * 8 + 1024;
}

// Threshold Phi (s x s, in place) and build its CSR in `scratch`; mode 1 absolute eps, 2 top-k.
cudaError_t dct_eps_threshold(double* Phi, int64_t s, int mode, double eps_value, void* scratch, int num_sms,
                              cudaStream_t st, const int64_t** rp_out, const int32_t** col_out,
                              const double** val_out) {
  const size_t N = (size_t)s * s;
  char* b = (char*)scratch;
  auto al = [](size_t v) { return (v + 255) / 256 * 256; };
  unsigned long long* kin = (unsigned long long*)b;
  b += al(N * 8);
  unsigned long long* kout = (unsigned long long*)b;
  b += al(N * 8);
  size_t temp = 0;
  cub::DeviceRadixSort::SortKeysDescending(nullptr, temp, kin, kout, (int)N);
  void* tmp = b;
  b += al(temp);
  int64_t* cnt = (int64_t*)b;
  b += al((size_t)(s + 1) * 8);
  int64_t* rp = (int64_t*)b;
  b += al((size_t)(s + 1) * 8);
  double* eps = (double*)b;
  b += 256;
  int32_t* col = (int32_t*)b;
  b += al(N * 4);
  double* val = (double*)b;
  cudaError_t e;
  if (mode == 2) {
    const int64_t k = (int64_t)eps_value;
    if (k < 1) return cudaErrorInvalidValue;
    k_abs_keys<<<num_sms * 8, 256, 0, st>>>(Phi, (int64_t)N, kin);
    e = cub::DeviceRadixSort::SortKeysDescending(tmp, temp, kin, kout, (int)N, 0, 64, st);
    if (e != cudaSuccess) return e;
    k_set_eps<<<1, 1, 0, st>>>(kout, k < (int64_t)N ? k : (int64_t)N, 0.0, 2, eps);
  } else {
    k_set_eps<<<1, 1, 0, st>>>(kout, 1, eps_value, 1, eps);
  }
  k_thresh_rows<<<num_sms * 8, 256, 0, st>>>(Phi, s, eps, cnt);
  k_scan_rows<<<1, 1024, 0, st>>>(cnt, s, rp);
  k_csr_fill<<<num_sms * 8, 256, 0, st>>>(Phi, s, eps, rp, col, val);
  *rp_out = rp;
  *col_out = col;
  *val_out = val;
  return cudaGetLastError();
}

cudaError_t dct_sparse_steps(int64_t s, const int64_t* rp, const int32_t* col, const double* val, double* Wa,
                             double* Wb, double* H, const SeriesParams* P, int K, int num_sms, cudaStream_t st) {
  // W_1 in Wa (dense_sym_init); W_k -> (k odd ? Wa : Wb) over W_{k-2}
  for (int k = 2; k < K; ++k) {
    const double* src = ((k - 1) & 1) ? Wa : Wb;
    double* out = (k & 1) ? Wa : Wb;
    const int64_t grid = s < (int64_t)num_sms * 16 ? s : (int64_t)num_sms * 16;
    k_sparse_sym_step<<<(unsigned)grid, 256, 0, st>>>(s, rp, col, val, src, out, H, P, k, k == K - 1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace cpa
