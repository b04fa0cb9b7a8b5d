// Batched fp32 path (BASELINE configs[2]: 65536 patch-group matrices, 64 x 64):
// the whole of Alg. 1 (T = I, eps = 0) for one matrix per
// 64-thread CTA (two warps), entirely on chip: X is read once, Y written once.
//
//   Gram G = A A^T (A = X if m <= n else X^T)   -- FFMA, smem operands
//   lambda_hat: T power steps on G (reading R6)  -- fp32, fixed order
//   c_k: K-node Chebyshev-Gauss rule        -- fp64 per matrix
//   W_1 = (2/L) G A - A; W_k = (4/L) G W_{k-1} - 2 W_{k-1} - W_{k-2}; Y += c_k W_k
//                                                             -- fused per step
//
// Every thread owns an 8x8 output tile (rows {4ty..4ty+3, 32+4ty..}, cols
// {4tx.., 32+4tx..}); W_{k-2} and Y stay in registers, G and W_{k-1} in
// shared memory (row stride 68 floats: conflict-free LDS.128 operand loads).
// Problems smaller than 64 x 64 are zero-padded (padding stays exactly 0).
#include "common.cuh"

namespace cpa {

constexpr int BT = 64;    // threads per matrix
constexpr int LDS = 68;   // smem row stride (floats)
constexpr int BKMAX = 128;  // largest K of the batched kernel (shared-memory budget: 4 CTAs / SM)

struct BatchedArgs {
  int64_t batch;
  int m, n;
  const float* X;
  float* Y;
  cpa_svt_kernel kern;
  int K, T;
  double safety, lam_override;
  float* lambda_out;
};

// acc[r][c] += sum_k A[k][row(r)] * B[k][col(c)], A/B in smem with stride LDS.
__device__ __forceinline__ void gemm64(const float* __restrict__ A, const float* __restrict__ B, int ty, int tx,
                                       float (&acc)[8][8]) {
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
#pragma unroll 1
  for (int k = 0; k < 64; ++k) {
    const float4 a0 = *reinterpret_cast<const float4*>(A + k * LDS + 4 * ty);
    const float4 a1 = *reinterpret_cast<const float4*>(A + k * LDS + 32 + 4 * ty);
    const float4 b0 = *reinterpret_cast<const float4*>(B + k * LDS + 4 * tx);
    const float4 b1 = *reinterpret_cast<const float4*>(B + k * LDS + 32 + 4 * tx);
    const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
  }
}

__device__ __forceinline__ int row_of(int ty, int r) { return r < 4 ? 4 * ty + r : 32 + 4 * ty + (r - 4); }
__device__ __forceinline__ int col_of(int tx, int c) { return c < 4 ? 4 * tx + c : 32 + 4 * tx + (c - 4); }

__global__ void __launch_bounds__(BT, 4) k_batched_f32(BatchedArgs a) {
  extern __shared__ __align__(16) float bsm[];
  float* sG = bsm;                // 64 x LDS
  float* sW = bsm + 64 * LDS;     // 64 x LDS
  float* sY = bsm + 128 * LDS;    // Y tile of thread t, element e at sY[e * BT + t] (conflict-free)
  __shared__ float sV[64];
  __shared__ float sRed[2];
  __shared__ double sH[BKMAX];
  __shared__ float sC[BKMAX];
  __shared__ double sLam[4];

  const int tid = threadIdx.x, ty = tid >> 3, tx = tid & 7, lane = tid & 31, warp = tid >> 5;
  const bool left = a.m <= a.n;
  const int s = left ? a.m : a.n;       // Gram side
  const int L = left ? a.n : a.m;       // long side
  const int K = a.K;
  const int64_t mn = (int64_t)a.m * a.n;

  for (int64_t b = blockIdx.x; b < a.batch; b += gridDim.x) {
    const float* X = a.X + b * mn;
    // ---- load A (s x L) into sW row-major and A^T into sG ([l][i]); zero padding
    for (int e = tid; e < 64 * 64; e += BT) {
      const int i = e >> 6, j = e & 63;  // A(i, j)
      float v = 0.f;
      if (i < s && j < L) v = left ? __ldg(X + (int64_t)i * a.n + j) : __ldg(X + (int64_t)j * a.n + i);
      sW[i * LDS + j] = v;
      sG[j * LDS + i] = v;
    }
    __syncthreads();
    float acc[8][8];
    // ---- Gram: G(i, j) = sum_l A(i, l) A(j, l)   (A^T in sG is [l][i])
    gemm64(sG, sG, ty, tx, acc);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) sG[row_of(ty, r) * LDS + col_of(tx, c)] = acc[r][c];
    __syncthreads();

    // ---- Lambda_max: power iteration (fp32, fixed reduction order) or override
    double lam_hat;
    if (a.lam_override > 0.0) {
      lam_hat = a.lam_override / a.safety;
    } else {
      sV[tid] = tid < s ? rsqrtf((float)s) : 0.f;
      __syncthreads();
      float nrm = 0.f;
      for (int t = 0; t < a.T; ++t) {
        float u = 0.f;
        for (int j = 0; j < 64; ++j) u = fmaf(sG[j * LDS + tid], sV[j], u);  // G symmetric: column tid
        float sq = u * u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) sRed[warp] = sq;
        __syncthreads();
        nrm = sqrtf(sRed[0] + sRed[1]);
        if (!(nrm > 0.f)) break;
        sV[tid] = u / nrm;
        __syncthreads();
      }
      lam_hat = nrm > 0.f ? (double)nrm : 0.0;
    }
    // ---- coefficients (fp64) for this matrix's Lambda_max
    const bool degen = !(lam_hat > kDegenerateLambda);
    const double lam = a.safety * lam_hat;
    const double tau = resolve_tau(a.kern, sqrt(lam_hat));
    for (int l = tid; l < K; l += BT) sH[l] = h_response(a.kern, lam / 2.0 * (cos(cheb_theta(l + 1, K)) + 1.0), tau);
    __syncthreads();
    for (int k = tid; k < K; k += BT) {
      double acc_c = 0.0;
      for (int l = 0; l < K; ++l) acc_c += cos(k * cheb_theta(l + 1, K)) * sH[l];
      sC[k] = degen ? 0.f : (float)(2.0 / K * acc_c);
    }
    if (tid == 0) sLam[0] = lam;
    __syncthreads();
    if (tid == 0 && a.lambda_out) a.lambda_out[b] = (float)lam;
    const float s2 = degen ? 0.f : (float)(2.0 / lam);
    const float s4 = 2.f * s2;

    // ---- recurrence: W_0 = A (in sW), wpp = own tile of W_{k-2} (registers), Y own tile (sY)
    float wpp[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) wpp[r][c] = sW[row_of(ty, r) * LDS + col_of(tx, c)];
    gemm64(sG, sW, ty, tx, acc);  // G symmetric: sG[k][i] = G(i, k)
    {
      const float h0 = 0.5f * sC[0], c1 = sC[1];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float w = s2 * acc[r][c] - wpp[r][c];  // W_1 = B_hat A
          sY[(r * 8 + c) * BT + tid] = h0 * wpp[r][c] + c1 * w;  // Y = c0/2 W_0 + c1 W_1
          acc[r][c] = w;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) sW[row_of(ty, r) * LDS + col_of(tx, c)] = acc[r][c];
    __syncthreads();
    for (int k = 2; k < K; ++k) {
      gemm64(sG, sW, ty, tx, acc);
      const float ck = sC[k];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float wp = sW[row_of(ty, r) * LDS + col_of(tx, c)];
          const float w = s4 * acc[r][c] - 2.f * wp - wpp[r][c];  // W_k = 2 B_hat W_{k-1} - W_{k-2}
          float* yp = sY + (r * 8 + c) * BT + tid;
          *yp = fmaf(ck, w, *yp);                                 // Y += c_k W_k
          wpp[r][c] = wp;
          acc[r][c] = w;
        }
      if (k + 1 < K) {
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) sW[row_of(ty, r) * LDS + col_of(tx, c)] = acc[r][c];
        __syncthreads();
      }
    }
    // ---- store Y (= Y_A if left, Y_A^T if right)
    float* Yb = a.Y + b * mn;
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int i = row_of(ty, r), j = col_of(tx, c);
        if (i < s && j < L) {
          const float yv = sY[(r * 8 + c) * BT + tid];
          if (left) Yb[(int64_t)i * a.n + j] = yv;
          else Yb[(int64_t)j * a.n + i] = yv;
        }
      }
    __syncthreads();
  }
}

cudaError_t launch_batched_f32(int64_t batch, int m, int n, const float* X, float* Y, const cpa_svt_kernel& k,
                               int K, int T, double safety, double lam_override, float* lambda_out, int num_sms,
                               cudaStream_t st, int* launches) {
  if (K > BKMAX) return cudaErrorNotSupported;
  BatchedArgs a{batch, m, n, X, Y, k, K, T, safety, lam_override, lambda_out};
  const size_t smem = (size_t)(128 * LDS + 64 * BT) * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(k_batched_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_batched_f32, BT, smem);
  if (e != cudaSuccess) return e;
  int64_t grid = (int64_t)num_sms * (per_sm > 0 ? per_sm : 1) * 64;
  if (grid > batch) grid = batch;
  k_batched_f32<<<(unsigned)grid, BT, smem, st>>>(a);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace cpa
