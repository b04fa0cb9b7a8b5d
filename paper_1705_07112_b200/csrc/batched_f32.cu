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
  const double* costab;   // cos(k theta_l), K x K, shared by every matrix (depends on K only)
};

// cos(k theta_l), theta_l = pi (l - 1/2) / K, for the coefficient rule of line 4
__global__ void k_costab(double* tab, int K) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < K * K; e += gridDim.x * blockDim.x)
    tab[e] = cos((e / K) * cheb_theta(e % K + 1, K));
}

// acc[r][c] = sum_k A[k][row(r)] * B[k][col(c)], A/B in smem with stride LDS.
// Packed dual-FP32 FMA (fma.rn.f32x2 -> SASS FFMA2 with a broadcast scalar operand):
// each instruction updates two adjacent columns, 1.6x the rate of 3-register FFMA on
// B200 (measured 64 vs 40 TFLOP/s) and bitwise the same per-element fma.rn.
__device__ __forceinline__ unsigned long long pack2(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
}
__device__ __forceinline__ void gemm64(const float* __restrict__ A, const float* __restrict__ B, int ty, int tx,
                                       float (&acc)[8][8]) {
  unsigned long long accp[8][4];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) accp[r][c] = 0ull;
#pragma unroll 2
  for (int k = 0; k < 64; ++k) {
    const float4 a0 = *reinterpret_cast<const float4*>(A + k * LDS + 4 * ty);
    const float4 a1 = *reinterpret_cast<const float4*>(A + k * LDS + 32 + 4 * ty);
    const float4 b0 = *reinterpret_cast<const float4*>(B + k * LDS + 4 * tx);
    const float4 b1 = *reinterpret_cast<const float4*>(B + k * LDS + 32 + 4 * tx);
    const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const unsigned long long b[4] = {pack2(b0.x, b0.y), pack2(b0.z, b0.w), pack2(b1.x, b1.y), pack2(b1.z, b1.w)};
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const unsigned long long aa = pack2(a[r], a[r]);
#pragma unroll
      for (int c = 0; c < 4; ++c) asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(accp[r][c]) : "l"(aa), "l"(b[c]));
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) unpack2(accp[r][c], acc[r][2 * c], acc[r][2 * c + 1]);
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
  // 64 x 64 matrices at 16-byte aligned addresses take the vector load path
  const bool full64 = a.m == 64 && a.n == 64 && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);

  for (int64_t b = blockIdx.x; b < a.batch; b += gridDim.x) {
    const float* X = a.X + b * mn;
    // ---- load A (s x L) into sW row-major and A^T into sG ([l][i]); zero padding.
    // All of the thread's global loads are issued before the first store (one round trip).
    if (full64) {
      float4 v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = __ldg(reinterpret_cast<const float4*>(X) + q * BT + tid);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = (q * BT + tid) * 4, i = e >> 6, j = e & 63;  // X(i, j..j+3), A = X
        *reinterpret_cast<float4*>(sW + i * LDS + j) = v[q];
        sG[j * LDS + i] = v[q].x; sG[(j + 1) * LDS + i] = v[q].y;
        sG[(j + 2) * LDS + i] = v[q].z; sG[(j + 3) * LDS + i] = v[q].w;
      }
    } else {
      for (int e0 = tid; e0 < 64 * 64; e0 += 8 * BT) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = e0 + q * BT, i = e >> 6, j = e & 63;  // A(i, j)
          v[q] = 0.f;
          if (e < 64 * 64 && i < s && j < L) v[q] = left ? __ldg(X + (int64_t)i * a.n + j) : __ldg(X + (int64_t)j * a.n + i);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = e0 + q * BT, i = e >> 6, j = e & 63;
          if (e < 64 * 64) {
            sW[i * LDS + j] = v[q];
            sG[j * LDS + i] = v[q];
          }
        }
      }
    }
    __syncthreads();
    float acc[8][8];
    // ---- Gram: G(i, j) = sum_l A(i, l) A(j, l)   (A^T in sG is [l][i])
    gemm64(sG, sG, ty, tx, acc);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        *reinterpret_cast<float4*>(sG + row_of(ty, r) * LDS + hh * 32 + 4 * tx) =
            make_float4(acc[r][4 * hh], acc[r][4 * hh + 1], acc[r][4 * hh + 2], acc[r][4 * hh + 3]);
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
        float u0 = 0.f, u1 = 0.f, u2 = 0.f, u3 = 0.f;  // four chains: the product is latency-bound
#pragma unroll 4
        for (int j = 0; j < 64; j += 4) {              // G symmetric: column tid
          u0 = fmaf(sG[j * LDS + tid], sV[j], u0);
          u1 = fmaf(sG[(j + 1) * LDS + tid], sV[j + 1], u1);
          u2 = fmaf(sG[(j + 2) * LDS + tid], sV[j + 2], u2);
          u3 = fmaf(sG[(j + 3) * LDS + tid], sV[j + 3], u3);
        }
        const float u = (u0 + u1) + (u2 + u3);
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
      const double* ct = a.costab + k * K;
      for (int l = 0; l < K; ++l) acc_c += __ldg(ct + l) * sH[l];
      sC[k] = degen ? 0.f : (float)(2.0 / K * acc_c);
    }
    if (tid == 0) sLam[0] = lam;
    __syncthreads();
    if (tid == 0 && a.lambda_out) a.lambda_out[b] = (float)lam;
    const float s2 = degen ? 0.f : (float)(2.0 / lam);
    const float s4 = 2.f * s2;

    // ---- recurrence: W_0 = A (in sW), wpp = own tile of W_{k-2} (registers), Y own tile (sY).
    // The thread's tile is two 4-wide column groups per row: every shared-memory access
    // of the epilogue is a 16-byte vector (the scalar version was bank-conflict bound).
    float4* sY4 = reinterpret_cast<float4*>(sY);  // [16 groups][BT threads]
    float wpp[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const float4 v = *reinterpret_cast<const float4*>(sW + row_of(ty, r) * LDS + hh * 32 + 4 * tx);
        wpp[r][4 * hh] = v.x; wpp[r][4 * hh + 1] = v.y; wpp[r][4 * hh + 2] = v.z; wpp[r][4 * hh + 3] = v.w;
      }
    gemm64(sG, sW, ty, tx, acc);  // G symmetric: sG[k][i] = G(i, k)
    {
      const float h0 = 0.5f * sC[0], c1 = sC[1];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float y[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = 4 * hh + q;
            const float w = s2 * acc[r][c] - wpp[r][c];  // W_1 = B_hat A
            y[q] = h0 * wpp[r][c] + c1 * w;               // Y = c0/2 W_0 + c1 W_1
            acc[r][c] = w;
          }
          sY4[(r * 2 + hh) * BT + tid] = make_float4(y[0], y[1], y[2], y[3]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        *reinterpret_cast<float4*>(sW + row_of(ty, r) * LDS + hh * 32 + 4 * tx) =
            make_float4(acc[r][4 * hh], acc[r][4 * hh + 1], acc[r][4 * hh + 2], acc[r][4 * hh + 3]);
    __syncthreads();
    for (int k = 2; k < K; ++k) {
      gemm64(sG, sW, ty, tx, acc);
      const float ck = sC[k];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const float4 wp4 = *reinterpret_cast<const float4*>(sW + row_of(ty, r) * LDS + hh * 32 + 4 * tx);
          float4 y4 = sY4[(r * 2 + hh) * BT + tid];
          const float wpv[4] = {wp4.x, wp4.y, wp4.z, wp4.w};
          float yv[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = 4 * hh + q;
            const float w = s4 * acc[r][c] - 2.f * wpv[q] - wpp[r][c];  // W_k = 2 B_hat W_{k-1} - W_{k-2}
            yv[q] = fmaf(ck, w, yv[q]);                                 // Y += c_k W_k
            wpp[r][c] = wpv[q];
            acc[r][c] = w;
          }
          sY4[(r * 2 + hh) * BT + tid] = make_float4(yv[0], yv[1], yv[2], yv[3]);
        }
      if (k + 1 < K) {
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
            *reinterpret_cast<float4*>(sW + row_of(ty, r) * LDS + hh * 32 + 4 * tx) =
                make_float4(acc[r][4 * hh], acc[r][4 * hh + 1], acc[r][4 * hh + 2], acc[r][4 * hh + 3]);
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
          const float yv = sY[((r * 2 + (c >> 2)) * BT + tid) * 4 + (c & 3)];
          if (left) Yb[(int64_t)i * a.n + j] = yv;
          else Yb[(int64_t)j * a.n + i] = yv;
        }
      }
    __syncthreads();
  }
}

cudaError_t launch_batched_f32(int64_t batch, int m, int n, const float* X, float* Y, const cpa_svt_kernel& k,
                               int K, int T, double safety, double lam_override, float* lambda_out, int num_sms,
                               cudaStream_t st, int* launches, double* costab) {
  if (K > BKMAX) return cudaErrorNotSupported;
  k_costab<<<(K * K + 255) / 256, 256, 0, st>>>(costab, K);
  if (launches) ++*launches;
  BatchedArgs a{batch, m, n, X, Y, k, K, T, safety, lam_override, lambda_out, costab};
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
