/*
 * cpa_svt.h -- C ABI of the B200-native CPA singular-value shrinkage library.
 *
 * Operation (Algorithm 1 with T = I and epsilon = 0; the
 * apply-to-X form of PAPER.md:278-307 eq. sing_shrink_from_eig_shrink):
 *
 *     Y = G_hat(X) = X H_hat(X^T X)        if m >  n   ("right", Gram n x n)
 *     Y = G_hat(X) = H_hat(X X^T) X        if m <= n   ("left",  Gram m x m)
 *
 * with H_hat(Phi) = c_0/2 Id + sum_{k=1}^{K-1} c_k Psi_k(B_hat),
 * B_hat = (2/Lambda_max) Phi - Id, the three-term recurrence
 * Psi_k = 2 B_hat Psi_{k-1} - Psi_{k-2}, and the K
 * Chebyshev-Gauss coefficients of PAPER.md:233 / 363 for the response h of
 * PAPER.md:496-519 (hard / soft / weighted soft).  Two evaluation orders of the
 * same polynomial are built (CPA_SVT_OPT_FORM):
 *   - the Alg. 1 s x s form (default for K > 2): the three-term recurrence on the
 *     s x s Gram, Psi_0 = Id, Psi_1 = B_hat, Psi_k = 2 B_hat Psi_{k-1} - Psi_{k-2}
 *     (PAPER.md:364-370), H_hat = c_0/2 Id + sum_k c_k Psi_k formed on the device,
 *     then ONE product Y = H_hat X (or X H_hat), Alg. 1 line 12.  For small s the
 *     same products run as two independent Chebyshev chains (even / odd k:
 *     Psi_k = 2 Psi_2 Psi_{k-2} - Psi_{|k-4|}, reading R28), with Psi_2
 *     formed from the power iteration's G^2 when that squaring ran (R29);
 *   - the apply-to-X form (line 12 distributed over the sum):
 *     W_0 = X,  W_1 = (2/L) G X - X,  W_k = (4/L) G W_{k-1} - 2 W_{k-1} - W_{k-2},
 *     Y = c_0/2 W_0 + c_1 W_1 + sum_{k>=2} c_k W_k.
 * Every recurrence step is one fused kernel (product + update + accumulation).
 *
 * Conventions (all entry points):
 *   - Every call returns cpa_svt_status; CPA_SVT_OK == 0.  Arguments are
 *     validated before any device work; on a non-OK status no output buffer
 *     has been written unless the status is CPA_SVT_E_CUDA / E_NCCL / E_DIVERGED.
 *   - Matrices are ROW-MAJOR with a leading dimension in ELEMENTS (ld >= cols).
 *   - X, Y, CSR arrays and lambda_out are DEVICE pointers on the handle's
 *     device, owned by the caller, valid until the handle's stream has
 *     executed the call.  Kernel specs, coefficient arrays, lambda and info
 *     structs are HOST pointers read (or written) before the call returns.
 *   - All device work is ordered on the handle's stream and is asynchronous,
 *     EXCEPT when `info` is non-NULL or `lam` asks for lambda back
 *     (lam->want_lambda) or CPA_SVT_OPT_DIVERGENCE is 2: then the call
 *     synchronises the stream before returning.  cpa_svt_apply_host is always
 *     synchronous.
 *   - Y must not alias X.  Y may be any caller buffer of the same shape.
 *   - Empty inputs are valid (dims < 0 are E_ARG): an X with m or n zero (a batch
 *     of zero matrices, a CSR row range with no rows) has an empty Y; the call
 *     validates its other arguments and returns CPA_SVT_OK without device work
 *     (X and Y may then be NULL).  In a sharded call a rank's block of the long
 *     dimension may be empty (long extent below the world size): that rank takes
 *     part in every collective with a zero partial Gram and writes nothing; the
 *     short dimension is global and must be >= 1.
 *   - The handle owns its workspace (Gram, two recurrence buffers, power
 *     iteration scratch, series parameters), grows it lazily and frees it in
 *     cpa_svt_free.  A handle is not thread-safe; use one per host thread.
 *   - Results are deterministic run to run for a fixed shape and world size
 *     (fixed reduction orders, no floating-point atomics on the dense path).
 */
#ifndef CPA_SVT_H
#define CPA_SVT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CPA_SVT_VERSION_MAJOR 0
#define CPA_SVT_VERSION_MINOR 1
/* Largest order K supported (number of coefficients c_0..c_{K-1}). */
#define CPA_SVT_KMAX 512

typedef struct cpa_svt_handle cpa_svt_handle; /* opaque */

typedef enum {
  CPA_SVT_OK = 0,
  CPA_SVT_E_ARG = 1,          /* NULL pointer, K < 2 or K > KMAX, dims < 0, ld < cols, Y aliases X, bad enum */
  CPA_SVT_E_DOMAIN = 2,       /* lambda_max override < 0 or non-finite, tau < 0, weight parameters invalid */
  CPA_SVT_E_DIVERGED = 3,     /* ||Y||_F > 1e3 sum|c_k| ||X||_F, or Y not finite (the series is
                                 bounded only for a Gram spectrum inside [0, Lambda_max]):
                                 Y HAS been written (and is meaningless).  Reported by calls that synchronise
                                 (info / want_lambda / apply_host, or CPA_SVT_OPT_DIVERGENCE = 2). */
  CPA_SVT_E_CUDA = 4,         /* a CUDA runtime call failed (cpa_svt_last_error has the text) */
  CPA_SVT_E_NCCL = 5,         /* an NCCL call failed or NCCL could not be loaded */
  CPA_SVT_E_NOMEM = 6,        /* workspace allocation failed */
  CPA_SVT_E_UNSUPPORTED = 7   /* valid request this build does not implement */
} cpa_svt_status;

/* Response family h(x; w(x)/rho, tau) of PAPER.md:496-519. */
typedef enum {
  CPA_SVT_HARD = 0,  /* h(x; 0, tau):          h = 1            if sqrt(x) > tau, else 0 */
  CPA_SVT_SOFT = 1,  /* h(x; 1/rho, 1/rho):    h = 1 - tau/sqrt(x) if sqrt(x) > tau, else 0 */
  CPA_SVT_WSOFT = 2  /* h(x; w(x)/rho, w/rho): h = 1 - w/sqrt(x)   if sqrt(x) > w,   else 0,
                        w(x) = w_c / (sqrt(max(x - w_shift, 0)) + w_eps)  (reading R10) */
} cpa_svt_kind;

typedef struct {
  int32_t kind;          /* cpa_svt_kind */
  int32_t tau_relative;  /* HARD/SOFT: if nonzero, the threshold is tau * sigma_max_hat, with
                            sigma_max_hat = sqrt(lambda_hat) (power-iteration estimate, reading R7) */
  double tau;            /* HARD/SOFT threshold on singular values, >= 0 */
  double w_c, w_shift, w_eps; /* WSOFT weight parameters, w_c >= 0, w_shift >= 0, w_eps > 0 */
} cpa_svt_kernel;

typedef enum { CPA_SVT_F64 = 0, CPA_SVT_F32 = 1 } cpa_svt_dtype;

typedef enum {
  CPA_SVT_MATH_NATIVE = 0, /* f64 only: DMMA (mma.sync f64) tensor tiles.  f32 + NATIVE is not built
                              (CPA_SVT_E_UNSUPPORTED): fp32 data runs on the tensor cores (below) */
  CPA_SVT_MATH_TF32 = 1,   /* f32 data, single-pass tcgen05 kind::tf32, operands rounded to nearest TF32
                              (Gram in 3xTF32).  Reduced accuracy: ~0.5-2e-4 relative Frobenius error
                              measured -- NOT the <= 1e-4 fp32 bar of the north star; use 3XTF32 for that */
  CPA_SVT_MATH_3XTF32 = 2  /* f32 data, tcgen05 kind::tf32 hi/lo split (near-fp32 accuracy, <= 1e-4) */
} cpa_svt_math;

/* Lambda_max of the Gram (Alg. 1 line 3): power iteration
 * v_0 = 1/sqrt(s), v_t = G v_{t-1}/||G v_{t-1}||, lambda_hat = ||G v_{T-1}||_2
 * after T = power_iters products; Lambda_max = safety * lambda_hat (reading R6).
 * If lambda_max > 0 on input the power iteration is skipped and that value is
 * used; then lambda_hat := lambda_max / safety.  On return (only if
 * want_lambda != 0) lambda_hat / lambda_max hold the values used. */
typedef struct {
  int32_t power_iters;   /* T >= 1 (ignored when lambda_max > 0 on input) */
  int32_t want_lambda;   /* nonzero: synchronise and write back lambda_hat / lambda_max */
  double safety;         /* >= 1; 1.01 in every BASELINE config */
  double lambda_max;     /* in: > 0 to override; out: value used */
  double lambda_hat;     /* out */
} cpa_svt_lambda;

/* Diagnostics (host).  Filled only when passed non-NULL; forces a sync. */
typedef struct {
  double lambda_hat, lambda_max, sigma_max_hat, tau_used;
  int32_t side;          /* 0 = left (G = X X^T), 1 = right (G = X^T X) */
  int32_t degenerate;    /* 1 if lambda_hat <= 1e-300: Y = 0 */
  float ms_gram, ms_allreduce, ms_power, ms_recurrence, ms_total;
  int32_t kernel_launches;  /* device kernels this call launched */
  int32_t form;          /* dense form that ran: 1 = apply-to-X, 2 = s x s symmetric, 3 = s x s full tiles,
                            4 = s x s in one thread block (fp64, s <= 64 and L <= 128, FORM auto) */
  int32_t rec_products;  /* s x s products the recurrence (Alg. 1 lines 8-11) launched for the dense
                            fp64 s x s forms (2 and 4): K - 2, or K - 3 when Psi_2 = 2 B_hat^2 - I was
                            formed from the power iteration's squaring (reading R29); 0 elsewhere */
  int32_t line12_in_recurrence;  /* 1: Alg. 1 line 12 (Y = H_hat X) ran inside the recurrence launch
                                    (m-chain mode, left side), its time in ms_recurrence */
} cpa_svt_info;

/* Multi-GPU sharding of the long dimension for cpa_svt_apply (handles with a communicator). */
typedef enum {
  CPA_SVT_SHARD_NONE = 0,  /* X is the whole matrix on every rank (replicas) */
  CPA_SVT_SHARD_COLS = 1,  /* left-apply (global m <= n): X is m x n_local, a column block */
  CPA_SVT_SHARD_ROWS = 2   /* right-apply (global m > n): X is m_local x n, a row block */
} cpa_svt_shard;

/* Create a handle bound to `device` and the CUDA stream `cuda_stream`
 * (a cudaStream_t; NULL = legacy default stream).  nccl_unique_id points to
 * the 128-byte ncclUniqueId created by cpa_svt_nccl_unique_id on rank 0 and
 * broadcast by the caller (required for world > 1; optional for world == 1,
 * where it creates a one-rank communicator so the sharded path with its
 * collectives runs on one GPU); the library creates its own NCCL communicator
 * (NCCL is loaded at run time).  The sharded calls below run their
 * collectives whenever the handle has a communicator. */
cpa_svt_status cpa_svt_init(cpa_svt_handle** h, int device, void* cuda_stream,
                            const void* nccl_unique_id, int rank, int world);
cpa_svt_status cpa_svt_free(cpa_svt_handle* h);

/* The handle's NCCL communicator as NCCL reports it (ncclCommCount / ncclCommUserRank):
 * *nranks = 0, *rank = -1 when the handle has none.  Host pointers.  E_ARG on NULL. */
cpa_svt_status cpa_svt_comm_info(const cpa_svt_handle* h, int* nranks, int* rank);

/* Writes a fresh 128-byte ncclUniqueId into out128 (call on rank 0 only). */
cpa_svt_status cpa_svt_nccl_unique_id(void* out128);

/* Pure host function, fp64: c_out[k] = (2/K) sum_{l=1}^{K} cos(k theta_l)
 * h((lambda_max/2)(cos theta_l + 1)), theta_l = pi (l - 1/2)/K, k = 0..K-1
 * (PAPER.md:233 eq. chebychev_coeff_shifted).  sigma_max_hat resolves a
 * relative tau.  c_out: host array of K doubles, caller-owned. */
cpa_svt_status cpa_svt_coeffs(const cpa_svt_kernel* k, int K, double lambda_max,
                              double sigma_max_hat, double* c_out);

/* Dense shrinkage of one matrix.  m, n: LOCAL shape of X (the shard when
 * world > 1).  long_global: global extent of the sharded dimension (ignored
 * for SHARD_NONE).  c: optional host array of K raw coefficients that
 * replaces line 4 (NULL = computed on the device from `k` and Lambda_max).
 * lam: required.  info: optional.  dtype/math: F64+NATIVE (DMMA), F32 with
 * TF32 / 3XTF32.  X and Y are dtype arrays.  With a communicator and a shard
 * mode the partial Grams are summed with one NCCL all-reduce (PAPER.md:278-307:
 * G = sum over column blocks of X_p X_p^T), Lambda_max and the coefficients are
 * broadcast from rank 0, and every rank applies the series to its own block.
 * All ranks must make the same call (same global shape, K, kernel, options);
 * argument errors are detected on every rank before the first collective. */
cpa_svt_status cpa_svt_apply(cpa_svt_handle* h, cpa_svt_dtype dtype, cpa_svt_math math,
                             int64_t m, int64_t n, cpa_svt_shard shard, int64_t long_global,
                             const void* X, int64_t ldx, void* Y, int64_t ldy,
                             const cpa_svt_kernel* k, int K, const double* c,
                             cpa_svt_lambda* lam, cpa_svt_info* info);

/* Same as cpa_svt_apply (world 1, SHARD_NONE) but X and Y are HOST arrays
 * (row-major, ld = n).  Copies X to handle-owned device memory, runs the
 * path, copies Y back, and synchronises.  Pinned host buffers give full
 * PCIe bandwidth; pageable ones work. */
cpa_svt_status cpa_svt_apply_host(cpa_svt_handle* h, cpa_svt_dtype dtype, cpa_svt_math math,
                                  int64_t m, int64_t n, const void* X_host, void* Y_host,
                                  const cpa_svt_kernel* k, int K, cpa_svt_lambda* lam,
                                  cpa_svt_info* info);

/* Sparse X (m x n, CSR, fp64): Y = X H_hat(X^T X), the n x n Gram never
 * formed.  c: optional host array of K raw coefficients replacing line 4 (as in
 * cpa_svt_apply; NULL = computed on the device from k and Lambda_max).  Each step runs Z = W_{k-1} X^T (m x m block rows) then
 * W_k = (4/L) Z X - 2 W_{k-1} - W_{k-2} fused with Y += c_k W_k.  X is
 * replicated on every rank (row_ptr int64[m+1], col int32[nnz] sorted per
 * row, val fp64[nnz], all device); this rank computes rows
 * [row_begin, row_end) of Y into Y (dense, (row_end-row_begin) x n, ld ldy).
 * Lambda_max: power iteration on X X^T (m-side), v -> X (X^T v) (reading R4). */
cpa_svt_status cpa_svt_apply_csr(cpa_svt_handle* h, int64_t m, int64_t n, int64_t nnz,
                                 const int64_t* row_ptr, const int32_t* col, const double* val,
                                 int64_t row_begin, int64_t row_end, double* Y, int64_t ldy,
                                 const cpa_svt_kernel* k, int K, const double* c, cpa_svt_lambda* lam,
                                 cpa_svt_info* info);

/* Batched fp32 shrinkage of `batch` independent m x n matrices stored
 * contiguously ([batch][m][n], row-major): Gram, power iteration, coefficients
 * and the recurrence per matrix inside one kernel (no host round trip).
 * lambda_out: optional device array of `batch` floats receiving Lambda_max.
 * Requires m, n <= 64 and K <= 128 (else CPA_SVT_E_UNSUPPORTED). */
cpa_svt_status cpa_svt_apply_batched(cpa_svt_handle* h, int64_t batch, int m, int n,
                                     const float* X, float* Y, const cpa_svt_kernel* k, int K,
                                     const cpa_svt_lambda* lam, float* lambda_out);

/* NEXT-2 component threshold of Alg. 1 line 2 (eq. threshold_components) for
 * CPA_SVT_OPT_TRANSFORM = 2 or 3 (DCT, block DCT): mode 0 keeps every component; 1 keeps |Phi_ij| >= value;
 * 2 keeps |Phi_ij| >= the value-th largest |Phi_ij| (ties kept; value >= 1).
 * Errors: E_ARG (null, mode), E_DOMAIN (value < 0, or < 1 for mode 2). */
cpa_svt_status cpa_svt_set_epsilon(cpa_svt_handle* h, int mode, double value);

/* NEXT-3: the paper's ADMM recovery with CPA shrinkage as the nuclear-norm prox
 * (eq. admm_algorithm_inp; synthetic experiment
 * PAPER.md:1095-1100 without the average-term constraint):
 *   min ||L||_* + eta ||Psi(L)||_1  s.t. L = D on the observed entries, L in [0, 1],
 * Psi = orthonormal 2-D DCT-II.  ADMM iterations (z, u start at 0):
 *   l = (K^T K)^-1 K^T (z - u);  z1 = CPA-shrink_soft(1/rho)(l + u1);  z2 = soft(Psi l + u2, eta/rho);
 *   z3 = observed D;  z4 = clip(l + u4, 0, 1);  u += K l - z;  stop: ||dl|| / ||l|| < tol.
 * D (m x n, row-major, ld n) and mask (m x n bytes, nonzero = observed) are device pointers;
 * L (m x n) receives the last l.  The shrinkage uses this handle's fp64 dense path (its form and
 * transform options apply), K terms and lam (power iterations / override) per call.  One host
 * sync per iteration.  Errors: E_ARG (null / sizes / K), E_DOMAIN (rho <= 0, eta < 0, tol < 0,
 * max_iter < 1), E_CUDA. */
typedef struct {
  double rho, eta, tol;   /* in */
  int32_t max_iter;       /* in, >= 1 */
  int32_t iters;          /* out: iterations run */
  double last_rel;        /* out: last ||l_{t+1} - l_t|| / ||l_{t+1}|| */
  double ms_shrink;       /* out: CUDA-event time inside the CPA shrinkage calls */
  double ms_total;        /* out: CUDA-event time of the whole loop */
  int32_t adaptive_eps;   /* in: 1 = threshold the transform-domain Gram of every shrinkage at the
                             recommended epsilon(E_t) (eq. recommendation_epsilon):
                             the k-th largest |Phi_ij|, k = (0.5e-4 | 1.5e-4 | 0.5e-3) s^2 for the
                             previous iteration's E > 0.03 | > 6e-4 | otherwise (first: 0.5e-4 s^2);
                             needs CPA_SVT_OPT_TRANSFORM 2 or 3 (else E_ARG); 0 = the handle's own
                             cpa_svt_set_epsilon setting */
  int32_t reserved;
} cpa_svt_admm;
cpa_svt_status cpa_svt_admm_recover(cpa_svt_handle* h, int64_t m, int64_t n, const double* D,
                                    const unsigned char* mask, int K, const cpa_svt_lambda* lam,
                                    cpa_svt_admm* opt, double* L);

/* Handle options (cpa_svt_set_option). */
typedef enum {
  CPA_SVT_OPT_FORM = 0      /* dense recurrence form: 0 = auto (fewest flops), 1 = apply-to-X
                               (W_k = Psi_k(B_hat) X, (K-1) 2 s^2 L flops), 2 = Alg. 1 literal s x s form
                               (H_hat = sum c_k Psi_k(B_hat) formed on the s x s Gram, then one product
                               Y = H_hat X); fp64 computes only the lower-triangle
                               tiles of each symmetric Psi_k (s^2 (s+1) flops per step), 3 = the s x s
                               form on full tiles (2 s^3 per step; cross-check).  Auto picks 2 whenever
                               K > 2 (fp64 and fp32/TF32; the TF32 s x s form is symmetric too). */,
  CPA_SVT_OPT_TRANSFORM = 1 /* NEXT-2, Alg. 1 line 1-2 with a sparsifying transform (PAPER.md:320-352,
                               628-630): 0 = T = I (default); 1 = one-level Haar DWT of the Gram index
                               with the high-frequency components of Phi set to 0 -- Alg. 1 then runs
                               on the low-pass half and line 12 applies B T^T H_hat(Phi_) T; 2 =
                               orthonormal DCT-II of the Gram index, Phi = T G T^T thresholded per
                               cpa_svt_set_epsilon, the recurrence on the sparse Phi_ (CSR) when a
                               threshold is set; 3 = the 8 x 8 block DCT (T =
                               blockdiag of 8 x 8 DCT-II blocks, a smaller last block when 8 does not
                               divide s), otherwise as 2.  fp64 dense, unsharded only (else
                               CPA_SVT_E_UNSUPPORTED). */,
  CPA_SVT_OPT_BATCHED = 2,  /* engine of cpa_svt_apply_batched: 0 = auto (tcgen05), 1 = fp32 FFMA (exact
                               fp32 products, apply-to-X form), 2 = tcgen05 3xTF32 (s x s form,
                               M = N = 64 MMAs, TMEM accumulators). */
  CPA_SVT_OPT_DIVERGENCE = 3 /* SPEC.md:215 check of apply / apply_host / apply_csr outputs (one extra pass
                               over X and Y): 0 = off, 1 = on, the verdict (CPA_SVT_E_DIVERGED) returned by
                               calls that synchronise anyway (default), 2 = on, every call synchronises and
                               returns it.  Sharded calls compare this rank's block of Y with its block of X.
                               cpa_svt_apply_batched is not checked. */
} cpa_svt_option;
cpa_svt_status cpa_svt_set_option(cpa_svt_handle* h, cpa_svt_option opt, int64_t value);

/* Per-phase device timing for measurement: when enabled, the library records a
 * CUDA event pair on the handle's stream around every launch it makes and
 * accumulates the elapsed time per phase (no host sync until read). */
typedef enum {
  CPA_SVT_PH_GRAM = 0,       /* Gram product (Alg. 1 line 1) */
  CPA_SVT_PH_ALLREDUCE = 1,  /* NCCL all-reduce of the Gram + Lambda broadcast */
  CPA_SVT_PH_POWER = 2,      /* power iteration + coefficients (lines 3-4) */
  CPA_SVT_PH_INIT = 3,       /* W_1 and Y init (lines 5-7) */
  CPA_SVT_PH_STEP = 4,       /* fused recurrence step (lines 8-11), one per k */
  CPA_SVT_PH_SPARSE_Z = 5,   /* sparse: Z = W_{k-1} X^T */
  CPA_SVT_PH_SPARSE_W = 6,   /* sparse: W_k = (4/L) Z X - 2 W_{k-1} - W_{k-2}, Y += c_k W_k */
  CPA_SVT_PH_BATCHED = 7,    /* batched kernel */
  CPA_SVT_PH_FINAL = 8,      /* s x s form: the final product Y = H_hat X (+ the divergence check) */
  CPA_SVT_PH_EXCHANGE = 9,   /* multi-GPU s x s form: per-step all-gather of the tile panels + unpack */
  CPA_SVT_PH_COUNT = 10
} cpa_svt_phase;
/* enable != 0: reset the accumulators and start recording; 0: stop. */
cpa_svt_status cpa_svt_profile(cpa_svt_handle* h, int enable);
/* Synchronise the stream, then write per-phase total ms and launch counts
 * (host arrays of CPA_SVT_PH_COUNT entries; either may be NULL). */
cpa_svt_status cpa_svt_profile_read(cpa_svt_handle* h, double* ms, int64_t* launches);

/* Kernel unit test hook (tests only): C (M x N, ld ldc, fp32) = A B on the
 * tcgen05 TF32 engine, A (M x Kd, K-major, ld lda), B K x N N-contiguous
 * (b_mn != 0, ld ldb) or N x K K-contiguous (b_mn == 0).  terms = 1 (TF32 of
 * the rna-rounded operands) or 3 (3xTF32).  All device pointers, ld % 4 == 0.
 * Synchronous. */
cpa_svt_status cpa_svt_debug_gemm_tf32(cpa_svt_handle* h, int M, int N, int Kd, const float* A, int64_t lda,
                                       const float* B, int64_t ldb, int b_mn, float* C, int64_t ldc, int terms);

const char* cpa_svt_status_string(cpa_svt_status s);
/* Text of the last error recorded on this handle ("" if none). */
const char* cpa_svt_last_error(const cpa_svt_handle* h);
/* Number of device kernels launched through this handle since init. */
int64_t cpa_svt_launch_count(const cpa_svt_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* CPA_SVT_H */
