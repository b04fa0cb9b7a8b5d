// C ABI of libcpasvt (include/cpa_svt.h): validation, side selection,
// workspace, launch sequence, NCCL plumbing.  All arithmetic of the method
// runs in the kernels of dense_f64.cu / power.cu / batched_f32.cu / sparse_f64.cu.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace cpa {
// dense_f64.cu
cudaError_t dense_gram_f64(const double* X, int64_t m, int64_t n, int64_t ldx, bool left, double* G,
                           cudaStream_t st, const double* gscale = nullptr, double* partial = nullptr,
                           int* tcount = nullptr);
size_t dense_gram_partial_doubles(int64_t s);
cudaError_t dense_cheb_launch(bool left, bool init, int64_t m, int64_t n, const double* G,
                              const double* Wsrc, int64_t ldsrc, const double* Wpp, int64_t ldpp,
                              double* Wout, int64_t ldout, double* Y, int64_t ldy, const SeriesParams* P,
                              int k, cudaStream_t st);
size_t dense_flow_sync_ints(int64_t m, int64_t n, int K);
size_t dense_flow_partial_doubles(int64_t m, int64_t n, int num_sms);
void dense_gram_chunk_range(int64_t kd, int q, int S, int64_t* k0, int64_t* k1);
bool small_f64_fits(int64_t m, int64_t n);
int small_f64_products(int64_t m, int64_t n, int K, int nsq, double lam_override);
cudaError_t launch_small_f64(const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t m, int64_t n,
                             SeriesParams* P, const cpa_svt_kernel& k, int K, int T, double safety,
                             double lam_override, const double* c_given, int nsq, cudaStream_t st, int check);
cudaError_t dense_gram_f64_chunk(const double* X, int64_t m, int64_t n, int64_t ldx, bool left, double* G,
                                 cudaStream_t st, double* partial, int* tcount, int q, int S);
cudaError_t dense_gemm_store(int64_t M, int64_t N, int64_t Kd, const double* A, int64_t lda, const double* B,
                             int64_t ldb, double* C, int64_t ldc, cudaStream_t st, double* partial = nullptr,
                             int* tcount = nullptr);
size_t dense_store_partial_doubles(int64_t M, int64_t N);
// transform.cu
size_t dct_eps_scratch_bytes(int64_t s);
cudaError_t dct_eps_threshold(double* Phi, int64_t s, int mode, double eps_value, void* scratch, int num_sms,
                              cudaStream_t st, const int64_t** rp_out, const int32_t** col_out,
                              const double** val_out);
cudaError_t dct_sparse_steps(int64_t s, const int64_t* rp, const int32_t* col, const double* val, double* Wa,
                             double* Wb, double* H, const SeriesParams* P, int K, int num_sms, cudaStream_t st);
// admm.cu
cudaError_t admm_dct(double* C, double* CT, int64_t n, int num_sms, cudaStream_t st);
cudaError_t block_dct_sandwich(const double* A, double* out, int64_t s, int inverse, cudaStream_t st);
cudaError_t admm_sub(const double* a, const double* b, double* out, int64_t N, cudaStream_t st);
cudaError_t admm_l(const double* z1, const double* u1, const double* pt, const uint8_t* mask, const double* D,
                   const double* u3, const double* z4, const double* u4, double* l, double* t, int64_t N,
                   cudaStream_t st);
int admm_tail_blocks();
cudaError_t admm_tail(const double* l, const double* lprev, const double* pl, const double* z1, const uint8_t* mask,
                      const double* D, double* z2, double* z4, double* u1, double* u2, double* u3, double* u4,
                      double thr, int64_t N, double* part, cudaStream_t st);
cudaError_t dense_haar_split(const double* X, int64_t m, int64_t n, int64_t ldx, bool left, double* AL, double* AH,
                             int num_sms, cudaStream_t st);
cudaError_t dense_haar_combine(const double* YL, const double* AH, const SeriesParams* P, int64_t m, int64_t n,
                               bool left, double* Y, int64_t ldy, int num_sms, cudaStream_t st);
cudaError_t dense_eye(double* I, int64_t s, cudaStream_t st);
size_t dense_sym_sync_ints(int64_t s, int K, int num_sms, int64_t L = 0);
size_t dense_sym_l12_partial_doubles(int64_t s, int64_t L, int num_sms);
int64_t dense_sym_ntri(int64_t s);
int64_t dense_sym_panel_tile0(int64_t s, int p, int P);
int64_t dense_sym_panel_slot(int64_t s, int P);
size_t dense_sym_panel_partial_doubles(int64_t s, int P, int num_sms);
cudaError_t dense_cheb_sym_panel(int64_t s, const double* G, double* W0, double* W1, double* W2, double* H,
                                 const SeriesParams* P, int K, int kstep, int64_t tile0, int64_t ntile,
                                 double* gout, int* sync, double* partial, int num_sms, cudaStream_t st);
cudaError_t dense_sym_unpack(const double* gbuf, int64_t s, int P, double* out, cudaStream_t st);
size_t dense_sym_partial_doubles(int64_t s, int num_sms, int m);
int dense_sym_use_chain(int64_t s, int K, int num_sms);
cudaError_t dense_sym_init(int64_t s, const double* G, double* Wa, double* H, const SeriesParams* P, int K,
                           int num_sms, cudaStream_t st, double* G2 = nullptr, const double* c2 = nullptr);
cudaError_t dense_cheb_sym(int64_t s, const double* G, double* W0, double* W1, double* W2, double* H,
                           const SeriesParams* P, int K, int* sync, double* partial, int num_sms, cudaStream_t st,
                           int m = 0, double* const* chain = nullptr, double* const* HX = nullptr,
                           bool psi2_given = false, const double* X = nullptr, int64_t ldx = 0, double* Y = nullptr,
                           int64_t ldy = 0, int64_t L = 0, double* l12_partial = nullptr);
cudaError_t dense_cheb_flow(bool left, int64_t m, int64_t n, const double* G, const double* X, int64_t ldx,
                            double* Wa, double* Wb, double* Y, int64_t ldy, const SeriesParams* P, int K, int* sync,
                            double* partial, int num_sms, cudaStream_t st);
// power.cu
cudaError_t launch_series(SeriesParams* P, const cpa_svt_kernel& k, int K, double safety, double lam_override,
                          const double* lam_src, const double* c_given, cudaStream_t st);
size_t power_dense_scratch_doubles(int64_t s);
size_t power_scale_offset(int64_t s);
int power_squarings(int64_t s, int T);
cudaError_t launch_diag_scale(const double* G, int64_t s, double* scale, cudaStream_t st);
cudaError_t launch_power_dense(const double* G, const double* G4, int pw, int64_t s, int T, double* scratch,
                               unsigned int* bar, SeriesParams* P, const cpa_svt_kernel& k, int K, double safety,
                               const double* c_given, int num_sms, cudaStream_t st);
int64_t power_rows_slot(int64_t s, int P);
size_t power_rows_scratch_doubles(int64_t s, int P, int num_sms);
cudaError_t launch_power_rows(const double* G, int64_t s, int t, int v, int P, double* scratch, int num_sms,
                              cudaStream_t st);
double* power_rows_buffer(double* scratch, int64_t s, int t, int P);
cudaError_t launch_power_rows_final(double* scratch, int64_t s, int T, int P, int num_sms, double** lam_hat,
                                    cudaStream_t st);
cudaError_t launch_power_dense_f32(const float* G, int64_t s, int64_t ld, int T, double* scratch, unsigned int* bar,
                                   SeriesParams* P, const cpa_svt_kernel& k, int K, double safety,
                                   const double* c_given, int num_sms, cudaStream_t st);
// tc_tf32.cu
cudaError_t tc_gemm(int mode, int terms, int M, int N, int Kd, const float* Ah, const float* Al, int64_t lda,
                    const float* Bh, const float* Bl, int64_t ldb, bool b_mn, float* out_f, float* out_h,
                    float* out_l, int out_split, int64_t ld_out, const float* wp, const float* wpp, int64_t ld_w,
                    float* y, int64_t ld_y, const SeriesParams* P, int k, int num_sms, cudaStream_t st,
                    int sym = 0);
cudaError_t tf32_sym_init(const float* G, int64_t s, int64_t ld, float* Wf, float* Wh, float* Wl, float* H,
                          const SeriesParams* P, int num_sms, cudaStream_t st);
cudaError_t tf32_sym_prep(const float* H, int64_t s, int64_t ld, float* Hh, float* Hl, int num_sms, cudaStream_t st);
cudaError_t tf32_prep(const float* X, int64_t m, int64_t n, int64_t ldx, bool transpose, float* Af, float* Ah,
                      float* Al, int64_t lda, int num_sms, cudaStream_t st);
cudaError_t tf32_finish(const float* Yi, int64_t ldi, int64_t m, int64_t n, bool transpose, float* Y, int64_t ldy,
                        int num_sms, cudaStream_t st);
cudaError_t tf32_eye(float* I, int64_t s, int64_t ld, int num_sms, cudaStream_t st);
cudaError_t tf32_panel_list(int64_t s, int terms, const int2** list, int* count, int* bn);
cudaError_t tc_gemm_panel(int terms, int s, const float* Ah, const float* Al, int64_t lda, const float* Bh,
                          const float* Bl, int64_t ldb, bool last, int64_t ld_out, const float* wp, const float* wpp,
                          int64_t ld_w, float* y, int64_t ld_y, const SeriesParams* P, int k, int64_t tile0,
                          int64_t ntile, float* gout, int num_sms, cudaStream_t st);
cudaError_t tf32_sym_unpack(const float* gbuf, int64_t s, int terms, int P, int64_t slot_tiles, int64_t ld, float* Wf,
                            float* Wh, float* Wl, float* H, cudaStream_t st);
cudaError_t launch_power_rows_f32(const float* G, int64_t s, int64_t ld, int t, int v, int P, double* scratch,
                                  int num_sms, cudaStream_t st);
// batched_f32.cu
cudaError_t launch_batched_f32(int64_t batch, int m, int n, const float* X, float* Y, const cpa_svt_kernel& k,
                               int K, int T, double safety, double lam_override, float* lambda_out,
                               int num_sms, cudaStream_t st, int* launches, double* costab);
cudaError_t launch_batched_tc(int64_t batch, int m, int n, const float* X, float* Y, const cpa_svt_kernel& k,
                               int K, int T, double safety, double lam_override, float* lambda_out,
                               int num_sms, cudaStream_t st, int* launches, double* costab);
// check.cu
size_t divergence_scratch_doubles();
cudaError_t divergence_check_f64(const double* X, int64_t xr, int64_t xc, int64_t ldx, const double* Y, int64_t yr,
                                 int64_t yc, int64_t ldy, double* scratch, SeriesParams* P, cudaStream_t st);
cudaError_t divergence_check_f32(const float* X, int64_t xr, int64_t xc, int64_t ldx, const float* Y, int64_t yr,
                                 int64_t yc, int64_t ldy, double* scratch, SeriesParams* P, cudaStream_t st);
// sparse_f64.cu
cudaError_t sparse_apply(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                         const double* val, int64_t row_begin, int64_t row_end, double* Y, int64_t ldy,
                         const cpa_svt_kernel& k, int K, int T, double safety, double lam_override,
                         SeriesParams* P, void* ws, size_t ws_bytes, size_t* ws_needed, int num_sms,
                         cudaStream_t st, int* launches, SparsePhaseHook hook, void* hook_ctx, const double* c_given);
}  // namespace cpa

using namespace cpa;

// ------------------------------------------------------------------ NCCL (run-time loaded)
namespace {
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  std::mutex mu;   // (handles created from several host threads)
  bool load() {
    std::lock_guard<std::mutex> lock(mu);
    if (lib) return true;
    lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return false;
    GetUniqueId = (decltype(GetUniqueId))dlsym(lib, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(lib, "ncclCommInitRank");
    CommDestroy = (decltype(CommDestroy))dlsym(lib, "ncclCommDestroy");
    AllReduce = (decltype(AllReduce))dlsym(lib, "ncclAllReduce");
    Broadcast = (decltype(Broadcast))dlsym(lib, "ncclBroadcast");
    AllGather = (decltype(AllGather))dlsym(lib, "ncclAllGather");
    GetErrorString = (decltype(GetErrorString))dlsym(lib, "ncclGetErrorString");
    CommCount = (decltype(CommCount))dlsym(lib, "ncclCommCount");
    CommUserRank = (decltype(CommUserRank))dlsym(lib, "ncclCommUserRank");
    return GetUniqueId && CommInitRank && CommDestroy && AllReduce && Broadcast && AllGather && GetErrorString &&
           CommCount && CommUserRank;
  }
};
NcclApi g_nccl;
}  // namespace

struct cpa_svt_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  int* dvote = nullptr;            // sharded calls: the ranks' pre-collective status vote (device int)
  int num_sms = 148;
  SeriesParams* P = nullptr;       // device
  unsigned int* bar = nullptr;     // device, 2 uints (grid barrier)
  double* d_c = nullptr;           // device, KMAX (caller coefficients)
  double* dchk = nullptr;          // device, divergence-check partial sums
  int div_mode = 1;                // CPA_SVT_OPT_DIVERGENCE: 0 off, 1 check (status on syncing calls), 2 check + sync
  void* ws = nullptr;              // workspace
  size_t ws_bytes = 0;
  void* hx = nullptr;              // apply_host device staging
  void* tws = nullptr;             // transform workspace (A_L, A_H, Y_L)
  void* aws = nullptr;             // ADMM workspace
  size_t aws_bytes = 0;
  size_t tws_bytes = 0;
  int transform = 0;               // CPA_SVT_OPT_TRANSFORM
  int eps_mode = 0;                // cpa_svt_set_epsilon: 0 keep all, 1 absolute, 2 top-k
  double eps_value = 0.0;
  int batched_engine = 0;          // CPA_SVT_OPT_BATCHED: 0 auto (tensor cores), 1 FFMA, 2 tcgen05
  size_t hx_bytes = 0;
  std::string err;
  int64_t launches = 0;
  // CPA_SVT_GUARD=1 (read at init; tests / debugging, compute-sanitizer being unavailable on
  // the pool): every workspace allocation carries a guard band filled with kGuardByte from the
  // end of what the current call uses, checked after every public call (E_CUDA on a change).
  bool guard = false;
  struct GuardBand { void** p; size_t from, to; };
  std::vector<GuardBand> guards;
  bool use_flow = true;            // persistent dataflow recurrence (CPA_SVT_FLOW=0: one launch per step)
  int form = 0;                    // CPA_SVT_OPT_FORM
  // profiling (cpa_svt_profile): event pairs per phase, resolved at read time
  // cpa_svt_apply_host pipeline: X arrives in kPipe k-chunks on copy_stream, each chunk's
  // split-K Gram unit starts when it lands; Y leaves in kPipe chunks as line 12 produces them
  static constexpr int kPipe = 4;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t pev[2 * kPipe] = {};
  const double* hp_X = nullptr;    // host X / Y of the call in flight (nullptr: no pipeline)
  double* hp_Y = nullptr;
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_used;
  double prof_ms[CPA_SVT_PH_COUNT] = {};
  int64_t prof_n[CPA_SVT_PH_COUNT] = {};
};

namespace {
// RAII: records an event pair around the launches of one phase when profiling.
struct Phase {
  cpa_svt_handle* h;
  int ph;
  cudaEvent_t e1 = nullptr;
  Phase(cpa_svt_handle* h_, int ph_, int n = 1) : h(h_), ph(ph_) {
    if (!h->prof) return;
    cudaEvent_t e0 = take();
    e1 = take();
    cudaEventRecord(e0, h->stream);
    h->ev_used.push_back({ph, {e0, e1}});
    h->prof_n[ph] += n;
  }
  cudaEvent_t take() {
    if (h->ev_pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
  }
  ~Phase() {
    if (e1) cudaEventRecord(e1, h->stream);
  }
};
// begin/end hook for phases spanning many launches (sparse path)
void phase_hook(void* ctx, int ph, int begin) {
  cpa_svt_handle* h = (cpa_svt_handle*)ctx;
  if (!h->prof) return;
  if (begin) {
    Phase p(h, ph);         // records the start event and reserves the pair ...
    p.e1 = nullptr;         // ... but the end event is recorded by the matching end call
  } else {
    cudaEventRecord(h->ev_used.back().second.second, h->stream);
  }
}
}  // namespace

#define CU(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      h->err = std::string(#call) + ": " + cudaGetErrorString(e_);                   \
      return CPA_SVT_E_CUDA;                                                         \
    }                                                                                \
  } while (0)

#define NC(call)                                                                     \
  do {                                                                               \
    ncclResult_t r_ = (call);                                                        \
    if (r_ != ncclSuccess) {                                                         \
      h->err = std::string(#call) + ": " + g_nccl.GetErrorString(r_);                \
      return CPA_SVT_E_NCCL;                                                         \
    }                                                                                \
  } while (0)

constexpr size_t kGuardBytes = 1 << 16;
constexpr unsigned char kGuardByte = 0xA5;

static cpa_svt_status grow(cpa_svt_handle* h, void** p, size_t* have, size_t need) {
  if (h->guard) {
    // allocation = capacity + guard band; the band of this call starts at `need`
    need = (need + 255) / 256 * 256;
    if (need > *have) {
      if (*p) {
        cudaStreamSynchronize(h->stream);
        cudaFree(*p);
        *p = nullptr;
        *have = 0;
      }
      if (cudaMalloc(p, need + kGuardBytes) != cudaSuccess) {
        cudaGetLastError();
        h->err = "workspace cudaMalloc (guarded)";
        return CPA_SVT_E_NOMEM;
      }
      *have = need;
    }
    if (cudaMemsetAsync((char*)*p + need, kGuardByte, *have + kGuardBytes - need, h->stream) != cudaSuccess)
      return CPA_SVT_E_CUDA;
    for (auto& g : h->guards)
      if (g.p == p) { g.from = need; g.to = *have + kGuardBytes; return CPA_SVT_OK; }
    h->guards.push_back({p, need, *have + kGuardBytes});
    return CPA_SVT_OK;
  }
  if (need <= *have) return CPA_SVT_OK;
  if (*p) {
    cudaStreamSynchronize(h->stream);
    cudaFree(*p);
    *p = nullptr;
    *have = 0;
  }
  cudaError_t e = cudaMalloc(p, need);
  if (e != cudaSuccess) {
    h->err = std::string("workspace cudaMalloc: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return CPA_SVT_E_NOMEM;
  }
  *have = need;
  return CPA_SVT_OK;
}

static cpa_svt_status check_kernel(const cpa_svt_kernel* k) {
  if (!k) return CPA_SVT_E_ARG;
  if (k->kind < CPA_SVT_HARD || k->kind > CPA_SVT_WSOFT) return CPA_SVT_E_ARG;
  if (k->kind != CPA_SVT_WSOFT) {
    if (!(k->tau >= 0.0) || !std::isfinite(k->tau)) return CPA_SVT_E_DOMAIN;
  } else {
    if (!(k->w_c >= 0.0) || !(k->w_shift >= 0.0) || !(k->w_eps > 0.0) || !std::isfinite(k->w_c))
      return CPA_SVT_E_DOMAIN;
  }
  return CPA_SVT_OK;
}

static cpa_svt_status check_lambda(const cpa_svt_lambda* lam) {
  if (!lam) return CPA_SVT_E_ARG;
  if (!(lam->safety >= 1.0) || !std::isfinite(lam->safety)) return CPA_SVT_E_DOMAIN;
  if (!std::isfinite(lam->lambda_max) || lam->lambda_max < 0.0) return CPA_SVT_E_DOMAIN;
  if (!(lam->lambda_max > 0.0) && lam->power_iters < 1) return CPA_SVT_E_ARG;
  return CPA_SVT_OK;
}

extern "C" {

const char* cpa_svt_status_string(cpa_svt_status s) {
  switch (s) {
    case CPA_SVT_OK: return "ok";
    case CPA_SVT_E_ARG: return "invalid argument";
    case CPA_SVT_E_DOMAIN: return "argument outside the method's domain";
    case CPA_SVT_E_DIVERGED: return "recurrence diverged";
    case CPA_SVT_E_CUDA: return "CUDA error";
    case CPA_SVT_E_NCCL: return "NCCL error";
    case CPA_SVT_E_NOMEM: return "out of device memory";
    case CPA_SVT_E_UNSUPPORTED: return "unsupported by this build";
  }
  return "unknown status";
}

const char* cpa_svt_last_error(const cpa_svt_handle* h) { return h ? h->err.c_str() : ""; }
int64_t cpa_svt_launch_count(const cpa_svt_handle* h) { return h ? h->launches : 0; }

cpa_svt_status cpa_svt_comm_info(const cpa_svt_handle* h, int* nranks, int* rank) {
  if (!h || !nranks || !rank) return CPA_SVT_E_ARG;
  *nranks = 0;
  *rank = -1;
  if (!h->comm) return CPA_SVT_OK;
  if (g_nccl.CommCount(h->comm, nranks) != ncclSuccess || g_nccl.CommUserRank(h->comm, rank) != ncclSuccess)
    return CPA_SVT_E_NCCL;
  return CPA_SVT_OK;
}

cpa_svt_status cpa_svt_nccl_unique_id(void* out128) {
  if (!out128) return CPA_SVT_E_ARG;
  if (!g_nccl.load()) return CPA_SVT_E_NCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return CPA_SVT_E_NCCL;
  memcpy(out128, &id, sizeof(id));
  return CPA_SVT_OK;
}

cpa_svt_status cpa_svt_init(cpa_svt_handle** out, int device, void* cuda_stream, const void* nccl_unique_id,
                            int rank, int world) {
  if (!out || world < 1 || rank < 0 || rank >= world) return CPA_SVT_E_ARG;
  if (world > 1 && !nccl_unique_id) return CPA_SVT_E_ARG;
  *out = nullptr;
  cpa_svt_handle* h = new cpa_svt_handle();
  h->device = device;
  h->stream = (cudaStream_t)cuda_stream;
  h->rank = rank;
  h->world = world;
  if (const char* f = getenv("CPA_SVT_FLOW")) h->use_flow = f[0] != '0';
  h->guard = env_on("CPA_SVT_GUARD");
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaMalloc(&h->P, sizeof(SeriesParams));
  if (e == cudaSuccess) e = cudaMalloc(&h->bar, 64);
  if (e == cudaSuccess) e = cudaMemset(h->bar, 0, 64);
  if (e == cudaSuccess) e = cudaMalloc(&h->d_c, CPA_SVT_KMAX * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&h->dchk, divergence_scratch_doubles() * sizeof(double));
  if (e == cudaSuccess) e = cudaMemset(h->dchk, 0, divergence_scratch_doubles() * sizeof(double));
  if (e != cudaSuccess) {
    cudaGetLastError();
    cpa_svt_free(h);
    return CPA_SVT_E_CUDA;
  }
  // a communicator whenever an id is given -- also for world == 1, so the shipped exchange
  // (all-reduce of the Gram, broadcast of the series parameters) runs on a single GPU too
  if (nccl_unique_id) {
    if (!g_nccl.load()) {
      cpa_svt_free(h);
      return CPA_SVT_E_NCCL;
    }
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    if (g_nccl.CommInitRank(&h->comm, world, id, rank) != ncclSuccess) {
      h->comm = nullptr;
      cpa_svt_free(h);
      return CPA_SVT_E_NCCL;
    }
    if (cudaMalloc(&h->dvote, sizeof(int)) != cudaSuccess) {
      cpa_svt_free(h);
      return CPA_SVT_E_NOMEM;
    }
  }
  *out = h;
  return CPA_SVT_OK;
}

cpa_svt_status cpa_svt_free(cpa_svt_handle* h) {
  if (!h) return CPA_SVT_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  else cudaDeviceSynchronize();
  if (h->comm) g_nccl.CommDestroy(h->comm);
  cudaFree(h->dvote);
  cudaFree(h->P);
  cudaFree(h->bar);
  cudaFree(h->d_c);
  cudaFree(h->dchk);
  cudaFree(h->ws);
  cudaFree(h->hx);
  cudaFree(h->tws);
  cudaFree(h->aws);
  for (auto& u : h->ev_used) {
    cudaEventDestroy(u.second.first);
    cudaEventDestroy(u.second.second);
  }
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  for (auto e : h->pev)
    if (e) cudaEventDestroy(e);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  delete h;
  return CPA_SVT_OK;
}

cpa_svt_status cpa_svt_set_option(cpa_svt_handle* h, cpa_svt_option opt, int64_t value) {
  if (!h) return CPA_SVT_E_ARG;
  if (opt == CPA_SVT_OPT_BATCHED) {
    if (value < 0 || value > 2) return CPA_SVT_E_ARG;
    h->batched_engine = (int)value;
    return CPA_SVT_OK;
  }
  if (opt == CPA_SVT_OPT_TRANSFORM) {
    if (value < 0 || value > 3) return CPA_SVT_E_ARG;
    h->transform = (int)value;
    return CPA_SVT_OK;
  }
  if (opt == CPA_SVT_OPT_DIVERGENCE) {
    if (value < 0 || value > 2) return CPA_SVT_E_ARG;
    h->div_mode = (int)value;
    return CPA_SVT_OK;
  }
  if (opt == CPA_SVT_OPT_FORM) {
    if (value < 0 || value > 3) return CPA_SVT_E_ARG;
    h->form = (int)value;
    return CPA_SVT_OK;
  }
  return CPA_SVT_E_ARG;
}

cpa_svt_status cpa_svt_set_epsilon(cpa_svt_handle* h, int mode, double value) {
  if (!h || mode < 0 || mode > 2) return CPA_SVT_E_ARG;
  if (!(value >= 0.0) || (mode == 2 && !(value >= 1.0))) return CPA_SVT_E_DOMAIN;
  h->eps_mode = mode;
  h->eps_value = value;
  return CPA_SVT_OK;
}

cpa_svt_status cpa_svt_profile(cpa_svt_handle* h, int enable) {
  if (!h) return CPA_SVT_E_ARG;
  if (enable) {
    for (int i = 0; i < CPA_SVT_PH_COUNT; ++i) { h->prof_ms[i] = 0.0; h->prof_n[i] = 0; }
    for (auto& u : h->ev_used) { h->ev_pool.push_back(u.second.first); h->ev_pool.push_back(u.second.second); }
    h->ev_used.clear();
  }
  h->prof = enable != 0;
  return CPA_SVT_OK;
}

cpa_svt_status cpa_svt_profile_read(cpa_svt_handle* h, double* ms, int64_t* launches) {
  if (!h) return CPA_SVT_E_ARG;
  CU(cudaSetDevice(h->device));
  CU(cudaStreamSynchronize(h->stream));
  for (auto& u : h->ev_used) {
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, u.second.first, u.second.second));
    h->prof_ms[u.first] += t;
    h->ev_pool.push_back(u.second.first);
    h->ev_pool.push_back(u.second.second);
  }
  h->ev_used.clear();
  for (int i = 0; i < CPA_SVT_PH_COUNT; ++i) {
    if (ms) ms[i] = h->prof_ms[i];
    if (launches) launches[i] = h->prof_n[i];
  }
  return CPA_SVT_OK;
}

cpa_svt_status cpa_svt_coeffs(const cpa_svt_kernel* k, int K, double lambda_max, double sigma_max_hat,
                              double* c_out) {
  if (!c_out || K < 1 || K > CPA_SVT_KMAX) return CPA_SVT_E_ARG;
  cpa_svt_status st = check_kernel(k);
  if (st != CPA_SVT_OK) return st;
  if (!(lambda_max > 0.0) || !std::isfinite(lambda_max) || !(sigma_max_hat >= 0.0)) return CPA_SVT_E_DOMAIN;
  const double tau = resolve_tau(*k, sigma_max_hat);
  std::vector<double> hv(K);
  for (int l = 0; l < K; ++l) hv[l] = h_response(*k, lambda_max / 2.0 * (cos(cheb_theta(l + 1, K)) + 1.0), tau);
  for (int kk = 0; kk < K; ++kk) {
    double acc = 0.0;
    for (int l = 0; l < K; ++l) acc += cos(kk * cheb_theta(l + 1, K)) * hv[l];
    c_out[kk] = 2.0 / K * acc;
  }
  return CPA_SVT_OK;
}

// Synchronises and reports Lambda / info when the caller asked for them (or when
// CPA_SVT_OPT_DIVERGENCE = 2); returns CPA_SVT_E_DIVERGED if the device check flagged the output.
static cpa_svt_status fill_info(cpa_svt_handle* h, cpa_svt_info* info, cpa_svt_lambda* lam, int side) {
  if (!info && !(lam && lam->want_lambda) && h->div_mode != 2) return CPA_SVT_OK;
  SeriesParams hp;
  CU(cudaMemcpyAsync(&hp, h->P, offsetof(SeriesParams, c), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  if (info) {
    info->lambda_hat = hp.lambda_hat;
    info->lambda_max = hp.lambda_max;
    info->sigma_max_hat = hp.sigma_hat;
    info->tau_used = hp.tau;
    info->side = side;
    info->degenerate = hp.degenerate;
    info->rec_products = 0;   // (set by the dense fp64 s x s path after this call)
    info->line12_in_recurrence = 0;
  }
  if (lam && lam->want_lambda) {
    lam->lambda_hat = hp.lambda_hat;
    lam->lambda_max = hp.lambda_max;
  }
  if (h->div_mode && hp.diverged) {
    h->err = "||Y||_F > 1e3 sum|c_k| ||X||_F (or non-finite Y): Lambda_max below the Gram's top eigenvalue?";
    return CPA_SVT_E_DIVERGED;
  }
  return CPA_SVT_OK;
}

// The divergence verdict of the last call (the stream must have been synchronised).
static cpa_svt_status read_verdict(cpa_svt_handle* h) {
  if (!h->div_mode) return CPA_SVT_OK;
  int32_t d = 0;
  CU(cudaMemcpy(&d, (const char*)h->P + offsetof(SeriesParams, diverged), sizeof(d), cudaMemcpyDeviceToHost));
  if (d) {
    h->err = "||Y||_F > 1e3 sum|c_k| ||X||_F (or non-finite Y): Lambda_max below the Gram's top eigenvalue?";
    return CPA_SVT_E_DIVERGED;
  }
  return CPA_SVT_OK;
}

// CPA_SVT_GUARD: every guard band still holds kGuardByte (synchronises).
static cpa_svt_status guard_check(cpa_svt_handle* h, cpa_svt_status st) {
  if (!h->guard) return st;
  CU(cudaStreamSynchronize(h->stream));
  std::vector<unsigned char> buf;
  for (auto& g : h->guards) {
    if (!*g.p) continue;
    buf.resize(g.to - g.from);
    CU(cudaMemcpy(buf.data(), (char*)*g.p + g.from, buf.size(), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < buf.size(); ++i)
      if (buf[i] != kGuardByte) {
        h->err = "workspace guard band overwritten at byte " + std::to_string(g.from + i) + " of a buffer whose call used " +
                 std::to_string(g.from) + " bytes";
        return CPA_SVT_E_CUDA;
      }
  }
  return st;
}

// SPEC.md:215 divergence check of the output against the input (check.cu); the verdict is read
// by fill_info / read_verdict.  Off with CPA_SVT_OPT_DIVERGENCE = 0.
// Sharded calls: every rank reaches this point before its first collective, whatever its local
// status (a workspace that failed to grow on one rank only); the worst status over the ranks is
// returned on all of them, so either every rank enqueues the collectives or none does (ADVICE r1:
// a rank returning early would leave its peers waiting inside NCCL).  One int all-reduce + a sync.
static cpa_svt_status rank_vote(cpa_svt_handle* h, cpa_svt_status local) {
  if (!h->comm || !h->dvote) return local;
  int v = (int)local;
  if (cudaMemcpyAsync(h->dvote, &v, sizeof(int), cudaMemcpyHostToDevice, h->stream) != cudaSuccess)
    return CPA_SVT_E_CUDA;
  if (g_nccl.AllReduce(h->dvote, h->dvote, 1, ncclInt32, ncclMax, h->comm, h->stream) != ncclSuccess)
    return CPA_SVT_E_NCCL;
  if (cudaMemcpyAsync(&v, h->dvote, sizeof(int), cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
      cudaStreamSynchronize(h->stream) != cudaSuccess)
    return CPA_SVT_E_CUDA;
  return (cpa_svt_status)v;
}

static cpa_svt_status check_f64(cpa_svt_handle* h, const double* X, int64_t xr, int64_t xc, int64_t ldx,
                                const double* Y, int64_t yr, int64_t yc, int64_t ldy, int* launches) {
  if (!h->div_mode) return CPA_SVT_OK;
  Phase p(h, CPA_SVT_PH_FINAL, 0);
  CU(divergence_check_f64(X, xr, xc, ldx, Y, yr, yc, ldy, h->dchk, h->P, h->stream));
  *launches += 1;
  return CPA_SVT_OK;
}

struct PhaseTimer {
  cudaEvent_t ev[6] = {};
  int n = 0;
  bool on = false;
  cudaStream_t st = nullptr;
  void start(bool enable, cudaStream_t s) {
    on = enable;
    st = s;
    if (!on) return;
    for (auto& e : ev) cudaEventCreate(&e);
    cudaEventRecord(ev[n++], st);
  }
  void mark() {
    if (on) cudaEventRecord(ev[n++], st);
  }
  float ms(int a, int b) {
    float t = 0.f;
    if (on && b < n) cudaEventElapsedTime(&t, ev[a], ev[b]);
    return t;
  }
  ~PhaseTimer() {
    if (on)
      for (auto& e : ev) cudaEventDestroy(e);
  }
};

// Alg. 1 lines 5-11 on (M x N) W_0 = Xsrc: the persistent dataflow kernel, or one
// launch per step (CPA_SVT_FLOW=0).  Y receives sum_k c_k W_k.
static cpa_svt_status run_recurrence_f64(cpa_svt_handle* h, bool left, int64_t M, int64_t N, const double* G,
                                         const double* Xsrc, int64_t ldx, double* Wa, double* Wb, double* Y,
                                         int64_t ldy, int K, double* part, int* sync, int* launches) {
  if (h->use_flow && K > 2) {
    Phase p(h, CPA_SVT_PH_STEP);
    CU(dense_cheb_flow(left, M, N, G, Xsrc, ldx, Wa, Wb, Y, ldy, h->P, K, sync, part, h->num_sms, h->stream));
    ++*launches;
    return CPA_SVT_OK;
  }
  {
    Phase p(h, CPA_SVT_PH_INIT);
    CU(dense_cheb_launch(left, true, M, N, G, Xsrc, ldx, nullptr, 0, K > 2 ? Wa : nullptr, N, Y, ldy, h->P, 1,
                         h->stream));
  }
  ++*launches;
  for (int kk = 2; kk < K; ++kk) {
    const double *src, *pp;
    double* out;
    int64_t ldsrc, ldpp;
    if (kk == 2) {
      src = Wa; ldsrc = N; pp = Xsrc; ldpp = ldx; out = Wb;
    } else {
      out = (kk & 1) ? Wa : Wb;      // W_k overwrites W_{k-2} in place
      src = (kk & 1) ? Wb : Wa;
      ldsrc = N; pp = out; ldpp = N;
    }
    if (kk == K - 1) out = nullptr;  // last W_k is never read again
    Phase p(h, CPA_SVT_PH_STEP);
    CU(dense_cheb_launch(left, false, M, N, G, src, ldsrc, pp, ldpp, out, N, Y, ldy, h->P, kk, h->stream));
    ++*launches;
  }
  return CPA_SVT_OK;
}

// Which dense form runs (CPA_SVT_OPT_FORM).  The s x s polynomial form of
// Alg. 1 with symmetric tiles costs (K-2) s^3 + 2 s^2 L_local against
// (K-1) 2 s^2 L_local for apply-to-X: fewer flops whenever K > 2 (s <= L).
// Form 3 (the s x s form on full tiles) is kept for cross-checks.
// With the multi-GPU panel split (P ranks) each rank does 1/P of the s x s recurrence.
static int dense_form(const cpa_svt_handle* h, int64_t s, int64_t L_local, int K, int panel_P = 1) {
  if (K <= 2 || h->form == 1) return 1;
  if (h->form == 2 || h->form == 3) return h->form;
  return (double)(K - 2) * s / panel_P + 2.0 * L_local < 2.0 * (K - 1) * L_local ? 2 : 1;
}
static cpa_svt_status apply_f64(cpa_svt_handle* h, int64_t m, int64_t n, cpa_svt_shard shard,
                                int64_t long_global, const double* X, int64_t ldx, double* Y, int64_t ldy,
                                const cpa_svt_kernel* k, int K, const double* c, cpa_svt_lambda* lam,
                                cpa_svt_info* info);

// NEXT-2 (reading R22): Alg. 1 with T = one-level Haar DWT of the Gram index and the
// high-frequency components of Phi zeroed.  In the transform basis Phi_ = blockdiag(G_L, 0)
// with G_L the Gram of the low-pass half A_L, so Alg. 1 runs on A_L unchanged and line 12
// recombines Y = T_L^T (H_hat(G_L) A_L) + h_hat(0) T_H^T A_H.
static cpa_svt_status apply_f64_haar(cpa_svt_handle* h, int64_t m, int64_t n, const double* X, int64_t ldx,
                                     double* Y, int64_t ldy, const cpa_svt_kernel* k, int K, const double* c,
                                     cpa_svt_lambda* lam, cpa_svt_info* info) {
  const bool left = m <= n;
  const int64_t s = left ? m : n, L = left ? n : m, nh = s / 2, nl = s - nh;
  const size_t nL = ((size_t)nl * L + 31) / 32 * 32, nH = ((size_t)nh * L + 31) / 32 * 32;
  cpa_svt_status st = grow(h, &h->tws, &h->tws_bytes, (2 * nL + nH) * sizeof(double) + 256);
  if (st != CPA_SVT_OK) return st;
  double* AL = (double*)h->tws;
  double* YL = AL + nL;
  double* AH = YL + nL;
  {
    Phase p(h, CPA_SVT_PH_GRAM);
    CU(dense_haar_split(X, m, n, ldx, left, AL, AH, h->num_sms, h->stream));
  }
  const int64_t ml = left ? nl : m, nn = left ? n : nl;   // A_L in X's orientation
  h->transform = 0;
  const int div_mode = h->div_mode;
  h->div_mode = 0;   // the check below covers the recombined output
  st = apply_f64(h, ml, nn, CPA_SVT_SHARD_NONE, 0, AL, nn, YL, nn, k, K, c, lam, info);
  h->transform = 1;
  h->div_mode = div_mode;
  if (st != CPA_SVT_OK) return st;
  int nlh = 2;
  {
    Phase p(h, CPA_SVT_PH_FINAL);
    CU(dense_haar_combine(YL, AH, h->P, m, n, left, Y, ldy, h->num_sms, h->stream));
  }
  st = check_f64(h, X, m, n, ldx, Y, m, n, ldy, &nlh);
  if (st != CPA_SVT_OK) return st;
  h->launches += nlh;
  if (info) {
    info->kernel_launches += nlh;
    info->side = left ? 0 : 1;
  }
  return fill_info(h, info, lam, left ? 0 : 1);
}

static cpa_svt_status apply_f64(cpa_svt_handle* h, int64_t m, int64_t n, cpa_svt_shard shard,
                                int64_t long_global, const double* X, int64_t ldx, double* Y, int64_t ldy,
                                const cpa_svt_kernel* k, int K, const double* c, cpa_svt_lambda* lam,
                                cpa_svt_info* info) {
  if (h->transform == 1) {
    if (shard != CPA_SVT_SHARD_NONE && h->comm != nullptr) return CPA_SVT_E_UNSUPPORTED;
    return apply_f64_haar(h, m, n, X, ldx, Y, ldy, k, K, c, lam, info);
  }
  // side selection (reading R3): left iff global m <= global n
  bool left;
  if (shard == CPA_SVT_SHARD_COLS) {
    if (m > long_global || long_global < n) return CPA_SVT_E_ARG;
    left = true;
  } else if (shard == CPA_SVT_SHARD_ROWS) {
    if (long_global <= n || long_global < m) return CPA_SVT_E_ARG;
    left = false;
  } else {
    left = m <= n;
  }
  const int64_t s = left ? m : n, L = left ? n : m;
  const bool sharded = shard != CPA_SVT_SHARD_NONE && h->comm != nullptr;
  const bool dct = h->transform == 2 || h->transform == 3;   // NEXT-2 DCT variants (Phi = C G C^T, thresholded)
  const bool bdct = h->transform == 3;     // 8 x 8 block DCT
  const bool sparse_eps = dct && h->eps_mode != 0;
  if (dct && sharded) return CPA_SVT_E_UNSUPPORTED;
  // validated before any device work or collective (see apply_tf32)
  if (!(lam->lambda_max > 0.0) && s * (int64_t)sizeof(double) > 200 * 1024) return CPA_SVT_E_UNSUPPORTED;
  // small problems (s <= 64, L <= 128, e.g. BASELINE configs[0]): all of Alg. 1 in one
  // thread block (small_f64.cu) -- the s x s form, automatic form selection only
  if (!sharded && !dct && h->form == 0 && small_f64_fits(m, n) && !env_on("CPA_SVT_NO_SMALL")) {
    if (h->hp_X) {
      CU(cudaMemcpyAsync((double*)X, h->hp_X, (size_t)m * n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
      h->hp_X = nullptr;
    }
    const double* c_small = nullptr;
    if (c) {
      CU(cudaMemcpyAsync(h->d_c, c, K * sizeof(double), cudaMemcpyHostToDevice, h->stream));
      c_small = h->d_c;
    }
    PhaseTimer tm;
    tm.start(info != nullptr, h->stream);
    {
      Phase p(h, CPA_SVT_PH_STEP);
      const int nsq = lam->lambda_max > 0.0 ? 0 : power_squarings(s, lam->power_iters);
      // (the SPEC.md:215 divergence check runs inside the kernel: X and Y pass through it anyway)
      CU(launch_small_f64(X, ldx, Y, ldy, m, n, h->P, *k, K, lam->power_iters, lam->safety, lam->lambda_max,
                          c_small, nsq, h->stream, h->div_mode != 0));
    }
    tm.mark();
    const int nl = 1;
    h->launches += nl;
    cpa_svt_status st = fill_info(h, info, lam, left ? 0 : 1);
    if (info) {
      info->ms_gram = info->ms_allreduce = info->ms_power = 0.0f;
      info->ms_recurrence = tm.ms(0, 1);
      info->ms_total = tm.ms(0, 1);
      info->kernel_launches = nl;
      info->form = 4;
      info->rec_products = small_f64_products(m, n, K, lam->lambda_max > 0.0 ? 0 : power_squarings(s, lam->power_iters),
                                              lam->lambda_max);
    }
    return st;
  }
  // Multi-GPU s x s recurrence (form 2, sharded): each rank computes a contiguous 1/P of the
  // lower tiles of every step and the steps' tiles are all-gathered (ncclAllGather, in place)
  // and unpacked into the full Psi_k on every rank -- instead of every rank evaluating the whole
  // s x s recurrence.  CPA_SVT_PANELS=1 forces it at world 1 (real NCCL all-gather of one rank);
  // CPA_SVT_PANEL_SIM=P runs P virtual ranks' panels one after the other on one GPU (tests of the
  // partition / pack / unpack; the slots are already in place, so no collective).
  int panel_sim = 0;
  if (const char* v = getenv("CPA_SVT_PANEL_SIM")) panel_sim = atoi(v);
  const bool panel_cand = K > 2 && !sparse_eps &&
                          ((sharded && (h->world > 1 || env_on("CPA_SVT_PANELS"))) || (panel_sim > 1 && h->world == 1));
  const int panel_cand_P = panel_cand ? (panel_sim > 1 && h->world == 1 ? panel_sim : h->world) : 1;
  // (the form choice sees the per-rank share of the s x s recurrence; sharded: from the global
  // long extent, so that every rank -- an empty block included -- takes the same form and so
  // enqueues the same collectives)
  const int64_t L_form = sharded ? std::max<int64_t>(1, (long_global + h->world - 1) / h->world) : L;
  const int form = dct ? 2 : dense_form(h, s, L_form, K, panel_cand_P);
  const bool poly = form != 1;
  const bool panels = panel_cand && form == 2;
  const int panel_P = panels ? panel_cand_P : 1;
  const size_t nGb = panels ? (size_t)panel_P * (size_t)dense_sym_panel_slot(s, panel_P) * 4096 : 0;
  // the panel form also shards the power iteration by rows of G (one all-gather of u per product)
  const size_t nPR = panels ? (size_t)((power_rows_scratch_doubles(s, panel_P, h->num_sms) + 31) / 32 * 32) : 0;
  if (h->hp_X && (sharded || dct || !poly)) {   // (the host pipeline covers the plain s x s form only)
    CU(cudaMemcpyAsync((double*)X, h->hp_X, (size_t)m * n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    h->hp_X = nullptr;
  }
  // workspace: G (s*s) | W_a | W_b | [I_s | H (s*s) in the poly forms] | power scratch | split-K partials | sync
  // (G^2 and G^4 for the squared power iteration live in W_a / W_b: free until the recurrence)
  const int64_t RM = poly ? s : m, RN = poly ? s : n;  // shape the recurrence runs on
  // every segment starts on a 256-byte boundary (16-byte vector paths, LL words)
  auto r32 = [](size_t v) { return (v + 31) / 32 * 32; };
  const size_t nG = r32((size_t)s * s), nW = r32((size_t)RM * RN), nPow = r32(power_dense_scratch_doubles(s));
  const size_t nX = poly ? 2 * nG : 0;
  // m-chain recurrence (form 2, one launch): 4m - 3 + m - 1 more s x s buffers (Psi_2 .. Psi_m, the
  // chains' rotations beside Wa / Wb / Is, the accumulators HX of all chains but the first)
  const int chain = form == 2 && !panels && !sparse_eps ? dense_sym_use_chain(s, K, h->num_sms) : 0;
  const size_t nCh = chain ? (size_t)(5 * chain - 4) * nG : 0;
  // line 12 folded into the m-chain launch (left side, device-resident Y, no transform; TMA needs
  // 16-byte rows of X): its units follow the last product's, row panel by row panel of H_hat
  const bool fold12 = chain && left && L > 0 && !h->hp_Y && !dct && h->transform == 0 && ldx % 2 == 0 &&
                      ((uintptr_t)X & 15) == 0 && !env_on("CPA_SVT_NO_L12_FOLD");
  const size_t nP12 = fold12 ? r32(dense_sym_l12_partial_doubles(s, n, h->num_sms)) : 0;
  const bool final_split = !env_on("CPA_SVT_FINAL_NOSPLIT");  // line-12 product split-K (default on)
  const size_t nPart = r32(std::max({dense_flow_partial_doubles(RM, RN, h->num_sms), dense_gram_partial_doubles(s),
                                     form == 2 ? dense_sym_partial_doubles(s, h->num_sms, chain) : (size_t)0,
                                     panels ? dense_sym_panel_partial_doubles(s, panel_P, h->num_sms) : (size_t)0,
                                     final_split && poly ? dense_store_partial_doubles(m, n) : (size_t)0}));
  const size_t nSync = std::max({dense_flow_sync_ints(RM, RN, K), (size_t)((s / 64 + 2) * (s / 64 + 2)),
                                 dense_sym_sync_ints(s, K, h->num_sms, fold12 ? n : 0), (size_t)1332});
  const size_t need = (nG + 2 * nW + nX + nPow + nPart + nGb + nPR + nCh + nP12) * sizeof(double) + nSync * sizeof(int) + 256;
  cpa_svt_status st = grow(h, &h->ws, &h->ws_bytes, need);
  if (sharded) st = rank_vote(h, st);
  if (st != CPA_SVT_OK) return st;
  double* G = (double*)h->ws;
  double* Wa = G + nG;
  double* Wb = Wa + nW;
  double* Is = Wb + nW;          // poly form: identity (W_0)
  double* H = Is + nG;           // poly form: H_hat
  double* pw = Wb + nW + nX;
  double* part = pw + nPow;
  double* gbuf = part + nPart;    // panel mode: P all-gather slots of packed 64 x 64 tiles
  double* prs = gbuf + nGb;       // panel mode: row-sharded power iteration scratch
  double* chb = prs + nPR;         // m-chain mode: 5m - 4 s x s buffers
  double* p12 = chb + nCh;         // line 12 in the m-chain launch: its split-K partials
  int* flow_sync = (int*)(p12 + nP12);
  const double* psi2_sq = nullptr;  // m-chain mode: c^2 (device) when chb holds c^2 G^2

  const double* c_dev = nullptr;
  if (c) {
    CU(cudaMemcpyAsync(h->d_c, c, K * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    c_dev = h->d_c;
  }
  PhaseTimer tm;
  tm.start(info != nullptr, h->stream);
  int launches = 0;
  // Alg. 1 line 1: partial Gram of this shard
  {
    Phase p(h, CPA_SVT_PH_GRAM);
    if (h->hp_X && !sharded && !dct) {
      // host pipeline: unit q of the split-K Gram waits only for the q-th k-range of X
      // (columns for the left Gram, rows for the right one) to land
      const int S = cpa_svt_handle::kPipe;
      for (int q = 0; q < S; ++q) {
        int64_t k0, k1;
        dense_gram_chunk_range(left ? n : m, q, S, &k0, &k1);
        if (k1 > k0) {
          if (left)
            CU(cudaMemcpy2DAsync((double*)X + k0, ldx * sizeof(double), h->hp_X + k0, n * sizeof(double),
                                 (k1 - k0) * sizeof(double), m, cudaMemcpyHostToDevice, h->copy_stream));
          else
            CU(cudaMemcpyAsync((double*)X + k0 * ldx, h->hp_X + k0 * n, (k1 - k0) * n * sizeof(double),
                               cudaMemcpyHostToDevice, h->copy_stream));
        }
        CU(cudaEventRecord(h->pev[q], h->copy_stream));
        CU(cudaStreamWaitEvent(h->stream, h->pev[q], 0));
        CU(dense_gram_f64_chunk(X, m, n, ldx, left, G, h->stream, part, flow_sync, q, S));
        ++launches;
      }
      --launches;
    } else if (L == 0) {   // an empty block of a sharded X: a zero partial Gram
      CU(cudaMemsetAsync(G, 0, (size_t)s * s * sizeof(double), h->stream));
      --launches;
    } else {
      CU(dense_gram_f64(X, m, n, ldx, left, G, h->stream, nullptr, part, flow_sync));
    }
  }
  ++launches;
  tm.mark();
  // exchange: G = sum_p G_p over NVLink (one all-reduce per shrinkage)
  if (sharded) {
    Phase p(h, CPA_SVT_PH_ALLREDUCE);
    NC(g_nccl.AllReduce(G, G, nG, ncclDouble, ncclSum, h->comm, h->stream));
  }
  tm.mark();
  // NEXT-2 DCT variant, Alg. 1 lines 1-2: Phi = C G C^T (two DMMA products), then the
  // component threshold into a CSR copy; G holds Phi_ from here on
  double *Cd = nullptr, *CTd = nullptr;
  const int64_t* csr_rp = nullptr;
  const int32_t* csr_col = nullptr;
  const double* csr_val = nullptr;
  if (dct) {
    const size_t nS = r32((size_t)s * s);
    st = grow(h, &h->tws, &h->tws_bytes, 2 * nS * sizeof(double) + (sparse_eps ? dct_eps_scratch_bytes(s) : 0) + 512);
    if (st != CPA_SVT_OK) return st;
    Cd = (double*)h->tws;
    CTd = Cd + nS;
    Phase p(h, CPA_SVT_PH_GRAM);
    if (bdct) {   // block-diagonal C: Phi = C G C^T block pair by block pair
      CU(block_dct_sandwich(G, Wa, s, 0, h->stream));
      CU(cudaMemcpyAsync(G, Wa, (size_t)s * s * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
      launches += 1;
    } else {
      CU(admm_dct(Cd, CTd, s, h->num_sms, h->stream));
      CU(dense_gemm_store(s, s, s, Cd, s, G, s, Wa, s, h->stream));    // C G
      CU(dense_gemm_store(s, s, s, Wa, s, CTd, s, G, s, h->stream));   // (C G) C^T
      launches += 3;
    }
    if (sparse_eps) {
      CU(dct_eps_threshold(G, s, h->eps_mode, h->eps_value, (void*)(CTd + nS), h->num_sms, h->stream, &csr_rp,
                           &csr_col, &csr_val));
      launches += 5;
    }
  }
  // Alg. 1 lines 3-4: Lambda_max and coefficients, on the device
  if (lam->lambda_max > 0.0) {
    Phase p(h, CPA_SVT_PH_POWER);
    CU(launch_series(h->P, *k, K, lam->safety, lam->lambda_max, nullptr, c_dev, h->stream));
  } else if (panels) {
    // row-sharded power iteration: rank p computes rows [s p / P, s (p+1) / P) of every product and
    // the products' slots are all-gathered (in place); virtual ranks one after another in the
    // simulation.  Same products as the replicated iteration (reading R6), another summation order.
    Phase p(h, CPA_SVT_PH_POWER);
    const int64_t pslot = power_rows_slot(s, panel_P);
    CU(cudaMemsetAsync(prs + 2 * panel_P * pslot + h->num_sms, 0, 2 * sizeof(double), h->stream));
    for (int t = 1; t <= lam->power_iters; ++t) {
      const int v0 = panel_sim > 1 ? 0 : h->rank, v1 = panel_sim > 1 ? panel_P : h->rank + 1;
      for (int v = v0; v < v1; ++v) {
        CU(launch_power_rows(G, s, t, v, panel_P, prs, h->num_sms, h->stream));
        ++launches;
      }
      if (panel_sim <= 1) {
        double* gb = power_rows_buffer(prs, s, t, panel_P);
        NC(g_nccl.AllGather(gb + (size_t)h->rank * pslot, gb, (size_t)pslot, ncclDouble, h->comm, h->stream));
      }
    }
    double* lam_dev = nullptr;
    CU(launch_power_rows_final(prs, s, lam->power_iters, panel_P, h->num_sms, &lam_dev, h->stream));
    CU(launch_series(h->P, *k, K, lam->safety, 0.0, lam_dev, c_dev, h->stream));
    launches += 2;
  } else {
    Phase p(h, CPA_SVT_PH_POWER);
    // Repeated squaring: v_{T-1} ~ G^{T-1} v_0 is reached with (T-1)/p products by
    // c^p G^p (p = 2^j, c = 2^-ilogb(max G_ii), exact) plus the remainder by G, then
    // lambda_hat = ||G v_{T-1}|| -- the same quantity as T plain products (reading R6);
    // j from the cost model power_squarings (j = 3 at c2).
    const double* G4 = nullptr;
    int gpow = 1;
    int nsq = power_squarings(s, lam->power_iters);
    if (const char* v = getenv("CPA_SVT_POWER_SQ"); v && *v) nsq = atoi(v);   // (experiments)
    if (nsq > 0 && nW >= nG) {
      double* sc = pw + power_scale_offset(s);  // scale slot inside the power scratch
      CU(launch_diag_scale(G, s, sc, h->stream));
      // m-chain mode: c^2 G^2 lands in the Psi_2 buffer, where the init turns it into Psi_2 =
      // 2 B_hat^2 - I (the recurrence then starts at k = 3); the later squarings use Wa / Wb
      double* first = (chain && K > 2 && !env_on("CPA_SVT_NO_PSI2_SQ")) ? chb : Wa;
      CU(dense_gram_f64(G, s, s, s, true, first, h->stream, sc, part, flow_sync));    // c^2 G^2
      launches += 2;
      if (first == chb) psi2_sq = sc;
      G4 = first;
      gpow = 2;
      for (int j = 1; j < nsq && 2 * gpow <= lam->power_iters - 1; ++j) {              // c^2p G^2p
        double* nxt = G4 == Wa ? Wb : Wa;
        CU(dense_gram_f64(G4, s, s, s, true, nxt, h->stream, nullptr, part, flow_sync));
        G4 = nxt;
        gpow *= 2;
        ++launches;
      }
    }
    CU(launch_power_dense(G, G4, gpow, s, lam->power_iters, pw, h->bar, h->P, *k, K, lam->safety, c_dev, h->num_sms,
                          h->stream));
  }
  ++launches;
  if (sharded) {
    Phase p(h, CPA_SVT_PH_ALLREDUCE, 0);
    NC(g_nccl.Broadcast(h->P, h->P, sizeof(SeriesParams), ncclChar, 0, h->comm, h->stream));
  }
  tm.mark();
  if (!poly) {
    // Alg. 1 lines 5-11 in the apply-to-X form: W_k = Psi_k(B_hat) X, Y = sum c_k W_k (no
    // collectives: an empty block has nothing to do)
    if (L > 0) {
      st = run_recurrence_f64(h, left, m, n, G, X, ldx, Wa, Wb, Y, ldy, K, part, flow_sync, &launches);
      if (st != CPA_SVT_OK) return st;
    }
  } else {
    // Alg. 1 literally: lines 5-11 on the s x s Gram with Psi_0 = Id (H_hat = sum c_k Psi_k),
    // then line 12: Y = H_hat X (left) or X H_hat (right) -- one product
    if (form == 2) {  // symmetric tiles (lower triangle computed, mirrored)
      {
        Phase p(h, CPA_SVT_PH_INIT);
        CU(dense_sym_init(s, G, Wa, H, h->P, K, h->num_sms, h->stream, psi2_sq ? chb : nullptr, psi2_sq));
        ++launches;
      }
      if (K > 2) {
        if (sparse_eps) {  // lines 8-11 on the sparse Phi_ (one launch per step)
          Phase p(h, CPA_SVT_PH_STEP);
          CU(dct_sparse_steps(s, csr_rp, csr_col, csr_val, Wa, Wb, H, h->P, K, h->num_sms, h->stream));
          launches += K - 2;
        } else if (panels) {
          double* Wr[3] = {Is, Wa, Wb};   // Psi_k lives in Wr[k % 3]; Wr[1] = Psi_1 from the init
          const int64_t slot = dense_sym_panel_slot(s, panel_P);
          for (int kk = 2; kk < K; ++kk) {
            const int v0 = panel_sim > 1 ? 0 : h->rank, v1 = panel_sim > 1 ? panel_P : h->rank + 1;
            for (int v = v0; v < v1; ++v) {
              const int64_t t0 = dense_sym_panel_tile0(s, v, panel_P), t1 = dense_sym_panel_tile0(s, v + 1, panel_P);
              Phase ps(h, CPA_SVT_PH_STEP);
              CU(dense_cheb_sym_panel(s, G, Wr[0], Wr[1], Wr[2], H, h->P, K, kk, t0, t1 - t0,
                                      gbuf + (size_t)v * slot * 4096, flow_sync, part, h->num_sms, h->stream));
              ++launches;
            }
            Phase px(h, CPA_SVT_PH_EXCHANGE);
            if (panel_sim <= 1)
              NC(g_nccl.AllGather(gbuf + (size_t)h->rank * slot * 4096, gbuf, (size_t)slot * 4096, ncclDouble,
                                  h->comm, h->stream));
            // Psi_k into its rotation buffer (over Psi_{k-3}); the last step's slots hold H_hat
            CU(dense_sym_unpack(gbuf, s, panel_P, kk == K - 1 ? H : Wr[kk % 3], h->stream));
            ++launches;
          }
        } else {
          Phase p(h, CPA_SVT_PH_STEP);
          if (chain) {   // Psi_1 (Wa, from the init) | Psi_2 .. Psi_m | rotations (Wb, Is, then chb); HX
            double* cb[12];
            cb[0] = Wa;
            double* nxt = chb;
            for (int i = 1; i < 4 * chain; ++i) {
              if (i == chain) cb[i] = Wb;
              else if (i == chain + 1) cb[i] = Is;
              else { cb[i] = nxt; nxt += nG; }
            }
            double* hx[2] = {nxt, nxt + nG};
            CU(dense_cheb_sym(s, G, Is, Wa, Wb, H, h->P, K, flow_sync, part, h->num_sms, h->stream, chain, cb, hx,
                              psi2_sq != nullptr, fold12 ? X : nullptr, ldx, Y, ldy, n, p12));
          } else {
            CU(dense_cheb_sym(s, G, Is, Wa, Wb, H, h->P, K, flow_sync, part, h->num_sms, h->stream));  // Is: 3rd W buffer
          }
          ++launches;
        }
      }
    } else {
      CU(dense_eye(Is, s, h->stream));
      ++launches;
      st = run_recurrence_f64(h, true, s, s, G, Is, s, Wa, Wb, H, s, K, part, flow_sync, &launches);
      if (st != CPA_SVT_OK) return st;
    }
    Phase p(h, CPA_SVT_PH_FINAL);
    // (split-K over the k = s dimension when the tiles alone leave slots idle: c2 111 -> 96 us)
    const double* Hm = H;
    if (bdct) {  // line 12 with T: Y = (C^T H C) X  or  X (C^T H C), C block diagonal
      CU(block_dct_sandwich(H, Wb, s, 1, h->stream));
      launches += 1;
      Hm = Wb;
    } else if (dct) {
      CU(dense_gemm_store(s, s, s, CTd, s, H, s, Wa, s, h->stream));
      CU(dense_gemm_store(s, s, s, Wa, s, Cd, s, Wb, s, h->stream));
      launches += 2;
      Hm = Wb;
    }
    double* fp = final_split ? part : nullptr;
    int* fs = final_split ? flow_sync : nullptr;
    if (h->hp_Y && !dct) {
      // host pipeline: Y leaves in chunks (column blocks for the left product, row blocks
      // for the right one) while the next chunk is computed
      const int S = cpa_svt_handle::kPipe;
      const int64_t Lc = left ? n : m;
      for (int q = 0; q < S; ++q) {
        const int64_t c0 = Lc * q / S / 64 * 64, c1 = q == S - 1 ? Lc : Lc * (q + 1) / S / 64 * 64;
        if (c1 <= c0) continue;
        if (left) {
          CU(dense_gemm_store(s, c1 - c0, s, Hm, s, X + c0, ldx, Y + c0, ldy, h->stream, fp, fs));
          CU(cudaEventRecord(h->pev[S + q], h->stream));
          CU(cudaStreamWaitEvent(h->copy_stream, h->pev[S + q], 0));
          CU(cudaMemcpy2DAsync(h->hp_Y + c0, n * sizeof(double), Y + c0, ldy * sizeof(double),
                               (c1 - c0) * sizeof(double), m, cudaMemcpyDeviceToHost, h->copy_stream));
        } else {
          CU(dense_gemm_store(c1 - c0, s, s, X + c0 * ldx, ldx, Hm, s, Y + c0 * ldy, ldy, h->stream, fp, fs));
          CU(cudaEventRecord(h->pev[S + q], h->stream));
          CU(cudaStreamWaitEvent(h->copy_stream, h->pev[S + q], 0));
          CU(cudaMemcpyAsync(h->hp_Y + c0 * n, Y + c0 * ldy, (c1 - c0) * n * sizeof(double),
                             cudaMemcpyDeviceToHost, h->copy_stream));
        }
        ++launches;
      }
      --launches;
      h->hp_Y = nullptr;   // delivered
    } else if (fold12 || L == 0) {
      --launches;   // (line 12 ran inside the recurrence launch / an empty block: no output)
    } else {
      if (left) CU(dense_gemm_store(s, n, s, Hm, s, X, ldx, Y, ldy, h->stream, fp, fs));
      else      CU(dense_gemm_store(m, s, s, X, ldx, Hm, s, Y, ldy, h->stream, fp, fs));
    }
    ++launches;
  }
  tm.mark();
  if (L > 0) {
    st = check_f64(h, X, m, n, ldx, Y, m, n, ldy, &launches);
    if (st != CPA_SVT_OK) return st;
  }
  h->launches += launches;
  st = fill_info(h, info, lam, left ? 0 : 1);
  if (info) {
    info->ms_gram = tm.ms(0, 1);
    info->ms_allreduce = tm.ms(1, 2);
    info->ms_power = tm.ms(2, 3);
    info->ms_recurrence = tm.ms(3, 4);
    info->ms_total = tm.ms(0, 4);
    info->kernel_launches = launches;
    info->form = form;
    info->rec_products = poly && K > 2 ? K - (psi2_sq ? 3 : 2) : 0;
    info->line12_in_recurrence = fold12 ? 1 : 0;
  }
  return st;
}

// fp32 data on the tcgen05 tensor cores: TF32 (rna operands) or 3xTF32 (hi/lo split).
static cpa_svt_status apply_tf32(cpa_svt_handle* h, int terms, int64_t m, int64_t n, cpa_svt_shard shard,
                                 int64_t long_global, const float* X, int64_t ldx, float* Y, int64_t ldy,
                                 const cpa_svt_kernel* k, int K, const double* c, cpa_svt_lambda* lam,
                                 cpa_svt_info* info) {
  bool left;
  if (shard == CPA_SVT_SHARD_COLS) {
    if (m > long_global || long_global < n) return CPA_SVT_E_ARG;
    left = true;
  } else if (shard == CPA_SVT_SHARD_ROWS) {
    if (long_global <= n || long_global < m) return CPA_SVT_E_ARG;
    left = false;
  } else {
    left = m <= n;
  }
  const bool sharded = shard != CPA_SVT_SHARD_NONE && h->comm != nullptr;
  const int64_t s = left ? m : n, L = left ? n : m;
  if (s > 2147483647 / 2 || L > 2147483647 / 2) return CPA_SVT_E_UNSUPPORTED;
  // every rank validates before the first collective is enqueued (a rank that returned
  // early would leave its peers waiting inside NCCL)
  if (!(lam->lambda_max > 0.0) && s * (int64_t)sizeof(double) > 200 * 1024) return CPA_SVT_E_UNSUPPORTED;
  const int64_t sp = (s + 3) / 4 * 4, Lp = (L + 3) / 4 * 4;
  // s x s form on full tiles (2(K-2) s^3 + 2 s^2 L) when it beats apply-to-X ((K-1) 2 s^2 L)
  const bool poly = K > 2 && h->form != 1;  // symmetric s x s form: fewer flops for any K > 2
  // multi-GPU s x s form by tile panels (as apply_f64): CPA_SVT_PANELS / CPA_SVT_PANEL_SIM for tests
  int panel_sim = 0;
  if (const char* v = getenv("CPA_SVT_PANEL_SIM")) panel_sim = atoi(v);
  const bool panels = poly && ((sharded && (h->world > 1 || env_on("CPA_SVT_PANELS"))) || (panel_sim > 1 && h->world == 1));
  const int panel_P = panels ? (panel_sim > 1 && h->world == 1 ? panel_sim : h->world) : 1;
  const int2* plist = nullptr;
  int pcount = 0, pbn = 0;
  if (panels && tf32_panel_list(s, terms, &plist, &pcount, &pbn) != cudaSuccess) return CPA_SVT_E_NOMEM;
  const int64_t pslot_tiles = panels ? (pcount + panel_P - 1) / panel_P : 0;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t nA = al((size_t)s * Lp * 4), nG = al((size_t)s * sp * 4);
  const size_t nPow = al(power_dense_scratch_doubles(s) * 8);
  const size_t nGb = panels ? al((size_t)panel_P * pslot_tiles * 128 * pbn * 4) : 0;
  const size_t nPR = panels ? al(power_rows_scratch_doubles(s, panel_P, h->num_sms) * 8) : 0;
  // X set (full, hi, lo) | Y_int | G (full, hi, lo) | apply: A set (3 x s*Lp)  poly: I set, B set, H (3 x s*sp each)
  // | power scratch | panel mode: all-gather slots, row-sharded power scratch
  const size_t need = 4 * nA + 3 * nG + (poly ? 9 * nG : 3 * nA) + nPow + nGb + nPR + 256;
  cpa_svt_status st = grow(h, &h->ws, &h->ws_bytes, need);
  if (sharded) st = rank_vote(h, st);
  if (st != CPA_SVT_OK) return st;
  char* b = (char*)h->ws;
  float* Xs[3] = {(float*)b, (float*)(b + nA), (float*)(b + 2 * nA)};
  float* Yi = (float*)(b + 3 * nA);
  float* Gf = (float*)(b + 4 * nA);
  float* Gh = (float*)(b + 4 * nA + nG);
  float* Gl = (float*)(b + 4 * nA + 2 * nG);
  char* rest = b + 4 * nA + 3 * nG;
  float* As[3];
  float* Is[3];
  float* Hs[3];
  double* pw;
  if (!poly) {
    for (int i = 0; i < 3; ++i) As[i] = (float*)(rest + i * nA);
    pw = (double*)(rest + 3 * nA);
  } else {
    for (int i = 0; i < 3; ++i) {
      Is[i] = (float*)(rest + i * nG);
      As[i] = (float*)(rest + (3 + i) * nG);
      Hs[i] = (float*)(rest + (6 + i) * nG);
    }
    pw = (double*)(rest + 9 * nG);
  }
  float* gbufF = (float*)((char*)pw + nPow);
  double* prs = (double*)((char*)gbufF + nGb);
  const double* c_dev = nullptr;
  if (c) {
    CU(cudaMemcpyAsync(h->d_c, c, K * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    c_dev = h->d_c;
  }
  PhaseTimer tm;
  tm.start(info != nullptr, h->stream);
  int launches = 0;
  if (L == 0) {   // an empty block of a sharded X: a zero partial Gram (the split copies are
                  // rebuilt from the reduced Gram below)
    Phase p(h, CPA_SVT_PH_GRAM);
    CU(cudaMemsetAsync(Gf, 0, (size_t)s * sp * sizeof(float), h->stream));
  } else {
    Phase p(h, CPA_SVT_PH_GRAM);
    CU(tf32_prep(X, m, n, ldx, !left, Xs[0], Xs[1], Xs[2], Lp, h->num_sms, h->stream));
    // Gram always 3xTF32: G(i,j) = sum_l A(i,l) A(j,l), both operands K-major
    // lower-triangle tiles only, mirrored (G exactly symmetric)
    CU(tc_gemm(0, 3, (int)s, (int)s, (int)L, Xs[1], Xs[2], Lp, Xs[1], Xs[2], Lp, false, Gf, Gh, Gl, 3, sp, nullptr,
               nullptr, 0, nullptr, 0, nullptr, 0, h->num_sms, h->stream, 1));
    launches += 2;
  }
  tm.mark();
  if (sharded) {
    Phase p(h, CPA_SVT_PH_ALLREDUCE);
    // the split copies are rebuilt from the reduced full Gram below
    NC(g_nccl.AllReduce(Gf, Gf, (size_t)s * sp, ncclFloat, ncclSum, h->comm, h->stream));
    CU(tf32_prep(Gf, s, sp, sp, false, Gf, Gh, Gl, sp, h->num_sms, h->stream));
    ++launches;
  }
  tm.mark();
  if (lam->lambda_max > 0.0) {
    Phase p(h, CPA_SVT_PH_POWER);
    CU(launch_series(h->P, *k, K, lam->safety, lam->lambda_max, nullptr, c_dev, h->stream));
  } else if (panels) {   // row-sharded power iteration (as apply_f64)
    Phase p(h, CPA_SVT_PH_POWER);
    const int64_t pslot = power_rows_slot(s, panel_P);
    CU(cudaMemsetAsync(prs + 2 * panel_P * pslot + h->num_sms, 0, 2 * sizeof(double), h->stream));
    for (int t = 1; t <= lam->power_iters; ++t) {
      const int v0 = panel_sim > 1 ? 0 : h->rank, v1 = panel_sim > 1 ? panel_P : h->rank + 1;
      for (int v = v0; v < v1; ++v) {
        CU(launch_power_rows_f32(Gf, s, sp, t, v, panel_P, prs, h->num_sms, h->stream));
        ++launches;
      }
      if (panel_sim <= 1) {
        double* gb = power_rows_buffer(prs, s, t, panel_P);
        NC(g_nccl.AllGather(gb + (size_t)h->rank * pslot, gb, (size_t)pslot, ncclDouble, h->comm, h->stream));
      }
    }
    double* lam_dev = nullptr;
    CU(launch_power_rows_final(prs, s, lam->power_iters, panel_P, h->num_sms, &lam_dev, h->stream));
    CU(launch_series(h->P, *k, K, lam->safety, 0.0, lam_dev, c_dev, h->stream));
  } else {
    Phase p(h, CPA_SVT_PH_POWER);
    CU(launch_power_dense_f32(Gf, s, sp, lam->power_iters, pw, h->bar, h->P, *k, K, lam->safety, c_dev, h->num_sms,
                              h->stream));
  }
  ++launches;
  if (sharded) {
    Phase p(h, CPA_SVT_PH_ALLREDUCE, 0);
    NC(g_nccl.Broadcast(h->P, h->P, sizeof(SeriesParams), ncclChar, 0, h->comm, h->stream));
  }
  tm.mark();
  // W_0 and the shape of the recurrence: apply-to-X (s x L, W_0 = A) or the s x s form (W_0 = Id)
  float** W0 = poly ? Is : Xs;
  const int64_t RN = poly ? s : L, ldr = poly ? sp : Lp;
  float* Yr = poly ? Hs[0] : Yi;
  float** sets[2] = {W0, As};
  if (poly) {
    // symmetric s x s form: W_1 = B_hat and H elementwise (no product), then lower-triangle
    // tiles per step with the TF32 operand copies mirrored; W_0 = I is read by step 2 only
    CU(tf32_eye(Is[0], s, sp, h->num_sms, h->stream));
    {
      Phase p(h, CPA_SVT_PH_INIT);
      CU(tf32_sym_init(Gf, s, sp, As[0], As[1], terms == 3 ? As[2] : nullptr, Hs[0], h->P, h->num_sms, h->stream));
    }
    launches += 2;
  }
  for (int kk = poly ? 2 : 1; kk < K && panels; ++kk) {
    // multi-GPU: this rank's 1/P of the step's lower tiles, packed; in-place all-gather; unpack the
    // full W_k (fp32 lower + TF32 hi / lo copies of both triangles), or H after the last step
    float** src = sets[(kk - 1) & 1];
    float** out = sets[kk & 1];
    const bool last = kk == K - 1;
    const size_t slotF = (size_t)pslot_tiles * 128 * pbn;
    const int v0 = panel_sim > 1 ? 0 : h->rank, v1 = panel_sim > 1 ? panel_P : h->rank + 1;
    for (int v = v0; v < v1; ++v) {
      const int64_t t0 = (int64_t)pcount * v / panel_P, t1 = (int64_t)pcount * (v + 1) / panel_P;
      Phase ps(h, CPA_SVT_PH_STEP);
      CU(tc_gemm_panel(terms, (int)s, Gh, Gl, sp, src[1], src[2], ldr, last, ldr, src[0], out[0], ldr, Yr, ldr, h->P,
                       kk, t0, t1 - t0, gbufF + (size_t)v * slotF, h->num_sms, h->stream));
      ++launches;
    }
    Phase px(h, CPA_SVT_PH_EXCHANGE);
    if (panel_sim <= 1)
      NC(g_nccl.AllGather(gbufF + (size_t)h->rank * slotF, gbufF, slotF, ncclFloat, h->comm, h->stream));
    CU(tf32_sym_unpack(gbufF, s, terms, panel_P, pslot_tiles, ldr, out[0], out[1], out[2], last ? Yr : nullptr,
                       h->stream));
    ++launches;
  }
  for (int kk = poly ? 2 : 1; kk < K && !panels && RN > 0; ++kk) {
    float** src = sets[(kk - 1) & 1];      // W_{k-1}: k=1 -> W_0
    float** out = sets[kk & 1];            // W_k overwrites W_{k-2} (k >= 2)
    const bool last = kk == K - 1;
    Phase p(h, kk == 1 ? CPA_SVT_PH_INIT : CPA_SVT_PH_STEP);
    CU(tc_gemm(kk == 1 ? 1 : 2, terms, (int)s, (int)RN, (int)s, Gh, Gl, sp, src[1], src[2], ldr, true,
               last ? nullptr : out[0], last ? nullptr : out[1], last ? nullptr : out[2], terms, ldr, src[0],
               kk == 1 ? nullptr : out[0], ldr, Yr, ldr, h->P, kk, h->num_sms, h->stream, poly ? 1 : 0));
    ++launches;
  }
  if (poly && L > 0) {
    // Alg. 1 line 12: Y = H_hat A, one tcgen05 product (H_hat split into hi/lo operands)
    Phase p(h, CPA_SVT_PH_FINAL);
    CU(tf32_sym_prep(Hs[0], s, sp, Hs[1], Hs[2], h->num_sms, h->stream));  // H lower -> full hi / lo
    CU(tc_gemm(0, terms, (int)s, (int)L, (int)s, Hs[1], Hs[2], sp, Xs[1], Xs[2], Lp, true, Yi, nullptr, nullptr, 1,
               Lp, nullptr, nullptr, 0, nullptr, 0, nullptr, 0, h->num_sms, h->stream));
    launches += 2;
  }
  if (L > 0) {
    CU(tf32_finish(Yi, Lp, m, n, !left, Y, ldy, h->num_sms, h->stream));
    ++launches;
  }
  tm.mark();
  if (h->div_mode && L > 0) {
    Phase p(h, CPA_SVT_PH_FINAL, 0);
    CU(divergence_check_f32(X, m, n, ldx, Y, m, n, ldy, h->dchk, h->P, h->stream));
    launches += 1;
  }
  h->launches += launches;
  st = fill_info(h, info, lam, left ? 0 : 1);
  if (info) {
    info->ms_gram = tm.ms(0, 1);
    info->ms_allreduce = tm.ms(1, 2);
    info->ms_power = tm.ms(2, 3);
    info->ms_recurrence = tm.ms(3, 4);
    info->ms_total = tm.ms(0, 4);
    info->kernel_launches = launches;
    info->form = poly ? 2 : 1;
  }
  return st;
}

cpa_svt_status cpa_svt_apply(cpa_svt_handle* h, cpa_svt_dtype dtype, cpa_svt_math math, int64_t m, int64_t n,
                             cpa_svt_shard shard, int64_t long_global, const void* X, int64_t ldx, void* Y,
                             int64_t ldy, const cpa_svt_kernel* k, int K, const double* c, cpa_svt_lambda* lam,
                             cpa_svt_info* info) {
  if (!h) return CPA_SVT_E_ARG;
  if (m < 0 || n < 0 || ldx < n || ldy < n || K < 2 || K > CPA_SVT_KMAX) return CPA_SVT_E_ARG;
  if (shard < CPA_SVT_SHARD_NONE || shard > CPA_SVT_SHARD_ROWS) return CPA_SVT_E_ARG;
  if ((dtype != CPA_SVT_F64 && dtype != CPA_SVT_F32) || math < CPA_SVT_MATH_NATIVE || math > CPA_SVT_MATH_3XTF32)
    return CPA_SVT_E_ARG;   // (bad enum; valid but unbuilt combinations are E_UNSUPPORTED below)
  // Empty inputs.  Without a shard mode (or a communicator) an empty X has an empty Y: nothing
  // to do, no device work.  In a sharded call the rank's block of the long dimension may be
  // empty (a long extent below the world size: dist.shard_range): that rank still takes part in
  // every collective with a zero partial Gram and its share of the s x s steps, and writes no
  // output; the short dimension is global and must be >= 1.
  const bool sharded_call = shard != CPA_SVT_SHARD_NONE && h->comm != nullptr;
  const bool empty_block = sharded_call && (shard == CPA_SVT_SHARD_COLS ? (n == 0 && m >= 1) : (m == 0 && n >= 1));
  if (!empty_block && (m >= 1 && n >= 1) && (!X || !Y || X == Y)) return CPA_SVT_E_ARG;
  if (!c) {
    cpa_svt_status st = check_kernel(k);
    if (st != CPA_SVT_OK) return st;
  }
  cpa_svt_status st = check_lambda(lam);
  if (st != CPA_SVT_OK) return st;
  const bool supported = (dtype == CPA_SVT_F64 && math == CPA_SVT_MATH_NATIVE) ||
                         (dtype == CPA_SVT_F32 && (math == CPA_SVT_MATH_TF32 || math == CPA_SVT_MATH_3XTF32) &&
                          !h->transform);
  if (!supported) return CPA_SVT_E_UNSUPPORTED;
  if ((m == 0 || n == 0) && !empty_block) {
    if (sharded_call) return CPA_SVT_E_ARG;   // (an empty short dimension: the global X is empty)
    if (info) {
      *info = cpa_svt_info{};
      info->side = m <= n ? 0 : 1;
      info->degenerate = 1;
    }
    if (lam && lam->want_lambda) {
      lam->lambda_hat = lam->lambda_max > 0.0 ? lam->lambda_max / lam->safety : 0.0;
      if (!(lam->lambda_max > 0.0)) lam->lambda_max = 0.0;
    }
    return CPA_SVT_OK;
  }
  if (cudaSetDevice(h->device) != cudaSuccess) return CPA_SVT_E_CUDA;
  cpa_svt_kernel kz{};
  if (!k) k = &kz;
  if (dtype == CPA_SVT_F64 && math == CPA_SVT_MATH_NATIVE)
    return guard_check(h, apply_f64(h, m, n, shard, long_global, (const double*)X, ldx, (double*)Y, ldy, k, K, c,
                                    lam, info));
  if (h->transform) return CPA_SVT_E_UNSUPPORTED;  // the transform variant is fp64-only
  if (dtype == CPA_SVT_F32 && (math == CPA_SVT_MATH_TF32 || math == CPA_SVT_MATH_3XTF32))
    return guard_check(h, apply_tf32(h, math == CPA_SVT_MATH_TF32 ? 1 : 3, m, n, shard, long_global, (const float*)X,
                                     ldx, (float*)Y, ldy, k, K, c, lam, info));
  return CPA_SVT_E_UNSUPPORTED;
}

cpa_svt_status cpa_svt_debug_gemm_tf32(cpa_svt_handle* h, int M, int N, int Kd, const float* A, int64_t lda,
                                       const float* B, int64_t ldb, int b_mn, float* C, int64_t ldc, int terms) {
  if (!h || !A || !B || !C || M < 1 || N < 1 || Kd < 1 || (terms != 1 && terms != 3)) return CPA_SVT_E_ARG;
  if (lda % 4 || ldb % 4 || ldc % 4) return CPA_SVT_E_ARG;
  if (cudaSetDevice(h->device) != cudaSuccess) return CPA_SVT_E_CUDA;
  const int64_t ra = M, ca = lda, rb = b_mn ? Kd : N, cb = ldb;
  const size_t na = (size_t)ra * ca, nb = (size_t)rb * cb;
  cpa_svt_status st = grow(h, &h->ws, &h->ws_bytes, (2 * na + 2 * nb) * 4 + 1024);
  if (st != CPA_SVT_OK) return st;
  float* Ah = (float*)h->ws;
  float* Al = Ah + ((na + 63) / 64) * 64;
  float* Bh = Al + ((na + 63) / 64) * 64;
  float* Bl = Bh + ((nb + 63) / 64) * 64;
  float* dummy = nullptr;
  CU(tf32_prep(A, ra, ca, lda, false, Ah /*full copy unused*/, Ah, Al, ca, h->num_sms, h->stream));
  CU(tf32_prep(B, rb, cb, ldb, false, Bh, Bh, Bl, cb, h->num_sms, h->stream));
  CU(tc_gemm(0, terms, M, N, Kd, Ah, Al, lda, Bh, Bl, ldb, b_mn != 0, C, dummy, dummy, 1, ldc, nullptr, nullptr, 0,
             nullptr, 0, nullptr, 0, h->num_sms, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return CPA_SVT_OK;
}

cpa_svt_status cpa_svt_apply_host(cpa_svt_handle* h, cpa_svt_dtype dtype, cpa_svt_math math, int64_t m, int64_t n,
                                  const void* X_host, void* Y_host, const cpa_svt_kernel* k, int K,
                                  cpa_svt_lambda* lam, cpa_svt_info* info) {
  if (!h || m < 0 || n < 0) return CPA_SVT_E_ARG;
  if (m == 0 || n == 0)   // an empty X: cpa_svt_apply validates the rest and returns (no device work)
    return cpa_svt_apply(h, dtype, math, m, n, CPA_SVT_SHARD_NONE, 0, nullptr, n, nullptr, n, k, K, nullptr, lam,
                         info);
  if (!X_host || !Y_host) return CPA_SVT_E_ARG;
  const size_t es = dtype == CPA_SVT_F64 ? 8 : 4;
  const size_t bytes = (size_t)m * n * es;
  if (cudaSetDevice(h->device) != cudaSuccess) return CPA_SVT_E_CUDA;
  cpa_svt_status st = grow(h, &h->hx, &h->hx_bytes, 2 * bytes + 256);
  if (st != CPA_SVT_OK) return st;
  char* dX = (char*)h->hx;
  char* dY = dX + ((bytes + 255) / 256) * 256;
  // fp64 s x s polynomial form (no transform): copies overlapped with the split-K Gram and
  // with line 12 (apply_f64); otherwise one copy each way around the call
  const int64_t s = std::min(m, n), L = std::max(m, n);
  const int64_t tri = ((s + 63) / 64) * ((s + 63) / 64 + 1) / 2;
  const bool pipe = dtype == CPA_SVT_F64 && math == CPA_SVT_MATH_NATIVE && h->transform == 0 && K > 2 &&
                    dense_form(h, s, L, K) != 1 && s >= 256 && tri < 1332 && !env_on("CPA_SVT_HOST_NOPIPE");
  if (pipe) {
    if (!h->copy_stream && cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
      return CPA_SVT_E_CUDA;
    for (auto& e : h->pev)
      if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return CPA_SVT_E_CUDA;
    // the previous call's work on dX / dY is ordered before this call's copies
    CU(cudaEventRecord(h->pev[0], h->stream));
    CU(cudaStreamWaitEvent(h->copy_stream, h->pev[0], 0));
    h->hp_X = (const double*)X_host;
    h->hp_Y = (double*)Y_host;
    st = cpa_svt_apply(h, dtype, math, m, n, CPA_SVT_SHARD_NONE, 0, dX, n, dY, n, k, K, nullptr, lam, info);
    const bool delivered = h->hp_Y == nullptr;
    h->hp_X = nullptr;
    h->hp_Y = nullptr;
    if (st != CPA_SVT_OK && st != CPA_SVT_E_DIVERGED) {
      cudaStreamSynchronize(h->copy_stream);
      return st;
    }
    if (!delivered) CU(cudaMemcpyAsync(Y_host, dY, bytes, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaStreamSynchronize(h->copy_stream));
    return guard_check(h, read_verdict(h));
  }
  CU(cudaMemcpyAsync(dX, X_host, bytes, cudaMemcpyHostToDevice, h->stream));
  st = cpa_svt_apply(h, dtype, math, m, n, CPA_SVT_SHARD_NONE, 0, dX, n, dY, n, k, K, nullptr, lam, info);
  if (st != CPA_SVT_OK && st != CPA_SVT_E_DIVERGED) return st;
  CU(cudaMemcpyAsync(Y_host, dY, bytes, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return guard_check(h, read_verdict(h));
}

// NEXT-3 (synthetic experiment PAPER.md:1095-1100): ADMM recovery of L from
// the observed entries of D.  K l = [l; Psi l; Omega l; l], Psi = C_m . C_n^T (orthonormal 2-D
// DCT), K^T K = (3 + mask) I; the nuclear prox is the CPA shrinkage (soft, tau = 1/rho) of this
// handle.  One host sync per iteration (the stopping test).
cpa_svt_status cpa_svt_admm_recover(cpa_svt_handle* h, int64_t m, int64_t n, const double* D, const uint8_t* mask,
                                    int K, const cpa_svt_lambda* lam, cpa_svt_admm* opt, double* L) {
  if (!h || !opt || !lam || m < 0 || n < 0 || K < 2 || K > CPA_SVT_KMAX) return CPA_SVT_E_ARG;
  const bool empty = m == 0 || n == 0;   // an empty D: nothing to recover, no device work
  if (!empty && (!D || !mask || !L)) return CPA_SVT_E_ARG;
  if (!(opt->rho > 0.0) || !(opt->eta >= 0.0) || !(opt->tol >= 0.0) || opt->max_iter < 1) return CPA_SVT_E_DOMAIN;
  cpa_svt_status st = check_lambda(lam);
  if (st != CPA_SVT_OK) return st;
  if (empty) {
    opt->iters = 0;
    opt->last_rel = 0.0;
    opt->ms_shrink = opt->ms_total = 0.0;
    return CPA_SVT_OK;
  }
  if (cudaSetDevice(h->device) != cudaSuccess) return CPA_SVT_E_CUDA;
  const int64_t N = m * n;
  auto r32 = [](size_t v) { return (v + 31) / 32 * 32; };
  const size_t nb = r32((size_t)N), nm = r32((size_t)(m * m)), nn = r32((size_t)(n * n));
  const int nparts = admm_tail_blocks();
  st = grow(h, &h->aws, &h->aws_bytes, (14 * nb + 2 * nm + 2 * nn + 2 * (size_t)nparts) * sizeof(double) + 256);
  if (st != CPA_SVT_OK) return st;
  double* p = (double*)h->aws;
  auto take = [&](size_t cnt) { double* q = p; p += cnt; return q; };
  double *Cm = take(nm), *CmT = take(nm), *Cn = take(nn), *CnT = take(nn);
  double *z1 = take(nb), *z2 = take(nb), *z4 = take(nb), *u1 = take(nb), *u2 = take(nb), *u3 = take(nb),
         *u4 = take(nb), *la = take(nb), *lb = take(nb), *pl = take(nb), *t = take(nb), *tmp = take(nb),
         *A1 = take(nb), *pt = take(nb);
  double* part = take(2 * (size_t)nparts);
  CU(admm_dct(Cm, CmT, m, h->num_sms, h->stream));
  CU(admm_dct(Cn, CnT, n, h->num_sms, h->stream));
  for (double* b : {z1, z2, z4, u1, u2, u3, u4, la})
    CU(cudaMemsetAsync(b, 0, (size_t)N * sizeof(double), h->stream));
  cpa_svt_kernel kern{};
  kern.kind = CPA_SVT_SOFT;
  kern.tau = 1.0 / opt->rho;
  kern.tau_relative = 0;
  cpa_svt_lambda lm = *lam;
  lm.want_lambda = 0;
  // adaptive epsilon (eq. recommendation_epsilon; reading R25): the k-th
  // largest |Phi_ij| with k from the previous iteration's error, the handle's setting restored after
  if (opt->adaptive_eps && h->transform != 2 && h->transform != 3) return CPA_SVT_E_ARG;
  const int saved_mode = h->eps_mode;
  const double saved_value = h->eps_value;
  const int64_t s_adm = std::min(m, n);
  auto eps_k = [&](double E) {
    const double frac = E > 0.3e-1 ? 0.5e-4 : (E > 6e-4 ? 1.5e-4 : 0.5e-3);
    return std::max(1.0, std::floor(frac * (double)s_adm * (double)s_adm));
  };
  double E_prev = INFINITY;
  cudaEvent_t e0, e1, ea, eb;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&ea); cudaEventCreate(&eb);
  cudaEventRecord(ea, h->stream);
  std::vector<double> hp(2 * (size_t)nparts);
  double ms_shrink = 0.0, rel = 0.0;
  double* l = la;
  double* lprev = lb;
  int it = 0;
  for (; it < opt->max_iter; ++it) {
    std::swap(l, lprev);   // lprev = l_t; l receives l_{t+1}
    // Psi^T (z2 - u2) = C_m^T (z2 - u2) C_n
    CU(admm_sub(z2, u2, tmp, N, h->stream));
    CU(dense_gemm_store(m, n, m, CmT, m, tmp, n, A1, n, h->stream));
    CU(dense_gemm_store(m, n, n, A1, n, Cn, n, pt, n, h->stream));
    CU(admm_l(z1, u1, pt, mask, D, u3, z4, u4, l, t, N, h->stream));
    // Psi l = C_m l C_n^T
    CU(dense_gemm_store(m, n, m, Cm, m, l, n, A1, n, h->stream));
    CU(dense_gemm_store(m, n, n, A1, n, CnT, n, pl, n, h->stream));
    // z1 = prox_{1/rho ||.||_*}(l + u1): the CPA shrinkage
    cudaEventRecord(e0, h->stream);
    if (opt->adaptive_eps) {
      h->eps_mode = 2;
      h->eps_value = eps_k(E_prev);
    }
    st = apply_f64(h, m, n, CPA_SVT_SHARD_NONE, 0, t, n, z1, n, &kern, K, nullptr, &lm, nullptr);
    if (opt->adaptive_eps) {
      h->eps_mode = saved_mode;
      h->eps_value = saved_value;
    }
    if (st != CPA_SVT_OK) return st;
    cudaEventRecord(e1, h->stream);
    CU(admm_tail(l, lprev, pl, z1, mask, D, z2, z4, u1, u2, u3, u4, opt->eta / opt->rho, N, part, h->stream));
    CU(cudaMemcpyAsync(hp.data(), part, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    ms_shrink += ms;
    double a = 0.0, b = 0.0;
    for (int i = 0; i < nparts; ++i) {
      a += hp[2 * i];
      b += hp[2 * i + 1];
    }
    rel = sqrt(a) / fmax(sqrt(b), 1e-300);
    E_prev = rel;
    h->launches += 9;
    if (rel < opt->tol) {
      ++it;
      break;
    }
  }
  cudaEventRecord(eb, h->stream);
  CU(cudaMemcpyAsync(L, l, (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  float mt = 0.f;
  cudaEventElapsedTime(&mt, ea, eb);
  cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(ea); cudaEventDestroy(eb);
  opt->iters = it;
  opt->last_rel = rel;
  opt->ms_shrink = ms_shrink;
  opt->ms_total = mt;
  return guard_check(h, CPA_SVT_OK);
}

cpa_svt_status cpa_svt_apply_batched(cpa_svt_handle* h, int64_t batch, int m, int n, const float* X, float* Y,
                                     const cpa_svt_kernel* k, int K, const cpa_svt_lambda* lam,
                                     float* lambda_out) {
  if (!h || batch < 0 || m < 0 || n < 0) return CPA_SVT_E_ARG;
  const bool empty = batch == 0 || m == 0 || n == 0;   // nothing to shrink: no device work
  if (!empty && (!X || !Y || (const void*)X == (void*)Y)) return CPA_SVT_E_ARG;
  if (K < 2 || K > CPA_SVT_KMAX) return CPA_SVT_E_ARG;
  cpa_svt_status st = check_kernel(k);
  if (st != CPA_SVT_OK) return st;
  st = check_lambda(lam);
  if (st != CPA_SVT_OK) return st;
  if (K > 128 || m > 64 || n > 64) return CPA_SVT_E_UNSUPPORTED;   // (the header's contract)
  if (empty) return CPA_SVT_OK;
  if (cudaSetDevice(h->device) != cudaSuccess) return CPA_SVT_E_CUDA;
  st = grow(h, &h->ws, &h->ws_bytes, 128 * 128 * sizeof(double));  // cos table
  if (st != CPA_SVT_OK) return st;
  int launches = 0;
  {
    Phase p(h, CPA_SVT_PH_BATCHED);
    if (h->batched_engine == 1)
      CU(launch_batched_f32(batch, m, n, X, Y, *k, K, lam->power_iters, lam->safety, lam->lambda_max, lambda_out,
                            h->num_sms, h->stream, &launches, (double*)h->ws));
    else
      CU(launch_batched_tc(batch, m, n, X, Y, *k, K, lam->power_iters, lam->safety, lam->lambda_max, lambda_out,
                           h->num_sms, h->stream, &launches, (double*)h->ws));
  }
  h->launches += launches;
  return guard_check(h, CPA_SVT_OK);
}

cpa_svt_status cpa_svt_apply_csr(cpa_svt_handle* h, int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                                 const int32_t* col, const double* val, int64_t row_begin, int64_t row_end,
                                 double* Y, int64_t ldy, const cpa_svt_kernel* k, int K, const double* c,
                                 cpa_svt_lambda* lam, cpa_svt_info* info) {
  if (!h || m < 0 || n < 0 || nnz < 0 || (nnz > 0 && (!col || !val))) return CPA_SVT_E_ARG;
  if (row_begin < 0 || row_end > m || row_begin > row_end || ldy < n || K < 2 || K > CPA_SVT_KMAX)
    return CPA_SVT_E_ARG;
  // an empty X (m or n zero): an empty Y, no device work (after the argument checks below)
  const bool empty = m == 0 || n == 0;
  if (!empty && (!row_ptr || (!Y && row_end > row_begin))) return CPA_SVT_E_ARG;
  if (m > 2147483647 || n > 2147483647) return CPA_SVT_E_ARG;
  cpa_svt_status st = CPA_SVT_OK;
  cpa_svt_kernel kz{};
  if (c) {   // raw coefficients replace line 4 (the kernel is not used)
    if (!k) k = &kz;
  } else {
    st = check_kernel(k);
    if (st != CPA_SVT_OK) return st;
  }
  st = check_lambda(lam);
  if (st != CPA_SVT_OK) return st;
  if (empty) {
    if (info) {
      *info = cpa_svt_info{};
      info->side = 1;
      info->degenerate = 1;
    }
    return CPA_SVT_OK;
  }
  if (cudaSetDevice(h->device) != cudaSuccess) return CPA_SVT_E_CUDA;
  const double* c_dev = nullptr;
  if (c) {
    CU(cudaMemcpyAsync(h->d_c, c, K * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    c_dev = h->d_c;
  }
  size_t need = 0;
  CU(sparse_apply(m, n, nnz, row_ptr, col, val, row_begin, row_end, Y, ldy, *k, K, lam->power_iters, lam->safety,
                  lam->lambda_max, h->P, nullptr, 0, &need, h->num_sms, h->stream, nullptr, nullptr, nullptr, c_dev));
  st = grow(h, &h->ws, &h->ws_bytes, need);
  if (st != CPA_SVT_OK) return st;
  PhaseTimer tm;
  tm.start(info != nullptr, h->stream);
  int launches = 0;
  CU(sparse_apply(m, n, nnz, row_ptr, col, val, row_begin, row_end, Y, ldy, *k, K, lam->power_iters, lam->safety,
                  lam->lambda_max, h->P, h->ws, h->ws_bytes, &need, h->num_sms, h->stream, &launches, phase_hook, h,
                  c_dev));
  tm.mark();
  if (h->div_mode && nnz > 0) {   // ||X||_F from the stored values; this rank's rows of Y
    CU(divergence_check_f64(val, 1, nnz, nnz, Y, row_end - row_begin, n, ldy, h->dchk, h->P, h->stream));
    launches += 1;
  }
  h->launches += launches;
  st = fill_info(h, info, lam, 1);
  if (info) {
    info->ms_total = info->ms_recurrence = tm.ms(0, 1);
    info->kernel_launches = launches;
  }
  return guard_check(h, st);
}

}  // extern "C"
