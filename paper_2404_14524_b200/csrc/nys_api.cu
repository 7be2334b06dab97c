// C ABI of libnysipm.so (include/nysipm.h) and the host-side drivers:
//   * sketch_impl  — Alg. 1 on the device
//   * pcg_impl     — PCG with device-resident scalars; the host only polls the
//                    convergence flag once per batch of iterations
//   * ipm_impl     — Alg. 3 / 4 / 5 + App. B for x >= 0
// Multi-GPU: A is column-sharded, m-space objects are replicated; the only exchanges are
// NCCL all-reduces of m-vectors (matvec partials), the m x l sketch, and a few scalars.
#include <dlfcn.h>

#include <chrono>
#include <cstdlib>
#include <condition_variable>
#include <mutex>
#include <cmath>
#include <cstring>
#include <stdexcept>

#include <nvtx3/nvToolsExt.h>

#include "k_vec.cuh"
#include "nccl.h"

using namespace nys;

namespace {
struct NysException {
  int code;
};
// NVTX range per phase of the hot path (visible in nsys / ncu --nvtx; header-only NVTX v3, a no-op
// without an attached tool)
struct NvtxRange {
  explicit NvtxRange(const char* s) { nvtxRangePushA(s); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

static constexpr size_t kGuardBytes = 64 * 1024;
static constexpr unsigned char kGuardByte = 0xA5;

void* nys_ctx::ws(const char* name, size_t bytes) {
  if (bytes == 0) bytes = 8;
  auto it = bufs.find(name);
  if (it != bufs.end() && it->second.second >= bytes) return it->second.first;
  if (it != bufs.end()) {
    if (debug_guard) cudaStreamSynchronize(stream);   // the guard check reads every live buffer
    cudaFree(it->second.first);
    bufs.erase(it);
  }
  void* p = nullptr;
  size_t alloc = bytes < 256 ? 256 : bytes;
  alloc = (alloc + 255) & ~size_t(255);
  cudaError_t e = cudaMalloc(&p, alloc + (debug_guard ? kGuardBytes : 0));
  if (e != cudaSuccess) {
    last_error = std::string("workspace '") + name + "': " + cudaGetErrorString(e);
    cudaGetLastError();
    throw NysException{NYS_ENOMEM};
  }
  if (debug_guard) {                                   // NaN poison + canary (stream-ordered)
    cudaMemsetAsync(p, 0xFF, alloc, stream);
    cudaMemsetAsync((char*)p + alloc, kGuardByte, kGuardBytes, stream);
  }
  bufs[name] = {p, alloc};
  ++ws_epoch;
  return p;
}

namespace {
__global__ void guard_check_kernel(const unsigned char* g, size_t n, unsigned char expect, unsigned int* flag) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (g[i] != expect) { atomicOr(flag, 1u); return; }
}
}  // namespace

int nys_ctx::check_guards() {
  if (!debug_guard) return NYS_OK;
  if (!guard_flag && cudaMalloc(&guard_flag, sizeof(unsigned int)) != cudaSuccess) return NYS_ENOMEM;
  for (auto& kv : bufs) {
    unsigned int h = 0;
    cudaMemsetAsync(guard_flag, 0, sizeof(unsigned int), stream);
    guard_check_kernel<<<64, 256, 0, stream>>>((const unsigned char*)kv.second.first + kv.second.second, kGuardBytes,
                                                kGuardByte, guard_flag);
    cudaMemcpyAsync(&h, guard_flag, sizeof(unsigned int), cudaMemcpyDeviceToHost, stream);
    if (cudaStreamSynchronize(stream) != cudaSuccess) { set_error("guard check: CUDA error"); return NYS_ECUDA; }
    if (h) {
      set_error("NYS_DEBUG_GUARD: out-of-bounds write past workspace '" + kv.first + "' (" +
                std::to_string(kv.second.second) + " bytes)");
      return NYS_ECUDA;
    }
  }
  return NYS_OK;
}

int nys_ctx::check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return NYS_ECUDA;
  }
  return NYS_OK;
}

// ------------------------------------------------------------------------------------------
// NCCL (dlopen'ed only for world > 1)
// ------------------------------------------------------------------------------------------
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) { err = "dlopen(libnccl.so.2) failed"; return false; }
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    getErrorString = (decltype(getErrorString))dlsym(h, "ncclGetErrorString");
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    if (!commInitRank || !allReduce || !commDestroy) { err = "NCCL symbols missing"; return false; }
    return true;
  }
};
NcclApi g_nccl;

// ------------------------------------------------------------------------------------------
// In-process loopback communicator: `world` contexts on ONE device, driven by `world` host
// threads, exchange through host-side barriers.  The sum/min is a fixed-order reduction over the
// ranks' device buffers (bitwise identical on every rank, as NCCL's), done only after every rank
// has synchronised its stream and arrived: no kernel ever waits on another rank's kernel.  It
// exists to run the multi-rank code path (sharding, replicated decisions, every all-reduce) where
// only one GPU is available; production multi-GPU runs use NCCL.
// ------------------------------------------------------------------------------------------
struct LoopComm {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;   // a rank's call failed: its peers leave their collectives with an error
  std::vector<double*> bufs;
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return false;
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || aborted; });
    }
    return !aborted;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};
// a failed collective call on one loopback rank must not leave its peers waiting forever
int loop_abort_on_error(nys_ctx* ctx, int rc) {
  if (ctx && ctx->debug_guard && (rc == NYS_OK || rc == NYS_NOTCONV || rc == NYS_EMAXITER)) {
    const int g = ctx->check_guards();
    if (g != NYS_OK) rc = g;
  }
  if (rc != NYS_OK && rc != NYS_EMAXITER && rc != NYS_NOTCONV && ctx && ctx->loop_comm)
    static_cast<LoopComm*>(ctx->loop_comm)->abort();
  return rc;
}

struct RankPtrs {
  const double* p[16];
};
__global__ void loop_reduce_kernel(RankPtrs R, int world, size_t count, int is_min, double* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double v = R.p[0][i];
    for (int r = 1; r < world; ++r) v = is_min ? fmin(v, R.p[r][i]) : v + R.p[r][i];
    out[i] = v;
  }
}

int loop_allreduce(nys_ctx* ctx, double* buf, size_t count, bool is_min) {
  LoopComm* c = (LoopComm*)ctx->loop_comm;
  NYS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  c->bufs[ctx->rank] = buf;
  if (!c->barrier()) { ctx->set_error("loopback all-reduce: a peer rank failed"); return NYS_ECUDA; }  // buffers final
  double* tmp = ctx->wsd("loop_tmp", count);
  RankPtrs R{};
  for (int r = 0; r < c->world; ++r) R.p[r] = c->bufs[r];
  int g = (int)((count + 255) / 256);
  if (g > 1024) g = 1024;
  loop_reduce_kernel<<<g, 256, 0, ctx->stream>>>(R, c->world, count, is_min ? 1 : 0, tmp);
  NYS_CUDA_TRY(ctx, cudaGetLastError());
  NYS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (!c->barrier()) { ctx->set_error("loopback all-reduce: a peer rank failed"); return NYS_ECUDA; }  // all read
  NYS_CUDA_TRY(ctx, cudaMemcpyAsync(buf, tmp, count * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  return NYS_OK;
}

int allreduce(nys_ctx* ctx, double* buf, size_t count, bool is_min = false) {
  if (!ctx->multi() || count == 0) return NYS_OK;
  if (ctx->loop_comm) return loop_allreduce(ctx, buf, count, is_min);
  ncclResult_t r = g_nccl.allReduce(buf, buf, count, ncclFloat64, is_min ? ncclMin : ncclSum,
                                    (ncclComm_t)ctx->nccl_comm, ctx->stream);
  if (r != ncclSuccess) {
    ctx->set_error(std::string("ncclAllReduce: ") + (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "?"));
    return NYS_ENCCL;
  }
  return NYS_OK;
}
int allreduce_slots(nys_ctx* ctx, int first, int count, bool is_min = false) {
  return allreduce(ctx, ctx->sc + first, (size_t)count, is_min);
}

inline int64_t even(int64_t v) { return (v + 1) & ~int64_t(1); }
// largest Nystrom rank: the sketch, factorisation (global-memory Cholesky and grid Jacobi above 256)
// and graph-path PCG kernels take up to 1024 columns (the paper runs ell = 800 on STL-10);
// the partial Cholesky preconditioner and the persistent PCG keep 256
constexpr int kMaxEll = 1024;
inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

int read_slots(nys_ctx* ctx) {
  NYS_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_sc, ctx->sc, S_COUNT * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  NYS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return NYS_OK;
}

// ------------------------------------------------------------------------------------------
// normal operator (A, d, e, delta) applied to p with the PCG epilogue (or plain)
// ------------------------------------------------------------------------------------------
struct NormalOp {
  int64_t m, n, lda;
  const double* A;
  const double* d;
  const double* e;
  double delta;
};

// w = N_delta v  where v = z + beta*p (beta slot / p may be null); p_out receives v.
// world > 1: local partial sum, all-reduce, then the replicated terms (+ PCG dot) are added
// by launch_finalize_terms (apply_normal_full).
int apply_normal(nys_ctx* ctx, const NormalOp& op, const double* z, const double* p, const double* beta,
                 double* p_out, double* w, bool pcg_alpha, const double* done) {
  MatvecCall c;
  c.mode = MV_FUSED;
  c.m = op.m; c.n = op.n; c.lda = op.lda; c.A = op.A;
  c.z = z; c.p = p; c.beta = beta; c.p_out = p_out; c.d = op.d; c.done = done;
  c.out = w;
  if (!ctx->multi()) {
    c.use_delta = true; c.delta = op.delta; c.e = op.e; c.pcg_alpha = pcg_alpha;
    return launch_matvec(ctx, c);
  }
  c.use_delta = false; c.pcg_alpha = false;
  NYS_TRY(launch_matvec(ctx, c));
  return allreduce(ctx, w, (size_t)op.m);
}
}  // namespace

namespace nys {
int launch_finalize_terms(nys_ctx* ctx, int64_t m, double* w, const double* v, double delta, const double* e,
                          bool pcg_alpha, const double* done);
}

namespace {
int apply_normal_full(nys_ctx* ctx, const NormalOp& op, const double* z, const double* p, const double* beta,
                      double* p_out, double* w, bool pcg_alpha, const double* done) {
  NYS_TRY(apply_normal(ctx, op, z, p, beta, p_out, w, pcg_alpha, done));
  if (ctx->multi()) {
    const double* v = p_out ? p_out : z;
    NYS_TRY(launch_finalize_terms(ctx, op.m, w, v, op.delta, op.e, pcg_alpha, done));
  }
  return NYS_OK;
}

// y = sgn * A u (+ add)   (N-only pass, summed over ranks)
int apply_A(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* u, double* out,
            double sgn, const double* add) {
  MatvecCall c;
  c.mode = MV_NONLY;
  c.m = m; c.n = n; c.lda = lda; c.A = A; c.u = u; c.out = out; c.sgn = sgn;
  if (!ctx->multi()) {
    c.add = add;
    return launch_matvec(ctx, c);
  }
  c.add = nullptr;
  NYS_TRY(launch_matvec(ctx, c));
  NYS_TRY(allreduce(ctx, out, (size_t)m));
  if (add) NYS_TRY(launch_axpby(ctx, m, 1.0, out, 1.0, add, out));
  return NYS_OK;
}

// T-only pass with an epilogue (local columns only: no exchange needed)
int apply_At(nys_ctx* ctx, const MatvecCall& c) { return launch_matvec(ctx, c); }

// ------------------------------------------------------------------------------------------
// Alg. 1: Nystrom factors from the sketch Y (m x l, ld mp) and Omega (ld mp)
// ------------------------------------------------------------------------------------------
// defer: no host read at all (one host round trip per outer iteration, ipm_impl): a failed Cholesky of
// Omega^T Y_nu or of a CholeskyQR pass only raises the device flag S_NYSFAIL; the caller discards the
// iteration when it sees the flag and re-runs it with defer = false (the nu x 10 retries of A4)
int nystrom_factor(nys_ctx* ctx, int64_t m, int ell, const double* Y, const double* Om, int64_t mp, double* U,
                   double* lam, nys_sketch_info* info, bool defer = false) {
  const int ldl = (int)even(ell);
  double* Ynu = ctx->wsd("nf_Ynu", (size_t)mp * ell);
  double* Bm = ctx->wsd("nf_B", (size_t)mp * ell);
  double* Qm = ctx->wsd("nf_Q", (size_t)mp * ell);
  double* G = ctx->wsd("nf_G", (size_t)ldl * ell);
  double* Gi = ctx->wsd("nf_Gi", (size_t)ldl * ell);
  double* R1 = ctx->wsd("nf_R1", (size_t)ldl * ell);
  double* R2 = ctx->wsd("nf_R2", (size_t)ldl * ell);
  double* R3 = ctx->wsd("nf_R3", (size_t)ldl * ell);
  double* Rt = ctx->wsd("nf_Rt", (size_t)ldl * ell);
  double* W = ctx->wsd("nf_W", (size_t)ldl * ell);
  double* sig = ctx->wsd("nf_sig", (size_t)ell);

  // NYS_FACT_TRACE: per-phase device times of this factorisation on stderr (development aid)
  const bool ftrace = getenv("NYS_FACT_TRACE") != nullptr;
  cudaEvent_t fev[8];
  int nfev = 0;
  auto fmark = [&]() {
    if (!ftrace || nfev >= 8) return;
    cudaEventCreate(&fev[nfev]);
    cudaEventRecord(fev[nfev++], ctx->stream);
  };
  fmark();
  NYS_TRY(launch_fro_nu(ctx, m, ell, Y, mp, 0));                      // line 3
  int retries = 0;
  for (;;) {
    NYS_TRY(launch_ynu(ctx, m, ell, Y, Om, Ynu, mp));                 // line 4
    GemmCall g;                                                        // Omega^T Y_nu
    g.M = ell; g.N = ell; g.K = m; g.A = Om; g.lda = mp; g.a_kmajor = true; g.B = Ynu; g.ldb = mp; g.C = G; g.ldc = ldl;
    NYS_TRY(launch_gemm(ctx, g));
    NYS_TRY(launch_set_slots(ctx, S_CHOLFAIL, 0.0));
    NYS_TRY(launch_chol_inv(ctx, ell, G, ldl, Gi, ldl, 0));           // line 5: C (in G), C^{-1}
    if (defer) { NYS_TRY(launch_flag_max(ctx, S_NYSFAIL, S_CHOLFAIL)); break; }
    NYS_TRY(read_slots(ctx));
    if (ctx->h_sc[S_CHOLFAIL] == 0.0) break;
    if (retries >= 3) {
      ctx->set_error("nys_sketch: Omega^T Y_nu not positive definite after 3 retries");
      return NYS_ECHOL;
    }
    ++retries;
    NYS_TRY(launch_set_slots(ctx, S_NU, ctx->h_sc[S_NU] * 10.0));     // A4
  }
  fmark();
  {                                                                    // line 6: B = Y_nu C^{-1}
    GemmCall g;
    g.M = m; g.N = ell; g.K = ell; g.A = Ynu; g.lda = mp; g.a_kmajor = false; g.B = Gi; g.ldb = ldl; g.C = Bm; g.ldc = mp;
    NYS_TRY(launch_gemm(ctx, g));
  }
  // line 7: thin SVD of B.  Shifted CholeskyQR3 (B = Q R), then one-sided Jacobi on R.
  NYS_TRY(launch_set_slots(ctx, S_SHIFT, (double)m, S_CHOLFAIL, 0.0));
  double* src = Bm;
  double* dst = Qm;
  double* Rs[3] = {R1, R2, R3};
  for (int pass = 0; pass < 3; ++pass) {
    GemmCall g;
    g.M = ell; g.N = ell; g.K = m; g.A = src; g.lda = mp; g.a_kmajor = true; g.B = src; g.ldb = mp; g.C = Rs[pass]; g.ldc = ldl;
    NYS_TRY(launch_gemm(ctx, g));
    NYS_TRY(launch_chol_inv(ctx, ell, Rs[pass], ldl, Gi, ldl, pass == 0 ? 1 : 0));
    GemmCall h;
    h.M = m; h.N = ell; h.K = ell; h.A = src; h.lda = mp; h.a_kmajor = false; h.B = Gi; h.ldb = ldl; h.C = dst; h.ldc = mp;
    NYS_TRY(launch_gemm(ctx, h));
    double* tmp = src; src = dst; dst = tmp;
  }
  // src now holds Q; R = R3 R2 R1
  fmark();
  NYS_TRY(launch_trmm_upper(ctx, ell, ldl, R2, R1, Rt));
  NYS_TRY(launch_trmm_upper(ctx, ell, ldl, R3, Rt, G));
  fmark();
  NYS_TRY(launch_jacobi_svd(ctx, ell, G, ldl, W, ldl, sig));
  fmark();
  {                                                                    // U = Q W
    GemmCall g;
    g.M = m; g.N = ell; g.K = ell; g.A = src; g.lda = mp; g.a_kmajor = false; g.B = W; g.ldb = ldl; g.C = U; g.ldc = mp;
    NYS_TRY(launch_gemm(ctx, g));
  }
  NYS_TRY(launch_lambda_from_sigma(ctx, ell, sig, lam));              // line 8
  fmark();
  if (ftrace) {
    cudaStreamSynchronize(ctx->stream);
    const char* names[] = {"nu+Gram+chol(C)", "B GEMM + CholQR3", "trmm", "jacobi", "U GEMM + lambda"};
    fprintf(stderr, "[fact] m=%lld ell=%d:", (long long)m, ell);
    for (int i = 0; i + 1 < nfev; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, fev[i], fev[i + 1]);
      fprintf(stderr, " %s %.3f ms;", names[i], ms);
    }
    fprintf(stderr, "\n");
    for (int i = 0; i < nfev; ++i) cudaEventDestroy(fev[i]);
  }
  if (info) NYS_TRY(launch_orth_err(ctx, m, ell, U, mp, S_TMP6));
  // a failed shifted CholeskyQR pass leaves Gi / R stale: U would be silently non-orthonormal, so the
  // flag is always checked: here, or (defer) through S_NYSFAIL with the caller's iteration read
  if (defer) return launch_flag_max(ctx, S_NYSFAIL, S_CHOLFAIL);
  NYS_TRY(read_slots(ctx));
  if (ctx->h_sc[S_CHOLFAIL] != 0.0) {
    ctx->set_error("nys_sketch: shifted CholeskyQR of B = Y_nu C^{-1} failed (B numerically rank deficient)");
    return NYS_ECHOL;
  }
  if (info) {
    info->nu = ctx->h_sc[S_NU];
    info->chol_retries = retries;
    info->orth_err = ctx->h_sc[S_TMP6];
    info->jacobi_sweeps = (int)ctx->h_sc[S_JSWEEPS];
  }
  return NYS_OK;
}

// Y = A (d o (A^T Omega)) (+ e o Omega), summed over ranks   (Alg. 1 line 2)
int sketch_Y(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d, const double* e,
             int ell, const double* Om, double* Y) {
  const int64_t mp = even(m), np_ = even(n);
  double* T = ctx->wsd("sk_T", (size_t)(np_ > 0 ? np_ : 2) * ell);
  {
    GemmCall g;  // T = diag(d) A^T Omega  (n x l)
    g.M = n; g.N = ell; g.K = m; g.A = A; g.lda = lda; g.a_kmajor = true; g.B = Om; g.ldb = mp; g.C = T; g.ldc = np_;
    g.row_scale = d;
    NYS_TRY(launch_gemm(ctx, g));
  }
  {
    GemmCall g;  // Y = A T (+ e o Omega)
    g.M = m; g.N = ell; g.K = n; g.A = A; g.lda = lda; g.a_kmajor = false; g.B = T; g.ldb = np_; g.C = Y; g.ldc = mp;
    if (!ctx->multi() && e) { g.addv = e; g.addm = Om; g.ldadd = mp; }
    if (n == 0) NYS_CUDA_TRY(ctx, cudaMemsetAsync(Y, 0, sizeof(double) * mp * ell, ctx->stream));
    else NYS_TRY(launch_gemm(ctx, g));
  }
  if (ctx->multi()) {
    NYS_TRY(allreduce(ctx, Y, (size_t)mp * ell));
    if (e) NYS_TRY(launch_add_eomega(ctx, m, ell, e, Om, Y, mp));
  }
  return NYS_OK;
}

// Alg. 1: sketch, then lines 3-8
int sketch_impl(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d, const double* e,
                int ell, const double* Om, double* U, double* lam, nys_sketch_info* info, bool defer = false) {
  NvtxRange nv("nystrom_sketch_and_factor");
  double* Y = ctx->wsd("sk_Y", (size_t)even(m) * ell);
  NYS_TRY(sketch_Y(ctx, m, n, A, lda, d, e, ell, Om, Y));
  return nystrom_factor(ctx, m, ell, Y, Om, even(m), U, lam, info, defer);
}

// ------------------------------------------------------------------------------------------
// Partial Cholesky preconditioner of rank ell for N_delta = N + delta I (f2)
// ------------------------------------------------------------------------------------------
int chol_build(nys_ctx* ctx, const NormalOp& op, int ell, CholFactors& F) {
  NvtxRange nv("partial_cholesky_build");
  const int64_t m = op.m, mp = even(m);
  F.m = m;
  F.ell = ell;
  F.diag = ctx->wsd("ch_diag", (size_t)mp);
  double* ones = ctx->wsd("ch_ones", (size_t)mp);
  NYS_CUDA_TRY(ctx, cudaMemsetAsync(ones, 0, (size_t)mp * sizeof(double), ctx->stream));
  NYS_TRY(launch_shift(ctx, m, ones, 1.0));
  {  // diag(N_delta) = sum_j d_j A_ij^2 + e_i + delta
    MatvecCall c;
    c.mode = MV_DIAG; c.m = m; c.n = op.n; c.lda = op.lda; c.A = op.A; c.d = op.d; c.z = ones;
    c.out = F.diag;
    if (!ctx->multi()) {
      c.use_delta = true; c.delta = op.delta; c.e = op.e;
      NYS_TRY(launch_matvec(ctx, c));
    } else {
      NYS_TRY(launch_matvec(ctx, c));
      NYS_TRY(allreduce(ctx, F.diag, (size_t)m));
      NYS_TRY(launch_finalize_terms(ctx, m, F.diag, ones, op.delta, op.e, false, nullptr));
    }
  }
  F.piv = (int64_t*)ctx->ws("ch_piv", (size_t)(ell > 0 ? ell : 1) * sizeof(int64_t));
  F.pivpos = (int*)ctx->ws("ch_pivpos", (size_t)mp * sizeof(int));
  NYS_TRY(launch_topl_select(ctx, F.diag, m, ell, F.piv, F.pivpos));
  F.dS = ctx->wsd("ch_dS", (size_t)mp);
  F.ldr = ell > 0 ? ell : 1;
  F.Rinv = ctx->wsd("ch_Rinv", (size_t)F.ldr * F.ldr);
  F.Zt = ctx->wsd("ch_Zt", (size_t)m * (ell > 0 ? ell : 1));
  if (ell > 0) {
    double* Om = ctx->wsd("ch_Om", (size_t)mp * ell);
    double* Y = ctx->wsd("ch_Y", (size_t)mp * ell);
    double* N11 = ctx->wsd("ch_N11", (size_t)ell * ell);
    double* Z = ctx->wsd("ch_Z", (size_t)mp * ell);
    NYS_TRY(launch_selection(ctx, m, ell, F.piv, Om, mp));
    NYS_TRY(sketch_Y(ctx, m, op.n, op.A, op.lda, op.d, op.e, ell, Om, Y));   // N E_P (+ e)
    NYS_TRY(launch_pivot_block(ctx, Y, mp, F.piv, ell, op.delta, N11));     // + delta; N11 = Y[P, :]
    NYS_TRY(launch_set_slots(ctx, S_CHOLFAIL, 0.0));
    NYS_TRY(launch_chol_inv(ctx, ell, N11, ell, F.Rinv, ell, 0));          // N11 = R^T R, R^{-1}
    NYS_TRY(read_slots(ctx));
    if (ctx->h_sc[S_CHOLFAIL] != 0.0) { ctx->set_error("partial Cholesky: N11 not positive definite"); return NYS_ECHOL; }
    GemmCall gz;  // Z = Y R^{-1}: rows P = L11 = R^T, rows Q = L21 = N21 L11^{-T}
    gz.M = m; gz.N = ell; gz.K = ell; gz.A = Y; gz.lda = mp; gz.a_kmajor = false; gz.B = F.Rinv; gz.ldb = ell;
    gz.C = Z; gz.ldc = mp;
    NYS_TRY(launch_gemm(ctx, gz));
    NYS_TRY(launch_transpose_u(ctx, m, ell, Z, mp, F.Zt));
  }
  return launch_chol_ds(ctx, m, ell, F.Zt, F.diag, F.pivpos, F.dS);
}

// ------------------------------------------------------------------------------------------
// PCG with device scalars (tolerance already in S_TOL via launch_pcg_setup)
// ------------------------------------------------------------------------------------------
struct PcgResult {
  int iters = 0;
  int status = 0;
  double rr = 0.0;
};

// One PCG iteration (it) of the fused single-GPU path: K1 -> update -> precond.
int pcg_iteration(nys_ctx* ctx, const NormalOp& op, int ell, const double* U, int64_t ldu, const double* s,
                  double* x, double* r, double* z, double* const* Pp, double* h, int it, int max_iter,
                  unsigned long long cond, const CholFactors* chol = nullptr) {
  const double* done = ctx->sc + S_DONE;
  const double* pold = (it == 0) ? nullptr : Pp[it & 1];
  double* pnew = Pp[(it + 1) & 1];
  MatvecCall c;
  c.mode = MV_FUSED; c.m = op.m; c.n = op.n; c.lda = op.lda; c.A = op.A; c.z = z; c.p = pold;
  c.beta = ctx->sc + S_BETA; c.p_out = pnew; c.d = op.d; c.done = done; c.delta = op.delta; c.e = op.e;
  c.pcg_fused = true;
  c.delta_from_slot = true;
  FusedPartials fp;
  c.fused_out = &fp;
  NYS_TRY(launch_matvec(ctx, c));
  if (chol) {  // partial Cholesky P^{-1} (Chol-IP-PMM): update computes rr only
    NYS_TRY(launch_pcg_update(ctx, 0, op.m, x, r, nullptr, pnew, nullptr, &fp, op.delta, op.e, nullptr, 0, 0, nullptr,
                              h, max_iter, cond, true, true));
    return launch_chol_apply(ctx, *chol, r, z, 1, 0);
  }
  NYS_TRY(launch_pcg_update(ctx, 0, op.m, x, r, nullptr, pnew, nullptr, &fp, op.delta, op.e, U, ldu, ell, s, h,
                            max_iter, cond, true));
  if (ell > 0) NYS_TRY(launch_pcg_precond(ctx, 0, op.m, r, z, U, ldu, ell, h));
  return NYS_OK;
}

// defer_slot >= 0 (single GPU): no host read; the iteration count, the breakdown flag and the graph-loop
// accounting are latched into device slots (launch_pcg_latch) for the caller's one read per outer
// iteration, and res.iters = -1
int pcg_impl(nys_ctx* ctx, const NormalOp& op, int ell, const double* U, int64_t ldu, const double* s,
             const double* rhs, double* x, int max_iter, PcgResult& res, const CholFactors* chol = nullptr,
             int defer_slot = -1) {
  NvtxRange nv("pcg_solve");
  const int64_t m = op.m;
  const int64_t mp = even(m);
  if (chol) ell = 0;  // no Nystrom factors on the partial-Cholesky path
  double* r = ctx->wsd("pcg_r", (size_t)mp);
  double* z = (ell > 0 || chol) ? ctx->wsd("pcg_z", (size_t)mp) : r;
  double* P0 = ctx->wsd("pcg_p0", (size_t)mp);
  double* P1 = ctx->wsd("pcg_p1", (size_t)mp);
  double* w = ctx->wsd("pcg_w", (size_t)mp);
  double* h = ctx->wsd("pcg_h", (size_t)(ell > 0 ? ell : 1));
  double* Pp[2] = {P0, P1};
  const double* done = ctx->sc + S_DONE;
  if (ctx->gloop) NYS_TRY(launch_set_slots(ctx, S_GITER, 0.0));   // delta lives in S_DELTA (control kernel)
  else NYS_TRY(launch_set_slots(ctx, S_DELTA, op.delta, S_GITER, 0.0));
  if (!chol && pcg_persistent_supported(ctx, m, op.n, ell)) {
    // the whole solve is ONE launch (k_pcg.cu): one CTA for small problems, else cooperative grid-wide
    if (pcg_small_supported(ctx, m, op.n, ell))
      NYS_TRY(launch_pcg_small(ctx, m, op.n, op.A, op.lda, op.d, op.e, U, ldu, ell, s, rhs, x, max_iter));
    else
      NYS_TRY(launch_pcg_persistent(ctx, m, op.n, op.A, op.lda, op.d, op.e, U, ldu, ell, s, rhs, x, max_iter));
    if (defer_slot >= 0) {
      res.iters = -1;
      res.status = 0;
      return launch_pcg_latch(ctx, defer_slot);
    }
    NYS_TRY(read_slots(ctx));
    res.iters = (int)ctx->h_sc[S_ITERS];
    res.status = (int)ctx->h_sc[S_STATUS];
    res.rr = ctx->h_sc[S_RR];
    ctx->matvecs += res.iters;
    return NYS_OK;
  }
  // the non-persistent PCG kernels read U ROW-major (contiguous rows): transpose once per solve
  if (ell > 0) {
    double* Ut = ctx->wsd("pcg_Ut", (size_t)m * ell);
    NYS_TRY(launch_transpose_u(ctx, m, ell, U, ldu, Ut));
    U = Ut;
    ldu = ell;
  }
  NYS_TRY(launch_pcg_update(ctx, 1, m, x, r, rhs, nullptr, nullptr, nullptr, op.delta, op.e, U, ldu, ell, s, h,
                            max_iter, 0ull, false, chol != nullptr));
  if (chol) NYS_TRY(launch_chol_apply(ctx, *chol, r, z, 1, 1));
  else if (ell > 0) NYS_TRY(launch_pcg_precond(ctx, 1, m, r, z, U, ldu, ell, h));
  if (!ctx->multi() && getenv("NYS_NO_GRAPH") == nullptr) {  // NYS_NO_GRAPH: eager loop (profiling)
    // iterations 0 and 1 eagerly (they size every workspace), then the rest of the loop as ONE
    // graph launch: a conditional WHILE node whose body is two iterations (p double-buffer
    // parity); pcg_update's last block clears the condition when PCG is done.
    for (int it = 0; it < 2; ++it) NYS_TRY(pcg_iteration(ctx, op, ell, U, ldu, s, x, r, z, Pp, h, it, max_iter, 0ull, chol));
    if (ctx->gloop) {
      // inside the graph-resident outer loop's capture: the WHILE node goes straight into the capturing
      // graph (its handle created there), its two-iteration body captured on a side stream, and the outer
      // capture continues after the node
      cudaStreamCaptureStatus cst;
      unsigned long long cid = 0;
      cudaGraph_t cg_ = nullptr;
      const cudaGraphNode_t* deps = nullptr;
      size_t ndeps = 0;
      NYS_CUDA_TRY(ctx, cudaStreamGetCaptureInfo(ctx->stream, &cst, &cid, &cg_, &deps, &ndeps));
      if (cst != cudaStreamCaptureStatusActive || cg_ == nullptr) {
        ctx->set_error("PCG: nested graph capture without an active capture");
        return NYS_ECUDA;
      }
      cudaGraphConditionalHandle hc;
      NYS_CUDA_TRY(ctx, cudaGraphConditionalHandleCreate(&hc, cg_, 1, cudaGraphCondAssignDefault));
      // the default applies only when the whole graph is launched: re-arm before every execution
      NYS_TRY(launch_set_cond(ctx, (unsigned long long)hc, 1u));
      NYS_CUDA_TRY(ctx, cudaStreamGetCaptureInfo(ctx->stream, &cst, &cid, &cg_, &deps, &ndeps));
      cudaGraphNodeParams gp = {};
      gp.type = cudaGraphNodeTypeConditional;
      gp.conditional.handle = hc;
      gp.conditional.type = cudaGraphCondTypeWhile;
      gp.conditional.size = 1;
      cudaGraphNode_t wn;
      NYS_CUDA_TRY(ctx, cudaGraphAddNode(&wn, cg_, deps, ndeps, &gp));
      cudaGraph_t body = gp.conditional.phGraph_out[0];
      if (!ctx->side_stream) NYS_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
      cudaStream_t main_stream = ctx->stream;
      ctx->stream = ctx->side_stream;
      int rc = NYS_OK;
      cudaError_t eb = cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
      if (eb == cudaSuccess) {
        rc = pcg_iteration(ctx, op, ell, U, ldu, s, x, r, z, Pp, h, 2, max_iter, (unsigned long long)hc, chol);
        if (rc == NYS_OK) rc = pcg_iteration(ctx, op, ell, U, ldu, s, x, r, z, Pp, h, 3, max_iter, (unsigned long long)hc, chol);
        cudaGraph_t bo = body;
        const cudaError_t ee = cudaStreamEndCapture(ctx->stream, &bo);
        if (rc == NYS_OK && ee != cudaSuccess) rc = NYS_ECUDA;
      }
      ctx->stream = main_stream;
      if (eb != cudaSuccess || rc != NYS_OK) {
        ctx->set_error("PCG: nested graph capture failed");
        return rc != NYS_OK ? rc : NYS_ECUDA;
      }
      NYS_CUDA_TRY(ctx, cudaStreamUpdateCaptureDependencies(ctx->stream, &wn, 1, cudaStreamSetCaptureDependencies));
      res.iters = -1;
      res.status = 0;
      return launch_pcg_latch(ctx, defer_slot);
    }
    // the key holds every value the captured kernels take as an argument: for the partial-Cholesky
    // path its rank, leading dimension and factor pointers too (a later build with a smaller rank
    // grows no workspace, so ws_epoch alone would not tell the graphs apart)
    char key[768];
    snprintf(key, sizeof(key), "pcg%s:%lld:%lld:%lld:%p:%p:%p:%p:%lld:%p:%d:%p:%d:%lld:%d:%d:%p:%p:%p:%p:%p",
             chol ? "C" : "N", (long long)m, (long long)op.n,
             (long long)op.lda, (const void*)op.A, (const void*)op.d, (const void*)op.e, (const void*)U,
             (long long)ldu, (const void*)s, ell, (const void*)x, max_iter, (long long)ctx->ws_epoch,
             chol ? chol->ell : -1, chol ? chol->ldr : -1, chol ? (const void*)chol->Zt : nullptr,
             chol ? (const void*)chol->dS : nullptr, chol ? (const void*)chol->Rinv : nullptr,
             chol ? (const void*)chol->piv : nullptr, chol ? (const void*)chol->pivpos : nullptr);
    auto itg = ctx->graphs.find(key);
    cudaGraphExec_t exec = nullptr;
    if (itg != ctx->graphs.end()) {
      exec = itg->second.second.first;
    } else {
      if (ctx->graphs.size() >= 64) {  // bounded cache (callers passing ever-new buffers)
        for (auto& kv : ctx->graphs) {
          cudaGraphExecDestroy(kv.second.second.first);
          cudaGraphDestroy(kv.second.second.second);
        }
        ctx->graphs.clear();
      }
      cudaGraph_t g;
      NYS_CUDA_TRY(ctx, cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle hcond;
      NYS_CUDA_TRY(ctx, cudaGraphConditionalHandleCreate(&hcond, g, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams gp = {};
      gp.type = cudaGraphNodeTypeConditional;
      gp.conditional.handle = hcond;
      gp.conditional.type = cudaGraphCondTypeWhile;
      gp.conditional.size = 1;
      cudaGraphNode_t node;
      NYS_CUDA_TRY(ctx, cudaGraphAddNode(&node, g, nullptr, 0, &gp));
      cudaGraph_t body = gp.conditional.phGraph_out[0];
      const int64_t l0 = ctx->launches, mv0 = ctx->matvecs;
      NYS_CUDA_TRY(ctx, cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      int rc1 = pcg_iteration(ctx, op, ell, U, ldu, s, x, r, z, Pp, h, 2, max_iter, (unsigned long long)hcond, chol);
      int rc2 = rc1 == NYS_OK ? pcg_iteration(ctx, op, ell, U, ldu, s, x, r, z, Pp, h, 3, max_iter, (unsigned long long)hcond, chol) : rc1;
      cudaGraph_t body_out = body;
      cudaError_t ec = cudaStreamEndCapture(ctx->stream, &body_out);
      ctx->launches = l0; ctx->matvecs = mv0;
      if (rc2 != NYS_OK) return rc2;
      if (ec != cudaSuccess) { ctx->set_error(std::string("PCG graph capture: ") + cudaGetErrorString(ec)); return NYS_ECUDA; }
      NYS_CUDA_TRY(ctx, cudaGraphInstantiate(&exec, g, 0));
      ctx->graphs[key] = {ctx->ws_epoch, {exec, g}};
    }
    NYS_CUDA_TRY(ctx, cudaGraphLaunch(exec, ctx->stream));
    if (defer_slot >= 0) {   // accounting and counts read later by the caller (S_GITACC, defer_slot)
      res.iters = -1;
      res.status = 0;
      return launch_pcg_latch(ctx, defer_slot);
    }
    NYS_TRY(read_slots(ctx));
    // accounting: each pcg_update run in the graph body stands for matvec + update + hred
    // (+ precond) launches of that iteration
    const int64_t body_updates = (int64_t)ctx->h_sc[S_GITER];
    ctx->launches += body_updates * (chol ? 7 : (ell > 0 ? 4 : 3));
    res.iters = (int)ctx->h_sc[S_ITERS];
    ctx->matvecs += res.iters > 2 ? res.iters - 2 : 0;
  } else {
    // multi-rank: every iteration all-reduces the matvec partial.  With NCCL the loop body is captured
    // ONCE as a CUDA graph of kBatch iterations (matvec, ncclAllReduce, finalize, update, precond; the
    // library's kernels return at once after convergence, the trailing all-reduces move stale data and
    // are harmless) and replayed with one host check per replay; the loopback communicator (host
    // barriers) cannot be captured and keeps the eager host loop.
    constexpr int kBatch = 8;
    auto one_iter = [&](int it) -> int {
      const double* pold = (it == 0) ? nullptr : Pp[it & 1];
      double* pnew = Pp[(it + 1) & 1];
      NYS_TRY(apply_normal_full(ctx, op, z, pold, ctx->sc + S_BETA, pnew, w, true, done));
      NYS_TRY(launch_pcg_update(ctx, 0, m, x, r, nullptr, pnew, w, nullptr, op.delta, op.e, U, ldu, ell, s, h,
                                max_iter, 0ull, false, chol != nullptr));
      if (chol) NYS_TRY(launch_chol_apply(ctx, *chol, r, z, 1, 0));
      else if (ell > 0) NYS_TRY(launch_pcg_precond(ctx, 0, m, r, z, U, ldu, ell, h));
      return NYS_OK;
    };
    const bool capture = ctx->nccl_comm != nullptr && ctx->loop_comm == nullptr && getenv("NYS_NO_GRAPH") == nullptr;
    int it = 0;
    if (capture) {
      for (; it < 2; ++it) NYS_TRY(one_iter(it));   // sizes every workspace before the capture
      NYS_TRY(read_slots(ctx));
      if (ctx->h_sc[S_DONE] == 0.0) {
        char key[768];
        snprintf(key, sizeof(key), "mpcg%s:%lld:%lld:%lld:%p:%p:%p:%p:%lld:%p:%d:%p:%d:%lld:%d:%d:%p:%p:%p:%p:%p:%p",
                 chol ? "C" : "N", (long long)m, (long long)op.n, (long long)op.lda, (const void*)op.A,
                 (const void*)op.d, (const void*)op.e, (const void*)U, (long long)ldu, (const void*)s, ell,
                 (const void*)x, max_iter, (long long)ctx->ws_epoch, chol ? chol->ell : -1, chol ? chol->ldr : -1,
                 chol ? (const void*)chol->Zt : nullptr, chol ? (const void*)chol->dS : nullptr,
                 chol ? (const void*)chol->Rinv : nullptr, chol ? (const void*)chol->piv : nullptr,
                 chol ? (const void*)chol->pivpos : nullptr, (const void*)rhs);
        char dkey[800];
        snprintf(dkey, sizeof(dkey), "%s:%.17g", key, op.delta);   // delta is a captured kernel argument here
        auto itg = ctx->graphs.find(dkey);
        cudaGraphExec_t exec = nullptr;
        if (itg != ctx->graphs.end()) {
          exec = itg->second.second.first;
        } else {
          if (ctx->graphs.size() >= 64) {
            for (auto& kv : ctx->graphs) {
              cudaGraphExecDestroy(kv.second.second.first);
              cudaGraphDestroy(kv.second.second.second);
            }
            ctx->graphs.clear();
          }
          const int64_t l0 = ctx->launches, mv0 = ctx->matvecs;
          NYS_CUDA_TRY(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
          int rc = NYS_OK;
          for (int b = 0; b < kBatch && rc == NYS_OK; ++b) rc = one_iter(2 + b);
          cudaGraph_t g = nullptr;
          const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &g);
          ctx->launches = l0; ctx->matvecs = mv0;
          if (rc != NYS_OK) { if (g) cudaGraphDestroy(g); return rc; }
          if (ec != cudaSuccess) { ctx->set_error(std::string("multi-rank PCG graph capture: ") + cudaGetErrorString(ec)); return NYS_ECUDA; }
          NYS_CUDA_TRY(ctx, cudaGraphInstantiate(&exec, g, 0));
          ctx->graphs[dkey] = {ctx->ws_epoch, {exec, g}};
        }
        for (;;) {
          NYS_CUDA_TRY(ctx, cudaGraphLaunch(exec, ctx->stream));
          ctx->launches += kBatch * (chol ? 7 : (ell > 0 ? 5 : 4));
          NYS_TRY(read_slots(ctx));
          if (ctx->h_sc[S_DONE] != 0.0) break;
        }
      }
    } else {
      int batch = 4;
      for (;;) {
        for (int b = 0; b < batch; ++b, ++it) NYS_TRY(one_iter(it));
        NYS_TRY(read_slots(ctx));
        if (ctx->h_sc[S_DONE] != 0.0) break;
        if (batch < 32) batch *= 2;
      }
    }
    res.iters = (int)ctx->h_sc[S_ITERS];
  }
  res.status = (int)ctx->h_sc[S_STATUS];
  res.rr = ctx->h_sc[S_RR];
  if (defer_slot >= 0) NYS_TRY(launch_pcg_latch(ctx, defer_slot));   // host-loop paths: counts known, latched too
  return NYS_OK;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

// ------------------------------------------------------------------------------------------
// finalize_terms for world > 1 (w := w + (delta + e) v ; optional pcg dot / alpha)
// ------------------------------------------------------------------------------------------
namespace nys {
__global__ void finalize_terms_kernel(int64_t m, double* w, const double* v, double delta, const double* e, int pcg,
                                      double* sc, double* part, unsigned int* counter, const double* done) {
  if (done && *done != 0.0) return;
  double dot = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const double s = w[i] + (delta + (e ? e[i] : 0.0)) * v[i];
    w[i] = s;
    dot = fma(v[i], s, dot);
  }
  if (!pcg) return;
  __shared__ double sh[32];
  __shared__ bool last;
  dot = warp_sum(dot);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) b += sh[i];
    part[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && warp_uniform_id() == 0) {
    __threadfence();
    const double pw = warp_sum_array(part, gridDim.x);
    if (threadIdx.x != 0) return;
    *counter = 0u;
    sc[S_PW] = pw;
    if (!(pw > 0.0) || !isfinite(pw)) { sc[S_STATUS] = (double)NYS_EBREAKDOWN; sc[S_DONE] = 1.0; sc[S_ALPHA] = 0.0; }
    else sc[S_ALPHA] = sc[S_RZ] / pw;
  }
}
int launch_finalize_terms(nys_ctx* ctx, int64_t m, double* w, const double* v, double delta, const double* e,
                          bool pcg_alpha, const double* done) {
  int g = (int)((m + 255) / 256);
  if (g > 2 * ctx->num_sms) g = 2 * ctx->num_sms;
  double* part = ctx->wsd("fin_part2", (size_t)g);
  finalize_terms_kernel<<<g, 256, 0, ctx->stream>>>(m, w, v, delta, e, pcg_alpha ? 1 : 0, ctx->sc, part,
                                                    ctx->counters + 4, done);
  ctx->launches++;
  return ctx->check_launch("finalize_terms");
}
}  // namespace nys

// ------------------------------------------------------------------------------------------
// Nys-IP-PMM driver
// ------------------------------------------------------------------------------------------
namespace {
// Omega_k (m x l, column-major ld = m semantics of the generator) into a buffer with ld = even(m)
int gen_omega(nys_ctx* ctx, int64_t m, int ell, uint64_t seed, uint64_t stream, double* Om) {
  const int64_t mp = even(m);
  if (mp == m) return launch_gaussian(ctx, Om, m * (int64_t)ell, seed, stream);
  double* tmp = ctx->wsd("ipm_Omtmp", (size_t)m * ell);
  NYS_TRY(launch_gaussian(ctx, tmp, m * (int64_t)ell, seed, stream));
  NYS_CUDA_TRY(ctx, cudaMemcpy2DAsync(Om, mp * 8, tmp, m * 8, m * 8, ell, cudaMemcpyDeviceToDevice, ctx->stream));
  return NYS_OK;
}

struct Dots {
  nys_ctx* ctx;
  int dot(int64_t n, const double* a, const double* b, int slot) {
    const double* aa[1] = {a};
    const double* bb[1] = {b};
    int out[1] = {slot};
    return launch_dots(ctx, n, 1, aa, bb, out, 5);
  }
};

// A-products of the driver for a dense A (structure 0) or the SVM-shaped A = [Xt, -Xt, I, -I]
// (structure 1; Xt = the dense block, never materialising the identity blocks).
struct AOps {
  nys_ctx* ctx;
  int structure;
  int64_t m, n, nd;        // n = variables; nd = columns of the dense block (n for structure 0)
  const double* A;         // dense block, column-major, lda
  int64_t lda;
  double *g, *atv, *uw, *addm, *dw, *e;  // structure-1/2 work vectors
  UnitBlocks UB;                          // structure 2
  int64_t r0 = 0, mr = 0;                 // structure 1: this rank's xi / s rows [r0, r0 + mr)
  // normal operator for the scaling d (n): dense -> (A, d); structured -> (Xt, d_w+ + d_w-, e)
  int normal_op(const double* d, double delta, NormalOp& op) {
    if (structure == 0) { op = NormalOp{m, n, lda, A, d, nullptr, delta}; return NYS_OK; }
    if (structure == 2) {                 // e = sum_k scale_k^2 d_unit (global: a replicated term)
      NYS_TRY(launch_unit_fold(ctx, UB, m, d + nd, nullptr, 1, e));
      if (ctx->multi()) NYS_TRY(allreduce(ctx, e, (size_t)m));
      op = NormalOp{m, nd, lda, A, d, e, delta};
      return NYS_OK;
    }
    NYS_TRY(launch_svm_scaling_fold(ctx, nd, m, r0, mr, d, dw, e));
    if (ctx->multi()) NYS_TRY(allreduce(ctx, e, (size_t)m));   // every row's d_xi + d_s, replicated
    op = NormalOp{m, nd, lda, A, dw, e, delta};
    return NYS_OK;
  }
  // out = A u (+ add)
  int Ax(const double* u, double* out, const double* add) {
    if (structure == 0) return apply_A(ctx, m, n, A, lda, u, out, 1.0, add);
    if (structure == 2) {
      if (!ctx->multi()) {              // unit part + add folded into the matvec's add vector
        NYS_TRY(launch_unit_fold(ctx, UB, m, u + nd, add, 0, addm));
        return apply_A(ctx, m, nd, A, lda, u, out, 1.0, addm);
      }
      NYS_TRY(launch_unit_fold(ctx, UB, m, u + nd, nullptr, 0, addm));   // local partial: before the all-reduce
      MatvecCall c;
      c.mode = MV_NONLY; c.m = m; c.n = nd; c.lda = lda; c.A = A; c.u = u; c.out = out; c.sgn = 1.0; c.add = addm;
      NYS_TRY(launch_matvec(ctx, c));
      NYS_TRY(allreduce(ctx, out, (size_t)m));
      if (add) NYS_TRY(launch_axpby(ctx, m, 1.0, out, 1.0, add, out));
      return NYS_OK;
    }
    if (!ctx->multi()) {
      NYS_TRY(launch_svm_fold(ctx, nd, m, r0, mr, u, add, uw, addm));
      return apply_A(ctx, m, nd, A, lda, uw, out, 1.0, addm);
    }
    NYS_TRY(launch_svm_fold(ctx, nd, m, r0, mr, u, nullptr, uw, addm));   // local partial: own rows only
    MatvecCall c;
    c.mode = MV_NONLY; c.m = m; c.n = nd; c.lda = lda; c.A = A; c.u = uw; c.out = out; c.sgn = 1.0; c.add = addm;
    NYS_TRY(launch_matvec(ctx, c));
    NYS_TRY(allreduce(ctx, out, (size_t)m));
    if (add) NYS_TRY(launch_axpby(ctx, m, 1.0, out, 1.0, add, out));
    return NYS_OK;
  }
  // structured: atv = A^T y (n-vector)
  int At_vec(const double* y) {
    MatvecCall mc;
    mc.mode = MV_TONLY; mc.m = m; mc.n = nd; mc.lda = lda; mc.A = A; mc.z = y; mc.tep = TE_PLAIN;
    mc.t1 = structure == 2 ? atv : g;
    NYS_TRY(apply_At(ctx, mc));
    if (structure == 2) return launch_unit_expand(ctx, UB, y, atv + nd);
    return launch_svm_expand(ctx, nd, r0, mr, g, y, atv);
  }
  int At_plain(const double* y, double* out) {
    if (structure == 0) {
      MatvecCall mc;
      mc.mode = MV_TONLY; mc.m = m; mc.n = n; mc.lda = lda; mc.A = A; mc.z = y; mc.tep = TE_PLAIN; mc.t1 = out;
      return apply_At(ctx, mc);
    }
    NYS_TRY(At_vec(y));
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(out, atv, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    return NYS_OK;
  }
  // out = c + q x - A^T y - z   (z may be null)
  int At_rd(const double* y, const double* c, const double* q, const double* x, const double* z, double* out) {
    if (structure == 0) {
      MatvecCall mc;
      mc.mode = MV_TONLY; mc.m = m; mc.n = n; mc.lda = lda; mc.A = A; mc.z = y; mc.tep = TE_RD;
      mc.t1 = out; mc.ta = c; mc.tb = q; mc.tc = x; mc.td = z;
      return apply_At(ctx, mc);
    }
    NYS_TRY(At_vec(y));
    return launch_epi_rd(ctx, n, c, q, x, atv, z, out);
  }
  // the residual products from ONE read of A (structure 0): ax = A x and rd = c + q x - A^T y - z
  // by the MV_BOTH pass (NYS_NO_MV_BOTH=1: the two separate passes)
  int Ax_At_rd(const double* x, double* ax, const double* y, const double* c, const double* q, const double* z,
               double* rd) {
    static const bool split = getenv("NYS_NO_MV_BOTH") != nullptr;
    if (structure != 0 || split) {
      NYS_TRY(Ax(x, ax, nullptr));
      return At_rd(y, c, q, x, z, rd);
    }
    MatvecCall mc;
    mc.mode = MV_BOTH; mc.m = m; mc.n = n; mc.lda = lda; mc.A = A;
    mc.z = y; mc.tep = TE_RD; mc.t1 = rd; mc.ta = c; mc.tb = q; mc.tc = x; mc.td = z;
    mc.u = x; mc.out = ax; mc.sgn = 1.0;
    NYS_TRY(launch_matvec(ctx, mc));
    if (ctx->multi()) NYS_TRY(allreduce(ctx, ax, (size_t)m));
    return NYS_OK;
  }
  // dx = d (A^T dy - r_d - xi_au); dz = (r_xz - z dx) / x
  int At_dx(const double* dy, const double* rd, const double* xiau, const double* rxz, const double* z,
            const double* x, const double* d, double* dx, double* dz) {
    if (structure == 0) {
      MatvecCall mc;
      mc.mode = MV_TONLY; mc.m = m; mc.n = n; mc.lda = lda; mc.A = A; mc.z = dy; mc.tep = TE_DX;
      mc.t1 = dx; mc.t2 = dz; mc.ta = rd; mc.tb = xiau; mc.tc = rxz; mc.td = z; mc.tx = x; mc.tdd = d;
      return apply_At(ctx, mc);
    }
    NYS_TRY(At_vec(dy));
    return launch_epi_dx(ctx, n, atv, rd, xiau, rxz, z, x, d, dx, dz);
  }
};

int ipm_impl(nys_ctx* ctx, const nys_qp* qp_in, const nys_options* opt, nys_solution* sol, nys_report* rep) {
  NvtxRange nv_solve("nys_ipppmm_solve");
  auto t_start = std::chrono::steady_clock::now();
  const int64_t m = qp_in->m, n = qp_in->n;
  const int64_t mp = even(m), np_ = even(n);
  const int ell = opt->ell;
  const int64_t launches0 = ctx->launches, matvecs0 = ctx->matvecs;
  // ---- problem data on the device --------------------------------------------------------
  const double *A = qp_in->A, *q = qp_in->q, *b = qp_in->b, *c = qp_in->c;
  int64_t lda = qp_in->lda;
  const int64_t ncolA = qp_in->structure >= 1 ? qp_in->nd : n;  // dense columns stored
  if (qp_in->host_ptrs) {
    const int64_t ldd = even(m);
    double* Ad = ctx->wsd("ipm_A", (size_t)ldd * (ncolA > 0 ? ncolA : 1));
    if (ncolA > 0)
      NYS_CUDA_TRY(ctx, cudaMemcpy2DAsync(Ad, ldd * 8, qp_in->A, qp_in->lda * 8, m * 8, ncolA, cudaMemcpyHostToDevice, ctx->stream));
    double* qd = ctx->wsd("ipm_q", (size_t)np_ + 2);
    double* cd = ctx->wsd("ipm_c", (size_t)np_ + 2);
    double* bd = ctx->wsd("ipm_b", (size_t)mp);
    if (n > 0) {
      NYS_CUDA_TRY(ctx, cudaMemcpyAsync(qd, qp_in->q, n * 8, cudaMemcpyHostToDevice, ctx->stream));
      NYS_CUDA_TRY(ctx, cudaMemcpyAsync(cd, qp_in->c, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(bd, qp_in->b, m * 8, cudaMemcpyHostToDevice, ctx->stream));
    A = Ad; lda = ldd; q = qd; b = bd; c = cd;
  }
  // ---- free / box variables (f1, (P~)/(D~)) ---------------------------------------
  const bool gen = qp_in->vtype != nullptr;
  const int8_t* vt = qp_in->vtype;
  const double* ub = qp_in->ub;
  if (gen && qp_in->host_ptrs && n > 0) {
    int8_t* vtd = (int8_t*)ctx->ws("ipm_vt", (size_t)np_ + 16);
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(vtd, qp_in->vtype, n, cudaMemcpyHostToDevice, ctx->stream));
    vt = vtd;
    if (qp_in->ub) {
      double* ubd = ctx->wsd("ipm_ub", (size_t)np_ + 2);
      NYS_CUDA_TRY(ctx, cudaMemcpyAsync(ubd, qp_in->ub, n * 8, cudaMemcpyHostToDevice, ctx->stream));
      ub = ubd;
    }
  }
  if (gen) {
    unsigned long long* bad = (unsigned long long*)ctx->ws("chk_bad", 8);
    unsigned long long hv = 0;
    NYS_CUDA_TRY(ctx, cudaMemsetAsync(bad, 0, 8, ctx->stream));
    NYS_TRY(launch_gen_check(ctx, n, vt, ub, bad));
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(&hv, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
    NYS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (hv != 0) {
      ctx->set_error("nys_ipppmm_solve: vtype not in {0,1,2} or ub_J not finite and > 0 (" + std::to_string(hv) +
                     " entries)");
      return NYS_EINVAL;
    }
  }
  // ---- iterate and work vectors ------------------------------------------------------------
  const size_t nn = (size_t)np_ + 2, mm = (size_t)mp;
  double *x = ctx->wsd("ipm_x", nn), *z = ctx->wsd("ipm_z", nn), *zeta = ctx->wsd("ipm_zeta", nn);
  double *d = ctx->wsd("ipm_d", nn), *rD = ctx->wsd("ipm_rD", nn), *rd = ctx->wsd("ipm_rd", nn);
  double *rxz = ctx->wsd("ipm_rxz", nn), *xiau = ctx->wsd("ipm_xiau", nn), *t = ctx->wsd("ipm_t", nn);
  double *dxp = ctx->wsd("ipm_dxp", nn), *dzp = ctx->wsd("ipm_dzp", nn), *dxc = ctx->wsd("ipm_dxc", nn);
  double *dzc = ctx->wsd("ipm_dzc", nn), *dx = ctx->wsd("ipm_dx", nn), *dz = ctx->wsd("ipm_dz", nn);
  double *ones = ctx->wsd("ipm_ones", nn);
  // general form: w, s, r_u, r_ws and the w / s directions (0 off J)
  double *w = nullptr, *sv = nullptr, *ru = nullptr, *rws = nullptr, *dwp = nullptr, *dsp = nullptr;
  double *dwc = nullptr, *dsc = nullptr, *dw = nullptr, *ds = nullptr;
  if (gen) {
    w = ctx->wsd("ipm_w", nn); sv = ctx->wsd("ipm_sv", nn); ru = ctx->wsd("ipm_ru", nn);
    rws = ctx->wsd("ipm_rws", nn); dwp = ctx->wsd("ipm_dwp", nn); dsp = ctx->wsd("ipm_dsp", nn);
    dwc = ctx->wsd("ipm_dwc", nn); dsc = ctx->wsd("ipm_dsc", nn); dw = ctx->wsd("ipm_dw", nn);
    ds = ctx->wsd("ipm_ds", nn);
  }
  double *y = ctx->wsd("ipm_y", mm), *lam = ctx->wsd("ipm_lam", mm), *ax = ctx->wsd("ipm_ax", mm);
  double *rP = ctx->wsd("ipm_rP", mm), *rp = ctx->wsd("ipm_rp", mm), *xi = ctx->wsd("ipm_xi", mm);
  double *dyp = ctx->wsd("ipm_dyp", mm), *dyc = ctx->wsd("ipm_dyc", mm), *u1 = ctx->wsd("ipm_u1", mm);
  // adaptive rank (f3, reading F1): workspace for the largest rank the run may reach
  int ell_cap = ell;
  if (ell > 0 && opt->precond != 1 && opt->ell_max > ell) {
    ell_cap = opt->ell_max;
    if (ell_cap > m) ell_cap = (int)m;
    if (ell_cap > kMaxEll) ell_cap = kMaxEll;
  }
  int ell_k = ell, ell_built = ell;      // rank of the next build / of the factors in use
  double lam_ell_cur = 0.0;
  // per-iteration phase timing with CUDA events (no stream synchronisation of its own: the events
  // are read after the iteration's residual read-back, which synchronises anyway)
  struct PhaseEvents {
    cudaEvent_t e[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    PhaseEvents() { for (auto& v : e) cudaEventCreate(&v); }
    ~PhaseEvents() { for (auto& v : e) if (v) cudaEventDestroy(v); }
    float ms(int a, int b) const { float t = 0.f; cudaEventElapsedTime(&t, e[a], e[b]); return t; }
  } pev;
  const int le = ell_cap > 0 ? ell_cap : 1;
  double *Om = ctx->wsd("ipm_Om", (size_t)mp * le), *U = ctx->wsd("ipm_U", (size_t)mp * le);
  double *lamh = ctx->wsd("ipm_lamh", (size_t)le), *scoef = ctx->wsd("ipm_s", (size_t)le);
  Dots D{ctx};
  AOps AO{ctx, qp_in->structure, m, n, ncolA, A, lda, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  if (AO.structure == 2) {
    AO.atv = ctx->wsd("svm_atv", nn);
    AO.addm = ctx->wsd("svm_addm", mm);
    AO.e = ctx->wsd("svm_e", mm);
    int64_t off = 0;
    AO.UB.nb = qp_in->n_unit_blocks;
    for (int k = 0; k < AO.UB.nb; ++k) {
      AO.UB.row0[k] = qp_in->unit_blocks[k].row0;
      AO.UB.count[k] = qp_in->unit_blocks[k].count;
      AO.UB.scale[k] = qp_in->unit_blocks[k].scale;
      AO.UB.off[k] = off;
      off += AO.UB.count[k];
    }
    AO.UB.total = off;
  }
  if (AO.structure == 1) {
    AO.r0 = qp_in->n_unit_blocks == 1 ? qp_in->unit_blocks[0].row0 : 0;
    AO.mr = qp_in->n_unit_blocks == 1 ? qp_in->unit_blocks[0].count : m;
    AO.g = ctx->wsd("svm_g", (size_t)even(ncolA) + 2);
    AO.atv = ctx->wsd("svm_atv", nn);
    AO.uw = ctx->wsd("svm_uw", (size_t)even(ncolA) + 2);
    AO.addm = ctx->wsd("svm_addm", mm);
    AO.dw = ctx->wsd("svm_dw", (size_t)even(ncolA) + 2);
    AO.e = ctx->wsd("svm_e", mm);
  }
  double n_total = (double)n;
  {
    // global variable count (for mu = x^T z / n)
    NYS_TRY(launch_set_slots(ctx, S_TMP5, (double)n));
    NYS_TRY(allreduce_slots(ctx, S_TMP5, 1));
    NYS_TRY(read_slots(ctx));
    n_total = ctx->h_sc[S_TMP5];
  }
  nys_report R{};
  R.max_records = rep ? rep->max_records : 0;
  R.records = rep ? rep->records : nullptr;
  double t_sketch = 0, t_pcg = 0;

  // ---- norms of b and c ------------------------------------------------------------------
  NYS_TRY(D.dot(m, b, b, S_BNORM));
  NYS_TRY(D.dot(n, c, c, S_TMP4));
  if (gen) {                                                         // t = -u_J / 2 ; ||u_J||^2 = 4 ||t||^2 (G1)
    NYS_TRY(launch_gen_half_u(ctx, n, vt, ub, -0.5, t));
    NYS_TRY(D.dot(n, t, t, S_TMP5));
  } else {
    NYS_TRY(launch_set_slots(ctx, S_TMP5, 0.0));
  }
  NYS_TRY(allreduce_slots(ctx, S_TMP4, 2));
  NYS_TRY(read_slots(ctx));
  const double bnorm = std::sqrt(ctx->h_sc[S_BNORM] + 4.0 * ctx->h_sc[S_TMP5]);
  if (gen) NYS_TRY(launch_set_slots(ctx, S_BNORM, bnorm * bnorm));  // ||[b; u_J]||^2 for the PCG tolerance (G1)
  const double cnorm = std::sqrt(ctx->h_sc[S_TMP4]);
  int total_inner = 0;

  // ---- initial point (App. B.2; u = 0) --------------------------------------
  nvtxRangePushA("initial_point");
  NYS_CUDA_TRY(ctx, cudaMemsetAsync(ones, 0, nn * sizeof(double), ctx->stream));
  NYS_TRY(launch_shift(ctx, n, ones, 1.0));
  NormalOp op0;
  NYS_TRY(AO.normal_op(ones, opt->init_delta, op0));
  const bool use_chol = opt->precond == 1;                            // Chol-IP-PMM (f2)
  CholFactors CF;
  if (ell > 0 || use_chol) {
    auto ts = std::chrono::steady_clock::now();
    if (use_chol) {
      NYS_TRY(chol_build(ctx, op0, ell, CF));
    } else {
      NYS_TRY(gen_omega(ctx, m, ell, opt->seed, 0, Om));               // stream 0
      NYS_TRY(sketch_impl(ctx, m, op0.n, op0.A, op0.lda, op0.d, op0.e, ell, Om, U, lamh, nullptr));
      NYS_TRY(launch_prec_coef(ctx, lamh, ell, opt->init_delta, scoef));
    }
    t_sketch += ms_since(ts);
  }
  const CholFactors* cfp = use_chol ? &CF : nullptr;
  auto tp = std::chrono::steady_clock::now();
  PcgResult pr;
  const double* rhs0 = b;
  if (gen) {                                                         // App. B.2: rhs = b - A u / 2
    NYS_TRY(AO.Ax(t, xi, b));
    rhs0 = xi;
  }
  NYS_TRY(D.dot(m, rhs0, rhs0, S_XINORM));
  NYS_TRY(launch_pcg_setup(ctx, 2, 0, 0, 0, S_XINORM, 0, 0, opt->init_tol_rel));
  NYS_TRY(pcg_impl(ctx, op0, ell, U, mp, scoef, rhs0, u1, opt->pcg_max_iter, pr, cfp));
  total_inner += pr.iters;
  NYS_TRY(AO.At_plain(u1, x));                                       // x~ = A^T u1 (+ u/2)
  if (gen) NYS_TRY(launch_axpby(ctx, n, 1.0, x, -1.0, t, x));
  NYS_TRY(launch_cpqx(ctx, n, c, q, x, t));                          // c + Q x~
  NYS_TRY(AO.Ax(t, xi, nullptr));                                    // A (c + Q x~)
  NYS_TRY(D.dot(m, xi, xi, S_XINORM));
  NYS_TRY(launch_pcg_setup(ctx, 2, 0, 0, 0, S_XINORM, 0, 0, opt->init_tol_rel));
  NYS_TRY(pcg_impl(ctx, op0, ell, U, mp, scoef, xi, y, opt->pcg_max_iter, pr, cfp));
  total_inner += pr.iters;
  t_pcg += ms_since(tp);
  NYS_TRY(AO.At_rd(y, c, q, x, nullptr, z));                         // z~ = c - A^T y~ + Q x~
  if (gen) {                                                         // App. B.2 with w, s (G2, G3)
    NYS_TRY(launch_gen_init_stats(ctx, n, vt, ub, x, z, w, sv, ctx->sc + S_G0));
    NYS_TRY(allreduce_slots(ctx, S_G0, 4, true));
    NYS_TRY(allreduce_slots(ctx, S_G4, 8));
    NYS_TRY(read_slots(ctx));
    const double* G = ctx->h_sc + S_G0;
    const double mx = G[0], mw = G[1], mz = G[2], ms = G[3], sx = G[4], sw = G[5], sz = G[6], ss = G[7];
    const double xz = G[8], ws = G[9], nij = G[10], nj = G[11];
    const double dp = std::max(-1.5 * std::min(mx, mw), 0.0);       // P:1468 over x~_IJ and w~_J
    const double dd = std::max(-1.5 * std::min(mz, ms), 0.0);       // P:1469 over z~_IJ and s~_J
    const double gam = xz + dd * sx + dp * sz + nij * dp * dd + ws + dd * sw + dp * ss + nj * dp * dd;
    const double den_p = sz + nij * dd + ss + nj * dd, den_d = sx + nij * dp + sw + nj * dp;   // G2
    const double dpt = dp + (den_p > 0 ? 0.5 * gam / den_p : 0.0);
    const double ddt = dd + (den_d > 0 ? 0.5 * gam / den_d : 0.0);
    NYS_TRY(launch_gen_init_apply(ctx, n, vt, x, z, w, sv, dpt, ddt));
    n_total = nij + nj;                                               // mu = (x^T z + w^T s) / (|IJ| + |J|)
  } else {
  NYS_TRY(launch_minsum(ctx, n, x, 0.0, S_TMP0, S_TMP1, 6));
  NYS_TRY(launch_minsum(ctx, n, z, 0.0, S_TMP2, S_TMP3, 7));
  NYS_TRY(D.dot(n, x, z, S_TMP4));
  if (ctx->multi()) {
    NYS_TRY(allreduce_slots(ctx, S_TMP0, 1, true));
    NYS_TRY(allreduce_slots(ctx, S_TMP2, 1, true));
    NYS_TRY(allreduce_slots(ctx, S_TMP1, 1));
    NYS_TRY(allreduce_slots(ctx, S_TMP3, 1));
    NYS_TRY(allreduce_slots(ctx, S_TMP4, 1));
  }
  NYS_TRY(read_slots(ctx));
  {
    const double minx = ctx->h_sc[S_TMP0], sumx = ctx->h_sc[S_TMP1];
    const double minz = ctx->h_sc[S_TMP2], sumz = ctx->h_sc[S_TMP3], xz = ctx->h_sc[S_TMP4];
    const double dp = std::max(-1.5 * minx, 0.0);
    const double dd = std::max(-1.5 * minz, 0.0);
    const double gamma = xz + dd * sumx + dp * sumz + n_total * dp * dd;  // P:1470 expanded
    const double sz = sumz + n_total * dd, sx = sumx + n_total * dp;  // A13
    double dpt = dp + (sz > 0 ? 0.5 * gamma / sz : 0.0);
    double ddt = dd + (sx > 0 ? 0.5 * gamma / sx : 0.0);
    if (minx + dpt <= 0.0) dpt += 1.0;                                // IPg
    if (minz + ddt <= 0.0) ddt += 1.0;
    NYS_TRY(launch_shift(ctx, n, x, dpt));
    NYS_TRY(launch_shift(ctx, n, z, ddt));
  }
  }
  nvtxRangePop();
  // ---- PMM parameters --------------------------------------------------------------
  NYS_CUDA_TRY(ctx, cudaMemcpyAsync(lam, y, m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  if (n > 0) NYS_CUDA_TRY(ctx, cudaMemcpyAsync(zeta, x, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  double rho = opt->rho0, delta = opt->delta0;

  auto residuals = [&](bool read = true) -> int {
    // r_P = b - A x ; r_D = c + Q x - A^T y - z ; ||r_P||^2, ||r_D||^2, x^T z
    NvtxRange nvr("residuals");
    NYS_TRY(AO.Ax_At_rd(x, ax, y, c, q, z, rD));
    NYS_TRY(launch_axpby(ctx, m, 1.0, b, -1.0, ax, rP));
    if (gen) {                                                        // G1: r_D += s ; r_U = u - x - w on J
      NYS_TRY(launch_axpby(ctx, n, 1.0, rD, 1.0, sv, rD));
      NYS_TRY(launch_gen_ru(ctx, n, vt, ub, x, w, ru));
      NYS_TRY(D.dot(n, ru, ru, S_TMP3));
      NYS_TRY(D.dot(n, w, sv, S_TMP4));
    } else {
      NYS_TRY(launch_set_slots(ctx, S_TMP3, 0.0, S_TMP4, 0.0));
    }
    NYS_TRY(D.dot(m, rP, rP, S_TMP0));
    NYS_TRY(D.dot(n, rD, rD, S_TMP1));
    NYS_TRY(D.dot(n, x, z, S_TMP2));
    NYS_TRY(allreduce_slots(ctx, S_TMP1, gen ? 4 : 2));
    if (!read) return NYS_OK;                                         // graph-resident loop: no host read
    NYS_TRY(read_slots(ctx));
    ctx->h_sc[S_TMP0] += ctx->h_sc[S_TMP3];                           // ||[r_P; r_U]||^2
    ctx->h_sc[S_TMP2] += ctx->h_sc[S_TMP4];                           // x^T z + w^T s
    return NYS_OK;
  };
  NYS_TRY(residuals());
  double nrP = std::sqrt(ctx->h_sc[S_TMP0]), nrD = std::sqrt(ctx->h_sc[S_TMP1]);
  double mu = n_total > 0 ? ctx->h_sc[S_TMP2] / n_total : 0.0;
  double nrP_ref = nrP, nrD_ref = nrD;
  int status = NYS_EMAXITER;
  int k = 0;
  int last_build = -1;          // outer iteration of the last preconditioner build (f3)
  int64_t base_its = -1, last_its = 0;
  // ---- graph-resident outer loop (f3) ------------------------------------------------
  // After iteration 0 (which sizes every workspace) the remaining outer iterations run as ONE graph launch:
  // a conditional WHILE node whose body is the iteration's kernel sequence (exactly the deferred host
  // loop's, with rho, delta, mu and the outer index read from device slots) followed by
  // ipm_control_kernel (record, PEU, termination test -> the WHILE condition) and the PEU copies.  The host
  // reads the device state once, when the graph returns.  Single GPU, standard form, Nystrom with a fixed
  // rank rebuilt every outer iteration (Alg. 3 as written), one-launch PCG (m <= 8192); NYS_NO_GRAPH_LOOP=1
  // keeps the host loop.  A Nystrom factorisation failure stops the graph, and the host loop re-runs that
  // iteration with its checks (A4 retries).
  const bool gl_ok = !ctx->multi() && !use_chol && !gen && ell > 0 && ell_cap == ell && opt->prec_refresh <= 1 &&
                     !(opt->prec_growth > 0.0) && !opt->verbose && getenv("NYS_NO_GRAPH_LOOP") == nullptr &&
                     getenv("NYS_NO_GRAPH") == nullptr;
  bool gl_tried = false;
  // test hook: NYS_INJECT_NYSFAIL=k raises the factorisation-failure flag in deferred outer iteration k
  static const int inject_k = getenv("NYS_INJECT_NYSFAIL") ? atoi(getenv("NYS_INJECT_NYSFAIL")) : -1;
  auto gl_body = [&]() -> int {   // one outer iteration, deferred checks, no host read
    NYS_TRY(launch_stamp(ctx, S_TS0));
    NYS_TRY(launch_scaling(ctx, n, q, x, z, rho, d));                // rho from S_RHO
    NormalOp op;
    NYS_TRY(AO.normal_op(d, delta, op));                               // op.delta unused: S_DELTA
    NYS_TRY(launch_set_slots(ctx, S_PCGBRK, 0.0, S_NYSFAIL, 0.0, S_GITACC, 0.0));
    NYS_TRY(gen_omega(ctx, m, ell, opt->seed, 0, Om));                 // stream S_KOUT + 1 (A6)
    NYS_TRY(sketch_impl(ctx, m, op.n, op.A, op.lda, op.d, op.e, ell, Om, U, lamh, nullptr, true));
    if (inject_k >= 0) NYS_TRY(launch_inject_nysfail(ctx, inject_k));   // test hook
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->sc + S_LAML, lamh + ell - 1, 8, cudaMemcpyDeviceToDevice, ctx->stream));
    NYS_TRY(launch_prec_coef(ctx, lamh, ell, delta, scoef));           // mu_prec = S_DELTA (A7)
    NYS_TRY(launch_stamp(ctx, S_TS1));
    PcgResult pr;
    NYS_TRY(launch_pred_rhs_n(ctx, n, x, z, zeta, rD, rho, d, rd, rxz, xiau, t));
    NYS_TRY(launch_pred_rhs_m(ctx, m, b, ax, y, lam, delta, rp));
    NYS_TRY(AO.Ax(t, xi, rp));
    NYS_TRY(D.dot(m, xi, xi, S_XINORM));
    NYS_TRY(launch_pcg_setup(ctx, 1, 0, opt->pcg_c, opt->pcg_floor, S_XINORM, S_BNORM, S_MUCUR, 0));
    NYS_TRY(launch_stamp(ctx, S_TS2));
    NYS_TRY(pcg_impl(ctx, op, ell, U, mp, scoef, xi, dyp, opt->pcg_max_iter, pr, nullptr, (int)S_PCGI0));
    NYS_TRY(launch_stamp(ctx, S_TS3));
    NYS_TRY(AO.At_dx(dyp, rd, xiau, rxz, z, x, d, dxp, dzp));
    NYS_TRY(launch_ratio(ctx, n, x, dxp, nullptr, nullptr, z, dzp, nullptr, nullptr, 8));
    NYS_TRY(launch_steps_post(ctx));
    NYS_TRY(launch_muaff(ctx, n, x, dxp, z, dzp, n_total, 9, w, dwp, sv, dsp));
    NYS_TRY(launch_corr_rhs(ctx, n, x, dxp, dzp, d, rxz, xiau, t));
    NYS_TRY(AO.Ax(t, xi, nullptr));
    NYS_TRY(D.dot(m, xi, xi, S_XINORM));
    NYS_TRY(launch_pcg_setup(ctx, 1, 0, opt->pcg_c, opt->pcg_floor, S_XINORM, S_BNORM, S_MUCUR, 0));
    NYS_TRY(launch_stamp(ctx, S_TS4));
    NYS_TRY(pcg_impl(ctx, op, ell, U, mp, scoef, xi, dyc, opt->pcg_max_iter, pr, nullptr, (int)S_PCGI1));
    NYS_TRY(launch_stamp(ctx, S_TS5));
    NYS_TRY(AO.At_dx(dyc, nullptr, xiau, rxz, z, x, d, dxc, dzc));
    NYS_TRY(launch_ratio(ctx, n, x, dx, dxp, dxc, z, dz, dzp, dzc, 8));
    NYS_TRY(launch_steps_post(ctx));
    NYS_TRY(launch_update_n(ctx, n, x, dx, z, dz));
    NYS_TRY(launch_update_m(ctx, m, y, dyp, dyc));
    return residuals(false);
  };
  // runs the graph loop from the current host state; gst: -1 not run (capture failed), else the stop code
  auto run_gloop = [&](int& gst) -> int {
    gst = -1;
    const int maxrec = std::max(1, opt->max_outer + 1);
    double* grec = ctx->wsd("gl_rec", (size_t)16 * maxrec);
    NYS_TRY(launch_set_slots(ctx, S_RHO, rho, S_DELTA, delta, S_OMU, mu));
    NYS_TRY(launch_set_slots(ctx, S_NRP, nrP, S_NRD, nrD, S_NRPREF, nrP_ref));
    NYS_TRY(launch_set_slots(ctx, S_NRDREF, nrD_ref, S_KOUT, (double)k, S_GSTOP, 0.0));
    NYS_TRY(launch_set_slots(ctx, S_INNER, 0.0, S_TSK, 0.0, S_TPCG, 0.0));
    NYS_TRY(launch_set_slots(ctx, S_GLACC, 0.0));
    NYS_TRY(launch_set_slots(ctx, S_MUCUR, mu, S_GPAR0, opt->tol, S_GPAR1, bnorm));
    NYS_TRY(launch_set_slots(ctx, S_GPAR2, cnorm, S_GPAR3, n_total, S_GPAR4, (double)opt->max_outer));
    NYS_TRY(launch_set_slots(ctx, S_GPAR5, opt->reg_floor, S_GPAR6, (double)maxrec));
    char key[512];
    snprintf(key, sizeof(key), "gloop:%lld:%lld:%lld:%p:%p:%p:%p:%lld:%d:%llu:%d:%lld:%.17g:%.17g:%d:%d:%.17g:",
             (long long)ctx->ws_epoch, (long long)m, (long long)n, (const void*)A, (const void*)q, (const void*)b,
             (const void*)c, (long long)lda, ell, (unsigned long long)opt->seed, qp_in->structure, (long long)ncolA,
             opt->pcg_c, opt->pcg_floor, opt->pcg_max_iter, qp_in->n_unit_blocks, n_total);
    std::string gkey(key);
    for (int ib = 0; ib < qp_in->n_unit_blocks; ++ib) {   // the unit blocks are kernel arguments (by value)
      char ub_[96];
      snprintf(ub_, sizeof(ub_), "%lld,%lld,%.17g;", (long long)qp_in->unit_blocks[ib].row0,
               (long long)qp_in->unit_blocks[ib].count, qp_in->unit_blocks[ib].scale);
      gkey += ub_;
    }
    cudaGraphExec_t exec = nullptr;
    int64_t body_launches = 0;
    auto itg = ctx->graphs.find(gkey);
    if (itg != ctx->graphs.end()) {
      exec = itg->second.second.first;
      body_launches = itg->second.first;
    } else {
      cudaGraph_t g;
      NYS_CUDA_TRY(ctx, cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle hc;
      NYS_CUDA_TRY(ctx, cudaGraphConditionalHandleCreate(&hc, g, 1u, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = hc;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t wnode;
      NYS_CUDA_TRY(ctx, cudaGraphAddNode(&wnode, g, nullptr, 0, &cp));
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      const int64_t l0 = ctx->launches, mv0 = ctx->matvecs;
      const int64_t ep0 = ctx->ws_epoch;
      NYS_CUDA_TRY(ctx, cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0,
                                                       cudaStreamCaptureModeThreadLocal));
      ctx->gloop = true;
      int rc = gl_body();
      if (rc == NYS_OK) rc = launch_ipm_control(ctx, grec, hc);
      if (rc == NYS_OK) rc = launch_cond_copy(ctx, S_CPLAM, lam, y, m);
      if (rc == NYS_OK) rc = launch_cond_copy(ctx, S_CPZETA, zeta, x, n);
      ctx->gloop = false;
      cudaGraph_t cap = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &cap);
      body_launches = ctx->launches - l0;
      ctx->launches = l0;
      ctx->matvecs = mv0;
      cudaError_t ie = cudaErrorUnknown;
      if (rc == NYS_OK && ce == cudaSuccess && ctx->ws_epoch == ep0) ie = cudaGraphInstantiate(&exec, g, 0);
      if (ie != cudaSuccess) {   // not capturable here (or a workspace grew): keep the host loop
        cudaGetLastError();
        cudaGraphDestroy(g);
        if (getenv("NYS_DEBUG"))
          fprintf(stderr, "[nys] graph loop not used (rc %d, capture %d, instantiate %d)\n", rc, (int)ce, (int)ie);
        return NYS_OK;
      }
      if (ctx->graphs.size() >= 64) {
        for (auto& kv : ctx->graphs) {
          cudaGraphExecDestroy(kv.second.second.first);
          cudaGraphDestroy(kv.second.second.second);
        }
        ctx->graphs.clear();
      }
      ctx->graphs[gkey] = std::make_pair(body_launches, std::make_pair(exec, g));
    }
    const int k0 = k;
    NYS_CUDA_TRY(ctx, cudaGraphLaunch(exec, ctx->stream));
    NYS_TRY(read_slots(ctx));
    gst = (int)ctx->h_sc[S_GSTOP];
    const int k1 = (int)ctx->h_sc[S_KOUT];
    rho = ctx->h_sc[S_RHO]; delta = ctx->h_sc[S_DELTA]; mu = ctx->h_sc[S_OMU];
    nrP = ctx->h_sc[S_NRP]; nrD = ctx->h_sc[S_NRD]; nrP_ref = ctx->h_sc[S_NRPREF]; nrD_ref = ctx->h_sc[S_NRDREF];
    const int inner = (int)ctx->h_sc[S_INNER];
    total_inner += inner;
    t_sketch += ctx->h_sc[S_TSK];
    t_pcg += ctx->h_sc[S_TPCG];
    ctx->matvecs += inner;                                             // one-launch PCG: one matvec per iteration
    ctx->launches += body_launches * (int64_t)(k1 - k0 + (gst == 2 || gst == 3 ? 1 : 0)) +
                     (int64_t)ctx->h_sc[S_GLACC] * (ell > 0 ? 4 : 3);
    if (k1 > k0) {
      std::vector<double> hr((size_t)16 * (k1 - k0));
      NYS_CUDA_TRY(ctx, cudaMemcpy(hr.data(), grec + (size_t)16 * k0, hr.size() * sizeof(double), cudaMemcpyDeviceToHost));
      for (int i = 0; i < k1 - k0; ++i) {
        const double* r = hr.data() + (size_t)16 * i;
        nys_iter_record rc2{};
        rc2.k = (int)r[0]; rc2.mu = r[1]; rc2.rel_p = r[2]; rc2.rel_d = r[3]; rc2.alpha_p = r[4]; rc2.alpha_d = r[5];
        rc2.pcg_pred = (int)r[6]; rc2.pcg_corr = (int)r[7]; rc2.rho = r[8]; rc2.delta = r[9];
        rc2.t_sketch_ms = r[10]; rc2.t_pcg_ms = r[11]; rc2.t_other_ms = 0.0; rc2.lam_ell = r[12];
        rc2.prec_built = 1; rc2.ell = ell;
        if (R.records && R.n_records < R.max_records) R.records[R.n_records++] = rc2;
      }
    }
    if (getenv("NYS_DEBUG")) fprintf(stderr, "[nys] graph loop: outer %d -> %d, stop code %d, %d PCG iterations\n", k0, k1, gst, inner);
    k = k1;
    return NYS_OK;
  };
  for (k = 0; k <= opt->max_outer; ++k) {
    const double rel_p = nrP / (1.0 + bnorm), rel_d = nrD / (1.0 + cnorm);
    if (rel_p <= opt->tol && rel_d <= opt->tol && mu <= opt->tol) { status = NYS_OK; break; }   // A11
    if (k == opt->max_outer) break;
    if (!std::isfinite(mu) || !std::isfinite(nrP) || !std::isfinite(nrD)) { status = NYS_EBREAKDOWN; break; }
    if (gl_ok && !gl_tried && k >= 1) {
      gl_tried = true;
      int gst = -1;
      NYS_TRY(run_gloop(gst));
      if (gst == 3) { status = NYS_EBREAKDOWN; break; }
      if (gst >= 0) { --k; continue; }   // the loop head re-tests TC / the cap at the new k, or re-runs a failed build
    }
    NvtxRange nv_outer("outer_iteration");
    // One host round trip per outer iteration (f3): the Nystrom build, both PCG solves and the step
    // run with deferred checks (device flags, latched counts) and everything is read with the
    // residuals at the end.  Attempt 1 re-runs the iteration with the host checks when attempt 0
    // raised S_NYSFAIL (the step was discarded on the device: the iterate is unchanged).
    const int last_build0 = last_build, ell_built0 = ell_built;
    const int64_t base_its0 = base_its;
    const bool no_defer = getenv("NYS_NO_DEFER") != nullptr || use_chol;
    nys_iter_record rec{};
    bool built_now = false;
    bool broke = false;
    const double delta_build = delta;
    const auto t_it = std::chrono::steady_clock::now();
    for (int attempt = 0; attempt < 2; ++attempt) {
    const bool defer = attempt == 0 && !no_defer;
    last_build = last_build0; ell_built = ell_built0; base_its = base_its0;
    rec = nys_iter_record{};
    rec.k = k; rec.mu = mu; rec.rel_p = rel_p; rec.rel_d = rel_d; rec.rho = rho; rec.delta = delta;
    if (gen) NYS_TRY(launch_gen_scaling(ctx, n, vt, q, x, z, w, sv, rho, d));
    else NYS_TRY(launch_scaling(ctx, n, q, x, z, rho, d));
    NormalOp op;
    NYS_TRY(AO.normal_op(d, delta, op));
    NYS_CUDA_TRY(ctx, cudaEventRecord(pev.e[0], ctx->stream));
    NYS_TRY(launch_set_slots(ctx, S_PCGBRK, 0.0, S_NYSFAIL, 0.0, S_GITACC, 0.0));
    built_now = false;
    if (use_chol) {                                                   // P:250-349, every iteration
      NYS_TRY(chol_build(ctx, op, ell, CF));
      rec.prec_built = 1;
    } else if (ell > 0) {                                             // P:759, Alg. 2
      const int refresh = opt->prec_refresh > 0 ? opt->prec_refresh : 1;
      const bool rebuild = last_build < 0 || k - last_build >= refresh ||
                           (opt->prec_growth > 0.0 && base_its > 0 && last_its > opt->prec_growth * base_its) ||
                           ell_k != ell_built;
      if (rebuild) {                                                  // f3: reuse between rebuilds
        NYS_TRY(gen_omega(ctx, m, ell_k, opt->seed, (uint64_t)k + 1, Om));
        NYS_TRY(sketch_impl(ctx, m, op.n, op.A, op.lda, op.d, op.e, ell_k, Om, U, lamh, nullptr, defer));
        if (defer && inject_k == k) NYS_TRY(launch_set_slots(ctx, S_NYSFAIL, 1.0));   // test hook
        last_build = k;
        base_its = -1;
        rec.prec_built = 1;
        ell_built = ell_k;
        built_now = true;
        // lambda_hat_ell into a device scalar slot: read with the iteration's residuals (F1 below)
        NYS_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->sc + S_LAML, lamh + ell_built - 1, 8, cudaMemcpyDeviceToDevice,
                                          ctx->stream));
      }
      NYS_TRY(launch_prec_coef(ctx, lamh, ell_built, delta, scoef));  // mu_prec = delta_k (A7)
    }
    NYS_CUDA_TRY(ctx, cudaEventRecord(pev.e[1], ctx->stream));
    NYS_TRY(launch_set_slots(ctx, S_MUCUR, mu));
    // ---- predictor ----
    nvtxRangePushA("predictor");
    if (gen) NYS_TRY(launch_gen_pred_rhs(ctx, n, vt, ub, x, z, w, sv, zeta, rD, rho, d, rd, rxz, ru, rws, xiau, t));
    else NYS_TRY(launch_pred_rhs_n(ctx, n, x, z, zeta, rD, rho, d, rd, rxz, xiau, t));
    NYS_TRY(launch_pred_rhs_m(ctx, m, b, ax, y, lam, delta, rp));
    NYS_TRY(AO.Ax(t, xi, rp));                                        // xi = r_p + A d (r_d + xi_au)
    NYS_TRY(D.dot(m, xi, xi, S_XINORM));
    NYS_TRY(launch_pcg_setup(ctx, 1, 0, opt->pcg_c, opt->pcg_floor, S_XINORM, S_BNORM, S_MUCUR, 0));
    rec.ell = use_chol ? ell : ell_built;
    NYS_CUDA_TRY(ctx, cudaEventRecord(pev.e[2], ctx->stream));
    NYS_TRY(pcg_impl(ctx, op, use_chol ? ell : ell_built, U, mp, scoef, xi, dyp, opt->pcg_max_iter, pr, cfp,
                     defer ? (int)S_PCGI0 : -1));
    NYS_CUDA_TRY(ctx, cudaEventRecord(pev.e[3], ctx->stream));
    if (pr.status == NYS_EBREAKDOWN) { broke = true; break; }
    rec.pcg_pred = pr.iters;
    NYS_TRY(AO.At_dx(dyp, rd, xiau, rxz, z, x, d, dxp, dzp));        // dx, dz (A15)
    if (gen) {
      NYS_TRY(launch_gen_recover(ctx, n, vt, x, z, w, sv, dxp, rxz, ru, rws, dzp, dwp, dsp));   // Alg. 4 line 3
      NYS_TRY(launch_gen_ratio(ctx, n, vt, x, z, w, sv, dxp, dzp, dwp, dsp, nullptr, nullptr, nullptr, nullptr,
                               nullptr, nullptr, nullptr, nullptr, 8));
    } else {
      NYS_TRY(launch_ratio(ctx, n, x, dxp, nullptr, nullptr, z, dzp, nullptr, nullptr, 8));
    }
    NYS_TRY(allreduce_slots(ctx, S_TMP0, 2, true));
    NYS_TRY(launch_steps_post(ctx));
    NYS_TRY(launch_muaff(ctx, n, x, dxp, z, dzp, n_total, 9, w, dwp, sv, dsp));
    if (ctx->multi()) {
      if (gen) NYS_TRY(allreduce_slots(ctx, S_TMP6, 2));
      else NYS_TRY(allreduce_slots(ctx, S_TMP7, 1));
      NYS_TRY(launch_muaff_post(ctx, n_total, gen ? 1 : 0));
    }
    nvtxRangePop();
    // ---- corrector ----
    nvtxRangePushA("corrector");
    if (gen) NYS_TRY(launch_gen_corr_rhs(ctx, n, vt, x, w, dxp, dzp, dwp, dsp, d, rxz, ru, rws, xiau, t));
    else NYS_TRY(launch_corr_rhs(ctx, n, x, dxp, dzp, d, rxz, xiau, t));
    NYS_TRY(AO.Ax(t, xi, nullptr));
    NYS_TRY(D.dot(m, xi, xi, S_XINORM));
    NYS_TRY(launch_pcg_setup(ctx, 1, 0, opt->pcg_c, opt->pcg_floor, S_XINORM, S_BNORM, S_MUCUR, 0));
    NYS_CUDA_TRY(ctx, cudaEventRecord(pev.e[4], ctx->stream));
    NYS_TRY(pcg_impl(ctx, op, use_chol ? ell : ell_built, U, mp, scoef, xi, dyc, opt->pcg_max_iter, pr, cfp,
                     defer ? (int)S_PCGI1 : -1));
    NYS_CUDA_TRY(ctx, cudaEventRecord(pev.e[5], ctx->stream));
    if (pr.status == NYS_EBREAKDOWN) { broke = true; break; }
    rec.pcg_corr = pr.iters;
    NYS_TRY(AO.At_dx(dyc, nullptr, xiau, rxz, z, x, d, dxc, dzc));
    nvtxRangePop();
    // ---- combine, stepsizes, update ----
    if (gen) {
      NYS_TRY(launch_gen_recover(ctx, n, vt, x, z, w, sv, dxc, rxz, ru, rws, dzc, dwc, dsc));
      NYS_TRY(launch_gen_ratio(ctx, n, vt, x, z, w, sv, dx, dz, dw, ds, dxp, dxc, dzp, dzc, dwp, dwc, dsp, dsc, 8));
    } else {
      NYS_TRY(launch_ratio(ctx, n, x, dx, dxp, dxc, z, dz, dzp, dzc, 8));
    }
    NYS_TRY(allreduce_slots(ctx, S_TMP0, 2, true));
    NYS_TRY(launch_steps_post(ctx));
    NYS_TRY(launch_update_n(ctx, n, x, dx, z, dz));
    if (gen) NYS_TRY(launch_update_n(ctx, n, w, dw, sv, ds));         // w += ap dw ; s += ad ds
    NYS_TRY(launch_update_m(ctx, m, y, dyp, dyc));
    NYS_TRY(residuals());                                             // synchronises: events complete
    if (defer) {
      if (ctx->h_sc[S_NYSFAIL] != 0.0) continue;                       // step discarded: re-run with host checks
      rec.pcg_pred = (int)ctx->h_sc[S_PCGI0];
      rec.pcg_corr = (int)ctx->h_sc[S_PCGI1];
      if (!ctx->multi()) {   // single-GPU accounting deferred by pcg_impl (multi-rank loops count as they go)
        const bool persistent = pcg_persistent_supported(ctx, m, op.n, use_chol ? 0 : ell_built) && !use_chol;
        ctx->matvecs += persistent ? rec.pcg_pred + rec.pcg_corr
                                   : std::max(rec.pcg_pred - 2, 0) + std::max(rec.pcg_corr - 2, 0);
        ctx->launches += (int64_t)ctx->h_sc[S_GITACC] * (ell_built > 0 ? 4 : 3);
      }
      if (ctx->h_sc[S_PCGBRK] != 0.0) { broke = true; break; }
    }
    break;
    }
    if (broke) { status = NYS_EBREAKDOWN; break; }
    last_its = (int64_t)rec.pcg_pred + rec.pcg_corr;
    if (base_its < 0) base_its = last_its;
    rec.t_sketch_ms = pev.ms(0, 1);
    rec.t_pcg_ms = pev.ms(2, 3) + pev.ms(4, 5);
    t_sketch += rec.t_sketch_ms;
    if (built_now) {
      lam_ell_cur = ctx->h_sc[S_LAML];
      if (ell_cap > ell_k && lam_ell_cur > opt->ell_tau * delta_build)   // F1: grow for the next build
        ell_k = std::min(2 * ell_k, ell_cap);
    }
    rec.lam_ell = use_chol ? 0.0 : lam_ell_cur;
    rec.alpha_p = ctx->h_sc[S_AP];
    rec.alpha_d = ctx->h_sc[S_AD];
    const double mu_new = n_total > 0 ? ctx->h_sc[S_TMP2] / n_total : 0.0;
    nrP = std::sqrt(ctx->h_sc[S_TMP0]);
    nrD = std::sqrt(ctx->h_sc[S_TMP1]);
    // ---- PEU (A12) ----
    // G5: no inequality at all (every variable free): mu = 0 and the reduction is complete (r = 1)
    double r = (mu > 0) ? std::min(std::max(1.0 - mu_new / mu, 0.0), 1.0) : (n_total > 0 ? 0.0 : 1.0);
    const bool p_imp = nrP <= 0.95 * nrP_ref;
    const bool d_imp = nrD <= 0.95 * nrD_ref;
    if (p_imp) {
      NYS_CUDA_TRY(ctx, cudaMemcpyAsync(lam, y, m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
      nrP_ref = nrP;
    }
    if (d_imp) {
      if (n > 0) NYS_CUDA_TRY(ctx, cudaMemcpyAsync(zeta, x, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
      nrD_ref = nrD;
    }
    delta = std::max(opt->reg_floor, (p_imp ? (1.0 - r) : (1.0 - 2.0 / 3.0 * r)) * delta);
    rho = std::max(opt->reg_floor, (d_imp ? (1.0 - r) : (1.0 - 2.0 / 3.0 * r)) * rho);
    total_inner += rec.pcg_pred + rec.pcg_corr;
    mu = mu_new;
    rec.t_other_ms = ms_since(t_it) - rec.t_sketch_ms - rec.t_pcg_ms;
    t_pcg += rec.t_pcg_ms;
    if (opt->verbose)
      fprintf(stderr, "[nys] k=%3d mu=%.3e rp=%.3e rd=%.3e ap=%.3f ad=%.3f pcg=%d/%d rho=%.2e delta=%.2e\n", k,
              rec.mu, rec.rel_p, rec.rel_d, rec.alpha_p, rec.alpha_d, rec.pcg_pred, rec.pcg_corr, rho, delta);
    if (R.records && R.n_records < R.max_records) R.records[R.n_records++] = rec;
  }
  // ---- objective and solution out ----------------------------------------------------------
  {
    double* qx = t;
    NYS_TRY(launch_mul(ctx, n, q, x, qx));
    NYS_TRY(D.dot(n, x, qx, S_TMP3));
    NYS_TRY(D.dot(n, c, x, S_TMP4));
    NYS_TRY(D.dot(m, b, y, S_TMP5));
    if (gen) {                                                        // u_J^T s_J
      NYS_TRY(launch_gen_half_u(ctx, n, vt, ub, 1.0, xiau));
      NYS_TRY(D.dot(n, xiau, sv, S_TMP6));
      NYS_TRY(allreduce_slots(ctx, S_TMP6, 1));
    } else {
      NYS_TRY(launch_set_slots(ctx, S_TMP6, 0.0));
    }
    NYS_TRY(allreduce_slots(ctx, S_TMP3, 2));
    NYS_TRY(read_slots(ctx));
    const double xqx = ctx->h_sc[S_TMP3], cx = ctx->h_sc[S_TMP4], by = ctx->h_sc[S_TMP5], us = ctx->h_sc[S_TMP6];
    if (sol) {
      sol->obj = 0.5 * xqx + cx;
      sol->dual_obj = by - 0.5 * xqx - us;
      const cudaMemcpyKind kind = qp_in->host_ptrs ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
      if (sol->x && n > 0) NYS_CUDA_TRY(ctx, cudaMemcpyAsync(sol->x, x, n * 8, kind, ctx->stream));
      if (sol->z && n > 0) NYS_CUDA_TRY(ctx, cudaMemcpyAsync(sol->z, z, n * 8, kind, ctx->stream));
      if (sol->y) NYS_CUDA_TRY(ctx, cudaMemcpyAsync(sol->y, y, m * 8, kind, ctx->stream));
      for (int k2 = 0; k2 < 2; ++k2) {                                // w, s (0 for the all-I form)
        double* dst = k2 == 0 ? sol->w : sol->s;
        if (!dst || n <= 0) continue;
        if (gen) NYS_CUDA_TRY(ctx, cudaMemcpyAsync(dst, k2 == 0 ? w : sv, n * 8, kind, ctx->stream));
        else if (qp_in->host_ptrs) memset(dst, 0, n * 8);
        else NYS_CUDA_TRY(ctx, cudaMemsetAsync(dst, 0, n * 8, ctx->stream));
      }
      NYS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    }
  }
  if (rep) {
    rep->status = status;
    rep->outer_iters = k;
    rep->inner_iters = total_inner;
    rep->rel_p = nrP / (1.0 + bnorm);
    rep->rel_d = nrD / (1.0 + cnorm);
    rep->mu = mu;
    rep->t_total_ms = ms_since(t_start);
    rep->t_sketch_ms = t_sketch;
    rep->t_pcg_ms = t_pcg;
    rep->t_other_ms = rep->t_total_ms - t_sketch - t_pcg;
    rep->n_records = R.n_records;
    rep->matvecs = ctx->matvecs - matvecs0;
    rep->kernel_launches = ctx->launches - launches0;
  }
  return status == NYS_EMAXITER ? NYS_EMAXITER : status;
}
}  // namespace

// ==========================================================================================
// extern "C" ABI
// ==========================================================================================
#define NYS_GUARD_BEGIN try {
#define NYS_GUARD_END                 \
  }                                   \
  catch (const NysException& ex) {    \
    return ex.code;                   \
  }                                   \
  catch (...) {                       \
    return NYS_ECUDA;                 \
  }

extern "C" {

const char* nys_strerror(int code) {
  switch (code) {
    case NYS_OK: return "ok";
    case NYS_NOTCONV: return "PCG did not converge within max_iter";
    case NYS_EINVAL: return "invalid argument";
    case NYS_ENONPOS: return "non-positive or non-finite scaling d_j";
    case NYS_ECHOL: return "sketch core not positive definite (Cholesky failed)";
    case NYS_EBREAKDOWN: return "PCG breakdown (p^T N p <= 0 or non-finite)";
    case NYS_EMAXITER: return "IP-PMM outer iteration limit reached";
    case NYS_ECUDA: return "CUDA error";
    case NYS_ENCCL: return "NCCL error";
    case NYS_ENOMEM: return "device allocation failed";
    default: return "unknown error";
  }
}

const char* nys_last_error(nys_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }

int64_t nys_kernel_launches(nys_ctx* ctx) { return ctx ? ctx->launches : 0; }

void nys_default_options(nys_options* o) {
  if (!o) return;
  o->tol = 1e-8;
  o->ell = 0;
  o->seed = 0;
  o->max_outer = 100;
  o->pcg_max_iter = 20000;
  o->rho0 = 8.0;
  o->delta0 = 8.0;
  o->reg_floor = 5e-10;
  o->pcg_c = 1e-3;
  o->pcg_floor = 1e-10;
  o->init_delta = 10.0;
  o->init_tol_rel = 1e-12;
  o->verbose = 0;
  o->prec_refresh = 1;
  o->prec_growth = 0.0;
  o->precond = 0;
  o->ell_max = 0;
  o->ell_tau = 10.0;
}

int nys_create(nys_ctx** out, int device, void* cuda_stream, const void* nccl_unique_id, int rank, int world) {
  if (!out) return NYS_EINVAL;
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return NYS_EINVAL;
  if (world > 1 && !nccl_unique_id) return NYS_EINVAL;
  nys_ctx* ctx = new nys_ctx();
  ctx->device = device;
  ctx->rank = rank;
  ctx->world = world;
  ctx->debug_guard = getenv("NYS_DEBUG_GUARD") != nullptr;
  auto fail = [&](int code) {
    *out = ctx;  // keep for nys_last_error; caller destroys
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) { ctx->set_error("cudaSetDevice failed"); return fail(NYS_ECUDA); }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) { ctx->set_error("cudaGetDeviceProperties failed"); return fail(NYS_ECUDA); }
  ctx->num_sms = prop.multiProcessorCount;
  if (cuda_stream) {
    ctx->stream = (cudaStream_t)cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) return fail(NYS_ECUDA);
    ctx->own_stream = true;
  }
  if (cudaMalloc(&ctx->sc, S_COUNT * sizeof(double)) != cudaSuccess) return fail(NYS_ENOMEM);
  if (cudaMalloc(&ctx->counters, kMaxCounters * sizeof(unsigned int)) != cudaSuccess) return fail(NYS_ENOMEM);
  cudaMemset(ctx->sc, 0, S_COUNT * sizeof(double));
  cudaMemset(ctx->counters, 0, kMaxCounters * sizeof(unsigned int));
  if (cudaMallocHost(&ctx->h_sc, S_COUNT * sizeof(double)) != cudaSuccess) return fail(NYS_ENOMEM);
  cudaEventCreate(&ctx->ev0);
  cudaEventCreate(&ctx->ev1);
  if (world > 1 && std::memcmp(nccl_unique_id, "NYSLOOP", 8) == 0) {  // loopback (one device)
    void* lc = nullptr;
    std::memcpy(&lc, (const char*)nccl_unique_id + 8, sizeof(void*));
    LoopComm* c = (LoopComm*)lc;
    if (!c || c->world != world) { ctx->set_error("loopback communicator / world mismatch"); return fail(NYS_EINVAL); }
    ctx->loop_comm = c;
  } else if (world > 1 || nccl_unique_id) {   // world = 1 with an id: a one-rank NCCL communicator
    ctx->coll = true;
    std::string err;
    if (!g_nccl.load(err)) { ctx->set_error(err); return fail(NYS_ENCCL); }
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    ncclComm_t comm;
    ncclResult_t r = g_nccl.commInitRank(&comm, world, id, rank);
    if (r != ncclSuccess) { ctx->set_error("ncclCommInitRank failed"); return fail(NYS_ENCCL); }
    ctx->nccl_comm = comm;
  }
  cudaDeviceSynchronize();
  *out = ctx;
  return NYS_OK;
}

static std::map<nys_ctx*, nys::CholFactors> g_chol;  // last nys_partial_cholesky per context
static std::mutex g_chol_mu;

int nys_loopback_comm_create(int world, void* out128) {
  if (world < 2 || world > 16 || !out128) return NYS_EINVAL;
  LoopComm* c = new LoopComm();
  c->world = world;
  c->bufs.assign(world, nullptr);
  std::memset(out128, 0, 128);
  std::memcpy(out128, "NYSLOOP", 8);
  std::memcpy((char*)out128 + 8, &c, sizeof(void*));
  return NYS_OK;
}

int nys_loopback_comm_destroy(void* id128) {
  if (!id128 || std::memcmp(id128, "NYSLOOP", 8) != 0) return NYS_EINVAL;
  LoopComm* c = nullptr;
  std::memcpy(&c, (const char*)id128 + 8, sizeof(void*));
  delete c;
  return NYS_OK;
}

int nys_nccl_unique_id(void* out128) {
  if (!out128) return NYS_EINVAL;
  std::string err;
  if (!g_nccl.load(err) || !g_nccl.getUniqueId) return NYS_ENCCL;
  ncclUniqueId id;
  if (g_nccl.getUniqueId(&id) != ncclSuccess) return NYS_ENCCL;
  std::memcpy(out128, &id, sizeof(id));
  return NYS_OK;
}

int nys_destroy(nys_ctx* ctx) {
  if (!ctx) return NYS_OK;
  {
    std::lock_guard<std::mutex> lk(g_chol_mu);
    g_chol.erase(ctx);
  }
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto& kv : ctx->bufs) cudaFree(kv.second.first);
  if (ctx->sc) cudaFree(ctx->sc);
  if (ctx->counters) cudaFree(ctx->counters);
  if (ctx->guard_flag) cudaFree(ctx->guard_flag);
  if (ctx->h_sc) cudaFreeHost(ctx->h_sc);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  for (auto& kv : ctx->graphs) {
    cudaGraphExecDestroy(kv.second.second.first);
    cudaGraphDestroy(kv.second.second.second);
  }
  if (ctx->nccl_comm && g_nccl.commDestroy) g_nccl.commDestroy((ncclComm_t)ctx->nccl_comm);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  if (ctx->side_stream) cudaStreamDestroy(ctx->side_stream);
  delete ctx;
  return NYS_OK;
}

static int check_A(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda) {
  if (!ctx) return NYS_EINVAL;
  if (m < 1 || n < 0 || lda < m || (lda & 1)) { ctx->set_error("bad m / n / lda (lda must be >= m and even)"); return NYS_EINVAL; }
  if (n > 0 && (!A || !aligned16(A))) { ctx->set_error("A must be a 16-byte aligned device pointer"); return NYS_EINVAL; }
  return NYS_OK;
}

static int nys_normal_matvec_body(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d,
                             const double* e, double delta, const double* v, double* w) {
  NYS_GUARD_BEGIN
  NYS_TRY(check_A(ctx, m, n, A, lda));
  if (!v || !w || (n > 0 && !d) || delta < 0 || v == w) { ctx->set_error("bad vector arguments"); return NYS_EINVAL; }
  cudaSetDevice(ctx->device);
  NormalOp op{m, n, lda, A, d, e, delta};
  NYS_TRY(apply_normal_full(ctx, op, v, nullptr, nullptr, nullptr, w, false, nullptr));
  return NYS_OK;
  NYS_GUARD_END
}

// a failing call on one loopback rank releases its peers (LoopComm::abort)
int nys_normal_matvec(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d,
                      const double* e, double delta, const double* v, double* w) {
  return loop_abort_on_error(ctx, nys_normal_matvec_body(ctx, m, n, A, lda, d, e, delta, v, w));
}

int nys_check_scaling(nys_ctx* ctx, int64_t n, const double* d, int64_t* bad_index) {
  NYS_GUARD_BEGIN
  if (!ctx || n < 0 || (n > 0 && !d)) return NYS_EINVAL;
  cudaSetDevice(ctx->device);
  unsigned long long* bad = (unsigned long long*)ctx->ws("chk_bad", 8);
  unsigned long long init = ~0ULL, hv = 0;
  NYS_CUDA_TRY(ctx, cudaMemcpyAsync(bad, &init, 8, cudaMemcpyHostToDevice, ctx->stream));
  NYS_TRY(launch_check_pos(ctx, n, d, bad));
  NYS_CUDA_TRY(ctx, cudaMemcpyAsync(&hv, bad, 8, cudaMemcpyDeviceToHost, ctx->stream));
  NYS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (bad_index) *bad_index = (hv == ~0ULL) ? -1 : (int64_t)hv;
  if (hv != ~0ULL) {
    ctx->set_error("d has a non-positive or non-finite entry at index " + std::to_string(hv));
    return NYS_ENONPOS;
  }
  return NYS_OK;
  NYS_GUARD_END
}

int nys_gaussian(nys_ctx* ctx, int64_t m, int ell, uint64_t seed, uint64_t stream, double* Omega) {
  NYS_GUARD_BEGIN
  if (!ctx || m < 0 || ell < 0 || (m * ell > 0 && !Omega)) return NYS_EINVAL;
  cudaSetDevice(ctx->device);
  return launch_gaussian(ctx, Omega, m * (int64_t)ell, seed, stream);
  NYS_GUARD_END
}

static int nys_sketch_body(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d, const double* e,
                      double delta, int ell, const double* Omega, double* U, double* lambda, nys_sketch_info* info) {
  NYS_GUARD_BEGIN
  NYS_TRY(check_A(ctx, m, n, A, lda));
  if (ell < 1 || ell > m || ell > kMaxEll || !(delta > 0) || !Omega || !U || !lambda || (n > 0 && !d)) {
    ctx->set_error("nys_sketch: need 1 <= ell <= min(m, 1024), delta > 0, non-null buffers");
    return NYS_EINVAL;
  }
  cudaSetDevice(ctx->device);
  NYS_CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  const int64_t mp = even(m);
  const double* Om = Omega;
  double* Uo = U;
  if (mp != m || !aligned16(Omega) || !aligned16(U)) {
    double* Omw = ctx->wsd("sk_Om_in", (size_t)mp * ell);
    NYS_CUDA_TRY(ctx, cudaMemcpy2DAsync(Omw, mp * 8, Omega, m * 8, m * 8, ell, cudaMemcpyDeviceToDevice, ctx->stream));
    Om = Omw;
    Uo = ctx->wsd("sk_U_out", (size_t)mp * ell);
  }
  nys_sketch_info tmp{};
  NYS_TRY(sketch_impl(ctx, m, n, A, lda, d, e, ell, Om, Uo, lambda, &tmp));
  if (Uo != U)
    NYS_CUDA_TRY(ctx, cudaMemcpy2DAsync(U, m * 8, Uo, mp * 8, m * 8, ell, cudaMemcpyDeviceToDevice, ctx->stream));
  NYS_CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  NYS_CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev1));
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  tmp.t_ms = ms;
  if (info) *info = tmp;
  return NYS_OK;
  NYS_GUARD_END
}

// a failing call on one loopback rank releases its peers (LoopComm::abort)
int nys_sketch(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d, const double* e,
               double delta, int ell, const double* Omega, double* U, double* lambda, nys_sketch_info* info) {
  return loop_abort_on_error(ctx, nys_sketch_body(ctx, m, n, A, lda, d, e, delta, ell, Omega, U, lambda, info));
}

static int nys_sketch_apply_body(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d,
                            const double* e, int ell, const double* Omega, double* Y) {
  NYS_GUARD_BEGIN
  NYS_TRY(check_A(ctx, m, n, A, lda));
  if (ell < 1 || !Omega || !Y || (n > 0 && !d)) { ctx->set_error("nys_sketch_apply: bad arguments"); return NYS_EINVAL; }
  cudaSetDevice(ctx->device);
  const int64_t mp = even(m);
  const double* Om = Omega;
  double* Yo = Y;
  if (mp != m || !aligned16(Omega) || !aligned16(Y)) {
    double* Omw = ctx->wsd("sk_Om_in", (size_t)mp * ell);
    NYS_CUDA_TRY(ctx, cudaMemcpy2DAsync(Omw, mp * 8, Omega, m * 8, m * 8, ell, cudaMemcpyDeviceToDevice, ctx->stream));
    Om = Omw;
    Yo = ctx->wsd("sk_Y_out", (size_t)mp * ell);
  }
  NYS_TRY(sketch_Y(ctx, m, n, A, lda, d, e, ell, Om, Yo));
  if (Yo != Y)
    NYS_CUDA_TRY(ctx, cudaMemcpy2DAsync(Y, m * 8, Yo, mp * 8, m * 8, ell, cudaMemcpyDeviceToDevice, ctx->stream));
  return NYS_OK;
  NYS_GUARD_END
}

// a failing call on one loopback rank releases its peers (LoopComm::abort)
int nys_sketch_apply(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d,
                     const double* e, int ell, const double* Omega, double* Y) {
  return loop_abort_on_error(ctx, nys_sketch_apply_body(ctx, m, n, A, lda, d, e, ell, Omega, Y));
}

static int nys_partial_cholesky_body(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d,
                                const double* e, double delta, int ell, int64_t* piv, double* L, double* dS) {
  NYS_GUARD_BEGIN
  NYS_TRY(check_A(ctx, m, n, A, lda));
  if (ell < 0 || ell > m || ell > 256 || !(delta > 0) || (n > 0 && !d)) {
    ctx->set_error("nys_partial_cholesky: bad arguments");
    return NYS_EINVAL;
  }
  cudaSetDevice(ctx->device);
  NormalOp op{m, n, lda, A, d, e, delta};
  CholFactors F;
  NYS_TRY(chol_build(ctx, op, ell, F));
  {
    // the factors nys_chol_precond_apply uses live in buffers only this call writes: chol_build's
    // ch_* workspaces are overwritten (or reallocated) by every later build on the context,
    // including each Chol-IP-PMM outer iteration
    const int64_t mp = even(m);
    const int le = ell > 0 ? ell : 1;
    CholFactors K = F;
    K.piv = (int64_t*)ctx->ws("abi_ch_piv", sizeof(int64_t) * le);
    K.pivpos = (int*)ctx->ws("abi_ch_pivpos", sizeof(int) * mp);
    K.Rinv = ctx->wsd("abi_ch_Rinv", (size_t)F.ldr * F.ldr);
    K.Zt = ctx->wsd("abi_ch_Zt", (size_t)m * le);
    K.dS = ctx->wsd("abi_ch_dS", (size_t)mp);
    K.diag = ctx->wsd("abi_ch_diag", (size_t)mp);
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(K.piv, F.piv, sizeof(int64_t) * le, cudaMemcpyDeviceToDevice, ctx->stream));
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(K.pivpos, F.pivpos, sizeof(int) * mp, cudaMemcpyDeviceToDevice, ctx->stream));
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(K.Rinv, F.Rinv, sizeof(double) * F.ldr * F.ldr, cudaMemcpyDeviceToDevice, ctx->stream));
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(K.Zt, F.Zt, sizeof(double) * m * le, cudaMemcpyDeviceToDevice, ctx->stream));
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(K.dS, F.dS, sizeof(double) * mp, cudaMemcpyDeviceToDevice, ctx->stream));
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(K.diag, F.diag, sizeof(double) * mp, cudaMemcpyDeviceToDevice, ctx->stream));
    std::lock_guard<std::mutex> lk(g_chol_mu);
    g_chol[ctx] = K;
  }
  if (piv && ell > 0)
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(piv, F.piv, sizeof(int64_t) * ell, cudaMemcpyDeviceToDevice, ctx->stream));
  if (L && ell > 0) NYS_TRY(launch_transpose_u(ctx, ell, (int)m, F.Zt, ell, L));   // row-major -> column-major
  if (dS) NYS_CUDA_TRY(ctx, cudaMemcpyAsync(dS, F.dS, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream));
  NYS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return NYS_OK;
  NYS_GUARD_END
}

// a failing call on one loopback rank releases its peers (LoopComm::abort)
int nys_partial_cholesky(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d,
                         const double* e, double delta, int ell, int64_t* piv, double* L, double* dS) {
  return loop_abort_on_error(ctx, nys_partial_cholesky_body(ctx, m, n, A, lda, d, e, delta, ell, piv, L, dS));
}

int nys_chol_precond_apply(nys_ctx* ctx, int64_t m, const double* v, double* out) {
  NYS_GUARD_BEGIN
  if (!ctx || !v || !out) return NYS_EINVAL;
  CholFactors F;
  {
    std::lock_guard<std::mutex> lk(g_chol_mu);
    auto it = g_chol.find(ctx);
    if (it == g_chol.end() || it->second.m != m) {
      ctx->set_error("nys_chol_precond_apply: no partial Cholesky factors of this size on the context");
      return NYS_EINVAL;
    }
    F = it->second;
  }
  cudaSetDevice(ctx->device);
  NYS_TRY(launch_chol_apply(ctx, F, v, out, 0, 0));
  return NYS_OK;
  NYS_GUARD_END
}

static int nys_pcg_solve_body(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d, const double* e,
                         double delta, int ell, const double* U, const double* lambda, double mu_prec, const double* rhs,
                         double* x, double tol_abs, int max_iter, nys_pcg_info* info) {
  NYS_GUARD_BEGIN
  NYS_TRY(check_A(ctx, m, n, A, lda));
  if (ell < 0 || ell > m || ell > kMaxEll || (ell > 0 && (!U || !lambda)) || !rhs || !x || max_iter < 0 || delta < 0 ||
      (n > 0 && !d) || (ell > 0 && !(mu_prec > 0))) {
    ctx->set_error("nys_pcg_solve: bad arguments");
    return NYS_EINVAL;
  }
  cudaSetDevice(ctx->device);
  NYS_CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  const int64_t mp = even(m);
  const double* Uu = U;
  if (ell > 0 && (mp != m || !aligned16(U))) {
    double* Uw = ctx->wsd("pcg_U_in", (size_t)mp * ell);
    NYS_CUDA_TRY(ctx, cudaMemcpy2DAsync(Uw, mp * 8, U, m * 8, m * 8, ell, cudaMemcpyDeviceToDevice, ctx->stream));
    Uu = Uw;
  }
  double* s = ctx->wsd("pcg_s", (size_t)(ell > 0 ? ell : 1));
  if (ell > 0) NYS_TRY(launch_prec_coef(ctx, lambda, ell, mu_prec, s));
  NYS_TRY(launch_pcg_setup(ctx, 0, tol_abs, 0, 0, 0, 0, 0, 0));
  NormalOp op{m, n, lda, A, d, e, delta};
  PcgResult pr;
  NYS_TRY(pcg_impl(ctx, op, ell, Uu, mp, s, rhs, x, max_iter, pr));
  // true residual at exit: ||rhs - N x||
  double* w = ctx->wsd("pcg_truew", (size_t)mp);
  NYS_TRY(apply_normal_full(ctx, op, x, nullptr, nullptr, nullptr, w, false, nullptr));
  NYS_TRY(launch_axpby(ctx, m, 1.0, rhs, -1.0, w, w));
  {
    const double* aa[1] = {w};
    const double* bb[1] = {w};
    int out[1] = {S_TMP6};
    NYS_TRY(launch_dots(ctx, m, 1, aa, bb, out, 10));
  }
  NYS_CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  NYS_TRY(read_slots(ctx));
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  const bool conv = std::sqrt(pr.rr) <= tol_abs;
  if (info) {
    info->iters = pr.iters;
    info->converged = conv ? 1 : 0;
    info->res_norm = std::sqrt(pr.rr);
    info->true_res_norm = std::sqrt(ctx->h_sc[S_TMP6]);
    info->t_ms = ms;
  }
  if (pr.status == NYS_EBREAKDOWN) { ctx->set_error("PCG breakdown"); return NYS_EBREAKDOWN; }
  return conv ? NYS_OK : NYS_NOTCONV;
  NYS_GUARD_END
}

// a failing call on one loopback rank releases its peers (LoopComm::abort)
int nys_pcg_solve(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d, const double* e,
                  double delta, int ell, const double* U, const double* lambda, double mu_prec, const double* rhs,
                  double* x, double tol_abs, int max_iter, nys_pcg_info* info) {
  return loop_abort_on_error(ctx, nys_pcg_solve_body(ctx, m, n, A, lda, d, e, delta, ell, U, lambda, mu_prec, rhs, x, tol_abs, max_iter, info));
}

static int nys_ipppmm_solve_body(nys_ctx* ctx, const nys_qp* qp, const nys_options* opt, nys_solution* sol, nys_report* rep) {
  NYS_GUARD_BEGIN
  if (!ctx || !qp || !opt) return NYS_EINVAL;
  if (qp->m < 1 || qp->n < 0 || qp->lda < qp->m || !qp->b || (qp->n > 0 && (!qp->A || !qp->q || !qp->c))) {
    ctx->set_error("nys_ipppmm_solve: bad problem");
    return NYS_EINVAL;
  }
  if (qp->structure == 1) {
    const bool one = qp->n_unit_blocks == 1 && qp->unit_blocks != nullptr;
    const int64_t r0 = one ? qp->unit_blocks[0].row0 : 0, mr = one ? qp->unit_blocks[0].count : qp->m;
    const bool ok = qp->nd >= 0 && (qp->n_unit_blocks == 0 || one) && r0 >= 0 && mr >= 0 && r0 + mr <= qp->m &&
                    (!one || qp->unit_blocks[0].scale == 1.0) && qp->n == 2 * qp->nd + 2 * mr &&
                    (ctx->multi() || (r0 == 0 && mr == qp->m));
    if (!ok) {
      ctx->set_error("nys_ipppmm_solve: structure 1 needs n = 2 nd + 2 count with this rank's xi / s rows given as one "
                     "unit block (row0, count, scale 1) inside [0, m) (single rank: the whole range)");
      return NYS_EINVAL;
    }
  }
  if (qp->structure == 2) {
    bool ok = qp->nd >= 1 && qp->n_unit_blocks >= 0 && qp->n_unit_blocks <= 8 &&
              (qp->n_unit_blocks == 0 || qp->unit_blocks != nullptr);
    int64_t tot = qp->nd;
    for (int k = 0; ok && k < qp->n_unit_blocks; ++k) {
      const nys_unit_block& u = qp->unit_blocks[k];
      ok = u.row0 >= 0 && u.count >= 0 && u.row0 + u.count <= qp->m && std::isfinite(u.scale) && u.scale != 0.0;
      tot += u.count;
    }
    if (!ok || tot != qp->n) {
      ctx->set_error("nys_ipppmm_solve: structure 2 needs nd >= 1, <= 8 unit blocks inside [0, m) with nonzero "
                     "scale, and n = nd + sum(count)");
      return NYS_EINVAL;
    }
  }
  if (qp->structure < 0 || qp->structure > 2) {
    ctx->set_error("nys_ipppmm_solve: unknown structure");
    return NYS_EINVAL;
  }
  if (!qp->host_ptrs) NYS_TRY(check_A(ctx, qp->m, qp->structure >= 1 ? qp->nd : qp->n, qp->A, qp->lda));
  if (opt->ell < 0 || opt->ell > qp->m || opt->ell > (opt->precond == 1 ? 256 : kMaxEll) || !(opt->tol > 0)) {
    ctx->set_error("nys_ipppmm_solve: bad options");
    return NYS_EINVAL;
  }
  cudaSetDevice(ctx->device);
  return ipm_impl(ctx, qp, opt, sol, rep);
  NYS_GUARD_END
}

// a failing call on one loopback rank releases its peers (LoopComm::abort)
int nys_ipppmm_solve(nys_ctx* ctx, const nys_qp* qp, const nys_options* opt, nys_solution* sol, nys_report* rep) {
  return loop_abort_on_error(ctx, nys_ipppmm_solve_body(ctx, qp, opt, sol, rep));
}

}  // extern "C"
