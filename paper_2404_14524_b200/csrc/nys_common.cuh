// Internal header of libnysipm.so (sm_100a).  Not part of the public ABI (include/nysipm.h).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "nysipm.h"

// ------------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------------
#define NYS_CUDA_TRY(ctx, expr)                                                            \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      (ctx)->set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                \
      return NYS_ECUDA;                                                                    \
    }                                                                                      \
  } while (0)

#define NYS_TRY(expr)               \
  do {                              \
    int _rc = (expr);               \
    if (_rc < 0) return _rc;        \
  } while (0)

// ------------------------------------------------------------------------------------------
// device scalar slots (one fp64 array in device memory per context)
// ------------------------------------------------------------------------------------------
namespace nys {
enum Slot : int {
  // PCG
  S_RZ = 0, S_PW, S_ALPHA, S_RR, S_BETA, S_TOL, S_DONE, S_ITERS, S_STATUS, S_MU, S_LAML,
  // reductions / IPM
  S_TMP0, S_TMP1, S_TMP2, S_TMP3, S_TMP4, S_TMP5, S_TMP6, S_TMP7,
  S_AP, S_AD, S_MUAFF, S_MUT, S_MUCUR, S_XINORM, S_BNORM,
  S_NU, S_SHIFT, S_CHOLFAIL, S_FRO, S_JSWEEPS, S_DELTA, S_GITER,
  // general-form initial point statistics (f1, gen_init_stats): 4 minima then 8 sums
  S_G0, S_G1, S_G2, S_G3, S_G4, S_G5, S_G6, S_G7, S_G8, S_G9, S_G10, S_G11,
  // one host round trip per outer iteration (ipm_impl): the two PCG solves' iteration counts, a
  // breakdown flag, a Nystrom-factorisation failure flag and the graph-path iteration accounting are
  // latched on the device and read with the iteration's residuals
  S_PCGI0, S_PCGI1, S_PCGBRK, S_NYSFAIL, S_GITACC,
  // graph-resident outer loop (f3, ipm_impl): the loop state lives on the device — rho, delta (S_DELTA),
  // mu, the residual norms and the PEU references, the outer index, a stop code, the PEU copy flags,
  // accumulated PCG iterations and phase times (globaltimer stamps), and the per-solve constants
  S_RHO, S_OMU, S_NRP, S_NRD, S_NRPREF, S_NRDREF, S_KOUT, S_GSTOP, S_CPLAM, S_CPZETA, S_INNER, S_TSK, S_TPCG,
  S_TS0, S_TS1, S_TS2, S_TS3, S_TS4, S_TS5,
  S_GPAR0, S_GPAR1, S_GPAR2, S_GPAR3, S_GPAR4, S_GPAR5, S_GPAR6, S_GLACC,
  S_COUNT = 96
};
constexpr int kMaxCounters = 64;
}  // namespace nys

// ------------------------------------------------------------------------------------------
// context
// ------------------------------------------------------------------------------------------
struct nys_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int rank = 0, world = 1;
  bool coll = false;               // a one-rank NCCL communicator (world = 1 with an id): multi-rank path
  bool multi() const { return world > 1 || coll; }
  bool gloop = false;              // capturing the graph-resident outer loop: per-iteration scalars from slots
  cudaStream_t side_stream = nullptr;  // nested captures (the PCG WHILE body inside the outer loop's body)
  void* nccl_comm = nullptr;
  void* loop_comm = nullptr;      // in-process loopback communicator (nys_loopback_comm_create)
  int num_sms = 148;
  int64_t launches = 0;
  int64_t matvecs = 0;
  std::string last_error;
  std::map<std::string, std::pair<void*, size_t>> bufs;
  double* sc = nullptr;           // device scalars [S_COUNT]
  unsigned int* counters = nullptr;  // device counters for last-block reductions
  double* h_sc = nullptr;         // pinned host mirror
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int64_t ws_epoch = 0;           // bumped whenever a workspace buffer is (re)allocated
  std::map<std::string, std::pair<int64_t, std::pair<cudaGraphExec_t, cudaGraph_t>>> graphs;  // PCG loop graphs
  // NYS_DEBUG_GUARD=1 (memcheck substitute; compute-sanitizer is closed on the GPU pool): every
  // workspace buffer is poisoned with NaN bytes when (re)allocated and followed by a 64 KiB canary,
  // verified after every ABI call (check_guards) -> an out-of-bounds write fails the call loudly,
  // a read of never-written workspace turns results into NaN (caught by the parity checks)
  bool debug_guard = false;
  unsigned int* guard_flag = nullptr;
  int check_guards();

  void set_error(const std::string& s) { last_error = s; }
  // named workspace, grown monotonically; contents are NOT preserved on growth
  void* ws(const char* name, size_t bytes);
  double* wsd(const char* name, size_t count) { return (double*)ws(name, count * sizeof(double)); }
  int check_launch(const char* what);
};

// ------------------------------------------------------------------------------------------
// PTX helpers (sm_90+/sm_100a): mbarrier, bulk async copy, cluster / DSMEM
// ------------------------------------------------------------------------------------------
namespace nys {
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
// generic-proxy shared-memory writes made visible to the async proxy (a later cp.async.bulk into
// the same stage must not be reordered before them)
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  const uint32_t a = smem_u32(bar);
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  const uint32_t a = smem_u32(bar);
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 1-D bulk async copy global -> shared (own CTA), completion on mbarrier (tx bytes)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// prefetch a contiguous global range into L2 (bulk, no completion tracking); 16-byte multiple
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t ncluster_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_cluster_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
// async remote store into a peer CTA's shared memory; completes `bytes` of transaction on the
// peer's mbarrier (the receiver waits with a plain cta-scope try_wait: no cluster-scope acquire,
// hence no L1 invalidation per wait)
__device__ __forceinline__ void st_async_f64(uint32_t cluster_addr, double v, uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(cluster_addr),
               "d"(v), "r"(cluster_bar)
               : "memory");
}
// gpu-scope ordering without full fences: release-RMW arrive, relaxed polling, one acquire fence
__device__ __forceinline__ unsigned int atom_add_acqrel_gpu(unsigned int* p, unsigned int v) {
  unsigned int old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_relaxed_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// acquire load: reading the value written by the last of a release sequence of red.release arrivals
// synchronises with all of them (no separate fence after the spin)
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// warp index broadcast from lane 0: lets the compiler prove warp-uniform branches, so shuffles
// inside them are not lowered to the slow WARPSYNC.COLLECTIVE path (cf. CUTLASS canonical_warp_idx_sync)
__device__ __forceinline__ int warp_uniform_id() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// deterministic warp-level sum / min of a global array (lane-strided L2 loads issued 8 at a time so
// that a round costs one L2 latency, not eight; fixed pairwise + xor trees)
__device__ __forceinline__ double warp_sum_array(const double* x, int n) {
  const int lane = threadIdx.x & 31;
  double a = 0.0;
  for (int i0 = lane; i0 < n; i0 += 256) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = (i0 + 32 * u < n) ? __ldcg(x + i0 + 32 * u) : 0.0;
    a += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}
__device__ __forceinline__ double warp_min_array(const double* x, int n) {
  const int lane = threadIdx.x & 31;
  double a = 1.0e300;
  for (int i0 = lane; i0 < n; i0 += 256) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = (i0 + 32 * u < n) ? __ldcg(x + i0 + 32 * u) : 1.0e300;
    a = fmin(a, fmin(fmin(fmin(v[0], v[1]), fmin(v[2], v[3])), fmin(fmin(v[4], v[5]), fmin(v[6], v[7]))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
  return a;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
}  // namespace nys

// ------------------------------------------------------------------------------------------
// internal launchers (implemented in k_*.cu)
// ------------------------------------------------------------------------------------------
namespace nys {

// Raise (never lower) a kernel's dynamic shared-memory limit on the context's device: several
// plans share one kernel instantiation with different stage counts, so the attribute must stay
// >= every plan's launch size.
int ensure_max_smem(nys_ctx* ctx, const void* fn, size_t bytes);

// MV_DIAG: out_i = sum_j d_j A_ij^2 (the diagonal of A D A^T; partial Cholesky)
// MV_BOTH: T-only pass on v (epilogue tep) AND out = sgn A u + add from the same read of A
enum MatvecMode { MV_FUSED = 0, MV_TONLY = 1, MV_NONLY = 2, MV_DIAG = 3, MV_BOTH = 4 };

// where the fused PCG matvec left its per-cluster w partials and per-CTA p^T N p partials
struct FusedPartials {
  const double* Wp = nullptr;
  int64_t wp_ld = 0;
  int nparts = 0;
  const double* pwp = nullptr;
  int npw = 0;
};
enum TEpilogue { TE_PLAIN = 0, TE_DX = 1, TE_RD = 2 };

struct MatvecCall {
  int mode = MV_FUSED;
  int64_t m = 0, n = 0, lda = 0;
  const double* A = nullptr;
  // operand vector v = z + (*beta) * p   (beta/p may be null)
  const double* z = nullptr;
  const double* p = nullptr;
  const double* beta = nullptr;
  double* p_out = nullptr;          // if set: v is written here (by cluster 0)
  const double* d = nullptr;        // FUSED: t_j = d_j (A^T v)_j
  const double* u = nullptr;        // NONLY: t_j = u_j
  // FUSED / NONLY finalize: out_i = sgn * (A t)_i + (delta + e_i) v_i + add_i ;
  // optional dot out^T v -> scalar slot (PCG: p^T w, then alpha = rz / pw)
  double* out = nullptr;
  double sgn = 1.0;
  double delta = 0.0;
  bool use_delta = false;
  const double* e = nullptr;
  const double* add = nullptr;
  bool pcg_alpha = false;           // compute pw and alpha (slots S_PW, S_ALPHA) ; breakdown -> S_STATUS
  // TONLY epilogue
  int tep = TE_PLAIN;
  double* t1 = nullptr;             // PLAIN: (A^T v)_j ; DX: dx ; RD: rD
  double* t2 = nullptr;             // DX: dz
  const double* ta = nullptr;       // DX: r_d (or null)   RD: c
  const double* tb = nullptr;       // DX: xi_au           RD: q
  const double* tc = nullptr;       // DX: r_xz            RD: x
  const double* td = nullptr;       // DX: z               RD: z (or null)
  const double* tx = nullptr;       // DX: x
  const double* tdd = nullptr;      // DX: d
  const double* done = nullptr;     // early-exit flag (device scalar), or null
  bool pcg_fused = false;           // FUSED for PCG (world == 1): partials only, consumed by pcg_update
  bool delta_from_slot = false;     // FUSED PCG: delta read from sc[S_DELTA] (graph-invariant)
  FusedPartials* fused_out = nullptr;
};
int launch_matvec(nys_ctx* ctx, const MatvecCall& c);

}  // namespace nys
