// launchers of k_vec.cu, k_gemm.cu and k_small.cu (internal)
#pragma once
#include "nys_common.cuh"

namespace nys {

// ------------------------------------------------------------------------------------------
// generic deterministic block reduction helpers
// ------------------------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void block_sum_to_part(double (&v)[NV], double* part, int stride) {
  __shared__ double sh[NV][32];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) sh[k][w] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int i = 0; i < nw; ++i) s += sh[k][i];
      part[(size_t)k * stride + blockIdx.x] = s;
    }
  }
}

__device__ __forceinline__ bool last_block_arrive(unsigned int* counter) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}



// k_vec.cu
int launch_gaussian(nys_ctx* ctx, double* O, int64_t total, uint64_t seed, uint64_t stream);
int launch_dots(nys_ctx* ctx, int64_t n, int nv, const double* const* a, const double* const* b, const int* out,
                int counter_slot);
int launch_muaff(nys_ctx* ctx, int64_t n, const double* x, const double* dx, const double* z, const double* dz,
                 double n_total, int counter_slot, const double* w = nullptr, const double* dw = nullptr,
                 const double* s = nullptr, const double* ds = nullptr);
int launch_muaff_post(nys_ctx* ctx, double n_total, int gen = 0);
int launch_ratio(nys_ctx* ctx, int64_t n, const double* x, double* dx, const double* dx1, const double* dx2,
                 const double* z, double* dz, const double* dz1, const double* dz2, int counter_slot);
int launch_steps_post(nys_ctx* ctx);
// graph-resident outer loop (ipm_impl, f3)
int launch_stamp(nys_ctx* ctx, int slot);
int launch_ipm_control(nys_ctx* ctx, double* rec, cudaGraphConditionalHandle h);
int launch_cond_copy(nys_ctx* ctx, int flag, double* dst, const double* src, int64_t len);
int launch_set_cond(nys_ctx* ctx, unsigned long long h, unsigned int v);
int launch_inject_nysfail(nys_ctx* ctx, int k);
// structure 2 (k_gen.cu): scaled identity blocks of A (nys_unit_block); off = column offsets in the unit part
struct UnitBlocks {
  int nb = 0;
  int64_t total = 0;
  int64_t row0[8], count[8], off[8];
  double scale[8];
};
int launch_unit_expand(nys_ctx* ctx, const UnitBlocks& U, const double* y, double* atv_unit);
int launch_unit_fold(nys_ctx* ctx, const UnitBlocks& U, int64_t m, const double* u_unit, const double* add, int diag,
                     double* out);
// general form (f1, k_gen.cu): vt[j] 0 = I, 1 = F, 2 = J
int launch_gen_scaling(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* q, const double* x, const double* z,
                       const double* w, const double* s, double rho, double* d);
int launch_gen_pred_rhs(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* ub, const double* x, const double* z,
                        const double* w, const double* s, const double* zeta, const double* rD, double rho,
                        const double* d, double* rd, double* rxz, double* ru, double* rws, double* xiau, double* t);
int launch_gen_corr_rhs(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* x, const double* w, const double* dxp,
                        const double* dzp, const double* dwp, const double* dsp, const double* d, double* rxz,
                        double* ru, double* rws, double* xiau, double* t);
int launch_gen_recover(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* x, const double* z, const double* w,
                       const double* s, const double* dx, const double* rxz, const double* ru, const double* rws,
                       double* dz, double* dw, double* ds);
int launch_gen_ratio(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* x, const double* z, const double* w,
                     const double* s, double* dx, double* dz, double* dw, double* ds, const double* dx1,
                     const double* dx2, const double* dz1, const double* dz2, const double* dw1, const double* dw2,
                     const double* ds1, const double* ds2, int counter_slot);
int launch_gen_ru(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* ub, const double* x, const double* w,
                  double* ru);
int launch_gen_init_stats(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* ub, double* x, double* z, double* w,
                          double* s, double* st);
int launch_gen_init_apply(nys_ctx* ctx, int64_t n, const int8_t* vt, double* x, double* z, double* w, double* s,
                          double dpt, double ddt);
int launch_gen_half_u(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* ub, double scale, double* v);
int launch_gen_check(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* ub, unsigned long long* bad);
int launch_pcg_update(nys_ctx* ctx, int init, int64_t m, double* x, double* r, const double* rhs, const double* p,
                      const double* w, const FusedPartials* fp, double delta, const double* e, const double* U,
                      int64_t ldu, int ell, const double* s, double* h, int max_iter,
                      unsigned long long cond = 0ull, bool delta_slot = false, bool ext_prec = false);
// U (m x ell, column-major, ld ldu) -> Ut row-major (row stride ell): the layout the graph-path PCG
// kernels read (contiguous rows)
int launch_transpose_u(nys_ctx* ctx, int64_t m, int ell, const double* U, int64_t ldu, double* Ut);
// k_chol.cu — partial Cholesky preconditioner (Chol-IP-PMM)
struct CholFactors {
  int64_t m = 0;
  int ell = 0;
  int64_t* piv = nullptr;   // ell pivots, value-descending
  int* pivpos = nullptr;    // m: position in piv, -1 off the pivots
  double* Rinv = nullptr;   // ell x ell upper, ld ldr: R^{-1} with R^T R = N11
  int ldr = 0;
  double* Zt = nullptr;     // m x ell ROW-major: rows P = L11 = R^T, rows Q = L21
  double* dS = nullptr;     // m: diag(S) on Q, 0 on P
  double* diag = nullptr;   // m: diag(N_delta)
};
int launch_topl_select(nys_ctx* ctx, const double* v, int64_t m, int ell, int64_t* piv, int* pivpos);
int launch_selection(nys_ctx* ctx, int64_t m, int ell, const int64_t* piv, double* Om, int64_t ldo);
int launch_pivot_block(nys_ctx* ctx, double* Y, int64_t ldy, const int64_t* piv, int ell, double delta, double* N11);
int launch_chol_ds(nys_ctx* ctx, int64_t m, int ell, const double* Zt, const double* dg, const int* pivpos, double* dS);
int launch_chol_apply(nys_ctx* ctx, const CholFactors& F, const double* v, double* out, int pcg, int init);
int launch_pcg_precond(nys_ctx* ctx, int init, int64_t m, const double* r, double* z, const double* U, int64_t ldu,
                       int ell, const double* h);
int launch_prec_coef(nys_ctx* ctx, const double* lam, int ell, double mu, double* s);
int launch_pcg_setup(nys_ctx* ctx, int mode, double tol_abs, double c, double floor_, int xi_slot, int b_slot,
                     int mu_slot, double init_rel);
int launch_scaling(nys_ctx* ctx, int64_t n, const double* q, const double* x, const double* z, double rho, double* d);
int launch_pred_rhs_n(nys_ctx* ctx, int64_t n, const double* x, const double* z, const double* zeta, const double* rD,
                      double rho, const double* d, double* rd, double* rxz, double* xiau, double* t);
int launch_pred_rhs_m(nys_ctx* ctx, int64_t m, const double* b, const double* ax, const double* y, const double* lam,
                      double delta, double* rp);
int launch_corr_rhs(nys_ctx* ctx, int64_t n, const double* x, const double* dxp, const double* dzp, const double* d,
                    double* rxz, double* xiau, double* t);
int launch_pcg_latch(nys_ctx* ctx, int slot);
int launch_flag_max(nys_ctx* ctx, int dst, int src);
int launch_update_n(nys_ctx* ctx, int64_t n, double* x, const double* dx, double* z, const double* dz);
int launch_update_m(nys_ctx* ctx, int64_t m, double* y, const double* dy1, const double* dy2);
int launch_axpby(nys_ctx* ctx, int64_t n, double a, const double* u, double b, const double* v, double* out);
int launch_mul(nys_ctx* ctx, int64_t n, const double* u, const double* v, double* out);
int launch_cpqx(nys_ctx* ctx, int64_t n, const double* c, const double* q, const double* x, double* t);
int launch_shift(nys_ctx* ctx, int64_t n, double* u, double s);
int launch_minsum(nys_ctx* ctx, int64_t n, const double* u, double shift, int min_slot, int sum_slot, int counter_slot);
int launch_svm_expand(nys_ctx* ctx, int64_t nd, int64_t r0, int64_t mr, const double* g, const double* y, double* atv);
int launch_svm_fold(nys_ctx* ctx, int64_t nd, int64_t m, int64_t r0, int64_t mr, const double* u, const double* add,
                    double* uw, double* addm);
int launch_svm_scaling_fold(nys_ctx* ctx, int64_t nd, int64_t m, int64_t r0, int64_t mr, const double* d, double* dw,
                            double* e);
int launch_epi_rd(nys_ctx* ctx, int64_t n, const double* c, const double* q, const double* x, const double* atv,
                  const double* z, double* out);
int launch_epi_dx(nys_ctx* ctx, int64_t n, const double* atv, const double* rd, const double* xiau, const double* rxz,
                  const double* z, const double* x, const double* d, double* dx, double* dz);
int launch_check_pos(nys_ctx* ctx, int64_t n, const double* d, unsigned long long* bad);
int launch_set_slots(nys_ctx* ctx, int k0, double v0, int k1 = -1, double v1 = 0, int k2 = -1, double v2 = 0);

// k_pcg.cu — persistent cooperative PCG (single GPU, m <= 8192)
bool pcg_small_supported(nys_ctx* ctx, int64_t m, int64_t n, int ell);
int launch_pcg_small(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d, const double* e,
                     const double* U, int64_t ldu, int ell, const double* s, const double* rhs, double* x, int max_iter);
// m > 8192 on one GPU: the persistent cluster PCG (k_pcgc.cu), dispatched by launch_pcg_persistent
bool pcg_cluster_supported(nys_ctx* ctx, int64_t m, int64_t n, int ell);
int launch_pcg_cluster(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d,
                       const double* e, const double* U, int64_t ldu, int ell, const double* s, const double* rhs,
                       double* x, int max_iter);
bool pcg_persistent_supported(nys_ctx* ctx, int64_t m, int64_t n, int ell);
int launch_pcg_persistent(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d,
                          const double* e, const double* U, int64_t ldu, int ell, const double* s, const double* rhs,
                          double* x, int max_iter);

// k_gemm.cu — fp64 DMMA GEMM  C(MxN, col-major) = Aop(MxK) * Bop(KxN)
//   a_kmajor = true : Aop(i,k) = A[i*lda + k]      (e.g. A^T of a column-major matrix)
//   a_kmajor = false: Aop(i,k) = A[i + k*lda]      (column-major)
//   Bop(k,j) = B[k + j*ldb]                         (column-major, K contiguous)
//   epilogue: C = row_scale o acc (+ add_scale * addv_i * addm(i,j))
struct GemmCall {
  int64_t M = 0, N = 0, K = 0;
  const double* A = nullptr;
  int64_t lda = 0;
  bool a_kmajor = false;
  const double* B = nullptr;
  int64_t ldb = 0;
  double* C = nullptr;
  int64_t ldc = 0;
  const double* row_scale = nullptr;  // length M or null
  const double* addv = nullptr;       // C(i,j) += addv[i] * addm[i + j*ldadd]
  const double* addm = nullptr;
  int64_t ldadd = 0;
  int splits = 0;                     // 0 = auto
};
int launch_gemm(nys_ctx* ctx, const GemmCall& g);

// k_small.cu — ell x ell dense routines (single CTA) and sketch helpers
int launch_fro_nu(nys_ctx* ctx, int64_t m, int ell, const double* Y, int64_t ldy, int retry_scale_slot);
int launch_add_eomega(nys_ctx* ctx, int64_t m, int ell, const double* e, const double* Om, double* Y, int64_t ld);
int launch_ynu(nys_ctx* ctx, int64_t m, int ell, const double* Y, const double* Om, double* Ynu, int64_t ld);
int launch_chol_inv(nys_ctx* ctx, int ell, double* G, int ldg, double* Rinv, int ldr, int shift_mode);
int launch_trmm_upper(nys_ctx* ctx, int ell, int ld, const double* R1, const double* R2, double* Out);  // R1 * R2
int launch_jacobi_svd(nys_ctx* ctx, int ell, const double* R, int ldr, double* V, int ldv, double* sigma);
int launch_lambda_from_sigma(nys_ctx* ctx, int ell, const double* sigma, double* lam);
int launch_orth_err(nys_ctx* ctx, int64_t m, int ell, const double* U, int64_t ldu, int slot);
}  // namespace nys
