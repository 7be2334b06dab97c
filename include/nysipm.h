/*
 * nysipm.h — C ABI of libnysipm.so, the B200 (sm_100a) hot path of Nys-IP-PMM
 * (Chu, Udell et al., arXiv 2404.14524; PAPER.md = the paper's text, cited as P:<line>).
 *
 * Scope: the inexact Newton solve inside each IP-PMM iteration —
 * PCG on the regularised normal equations (N_k + delta_k I) dy = xi with
 * N_k = A (Q + Theta_k^{-1} + rho_k I)^{-1} A^T, preconditioned by the randomized
 * Nystrom preconditioner (Alg. 1-2) — plus the outer Nys-IP-PMM driver for the
 * primal-dual pair (P)/(D) with x >= 0 (Alg. 3-5; App. B).
 *
 * Conventions shared by every call
 *   - All arithmetic is IEEE fp64.  Sizes and leading dimensions are int64.
 *   - A is the caller's dense fp64 matrix, COLUMN-MAJOR, m rows x n columns, leading
 *     dimension lda >= m, lda EVEN, base pointer 16-byte aligned (the single-pass matvec
 *     streams column segments with 1-D bulk-async copies that need 16-byte alignment).
 *     m <= 138240 (= 16 x 8640: a column is split over at most a 16-CTA cluster); larger m
 *     returns NYS_EINVAL.
 *     With world > 1 each rank passes ITS column shard (m x n_local) and the m-space
 *     results are summed over ranks (A = [A_0, A_1, ...]).
 *   - Unless a call says otherwise, every pointer is a DEVICE pointer on the context's
 *     device, owned by the caller; the library never frees or retains it after the call.
 *   - Work is enqueued on the context's stream.  Calls that need a scalar decision
 *     (pcg_solve, sketch's Cholesky check, ipppmm_solve) synchronise that stream before
 *     returning; normal_matvec does not (it returns as soon as the work is enqueued).
 *   - The library owns its workspace (allocated lazily, grown monotonically, freed by
 *     nys_destroy).  No allocation happens inside the PCG loop.
 *   - Return value: NYS_OK (0) or a negative error code below; nys_strerror() names it.
 *     NYS_NOTCONV (> 0) is a warning: the result is returned and valid as an iterate.
 */
#ifndef NYSIPM_H
#define NYSIPM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NYS_OK          0
#define NYS_NOTCONV     1    /* PCG hit max_iter; info.converged = 0                */
#define NYS_EINVAL     -1    /* bad size / pointer / alignment / delta <= 0 / ell range     */
#define NYS_ENONPOS    -2    /* some d_j <= 0 or non-finite                           */
#define NYS_ECHOL      -3    /* Omega^T Y_nu not PD after nu *= 10 retries       */
#define NYS_EBREAKDOWN -4    /* PCG: p^T N p <= 0 or non-finite               */
#define NYS_EMAXITER   -5    /* IP-PMM outer iteration limit                         */
#define NYS_ECUDA      -6    /* CUDA runtime error (message via nys_last_error)              */
#define NYS_ENCCL      -7    /* NCCL error                                                   */
#define NYS_ENOMEM     -8    /* device allocation failed                                     */

typedef struct nys_ctx nys_ctx;

/* Create a context bound to `device` and `cuda_stream` (a cudaStream_t; NULL -> the library
 * creates and owns a non-blocking stream).  nccl_unique_id: NULL for a single GPU, else a
 * pointer to the 128-byte ncclUniqueId shared by all `world` ranks (rank in [0, world)).
 * world = 1 with a non-NULL id creates a ONE-rank NCCL communicator and every call takes the
 * multi-rank path (local partials, ncclAllReduce, replicated terms): validation of the NCCL
 * plumbing on a single GPU.  NCCL (libnccl.so.2) is loaded with dlopen only when an id is given. */
int nys_create(nys_ctx** out, int device, void* cuda_stream,
               const void* nccl_unique_id, int rank, int world);
int nys_destroy(nys_ctx* ctx);
/* Fill out128 (128 bytes) with a fresh ncclUniqueId (rank 0 calls this and broadcasts it
 * through the caller's own channel, e.g. torch.distributed).  dlopens libnccl.so.2. */
int nys_nccl_unique_id(void* out128);

/* ---------------------------------------------------------------------------------------
 * nys_partial_cholesky — the partial Cholesky preconditioner of Chol-IP-PMM (SURVEY
 * §8(f) f2) for N_delta = A diag(d) A^T + diag(e) + delta I (summed over ranks), rank ell:
 *   piv (device, ell int64, may be NULL): the pivots = indices of the ell largest diagonal entries of
 *       N_delta (reading C1: original diagonal, ties -> smaller index), value-descending;
 *   L   (device, m x ell column-major, ld m, may be NULL): rows piv = L11 (lower Cholesky factor of
 *       N_delta[piv, piv], pivot order), other rows = L21 = N_delta[Q, piv] L11^{-T};
 *   dS  (device, m, may be NULL): diag(S) of the Schur complement on the non-pivot rows, 0 on piv.
 * The factors are also kept in the context for nys_chol_precond_apply.  NYS_ECHOL if N_delta[piv,piv]
 * is not positive definite.  Synchronises the stream. */
int nys_partial_cholesky(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d,
                         const double* e, double delta, int ell, int64_t* piv, double* L, double* dS);
/* out = P_Chol^{-1} v (eq. P:309-322) with the factors of the last nys_partial_cholesky call on this
 * context (m must match).  v, out: device m-vectors. */
int nys_chol_precond_apply(nys_ctx* ctx, int64_t m, const double* v, double* out);

/* In-process LOOPBACK communicator for `world` ranks on ONE device (validation of the multi-rank
 * path where a single GPU is available).  Fills the 128-byte id that nys_create takes in place of
 * an NCCL unique id; each rank is then driven by its own host thread.  All-reduces synchronise the
 * rank's stream, meet at a host barrier and sum the ranks' device buffers in rank order (bitwise
 * identical on every rank); no kernel waits on another rank.  Destroy after every context using it
 * has been destroyed.  2 <= world <= 16.  Returns NYS_EINVAL on bad arguments. */
int nys_loopback_comm_create(int world, void* out128);
int nys_loopback_comm_destroy(void* id128);
const char* nys_strerror(int code);
/* Last detailed error message of this context (CUDA/NCCL string, offending index...). */
const char* nys_last_error(nys_ctx* ctx);

/* ---------------------------------------------------------------------------------------
 * nys_normal_matvec — w = sum_ranks A diag(d) A^T v + e o v + delta v
 *   The regularised normal-equation operator of IP-PMM applied to one vector, in ONE pass
 *   over A: t = d o (A^T v) and A t are computed from the same on-chip column panel.
 *   m, n, A, lda : see conventions (n = local column count on this rank)
 *   d            : n-vector, d_j = 1/(q_j + z_j/x_j + rho) > 0  (not checked here; see
 *                  nys_check_scaling)
 *   e            : m-vector diagonal term (unit columns of A) or NULL
 *   delta        : >= 0
 *   v            : m-vector (replicated over ranks);  w : m-vector out (may not alias v)
 *   Errors: NYS_EINVAL on bad sizes/alignment; NYS_ECUDA / NYS_ENCCL.
 * ------------------------------------------------------------------------------------- */
int nys_normal_matvec(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda,
                      const double* d, const double* e, double delta,
                      const double* v, double* w);

/* Validate a scaling vector: returns NYS_ENONPOS and stores the first offending index in
 * *bad_index (or -1) if some d_j <= 0 or non-finite.  Synchronises. */
int nys_check_scaling(nys_ctx* ctx, int64_t n, const double* d, int64_t* bad_index);

typedef struct {
  double nu;             /* final shift nu of Alg. 1 line 3 (after retries)              */
  int    chol_retries;   /* number of nu <- 10 nu retries                     */
  double orth_err;       /* ||U^T U - I||_F of the returned U                             */
  double t_ms;           /* device time of the whole call                                  */
  int    jacobi_sweeps;  /* sweeps of the ell x ell one-sided Jacobi SVD                   */
} nys_sketch_info;

/* ---------------------------------------------------------------------------------------
 * nys_sketch — randomized Nystrom approximation N_hat = U diag(lambda) U^T of
 *   N = A diag(d) A^T (+ diag(e))   — Alg. 1; delta is NOT added to the sketch
 *   (SURVEY A1), it is only validated (> 0) since Alg. 2 pairs it with the factors.
 *   Omega  : m x ell column-major Gaussian test matrix (ld = m), identical on all ranks
 *   U      : m x ell column-major out (ld = m), orthonormal columns
 *   lambda : ell out, descending, >= 0  (lambda_hat = max{0, Sigma^2 - nu})
 *   info   : may be NULL
 *   Steps: Y = A(d o (A^T Omega)) (+ e o Omega) [fp64 DMMA GEMMs, allreduce over ranks];
 *   nu = eps(||Y||_F); Y_nu = Y + nu Omega; C = chol(Omega^T Y_nu); B = Y_nu C^{-1};
 *   thin SVD of B by shifted CholeskyQR3 + one-sided Jacobi on the ell x ell factor.
 *   Errors: NYS_EINVAL (ell < 1, ell > m, ell > 1024, delta <= 0), NYS_ECHOL.
 * ------------------------------------------------------------------------------------- */
int nys_sketch(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda,
               const double* d, const double* e, double delta, int ell,
               const double* Omega, double* U, double* lambda, nys_sketch_info* info);

/* ---------------------------------------------------------------------------------------
 * nys_sketch_apply — the sketch step of Alg. 1 on its own (line 2):
 *   Y = A diag(d) A^T Omega (+ e o Omega), summed over ranks; delta is not added (A1).
 *   Omega, Y : m x ell column-major (ld = m).  Two fp64 DMMA GEMMs (T = d o A^T Omega, Y = A T).
 * ------------------------------------------------------------------------------------- */
int nys_sketch_apply(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda,
                     const double* d, const double* e, int ell, const double* Omega, double* Y);

/* Fill Omega (m x ell, column-major, ld = m) with the counter-based Gaussian test matrix of
 * Philox4x32-10 keyed by seed, counter = (pair index, stream), Box-Muller. */
int nys_gaussian(nys_ctx* ctx, int64_t m, int ell, uint64_t seed, uint64_t stream, double* Omega);

typedef struct {
  int    iters;          /* PCG iterations (operator applications in the loop)            */
  int    converged;      /* 1 iff ||r|| <= tol_abs                                         */
  double res_norm;       /* recursive residual norm at exit                                */
  double true_res_norm;  /* ||rhs - (N + delta I) x|| recomputed at exit                   */
  double t_ms;           /* device time of the call                                        */
} nys_pcg_info;

/* ---------------------------------------------------------------------------------------
 * nys_pcg_solve — PCG on (A diag(d) A^T + e + delta I) x = rhs with the Nystrom
 *   preconditioner P^{-1} = (lam_l + mu) U (Lam + mu I)^{-1} U^T + (I - U U^T)
 *   ell      : 0 -> no preconditioner (CG-IP-PMM); else U (m x ell, ld = m) and
 *              lambda (ell, descending) from nys_sketch
 *   mu_prec  : the preconditioner shift, = delta_k in Nys-IP-PMM
 *   rhs      : m-vector;  x : m-vector out (zero initial guess)
 *   tol_abs  : stop when the recursive residual ||r||_2 <= tol_abs
 *   max_iter : iteration cap; on exhaustion returns NYS_NOTCONV with x valid
 *   Errors: NYS_EBREAKDOWN, NYS_EINVAL.
 * ------------------------------------------------------------------------------------- */
int nys_pcg_solve(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda,
                  const double* d, const double* e, double delta,
                  int ell, const double* U, const double* lambda, double mu_prec,
                  const double* rhs, double* x, double tol_abs, int max_iter,
                  nys_pcg_info* info);

/* ---------------------------------------------------------------------------------------
 * nys_ipppmm_solve — Nys-IP-PMM (Alg. 3) for
 *     (P) min 1/2 x^T diag(q) x + c^T x  s.t.  A x = b, x >= 0
 *   with Mehrotra predictor-corrector (Alg. 5), Newton system via normal equations (Alg. 4),
 *   initial point (App. B.2), stepsizes (App. B.3); PEU / TC readings of SURVEY §8(c)
 *   A11-A12.  The preconditioner is rebuilt every outer iteration from a fresh
 *   Omega_k (Philox, stream k+1; the initial point uses stream 0).
 * ------------------------------------------------------------------------------------- */
typedef struct nys_unit_block {
  int64_t row0;          /* row of the block's first column                                 */
  int64_t count;         /* columns in the block (rows row0 .. row0 + count - 1)           */
  double  scale;         /* nonzero entry of every column (e.g. +1, -1)                     */
} nys_unit_block;

typedef struct {
  int64_t m, n;          /* rows; LOCAL column count on this rank                          */
  const double* A;       /* m x n column-major, lda (see conventions)                      */
  int64_t lda;
  const double* q;       /* n (local), diag(Q) >= 0                                        */
  const double* b;       /* m (replicated)                                                 */
  const double* c;       /* n (local)                                                      */
  int host_ptrs;         /* 1: A, q, b, c are HOST pointers (copied in by the library)     */
  int structure;         /* 0: A is dense m x n.  1: SVM-shaped (BASELINE configs[2], SURVEY
                            A23): A = [Xt, -Xt, I_m, -I_m] with the dense block Xt (m x nd,
                            column-major, lda) passed in `A`; n = 2 nd + 2 m variables ordered
                            [w+, w-, xi, s].  The identity blocks are never materialised: they
                            contribute the diagonal term e = d_xi + d_s of the normal operator.
                            Multi-rank: each rank passes its feature columns Xt_g (nd_g) and owns
                            the xi / s variables of ONE row range, given as a single unit block
                            (row0, count, scale = 1) in unit_blocks; then n = 2 nd + 2 count,
                            variables [w+_g, w-_g, xi_rows, s_rows], and the row ranges of the
                            ranks partition [0, m).  No unit block: the whole range [0, m).
                            2: dense block + scaled identity blocks (below).                    */
  int64_t nd;            /* structure 1 / 2: number of dense columns stored in `A`          */
  /* Free and box-constrained variables, problem (P~)/(D~) (Alg. 5; SURVEY
   * §8(f) f1).  vtype == NULL: every variable is in I (x >= 0), the form (P)/(D).  Otherwise
   * vtype[j] (n local entries, int8) is 0 for j in I (x_j >= 0), 1 for j in F (free), 2 for j in J
   * (0 <= x_j <= ub[j]); ub (n local doubles) is read on J only and may be NULL when no entry is 2.
   * Same memory space as A (host_ptrs).  Works with every `structure`.  With every variable free
   * the duality measure is identically 0 and the method reduces to the proximal method of
   * multipliers on the equality-constrained QP (reading G5).                          */
  const int8_t* vtype;
  const double* ub;
  /* structure 2: A = [B, S_0, ..., S_{K-1}] with the dense block B (m x nd, column-major, lda) in
   * `A` and K <= 8 scaled identity blocks S_k = scale_k [e_{row0_k}, ..., e_{row0_k + count_k - 1}]
   * (never materialised); variables ordered [B columns, S_0 columns, S_1 columns, ...], so
   * n = nd + sum_k count_k (this rank's local columns; each rank passes its own blocks).  The blocks
   * contribute the diagonal term e_i = sum_k scale_k^2 d_j of the normal operator and the
   * elementwise parts of A u and A^T y.  This is the shape of the paper's own QP formulations:
   * dual SVM A = [I_d, -X diag(y); 0, y^T] (App. C.2: dense block [-X diag(y); y^T],
   * one identity block) and the factor-model portfolio (App. C.1: identity blocks for
   * the free factor variables and the slacks).  unit_blocks is a HOST array.                    */
  int n_unit_blocks;
  const struct nys_unit_block* unit_blocks;
} nys_qp;

typedef struct {
  double tol;            /* 1e-8                                                   */
  int    ell;            /* fixed sketch size; 0 = CG-IP-PMM                        */
  uint64_t seed;         /* Omega seed                                                      */
  int    max_outer;      /* 100                                                            */
  int    pcg_max_iter;   /* 20000 (SURVEY A10')                                             */
  double rho0, delta0;   /* 8, 8                                                    */
  double reg_floor;      /* 5e-10 (Tables 5-6)                                              */
  double pcg_c;          /* 1e-3  (A8': tau = max(floor(1+|b|), min(0.1|xi|, c mu (1+|b|))))*/
  double pcg_floor;      /* 1e-10                                                          */
  double init_delta;     /* 10                                                     */
  double init_tol_rel;   /* 1e-12 (A14'')                                                  */
  int    verbose;        /* 1: print one line per outer iteration to stderr                */
  /* Preconditioner reuse (the paper's future work, "reusing the
   * preconditioner between iterations").  The Nystrom factors (U, lambda) are rebuilt at outer
   * iteration k when k - k_last >= prec_refresh, or (prec_growth > 0) when the previous outer
   * iteration's PCG count (predictor + corrector) exceeded prec_growth x the count of the iteration
   * that followed the last rebuild.  Between rebuilds only mu_prec = delta_k is updated.
   * prec_refresh = 1, prec_growth = 0 is Alg. 3 as written (a fresh sketch every iteration).      */
  int    prec_refresh;   /* 1                                                              */
  double prec_growth;    /* 0 (off)                                                         */
  /* 0: randomized Nystrom P^{-1} (Nys-IP-PMM).  1: the partial Cholesky preconditioner of rank
   * ell (Chol-IP-PMM, the paper's comparison arm), built every outer
   * iteration from diag(N_delta): pivots = the ell largest diagonal entries (reading C1).       */
  int    precond;        /* 0                                                              */
  /* Adaptive Nystrom rank (the paper's future work "tuning the rank", P:1102;
   * reading F1): when ell_max > ell, after a build with rank ell_k whose lambda_hat_ell exceeds
   * ell_tau * delta_k (mu_prec, A7) the next build (forced at the next outer iteration) uses
   * min(2 ell_k, ell_max, m, 1024).  The rank never shrinks.  0 = fixed rank.                   */
  int    ell_max;        /* 0                                                              */
  double ell_tau;        /* 10                                                             */
} nys_options;

/* Fill *opt with the defaults above. */
void nys_default_options(nys_options* opt);

typedef struct {
  int    k;              /* outer iteration                                                */
  double mu, rel_p, rel_d;
  double alpha_p, alpha_d;
  int    pcg_pred, pcg_corr;
  double rho, delta;     /* parameters used in this iteration                              */
  double t_sketch_ms, t_pcg_ms, t_other_ms;
  int    prec_built;     /* 1: the Nystrom preconditioner was (re)built this iteration     */
  int    ell;            /* rank of the preconditioner used in this iteration              */
  double lam_ell;        /* its lambda_hat_ell (0 when ell = 0 or partial Cholesky)         */
} nys_iter_record;

typedef struct {
  double* x;             /* n (local) out — device pointer, or host if qp.host_ptrs        */
  double* y;             /* m out                                                          */
  double* z;             /* n (local) out                                                  */
  double obj;            /* 1/2 x^T Q x + c^T x  (summed over ranks)                       */
  double dual_obj;       /* b^T y - 1/2 x^T Q x  (- u_J^T s_J with box variables)           */
  double* w;             /* n (local) out or NULL: the upper-bound slack (0 off J)          */
  double* s;             /* n (local) out or NULL: the upper-bound dual (0 off J)           */
} nys_solution;

typedef struct {
  int    status;         /* NYS_OK (optimal), NYS_EMAXITER, or an error code               */
  int    outer_iters;
  int    inner_iters;    /* total PCG iterations incl. the initial point                  */
  double rel_p, rel_d, mu;
  double t_total_ms, t_sketch_ms, t_pcg_ms, t_other_ms;
  int    n_records;      /* records written (<= max_records)                              */
  int    max_records;    /* capacity of `records` (caller-owned host array, may be 0)      */
  nys_iter_record* records;
  int64_t matvecs;       /* fused normal matvecs launched                                  */
  int64_t kernel_launches; /* library kernel launches during the call                    */
} nys_report;

int nys_ipppmm_solve(nys_ctx* ctx, const nys_qp* qp, const nys_options* opt,
                     nys_solution* sol, nys_report* rep);

/* Accounting of library kernel launches since context creation (bench "gpu_launches"). */
int64_t nys_kernel_launches(nys_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* NYSIPM_H */
