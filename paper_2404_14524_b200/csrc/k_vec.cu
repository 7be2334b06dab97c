// Vector kernels of the hot path: PCG updates with the fused Nystrom preconditioner apply,
// IPM elementwise work of Alg. 4 / Alg. 5, deterministic reductions, the Gaussian test
// matrix generator.  All reductions are two-level (block partials + last-block sum in a
// fixed order) so results are bitwise reproducible run to run.
#include "k_vec.cuh"

namespace nys {

// ------------------------------------------------------------------------------------------
// Philox4x32-10 + Box-Muller (Salmon et al. SC'11).  Same published generator as
// the oracle's numpy implementation (no shared code).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                             uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
  const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
  const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
  c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
}

__global__ void gaussian_kernel(double* __restrict__ O, int64_t total, uint64_t seed, uint64_t stream,
                                const double* kslot) {
  if (kslot != nullptr) stream = (uint64_t)(*kslot) + 1u;   // graph-resident loop: stream k + 1 (A6)
  const int64_t npairs = (total + 1) >> 1;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs; p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c0 = (uint32_t)p, c1 = (uint32_t)((uint64_t)p >> 32), c2 = (uint32_t)stream, c3 = (uint32_t)(stream >> 32);
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
      philox_round(c0, c1, c2, c3, k0, k1);
    }
    const uint64_t a = ((((uint64_t)c0) << 32) | c1) >> 11;
    const uint64_t b = ((((uint64_t)c2) << 32) | c3) >> 11;
    const double u1 = ((double)a + 0.5) * 0x1p-53;
    const double u2 = (double)b * 0x1p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double th = 2.0 * 3.141592653589793 * u2;
    const int64_t L = 2 * p;
    O[L] = r * cos(th);
    if (L + 1 < total) O[L + 1] = r * sin(th);
  }
}

int launch_gaussian(nys_ctx* ctx, double* O, int64_t total, uint64_t seed, uint64_t stream) {
  if (total <= 0) return NYS_OK;
  int64_t npairs = (total + 1) / 2;
  int grid = (int)((npairs + 255) / 256);
  if (grid > 8 * ctx->num_sms) grid = 8 * ctx->num_sms;
  gaussian_kernel<<<grid, 256, 0, ctx->stream>>>(O, total, seed, stream, ctx->gloop ? ctx->sc + S_KOUT : nullptr);
  ctx->launches++;
  return ctx->check_launch("gaussian");
}

// ------------------------------------------------------------------------------------------
// dots: out_slot[k] = sum_i a_k[i] * b_k[i]   (b_k == nullptr -> a_k[i]^2), k < 4
// optional affine pre-map: a_k[i] + alpha_k * da_k[i]  (for mu_aff)
// ------------------------------------------------------------------------------------------
struct DotArgs {
  int nv;
  int64_t n;
  const double* a[4];
  const double* b[4];
  const double* da[4];
  const double* db[4];
  int sa[4], sb[4];   // slot indices of the step lengths for da / db (-1 = none)
  int out[4];
  double* sc;
  double* part;
  unsigned int* counter;
  int post;           // post-processing of the slots on the last block
  double post_a;
};

enum DotPost { DP_NONE = 0, DP_MUAFF = 1 };

__global__ void __launch_bounds__(256) dots_kernel(const DotArgs D) {
  double v[4] = {0, 0, 0, 0};
  double al[4], bl[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    al[k] = (k < D.nv && D.sa[k] >= 0) ? D.sc[D.sa[k]] : 0.0;
    bl[k] = (k < D.nv && D.sb[k] >= 0) ? D.sc[D.sb[k]] : 0.0;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < D.n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < D.nv) {
        double x = D.a[k][i];
        if (D.da[k]) x += al[k] * D.da[k][i];
        double y = x;
        if (D.b[k]) {
          y = D.b[k][i];
          if (D.db[k]) y += bl[k] * D.db[k][i];
        }
        v[k] = fma(x, y, v[k]);
      }
    }
  }
  block_sum_to_part<4>(v, D.part, gridDim.x);
  if (last_block_arrive(D.counter)) {
    const int wk = warp_uniform_id();
    if (wk < D.nv) {
      const double v0 = warp_sum_array(D.part + (size_t)wk * gridDim.x, gridDim.x);
      if ((threadIdx.x & 31) == 0) D.sc[D.out[wk]] = v0;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    *D.counter = 0u;
    if (D.post == DP_MUAFF) {
      // mu_aff = (x + ap dx)^T (z + ad dz) / n_total ; mu~ = mu_aff^3 / mu^2
      const double muaff = D.post_a > 0 ? (D.sc[D.out[0]] + (D.nv > 1 ? D.sc[D.out[1]] : 0.0)) / D.post_a : 0.0;
      const double mu = D.sc[S_MUCUR];
      D.sc[S_MUAFF] = muaff;
      D.sc[S_MUT] = muaff * muaff * muaff / (mu * mu);
    }
  }
}

static int reduce_grid(nys_ctx* ctx, int64_t n) {
  // one 256-row tile per block while that stays under two blocks per SM (the reductions are
  // latency-bound at the IPM's n: more blocks in flight, one element per thread)
  int g = (int)((n + 255) / 256);
  if (const char* e = getenv("NYS_REDUCE_ROWS")) g = (int)((n + atoi(e) - 1) / atoi(e));
  if (g < 1) g = 1;
  if (g > 2 * ctx->num_sms) g = 2 * ctx->num_sms;
  return g;
}

int launch_dots(nys_ctx* ctx, int64_t n, int nv, const double* const* a, const double* const* b, const int* out,
                int counter_slot) {
  DotArgs D{};
  D.nv = nv; D.n = n;
  for (int k = 0; k < 4; ++k) { D.sa[k] = -1; D.sb[k] = -1; }
  for (int k = 0; k < nv; ++k) { D.a[k] = a[k]; D.b[k] = b ? b[k] : nullptr; D.out[k] = out[k]; }
  D.sc = ctx->sc;
  const int g = reduce_grid(ctx, n);
  D.part = ctx->wsd("dot_part", (size_t)4 * g);
  D.counter = ctx->counters + counter_slot;
  D.post = DP_NONE;
  dots_kernel<<<g, 256, 0, ctx->stream>>>(D);
  ctx->launches++;
  return ctx->check_launch("dots");
}

int launch_muaff(nys_ctx* ctx, int64_t n, const double* x, const double* dx, const double* z, const double* dz,
                 double n_total, int counter_slot, const double* w, const double* dw, const double* s,
                 const double* ds) {
  DotArgs D{};
  D.nv = w ? 2 : 1; D.n = n;
  for (int k = 0; k < 4; ++k) { D.sa[k] = -1; D.sb[k] = -1; }
  D.a[0] = x; D.da[0] = dx; D.sa[0] = S_AP;
  D.b[0] = z; D.db[0] = dz; D.sb[0] = S_AD;
  D.out[0] = S_TMP7;
  if (w) {  // general form (f1): + (w + ap dw)^T (s + ad ds) on J (w, s, dw, ds are 0 off J)
    D.a[1] = w; D.da[1] = dw; D.sa[1] = S_AP;
    D.b[1] = s; D.db[1] = ds; D.sb[1] = S_AD;
    D.out[1] = S_TMP6;
  }
  D.sc = ctx->sc;
  const int g = reduce_grid(ctx, n);
  D.part = ctx->wsd("dot_part", (size_t)4 * g);
  D.counter = ctx->counters + counter_slot;
  D.post = ctx->multi() ? DP_NONE : DP_MUAFF;
  D.post_a = n_total;
  dots_kernel<<<g, 256, 0, ctx->stream>>>(D);
  ctx->launches++;
  return ctx->check_launch("muaff");
}

__global__ void muaff_post_kernel(double* sc, double n_total, int gen) {
  const double muaff = n_total > 0 ? (sc[S_TMP7] + (gen ? sc[S_TMP6] : 0.0)) / n_total : 0.0;
  const double mu = sc[S_MUCUR];
  sc[S_MUAFF] = muaff;
  sc[S_MUT] = muaff * muaff * muaff / (mu * mu);
}
int launch_muaff_post(nys_ctx* ctx, double n_total, int gen) {
  muaff_post_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sc, n_total, gen);
  ctx->launches++;
  return ctx->check_launch("muaff_post");
}

// ------------------------------------------------------------------------------------------
// ratio test: min over dv_i < 0 of -v_i / dv_i for two pairs -> raw minima in
// slots (S_TMP0, S_TMP1); alpha = 0.995 min(1, .) applied by steps_post (after a possible
// cross-rank min).  Optionally forms dv = dv1 + dv2 on the fly and stores it.
// ------------------------------------------------------------------------------------------
struct RatioArgs {
  int64_t n;
  const double* x;
  double* dx;
  const double* dx1;
  const double* dx2;
  const double* z;
  double* dz;
  const double* dz1;
  const double* dz2;
  double* sc;
  double* part;
  unsigned int* counter;
};

__global__ void __launch_bounds__(256) ratio_kernel(const RatioArgs R) {
  double mp = 1.0e300, md = 1.0e300;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R.n; i += (int64_t)gridDim.x * blockDim.x) {
    double dx, dz;
    if (R.dx1) { dx = R.dx1[i] + R.dx2[i]; R.dx[i] = dx; } else dx = R.dx[i];
    if (R.dz1) { dz = R.dz1[i] + R.dz2[i]; R.dz[i] = dz; } else dz = R.dz[i];
    if (dx < 0.0) mp = fmin(mp, -R.x[i] / dx);
    if (dz < 0.0) md = fmin(md, -R.z[i] / dz);
  }
  __shared__ double sh[2][32];
  mp = warp_min(mp);
  md = warp_min(md);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sh[0][w] = mp; sh[1][w] = md; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 1.0e300, b = 1.0e300;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { a = fmin(a, sh[0][i]); b = fmin(b, sh[1][i]); }
    R.part[blockIdx.x] = a;
    R.part[gridDim.x + blockIdx.x] = b;
  }
  if (last_block_arrive(R.counter) && warp_uniform_id() == 0) {
    const double a = warp_min_array(R.part, gridDim.x);
    const double b = warp_min_array(R.part + gridDim.x, gridDim.x);
    if (threadIdx.x != 0) return;
    *R.counter = 0u;
    R.sc[S_TMP0] = a;
    R.sc[S_TMP1] = b;
  }
}

__global__ void steps_post_kernel(double* sc) {
  sc[S_AP] = 0.995 * fmin(1.0, sc[S_TMP0]);
  sc[S_AD] = 0.995 * fmin(1.0, sc[S_TMP1]);
}

int launch_ratio(nys_ctx* ctx, int64_t n, const double* x, double* dx, const double* dx1, const double* dx2,
                 const double* z, double* dz, const double* dz1, const double* dz2, int counter_slot) {
  RatioArgs R{};
  R.n = n; R.x = x; R.dx = dx; R.dx1 = dx1; R.dx2 = dx2; R.z = z; R.dz = dz; R.dz1 = dz1; R.dz2 = dz2;
  R.sc = ctx->sc;
  const int g = reduce_grid(ctx, n);
  R.part = ctx->wsd("ratio_part", (size_t)2 * g);
  R.counter = ctx->counters + counter_slot;
  ratio_kernel<<<g, 256, 0, ctx->stream>>>(R);
  ctx->launches++;
  return ctx->check_launch("ratio");
}
int launch_steps_post(nys_ctx* ctx) {
  steps_post_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sc);
  ctx->launches++;
  return ctx->check_launch("steps_post");
}

// ------------------------------------------------------------------------------------------
// PCG kernels.  Rows are processed in chunks of 64 (a block owns `nsub` consecutive chunks).
// ------------------------------------------------------------------------------------------
// update:  alpha = rz / p^T w  (p^T w from the matvec's per-CTA partials, summed identically by
//          every block) ; w_i = sum_c Wp[c][i] + (delta + e_i) p_i  (or given) ;
//          x += alpha p ; r -= alpha w  |  (init) x = 0, r = rhs ;
//          rr = r^T r ; g = U^T r ; last block: convergence test, h = s o g  (P^{-1} coefficients)
struct PcgUpdArgs {
  unsigned long long cond;  // cudaGraphConditionalHandle of the enclosing WHILE node (0 = none)
  int init;
  int64_t m;
  double* x;
  double* r;
  const double* rhs;
  const double* p;
  const double* w;      // given w (multi-GPU path) or null
  const double* Wp;     // fused partials (world == 1)
  int64_t wp_ld;
  int nparts;
  const double* pwp;
  int npw;
  double delta;
  int delta_slot;       // 1: delta = sc[S_DELTA]
  const double* e;
  const double* U;
  int64_t ldu;
  int ell;
  const double* s;
  double* h;
  double* sc;
  double* part;         // (1 + ell) x grid
  unsigned int* counter;
  int max_iter;
  int64_t rows_per_block;
  int ext_prec;         // 1: an external preconditioner (partial Cholesky) sets rz / beta
};

// Row-parallel update: a block owns `rows_per_block` consecutive rows, one row per thread per
// 256-row tile (no serial 16-row chunks).  w_i sums the matvec's partial rows with independent
// L2 loads; U^T r partials: for every column a warp reduces its 32 rows with shuffles and
// accumulates in its own shared-memory row (tile after tile), then the 8 warp rows are summed in
// a fixed order -> one (1 + ell)-row of block partials.  pcg_hred_kernel (one block per column)
// finishes the reduction: rr, the convergence test, h = s o (U^T r).
// BIG (ell > 256, up to 1024): the per-warp rows of U^T r partials live in dynamic shared memory and the
// U^T r pass runs over column chunks of 256 (lane L of a warp covers chunk columns L, L + 32, ...)
template <bool BIG>
__global__ void __launch_bounds__(256) pcg_update_kernel(const PcgUpdArgs A) {
  if (A.cond != 0ull && blockIdx.x == 0 && threadIdx.x == 0) A.sc[S_GITER] += 1.0;  // launch accounting
  if (A.sc[S_DONE] != 0.0) {  // converged / max_iter / breakdown: end the graph-resident loop
    if (A.cond != 0ull && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(A.cond, 0u);
    return;
  }
  const double delta = A.delta_slot ? A.sc[S_DELTA] : A.delta;
  __shared__ double wred_s[BIG ? 1 : 8 * 257];  // [warp][1 + c] : rr and U^T r partials of this block
  extern __shared__ double wred_d[];
  const int wld = BIG ? 1 + A.ell : 257;
  double* wred = BIG ? wred_d : wred_s;
  __shared__ double rsh[256];
  __shared__ double s_alpha;
  __shared__ int s_ok;
  const int tid = threadIdx.x, warp = warp_uniform_id(), lane = tid & 31;
  if (!A.init) {
    if (warp == 0) {
      double pw;
      if (A.w != nullptr) pw = A.sc[S_PW];
      else pw = warp_sum_array(A.pwp, A.npw);
      if (lane == 0) {
        const bool ok = (pw > 0.0) && isfinite(pw);
        s_ok = ok ? 1 : 0;
        s_alpha = ok ? A.sc[S_RZ] / pw : 0.0;
        if (blockIdx.x == 0) {
          A.sc[S_PW] = pw;
          A.sc[S_ALPHA] = s_alpha;
        }
      }
    }
  }
  const int ncol = 1 + A.ell;
  for (int c = lane; c < ncol; c += 32) wred[warp * wld + c] = 0.0;
  __syncthreads();
  if (!A.init && !s_ok) {
    if (blockIdx.x == 0 && tid == 0) { A.sc[S_STATUS] = (double)NYS_EBREAKDOWN; A.sc[S_DONE] = 1.0; }
    return;
  }
  const double alpha = A.init ? 0.0 : s_alpha;
  const int64_t lo = (int64_t)blockIdx.x * A.rows_per_block;
  int64_t hi = lo + A.rows_per_block;
  if (hi > A.m) hi = A.m;
  for (int64_t t0 = lo; t0 < hi; t0 += 256) {
    const int64_t i = t0 + tid;
    double ri = 0.0;
    if (i < hi) {
      if (A.init) {
        ri = A.rhs[i];
        A.x[i] = 0.0;
      } else {
        const double pi = A.p[i];
        double wi;
        if (A.w != nullptr) {
          wi = A.w[i];
        } else {
          double acc = 0.0;
          for (int c0 = 0; c0 < A.nparts; c0 += 8) {   // 8 independent L2 loads per round
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = (c0 + u < A.nparts) ? __ldcg(A.Wp + (size_t)(c0 + u) * A.wp_ld + i) : 0.0;
            acc += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
          }
          wi = acc + (delta + (A.e ? A.e[i] : 0.0)) * pi;
        }
        A.x[i] = fma(alpha, pi, A.x[i]);
        ri = fma(-alpha, wi, A.r[i]);
      }
      A.r[i] = ri;
    }
    // rr: this warp's 32 rows
    const double rrw = warp_sum(ri * ri);
    if (lane == 0) wred[warp * wld] += rrw;
    rsh[tid] = ri;  // rows past hi hold 0
    __syncthreads();
    // U^T r with U stored ROW-major (Ut[i][c], row stride ldu): warp w takes tile rows w, w+8, ...;
    // lane L accumulates columns L, L+32, ... (contiguous 256-B reads of each row, no shuffles)
    for (int c0 = 0; c0 < (BIG ? A.ell : 1); c0 += 256) {
      double gacc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) gacc[k] = 0.0;
      const int tile_rows = (int)((hi - t0) < 256 ? (hi - t0) : 256);
      for (int rr0 = warp; rr0 < tile_rows; rr0 += 32) {
        double uv[4][8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int row = rr0 + 8 * q;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int c = c0 + lane + 32 * k;
            uv[q][k] = (row < tile_rows && c < A.ell) ? A.U[(size_t)(t0 + row) * A.ldu + c] : 0.0;
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int row = rr0 + 8 * q;
          const double rv = (row < tile_rows) ? rsh[row] : 0.0;
#pragma unroll
          for (int k = 0; k < 8; ++k) gacc[k] = fma(uv[q][k], rv, gacc[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int c = c0 + lane + 32 * k;
        if (c < A.ell) wred[warp * wld + 1 + c] += gacc[k];
      }
    }
    __syncthreads();
  }
  __syncthreads();
  for (int c = tid; c < ncol; c += 256) {
    const double v = ((wred[0 * wld + c] + wred[1 * wld + c]) + (wred[2 * wld + c] + wred[3 * wld + c])) +
                     ((wred[4 * wld + c] + wred[5 * wld + c]) + (wred[6 * wld + c] + wred[7 * wld + c]));
    A.part[(size_t)c * gridDim.x + blockIdx.x] = v;
  }
}

// column c of the block partials -> rr (c = 0: convergence test, PCG bookkeeping) or h_{c-1}
__global__ void __launch_bounds__(256) pcg_hred_kernel(const PcgUpdArgs A, int G) {
  if (A.sc[S_DONE] != 0.0) return;
  __shared__ double ws[8];
  const int c = blockIdx.x, tid = threadIdx.x, warp = warp_uniform_id(), lane = tid & 31;
  const double* src = A.part + (size_t)c * G;
  double acc = 0.0;
  for (int k0 = tid; k0 < G; k0 += 1024) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (k0 + 256 * u < G) ? __ldcg(src + k0 + 256 * u) : 0.0;
    acc += (v[0] + v[1]) + (v[2] + v[3]);
  }
  acc = warp_sum(acc);
  if (lane == 0) ws[warp] = acc;
  __syncthreads();
  if (tid != 0) return;
  const double tot = ((ws[0] + ws[1]) + (ws[2] + ws[3])) + ((ws[4] + ws[5]) + (ws[6] + ws[7]));
  if (c > 0) {
    A.h[c - 1] = A.s[c - 1] * tot;
    return;
  }
  const double rrt = tot;
  A.sc[S_RR] = rrt;
  double iters = A.sc[S_ITERS];
  if (!A.init) iters += 1.0;
  A.sc[S_ITERS] = iters;
  const double tol = A.sc[S_TOL];
  int cv = (sqrt(rrt) <= tol) ? 1 : 0;
  if (!isfinite(rrt)) { A.sc[S_STATUS] = (double)NYS_EBREAKDOWN; cv = 1; }
  if (cv || iters >= (double)A.max_iter) {
    A.sc[S_DONE] = 1.0;
    if (A.cond != 0ull) cudaGraphSetConditional(A.cond, 0u);
  }
  if (A.ell == 0 && !A.ext_prec && !cv) {  // P = I: z = r, rz_new = rr
    const double rzold = A.sc[S_RZ];
    A.sc[S_BETA] = A.init ? 0.0 : rrt / rzold;
    A.sc[S_RZ] = rrt;
  }
}

struct PcgPrecArgs {
  int init;
  int64_t m;
  const double* r;
  double* z;
  const double* U;
  int64_t ldu;
  int ell;
  const double* h;
  double* sc;
  double* part;
  unsigned int* counter;
  int nsub;
};

// z = r + U h with U stored ROW-major (Ut[i][c], row stride ldu): one warp per row, lane L
// covering columns L, L+32, ... (contiguous reads), 4 rows in flight per warp, a shuffle sum per
// row; rz = r^T z partials, the last block finishes rz and beta.
// KH = columns per lane / 32: 8 for ell <= 256, 32 up to 1024 (the small variant keeps the unrolled
// loop and the register footprint of the common case)
template <int KH>
__global__ void __launch_bounds__(256) pcg_precond_kernel(const PcgPrecArgs A) {
  if (A.sc[S_DONE] != 0.0) return;
  __shared__ double hsh[32 * KH];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int c = tid; c < A.ell; c += blockDim.x) hsh[c] = __ldcg(A.h + c);
  __syncthreads();
  double hl[KH];
#pragma unroll
  for (int k = 0; k < KH; ++k) hl[k] = (lane + 32 * k < A.ell) ? hsh[lane + 32 * k] : 0.0;
  const int64_t nw = (int64_t)gridDim.x * 8;
  const int64_t w0 = (int64_t)blockIdx.x * 8 + (tid >> 5);
  double rz = 0.0;
  for (int64_t i0 = w0; i0 < A.m; i0 += 4 * nw) {
    double acc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + q * nw;
      double a = 0.0;
      if (i < A.m) {
#pragma unroll
        for (int k = 0; k < KH; ++k) {
          const int c = lane + 32 * k;
          if (c < A.ell) a = fma(A.U[(size_t)i * A.ldu + c], hl[k], a);
        }
      }
      acc[q] = a;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + q * nw;
      const double us = warp_sum(acc[q]);
      if (lane == 0 && i < A.m) {
        const double ri = A.r[i];
        const double zi = ri + us;
        A.z[i] = zi;
        rz = fma(ri, zi, rz);
      }
    }
  }
  double v[1] = {rz};
  block_sum_to_part<1>(v, A.part, gridDim.x);
  if (last_block_arrive(A.counter) && warp_uniform_id() == 0) {
    const double rzn = warp_sum_array(A.part, gridDim.x);
    if (threadIdx.x != 0) return;
    const double rzo = A.sc[S_RZ];
    A.sc[S_BETA] = A.init ? 0.0 : rzn / rzo;
    A.sc[S_RZ] = rzn;
    if (!(rzn > 0.0) || !isfinite(rzn)) { A.sc[S_STATUS] = (double)NYS_EBREAKDOWN; A.sc[S_DONE] = 1.0; }
    *A.counter = 0u;
  }
}

// Ut[i][c] = U[c][i]  (m x ell column-major, ld ldu  ->  row-major, row stride ell), 32x32 tiles
__global__ void transpose_u_kernel(int64_t m, int ell, const double* U, int64_t ldu, double* Ut) {
  __shared__ double t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: 8 rows of 32
  for (int cc = ty; cc < 32; cc += 8) {
    const int c = c0 + cc;
    const int64_t i = i0 + tx;
    t[cc][tx] = (c < ell && i < m) ? U[(size_t)c * ldu + i] : 0.0;
  }
  __syncthreads();
  for (int ii = ty; ii < 32; ii += 8) {
    const int64_t i = i0 + ii;
    const int c = c0 + tx;
    if (i < m && c < ell) Ut[(size_t)i * ell + c] = t[tx][ii];
  }
}
int launch_transpose_u(nys_ctx* ctx, int64_t m, int ell, const double* U, int64_t ldu, double* Ut) {
  if (m <= 0 || ell <= 0) return NYS_OK;
  dim3 grid((unsigned)((m + 31) / 32), (unsigned)((ell + 31) / 32));
  transpose_u_kernel<<<grid, 256, 0, ctx->stream>>>(m, ell, U, ldu, Ut);
  ctx->launches++;
  return ctx->check_launch("transpose_u");
}

int launch_pcg_update(nys_ctx* ctx, int init, int64_t m, double* x, double* r, const double* rhs, const double* p,
                      const double* w, const FusedPartials* fp, double delta, const double* e, const double* U,
                      int64_t ldu, int ell, const double* s, double* h, int max_iter, unsigned long long cond,
                      bool delta_slot, bool ext_prec) {
  PcgUpdArgs A{};
  A.ext_prec = ext_prec ? 1 : 0;
  A.cond = cond;
  A.delta_slot = delta_slot ? 1 : 0;
  A.init = init; A.m = m; A.x = x; A.r = r; A.rhs = rhs; A.p = p; A.w = w;
  if (fp) { A.Wp = fp->Wp; A.wp_ld = fp->wp_ld; A.nparts = fp->nparts; A.pwp = fp->pwp; A.npw = fp->npw; }
  A.delta = delta; A.e = e;
  A.U = U; A.ldu = ldu; A.ell = ell; A.s = s; A.h = h; A.sc = ctx->sc; A.max_iter = max_iter;
  // one 256-row tile per block while that gives <= 8 blocks per SM, else 256-row tiles in a loop
  int64_t rpb = 256;
  if ((m + rpb - 1) / rpb > 8LL * ctx->num_sms) rpb = ((m + 8LL * ctx->num_sms - 1) / (8LL * ctx->num_sms) + 255) / 256 * 256;
  int g = (int)((m + rpb - 1) / rpb);
  if (g < 1) g = 1;
  A.rows_per_block = rpb;
  A.part = ctx->wsd("pcg_upd_part", (size_t)(1 + ell) * g);
  A.counter = ctx->counters + 1;
  if (ell > 256) {
    const size_t sm = (size_t)8 * (1 + ell) * sizeof(double);
    NYS_TRY(ensure_max_smem(ctx, (const void*)pcg_update_kernel<true>, sm));
    pcg_update_kernel<true><<<(unsigned)g, 256, sm, ctx->stream>>>(A);
  } else {
    pcg_update_kernel<false><<<(unsigned)g, 256, 0, ctx->stream>>>(A);
  }
  ctx->launches++;
  NYS_TRY(ctx->check_launch("pcg_update"));
  pcg_hred_kernel<<<(unsigned)(1 + ell), 256, 0, ctx->stream>>>(A, g);
  ctx->launches++;
  return ctx->check_launch("pcg_hred");
}

int launch_pcg_precond(nys_ctx* ctx, int init, int64_t m, const double* r, double* z, const double* U, int64_t ldu,
                       int ell, const double* h) {
  PcgPrecArgs A{};
  A.init = init; A.m = m; A.r = r; A.z = z; A.U = U; A.ldu = ldu; A.ell = ell; A.h = h; A.sc = ctx->sc;
  int64_t g = (m + 31) / 32;  // 8 warps per block, 4 rows per warp
  if (g > 4 * ctx->num_sms) g = 4 * ctx->num_sms;
  if (g < 1) g = 1;
  A.nsub = 0;
  A.part = ctx->wsd("pcg_prec_part", (size_t)g);
  A.counter = ctx->counters + 2;
  if (ell > 256) pcg_precond_kernel<32><<<(unsigned)g, 256, 0, ctx->stream>>>(A);
  else pcg_precond_kernel<8><<<(unsigned)g, 256, 0, ctx->stream>>>(A);
  ctx->launches++;
  return ctx->check_launch("pcg_precond");
}

// s_i = (lam_l + mu) / (lam_i + mu) - 1
__global__ void prec_coef_kernel(const double* lam, int ell, double mu, double* s, const double* muslot) {
  if (muslot != nullptr) mu = *muslot;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ell) s[i] = (lam[ell - 1] + mu) / (lam[i] + mu) - 1.0;
}
int launch_prec_coef(nys_ctx* ctx, const double* lam, int ell, double mu, double* s) {
  if (ell <= 0) return NYS_OK;
  prec_coef_kernel<<<(ell + 127) / 128, 128, 0, ctx->stream>>>(lam, ell, mu, s, ctx->gloop ? ctx->sc + S_DELTA : nullptr);
  ctx->launches++;
  return ctx->check_launch("prec_coef");
}

// PCG tolerance (A8'): tau = max(floor (1+|b|), min(0.1 |xi|, c mu (1+|b|))) from device scalars
__global__ void pcg_setup_kernel(double* sc, int mode, double tol_abs, double c, double floor_, int xi_slot,
                                 int b_slot, int mu_slot, double init_rel) {
  double tol;
  if (mode == 0) {
    tol = tol_abs;
  } else if (mode == 1) {
    const double xin = sqrt(sc[xi_slot]);
    const double bn = sqrt(sc[b_slot]);
    const double mu = sc[mu_slot];
    tol = fmax(floor_ * (1.0 + bn), fmin(0.1 * xin, c * mu * (1.0 + bn)));
  } else {  // initial point: init_rel * |rhs|
    tol = init_rel * sqrt(sc[xi_slot]);
  }
  sc[S_TOL] = tol;
  sc[S_DONE] = 0.0;
  sc[S_ITERS] = 0.0;
  sc[S_STATUS] = 0.0;
  sc[S_RZ] = 0.0;
  sc[S_BETA] = 0.0;
  sc[S_ALPHA] = 0.0;
}
int launch_pcg_setup(nys_ctx* ctx, int mode, double tol_abs, double c, double floor_, int xi_slot, int b_slot,
                     int mu_slot, double init_rel) {
  pcg_setup_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sc, mode, tol_abs, c, floor_, xi_slot, b_slot, mu_slot, init_rel);
  ctx->launches++;
  return ctx->check_launch("pcg_setup");
}

// ------------------------------------------------------------------------------------------
// IPM elementwise kernels (Alg. 4 / Alg. 5 for I-only variables)
// ------------------------------------------------------------------------------------------
// d_j = 1 / (q_j + z_j / x_j + rho)
__global__ void scaling_kernel(int64_t n, const double* q, const double* x, const double* z, double rho, double* d,
                               const double* rslot) {
  if (rslot != nullptr) rho = *rslot;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    d[j] = 1.0 / (q[j] + z[j] / x[j] + rho);
}

// predictor: r_d = c + q x - A^T y - z + rho (x - zeta) = rD + rho (x - zeta)
// [rD = dual residual at the current iterate]; r_xz = -x z ; xi_au = -r_xz / x (= z) ;
// t = d (r_d + xi_au)
__global__ void pred_rhs_n_kernel(int64_t n, const double* x, const double* z, const double* zeta, const double* rD,
                                  double rho, const double* d, double* rd, double* rxz, double* xiau, double* t,
                                  const double* rslot) {
  if (rslot != nullptr) rho = *rslot;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double xj = x[j], zj = z[j];
    const double r = rD[j] + rho * (xj - zeta[j]);
    const double rx = -xj * zj;
    const double xa = -rx / xj;
    rd[j] = r;
    rxz[j] = rx;
    xiau[j] = xa;
    t[j] = d[j] * (r + xa);
  }
}
// r_p = b - A x - delta (y - lambda) [ax = A x given]
__global__ void pred_rhs_m_kernel(int64_t m, const double* b, const double* ax, const double* y, const double* lam,
                                  double delta, double* rp, const double* dslot) {
  if (dslot != nullptr) delta = *dslot;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    rp[i] = b[i] - ax[i] - delta * (y[i] - lam[i]);
}
// corrector: r_d = r_p = 0 ; r_xz = mu~ - dxp dzp ; xi_au = -r_xz / x ; t = d xi_au
__global__ void corr_rhs_kernel(int64_t n, const double* x, const double* dxp, const double* dzp, const double* sc,
                                const double* d, double* rxz, double* xiau, double* t) {
  const double mut = sc[S_MUT];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double rx = mut - dxp[j] * dzp[j];
    const double xa = -rx / x[j];
    rxz[j] = rx;
    xiau[j] = xa;
    t[j] = d[j] * xa;
  }
}
// iterate update: x += ap dx ; z += ad dz   (n-space)  and  y += ad dy (m-space)
__global__ void update_n_kernel(int64_t n, double* x, const double* dx, double* z, const double* dz, const double* sc) {
  if (sc[S_PCGBRK] != 0.0 || sc[S_NYSFAIL] != 0.0) return;   // discarded iteration: the iterate stays
  const double ap = sc[S_AP], ad = sc[S_AD];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    x[j] = fma(ap, dx[j], x[j]);
    z[j] = fma(ad, dz[j], z[j]);
  }
}
__global__ void update_m_kernel(int64_t m, double* y, const double* dy1, const double* dy2, const double* sc) {
  if (sc[S_PCGBRK] != 0.0 || sc[S_NYSFAIL] != 0.0) return;
  const double ad = sc[S_AD];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(ad, dy1[i] + dy2[i], y[i]);
}
// r = b - ax  (m) ;  generic axpby: out = a*u + b*v
__global__ void axpby_kernel(int64_t n, double a, const double* u, double b, const double* v, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * u[i] + (v ? b * v[i] : 0.0);
}
// out = u o v
__global__ void mul_kernel(int64_t n, const double* u, const double* v, double* out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    out[j] = u[j] * v[j];
}
// t = c + q o x  (initial point rhs) ; shift: out = u + s (scalar)
__global__ void cpqx_kernel(int64_t n, const double* c, const double* q, const double* x, double* t) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    t[j] = c[j] + q[j] * x[j];
}
__global__ void shift_kernel(int64_t n, double* u, double s) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    u[j] += s;
}
// min of a vector (raw) -> slot ; sums -> slot : generic "minsum"
__global__ void __launch_bounds__(256) minsum_kernel(int64_t n, const double* u, double shift, double* sc, int min_slot,
                                                     int sum_slot, double* part, unsigned int* counter) {
  double mn = 1.0e300, sm = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double v = u[j];
    mn = fmin(mn, v);
    sm += v + shift;
  }
  __shared__ double sh[2][32];
  mn = warp_min(mn);
  sm = warp_sum(sm);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sh[0][w] = mn; sh[1][w] = sm; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 1.0e300, b = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { a = fmin(a, sh[0][i]); b += sh[1][i]; }
    part[blockIdx.x] = a;
    part[gridDim.x + blockIdx.x] = b;
  }
  if (last_block_arrive(counter) && warp_uniform_id() == 0) {
    const double a = warp_min_array(part, gridDim.x);
    const double b = warp_sum_array(part + gridDim.x, gridDim.x);
    if (threadIdx.x != 0) return;
    *counter = 0u;
    if (min_slot >= 0) sc[min_slot] = a;
    if (sum_slot >= 0) sc[sum_slot] = b;
  }
}

static int ew_grid(nys_ctx* ctx, int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g < 1) g = 1;
  if (g > 4 * ctx->num_sms) g = 4 * ctx->num_sms;
  return (int)g;
}

int launch_scaling(nys_ctx* ctx, int64_t n, const double* q, const double* x, const double* z, double rho, double* d) {
  if (n <= 0) return NYS_OK;
  scaling_kernel<<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, q, x, z, rho, d, ctx->gloop ? ctx->sc + S_RHO : nullptr);
  ctx->launches++;
  return ctx->check_launch("scaling");
}
int launch_pred_rhs_n(nys_ctx* ctx, int64_t n, const double* x, const double* z, const double* zeta, const double* rD,
                      double rho, const double* d, double* rd, double* rxz, double* xiau, double* t) {
  if (n <= 0) return NYS_OK;
  pred_rhs_n_kernel<<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, x, z, zeta, rD, rho, d, rd, rxz, xiau, t,
                                                               ctx->gloop ? ctx->sc + S_RHO : nullptr);
  ctx->launches++;
  return ctx->check_launch("pred_rhs_n");
}
int launch_pred_rhs_m(nys_ctx* ctx, int64_t m, const double* b, const double* ax, const double* y, const double* lam,
                      double delta, double* rp) {
  pred_rhs_m_kernel<<<ew_grid(ctx, m), 256, 0, ctx->stream>>>(m, b, ax, y, lam, delta, rp,
                                                               ctx->gloop ? ctx->sc + S_DELTA : nullptr);
  ctx->launches++;
  return ctx->check_launch("pred_rhs_m");
}
int launch_corr_rhs(nys_ctx* ctx, int64_t n, const double* x, const double* dxp, const double* dzp, const double* d,
                    double* rxz, double* xiau, double* t) {
  if (n <= 0) return NYS_OK;
  corr_rhs_kernel<<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, x, dxp, dzp, ctx->sc, d, rxz, xiau, t);
  ctx->launches++;
  return ctx->check_launch("corr_rhs");
}
int launch_update_n(nys_ctx* ctx, int64_t n, double* x, const double* dx, double* z, const double* dz) {
  if (n <= 0) return NYS_OK;
  update_n_kernel<<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, x, dx, z, dz, ctx->sc);
  ctx->launches++;
  return ctx->check_launch("update_n");
}
int launch_update_m(nys_ctx* ctx, int64_t m, double* y, const double* dy1, const double* dy2) {
  update_m_kernel<<<ew_grid(ctx, m), 256, 0, ctx->stream>>>(m, y, dy1, dy2, ctx->sc);
  ctx->launches++;
  return ctx->check_launch("update_m");
}
int launch_axpby(nys_ctx* ctx, int64_t n, double a, const double* u, double b, const double* v, double* out) {
  if (n <= 0) return NYS_OK;
  axpby_kernel<<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, a, u, b, v, out);
  ctx->launches++;
  return ctx->check_launch("axpby");
}
int launch_mul(nys_ctx* ctx, int64_t n, const double* u, const double* v, double* out) {
  if (n <= 0) return NYS_OK;
  mul_kernel<<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, u, v, out);
  ctx->launches++;
  return ctx->check_launch("mul");
}
int launch_cpqx(nys_ctx* ctx, int64_t n, const double* c, const double* q, const double* x, double* t) {
  if (n <= 0) return NYS_OK;
  cpqx_kernel<<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, c, q, x, t);
  ctx->launches++;
  return ctx->check_launch("cpqx");
}
int launch_shift(nys_ctx* ctx, int64_t n, double* u, double s) {
  if (n <= 0) return NYS_OK;
  shift_kernel<<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, u, s);
  ctx->launches++;
  return ctx->check_launch("shift");
}
int launch_minsum(nys_ctx* ctx, int64_t n, const double* u, double shift, int min_slot, int sum_slot, int counter_slot) {
  const int g = reduce_grid(ctx, n);
  double* part = ctx->wsd("minsum_part", (size_t)2 * g);
  minsum_kernel<<<g, 256, 0, ctx->stream>>>(n, u, shift, ctx->sc, min_slot, sum_slot, part, ctx->counters + counter_slot);
  ctx->launches++;
  return ctx->check_launch("minsum");
}

// ------------------------------------------------------------------------------------------
// SVM-structured A = [Xt, -Xt, I, -I]: variables [w+ (nd), w- (nd), xi (mr), s (mr)], the
// xi / s variables of this rank being those of rows [r0, r0 + mr) (single rank: r0 = 0, mr = m)
// ------------------------------------------------------------------------------------------
// A^T y = [Xt^T y ; -Xt^T y ; y_rows ; -y_rows]   from g = Xt^T y
__global__ void svm_expand_kernel(int64_t nd, int64_t r0, int64_t mr, const double* g, const double* y, double* atv) {
  const int64_t n = 2 * nd + 2 * mr;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double v;
    if (j < nd) v = g[j];
    else if (j < 2 * nd) v = -g[j - nd];
    else if (j < 2 * nd + mr) v = y[r0 + j - 2 * nd];
    else v = -y[r0 + j - 2 * nd - mr];
    atv[j] = v;
  }
}
// A u = Xt (u_w+ - u_w-) + (u_xi - u_s on the own rows) :  uw (nd) and the diagonal part addm (m) (+ add)
__global__ void svm_fold_kernel(int64_t nd, int64_t m, int64_t r0, int64_t mr, const double* u, const double* add,
                                double* uw, double* addm) {
  const int64_t tot = nd + m;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < tot; j += (int64_t)gridDim.x * blockDim.x) {
    if (j < nd) uw[j] = u[j] - u[nd + j];
    else {
      const int64_t i = j - nd, k = i - r0;
      const double un = (k >= 0 && k < mr) ? u[2 * nd + k] - u[2 * nd + mr + k] : 0.0;
      addm[i] = un + (add ? add[i] : 0.0);
    }
  }
}
// normal operator of the structured A: N = Xt diag(d_w+ + d_w-) Xt^T + diag(d_xi + d_s) (own rows; the
// other rows' terms come from their ranks through the all-reduce)
__global__ void svm_scaling_fold_kernel(int64_t nd, int64_t m, int64_t r0, int64_t mr, const double* d, double* dw,
                                        double* e) {
  const int64_t tot = nd + m;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < tot; j += (int64_t)gridDim.x * blockDim.x) {
    if (j < nd) dw[j] = d[j] + d[nd + j];
    else {
      const int64_t i = j - nd, k = i - r0;
      e[i] = (k >= 0 && k < mr) ? d[2 * nd + k] + d[2 * nd + mr + k] : 0.0;
    }
  }
}
// generic IPM epilogues on an explicit A^T v (n-vector)
__global__ void epi_rd_kernel(int64_t n, const double* c, const double* q, const double* x, const double* atv,
                              const double* z, double* out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    out[j] = c[j] + q[j] * x[j] - atv[j] - (z ? z[j] : 0.0);
}
__global__ void epi_dx_kernel(int64_t n, const double* atv, const double* rd, const double* xiau, const double* rxz,
                              const double* z, const double* x, const double* d, double* dx, double* dz) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double v = d[j] * (atv[j] - (rd ? rd[j] : 0.0) - xiau[j]);
    dx[j] = v;
    dz[j] = (rxz[j] - z[j] * v) / x[j];
  }
}
int launch_svm_expand(nys_ctx* ctx, int64_t nd, int64_t r0, int64_t mr, const double* g, const double* y, double* atv) {
  if (2 * nd + 2 * mr <= 0) return NYS_OK;
  svm_expand_kernel<<<ew_grid(ctx, 2 * nd + 2 * mr), 256, 0, ctx->stream>>>(nd, r0, mr, g, y, atv);
  ctx->launches++;
  return ctx->check_launch("svm_expand");
}
int launch_svm_fold(nys_ctx* ctx, int64_t nd, int64_t m, int64_t r0, int64_t mr, const double* u, const double* add,
                    double* uw, double* addm) {
  svm_fold_kernel<<<ew_grid(ctx, nd + m), 256, 0, ctx->stream>>>(nd, m, r0, mr, u, add, uw, addm);
  ctx->launches++;
  return ctx->check_launch("svm_fold");
}
int launch_svm_scaling_fold(nys_ctx* ctx, int64_t nd, int64_t m, int64_t r0, int64_t mr, const double* d, double* dw,
                            double* e) {
  svm_scaling_fold_kernel<<<ew_grid(ctx, nd + m), 256, 0, ctx->stream>>>(nd, m, r0, mr, d, dw, e);
  ctx->launches++;
  return ctx->check_launch("svm_scaling_fold");
}
int launch_epi_rd(nys_ctx* ctx, int64_t n, const double* c, const double* q, const double* x, const double* atv,
                  const double* z, double* out) {
  if (n <= 0) return NYS_OK;
  epi_rd_kernel<<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, c, q, x, atv, z, out);
  ctx->launches++;
  return ctx->check_launch("epi_rd");
}
int launch_epi_dx(nys_ctx* ctx, int64_t n, const double* atv, const double* rd, const double* xiau, const double* rxz,
                  const double* z, const double* x, const double* d, double* dx, double* dz) {
  if (n <= 0) return NYS_OK;
  epi_dx_kernel<<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, atv, rd, xiau, rxz, z, x, d, dx, dz);
  ctx->launches++;
  return ctx->check_launch("epi_dx");
}

// positivity check of d (nys_check_scaling): first bad index -> slot
__global__ void check_pos_kernel(int64_t n, const double* d, unsigned long long* bad) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double v = d[j];
    if (!(v > 0.0) || !isfinite(v)) atomicMin(bad, (unsigned long long)j);
  }
}
int launch_check_pos(nys_ctx* ctx, int64_t n, const double* d, unsigned long long* bad) {
  if (n <= 0) return NYS_OK;
  check_pos_kernel<<<ew_grid(ctx, n), 256, 0, ctx->stream>>>(n, d, bad);
  ctx->launches++;
  return ctx->check_launch("check_pos");
}

// set scalar slots from host values (one tiny kernel, stream ordered)
__global__ void set_slots_kernel(double* sc, int k0, double v0, int k1, double v1, int k2, double v2) {
  if (k0 >= 0) sc[k0] = v0;
  if (k1 >= 0) sc[k1] = v1;
  if (k2 >= 0) sc[k2] = v2;
}
// latch a finished PCG solve: iteration count into `slot`, graph-loop iterations accumulated, breakdown flag
__global__ void pcg_latch_kernel(double* sc, int slot) {
  sc[slot] = sc[S_ITERS];
  sc[S_GITACC] += sc[S_GITER];
  if (sc[S_STATUS] == (double)NYS_EBREAKDOWN) sc[S_PCGBRK] = 1.0;
}
int launch_pcg_latch(nys_ctx* ctx, int slot) {
  pcg_latch_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sc, slot);
  ctx->launches++;
  return ctx->check_launch("pcg_latch");
}
__global__ void flag_max_kernel(double* sc, int dst, int src) { sc[dst] = fmax(sc[dst], sc[src]); }
int launch_flag_max(nys_ctx* ctx, int dst, int src) {
  flag_max_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sc, dst, src);
  ctx->launches++;
  return ctx->check_launch("flag_max");
}
int launch_set_slots(nys_ctx* ctx, int k0, double v0, int k1, double v1, int k2, double v2) {
  set_slots_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sc, k0, v0, k1, v1, k2, v2);
  ctx->launches++;
  return ctx->check_launch("set_slots");
}

}  // namespace nys

// ------------------------------------------------------------------------------------------
// graph-resident outer loop (f3): the host loop's end-of-iteration logic on the device
// ------------------------------------------------------------------------------------------
namespace nys {
__global__ void stamp_kernel(double* sc, int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  sc[slot] = (double)t;
}
int launch_stamp(nys_ctx* ctx, int slot) {
  stamp_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sc, slot);
  ctx->launches++;
  return ctx->check_launch("stamp");
}

// One thread, after the iteration's residual norms are in S_TMP0..4: the iteration record, the PEU
// (reading A12: the factor 1 - r when the residual improved to <= 0.95 of its reference, else
// 1 - 2r/3, floored), the copies lambda <- y / zeta <- x flagged for cond_copy_kernel, the termination
// criterion of the next iteration (A11) and the iteration cap — the same arithmetic and order as the host
// loop of ipm_impl — then the WHILE condition.  Stop codes: 1 converged, 2 Nystrom factorisation failure
// (the host re-runs the iteration with its checks), 3 breakdown / non-finite, 4 iteration cap.
__global__ void ipm_control_kernel(double* sc, double* rec, cudaGraphConditionalHandle h) {
  const double tol = sc[S_GPAR0], bnorm = sc[S_GPAR1], cnorm = sc[S_GPAR2], n_total = sc[S_GPAR3];
  const double max_outer = sc[S_GPAR4], floor_ = sc[S_GPAR5], max_rec = sc[S_GPAR6];
  const int k = (int)sc[S_KOUT];
  if (sc[S_NYSFAIL] != 0.0 || sc[S_PCGBRK] != 0.0) {
    sc[S_GSTOP] = sc[S_NYSFAIL] != 0.0 ? 2.0 : 3.0;
    sc[S_CPLAM] = 0.0;   // the discarded iteration copies nothing
    sc[S_CPZETA] = 0.0;
    cudaGraphSetConditional(h, 0u);
    return;
  }
  const double tsk = (sc[S_TS1] - sc[S_TS0]) * 1e-6;
  const double tpcg = ((sc[S_TS3] - sc[S_TS2]) + (sc[S_TS5] - sc[S_TS4])) * 1e-6;
  const double mu = sc[S_OMU], nrP = sc[S_NRP], nrD = sc[S_NRD];
  const double rho = sc[S_RHO], delta = sc[S_DELTA];
  const double pred = sc[S_PCGI0], corr = sc[S_PCGI1];
  if (k < max_rec) {
    double* r = rec + (size_t)k * 16;
    r[0] = k; r[1] = mu; r[2] = nrP / (1.0 + bnorm); r[3] = nrD / (1.0 + cnorm);
    r[4] = sc[S_AP]; r[5] = sc[S_AD]; r[6] = pred; r[7] = corr; r[8] = rho; r[9] = delta;
    r[10] = tsk; r[11] = tpcg; r[12] = sc[S_LAML];
  }
  const double mu_new = n_total > 0 ? (sc[S_TMP2] + sc[S_TMP4]) / n_total : 0.0;
  const double nrPn = sqrt(sc[S_TMP0] + sc[S_TMP3]), nrDn = sqrt(sc[S_TMP1]);
  const double rr = (mu > 0) ? fmin(fmax(1.0 - mu_new / mu, 0.0), 1.0) : (n_total > 0 ? 0.0 : 1.0);
  const bool p_imp = nrPn <= 0.95 * sc[S_NRPREF];
  const bool d_imp = nrDn <= 0.95 * sc[S_NRDREF];
  sc[S_CPLAM] = p_imp ? 1.0 : 0.0;
  sc[S_CPZETA] = d_imp ? 1.0 : 0.0;
  if (p_imp) sc[S_NRPREF] = nrPn;
  if (d_imp) sc[S_NRDREF] = nrDn;
  sc[S_DELTA] = fmax(floor_, (p_imp ? (1.0 - rr) : (1.0 - 2.0 / 3.0 * rr)) * delta);
  sc[S_RHO] = fmax(floor_, (d_imp ? (1.0 - rr) : (1.0 - 2.0 / 3.0 * rr)) * rho);
  sc[S_INNER] += pred + corr;
  sc[S_GLACC] += sc[S_GITACC];   // graph-path PCG iterations run by the nested WHILE bodies (accounting)
  sc[S_TSK] += tsk;
  sc[S_TPCG] += tpcg;
  sc[S_OMU] = mu_new;
  sc[S_MUCUR] = mu_new;
  sc[S_NRP] = nrPn;
  sc[S_NRD] = nrDn;
  sc[S_KOUT] = k + 1;
  double stop = 0.0;
  if (nrPn / (1.0 + bnorm) <= tol && nrDn / (1.0 + cnorm) <= tol && mu_new <= tol) stop = 1.0;   // A11
  else if (k + 1 >= max_outer) stop = 4.0;
  else if (!isfinite(mu_new) || !isfinite(nrPn) || !isfinite(nrDn)) stop = 3.0;
  sc[S_GSTOP] = stop;
  cudaGraphSetConditional(h, stop == 0.0 ? 1u : 0u);
}
int launch_ipm_control(nys_ctx* ctx, double* rec, cudaGraphConditionalHandle h) {
  ipm_control_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sc, rec, h);
  ctx->launches++;
  return ctx->check_launch("ipm_control");
}
// dst <- src when the flag slot is set (the PEU's lambda <- y and zeta <- x)
__global__ void cond_copy_kernel(const double* sc, int flag, double* dst, const double* src, int64_t len) {
  if (sc[flag] == 0.0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
int launch_cond_copy(nys_ctx* ctx, int flag, double* dst, const double* src, int64_t len) {
  if (len <= 0) return NYS_OK;
  cond_copy_kernel<<<ew_grid(ctx, len), 256, 0, ctx->stream>>>(ctx->sc, flag, dst, src, len);
  ctx->launches++;
  return ctx->check_launch("cond_copy");
}
}  // namespace nys

namespace nys {
// test hook (NYS_INJECT_NYSFAIL=k): raise the factorisation-failure flag in outer iteration k
__global__ void inject_nysfail_kernel(double* sc, int k) {
  if ((int)sc[S_KOUT] == k) sc[S_NYSFAIL] = 1.0;
}
int launch_inject_nysfail(nys_ctx* ctx, int k) {
  inject_nysfail_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sc, k);
  ctx->launches++;
  return ctx->check_launch("inject_nysfail");
}
// re-arm a WHILE node's condition (a nested conditional node gets its default only at graph launch)
__global__ void set_cond_kernel(cudaGraphConditionalHandle h, unsigned int v) { cudaGraphSetConditional(h, v); }
int launch_set_cond(nys_ctx* ctx, unsigned long long h, unsigned int v) {
  set_cond_kernel<<<1, 1, 0, ctx->stream>>>((cudaGraphConditionalHandle)h, v);
  ctx->launches++;
  return ctx->check_launch("set_cond");
}
}  // namespace nys
