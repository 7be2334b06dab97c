// Small dense kernels of Alg. 1: the shift nu = eps(||Y||_F), Y_nu, the
// ell x ell Cholesky + triangular inverse (lines 5-6), triangular products, and the thin SVD
// of B = Y_nu C^{-1} finished on the ell x ell triangular factor by one-sided Jacobi.
// All ell x ell routines run in ONE CTA (1024 threads) with the matrices in shared memory
// when they fit, else in an L2-resident global workspace.
#include <algorithm>
#include <cooperative_groups.h>

#include "k_vec.cuh"

namespace cg = cooperative_groups;

namespace nys {

// ------------------------------------------------------------------------------------------
// ||Y||_F and nu = eps(||Y||_F) = 2^(floor(log2 ||Y||_F) - 52)
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) fro_kernel(int64_t m, int ell, const double* Y, int64_t ldy, double* part,
                                                  unsigned int* counter, double* sc) {
  double acc = 0.0;
  const int64_t total = m * (int64_t)ell;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    const double v = Y[i + j * ldy];
    acc = fma(v, v, acc);
  }
  acc = warp_sum(acc);
  __shared__ double sh[32];
  __shared__ bool last;
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    part[blockIdx.x] = s;
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last && warp_uniform_id() == 0) {
    __threadfence();
    const double s = warp_sum_array(part, gridDim.x);
    if (threadIdx.x != 0) return;
    *counter = 0u;
    const double f = sqrt(s);
    sc[S_FRO] = f;
    double nu;
    if (f > 0.0 && isfinite(f)) {
      nu = ldexp(1.0, ilogb(f) - 52);
      if (nu == 0.0) nu = 4.9406564584124654e-324;
    } else {
      nu = 4.9406564584124654e-324;
    }
    sc[S_NU] = nu;
  }
}

int launch_fro_nu(nys_ctx* ctx, int64_t m, int ell, const double* Y, int64_t ldy, int /*unused*/) {
  int64_t total = m * ell;
  int g = (int)((total + 1023) / 1024);
  if (g > 2 * ctx->num_sms) g = 2 * ctx->num_sms;
  if (g < 1) g = 1;
  double* part = ctx->wsd("fro_part", (size_t)g);
  fro_kernel<<<g, 256, 0, ctx->stream>>>(m, ell, Y, ldy, part, ctx->counters + 3, ctx->sc);
  ctx->launches++;
  return ctx->check_launch("fro");
}

// Y_nu = Y + nu Omega
__global__ void ynu_kernel(int64_t m, int ell, const double* Y, const double* Om, double* Ynu, int64_t ld,
                           const double* sc) {
  const double nu = sc[S_NU];
  const int64_t total = m * (int64_t)ell;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    Ynu[i + j * ld] = fma(nu, Om[i + j * ld], Y[i + j * ld]);
  }
}
int launch_ynu(nys_ctx* ctx, int64_t m, int ell, const double* Y, const double* Om, double* Ynu, int64_t ld) {
  int64_t total = m * ell;
  int g = (int)((total + 255) / 256);
  if (g > 4 * ctx->num_sms) g = 4 * ctx->num_sms;
  if (g < 1) g = 1;
  ynu_kernel<<<g, 256, 0, ctx->stream>>>(m, ell, Y, Om, Ynu, ld, ctx->sc);
  ctx->launches++;
  return ctx->check_launch("ynu");
}

// Y += e o Omega (multi-GPU sketch: the diagonal term is added once, after the all-reduce)
__global__ void add_eomega_kernel(int64_t m, int ell, const double* e, const double* Om, double* Y, int64_t ld) {
  const int64_t total = m * (int64_t)ell;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q % m, j = q / m;
    Y[i + j * ld] = fma(e[i], Om[i + j * ld], Y[i + j * ld]);
  }
}
int launch_add_eomega(nys_ctx* ctx, int64_t m, int ell, const double* e, const double* Om, double* Y, int64_t ld) {
  int64_t total = m * ell;
  int g = (int)((total + 255) / 256);
  if (g > 4 * ctx->num_sms) g = 4 * ctx->num_sms;
  if (g < 1) g = 1;
  add_eomega_kernel<<<g, 256, 0, ctx->stream>>>(m, ell, e, Om, Y, ld);
  ctx->launches++;
  return ctx->check_launch("add_eomega");
}

// ------------------------------------------------------------------------------------------
// Cholesky G = R^T R (R upper) of the symmetrised G (+ optional CholeskyQR shift), and R^{-1}.
// G (ell x ell, ld ldg) is overwritten with R (upper; strict lower zeroed).
// shift_mode 0: none (Alg. 1 line 5, A3 symmetrisation).
// shift_mode 1: shifted CholeskyQR (Fukaya et al. 2020): s = 11 (m ell + ell(ell+1)) u tr(G)
//               with m passed in sc[S_SHIFT] as a double on entry.
// Failure (non-positive / non-finite pivot) sets sc[S_CHOLFAIL] = 1.
// ------------------------------------------------------------------------------------------
template <bool SM>
__global__ void __launch_bounds__(256) chol_inv_kernel(int ell, double* G, int ldg, double* Rinv, int ldr,
                                                       int shift_mode, double* sc, double* gws) {
  extern __shared__ double csm[];
  const int n = ell;
  const int lx = n | 1;                   // odd leading dimension of X: conflict-free column access
  double* W = SM ? csm : gws;             // n x n, ld n : the factor
  double* X = W + (size_t)n * n;          // n x n, ld lx : R^{-1}
  __shared__ double rsq_s[SM ? 256 : 1];
  __shared__ double rowk_s[SM ? 256 : 1];  // row k gathered once per step (a strided, bank-conflicted read otherwise)
  double* rsq = SM ? rsq_s : X + (size_t)n * lx;          // global variant (ell > 113): after X in gws
  double* rowk = SM ? rowk_s : rsq + n;
  __shared__ double shift;
  const int tid = threadIdx.x, warp = warp_uniform_id(), lane = tid & 31, nw = blockDim.x >> 5;
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e % n, j = e / n;
    W[i + j * n] = 0.5 * (G[i + j * ldg] + G[j + i * ldg]);
  }
  for (int e = tid; e < n * lx; e += blockDim.x) X[e] = 0.0;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    if (shift_mode == 1) {
      double tr = 0.0;
      for (int i = 0; i < n; ++i) tr += W[i + i * n];
      s = 11.0 * (sc[S_SHIFT] * n + (double)n * (n + 1)) * 0x1p-53 * tr;
    }
    shift = s;
  }
  __syncthreads();
  if (shift_mode == 1) {
    for (int i = tid; i < n; i += blockDim.x) W[i + i * n] += shift;
    __syncthreads();
  }
  // right-looking Cholesky, one barrier per step: the trailing update uses the UNSCALED row k
  // (a_ij -= a_ki a_kj / a_kk); rows are scaled by 1/sqrt(a_kk) at the end -> R^T R = G.
  for (int k = 0; k < n; ++k) {
    const double piv = W[k + k * n];
    if (!(piv > 0.0) || !isfinite(piv)) {  // uniform: every thread reads the same pivot
      if (tid == 0) sc[S_CHOLFAIL] = 1.0;
      return;
    }
    for (int i = k + 1 + tid; i < n; i += blockDim.x) rowk[i] = W[k + i * n];
    __syncthreads();
    const double inv = 1.0 / piv;
    for (int j = k + 1 + warp; j < n; j += nw) {
      const double akj = rowk[j] * inv;
      for (int i = k + 1 + lane; i <= j; i += 32) W[i + j * n] = fma(-rowk[i], akj, W[i + j * n]);
    }
    __syncthreads();
  }
  for (int i = tid; i < n; i += blockDim.x) rsq[i] = 1.0 / sqrt(W[i + i * n]);
  __syncthreads();
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e % n, j = e / n;
    W[i + j * n] = (i < j) ? W[i + j * n] * rsq[i] : (i == j ? W[i + j * n] * rsq[i] : 0.0);
  }
  __syncthreads();
  // X = R^{-1} by back substitution with every (k, j) update in parallel:
  // X = I; for i = n-1..0: X(i, j>=i) /= R(i,i);  X(k<i, j>=i) -= R(k,i) X(i,j)
  for (int j = tid; j < n; j += blockDim.x) X[j + j * lx] = 1.0;
  __syncthreads();
  for (int i = n - 1; i >= 0; --i) {
    const double inv = 1.0 / W[i + i * n];
    for (int j = i + tid; j < n; j += blockDim.x) X[i + j * lx] *= inv;
    __syncthreads();
    for (int j = i + warp; j < n; j += nw) {   // warps over columns, lanes over rows (no index decode)
      const double xij = X[i + j * lx];
      for (int k = lane; k < i; k += 32) X[k + j * lx] = fma(-W[k + i * n], xij, X[k + j * lx]);
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e % n, j = e / n;
    G[i + j * ldg] = W[i + j * n];
    Rinv[i + j * ldr] = X[i + j * lx];
  }
}

// Same contract as chol_inv_kernel for ell up to 226 in ONE CTA: the upper triangle is held PACKED
// in shared memory (column-major upper packing, idx(i, j) = j (j + 1) / 2 + i, ell (ell + 1) / 2
// doubles = 205 KB at ell = 226) and R is inverted IN PLACE (the column-oriented upper-triangular
// inverse: column j of R^{-1} = -R^{-1}_jj T_{0:j,0:j} R_{0:j,j} with T the already inverted block),
// instead of the ell^2 + ell^2 layout the unpacked kernel needs (which fits only ell <= 113).
__device__ __forceinline__ int pidx(int i, int j) { return j * (j + 1) / 2 + i; }
__global__ void __launch_bounds__(1024) chol_inv_packed_kernel(int ell, double* G, int ldg, double* Rinv, int ldr,
                                                              int shift_mode, double* sc) {
  extern __shared__ double pk[];
  const int n = ell;
  __shared__ double rsq[256];
  __shared__ double tmp[256];
  __shared__ double row[256];   // row k / row i of the packed matrix (a strided gather done once per step)
  __shared__ double shift;
  const int tid = threadIdx.x, warp = warp_uniform_id(), lane = tid & 31, nw = blockDim.x >> 5;
  for (int j = warp; j < n; j += nw)
    for (int i = lane; i <= j; i += 32) pk[pidx(i, j)] = 0.5 * (G[i + (size_t)j * ldg] + G[j + (size_t)i * ldg]);
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    if (shift_mode == 1) {
      double tr = 0.0;
      for (int i = 0; i < n; ++i) tr += pk[pidx(i, i)];
      s = 11.0 * (sc[S_SHIFT] * n + (double)n * (n + 1)) * 0x1p-53 * tr;
    }
    shift = s;
  }
  __syncthreads();
  if (shift_mode == 1) {
    for (int i = tid; i < n; i += blockDim.x) pk[pidx(i, i)] += shift;
    __syncthreads();
  }
  for (int k = 0; k < n; ++k) {  // right-looking, unscaled row k (as chol_inv_kernel)
    const double piv = pk[pidx(k, k)];
    if (!(piv > 0.0) || !isfinite(piv)) {
      if (tid == 0) sc[S_CHOLFAIL] = 1.0;
      return;
    }
    for (int i = k + 1 + tid; i < n; i += blockDim.x) row[i] = pk[pidx(k, i)];
    __syncthreads();
    const double inv = 1.0 / piv;
    for (int j = k + 1 + warp; j < n; j += nw) {
      const double akj = row[j] * inv;
      double* colj = pk + pidx(0, j);
      for (int i = k + 1 + lane; i <= j; i += 32) colj[i] = fma(-row[i], akj, colj[i]);
    }
    __syncthreads();
  }
  for (int i = tid; i < n; i += blockDim.x) rsq[i] = 1.0 / sqrt(pk[pidx(i, i)]);
  __syncthreads();
  for (int j = warp; j < n; j += nw)
    for (int i = lane; i <= j; i += 32) pk[pidx(i, j)] *= rsq[i];
  __syncthreads();
  for (int e = tid; e < n * n; e += blockDim.x) {  // R out (lower zeroed)
    const int i = e % n, j = e / n;
    G[i + (size_t)j * ldg] = (i <= j) ? pk[pidx(i, j)] : 0.0;
  }
  __syncthreads();
  // in-place inverse, right to left (every (k, j) update of a step in parallel): at step i the
  // column above the diagonal still holds R(0:i, i) -> tmp; row i (holding the accumulated X(i, j > i))
  // is scaled by 1 / R(i, i); then X(k < i, j >= i) -= R(k, i) X(i, j) with X(k, i) starting at 0.
  for (int i = n - 1; i >= 0; --i) {
    for (int k = tid; k < i; k += blockDim.x) tmp[k] = pk[pidx(k, i)];
    const double inv = 1.0 / pk[pidx(i, i)];
    __syncthreads();
    for (int j = i + 1 + tid; j < n; j += blockDim.x) {
      const double x = pk[pidx(i, j)] * inv;
      pk[pidx(i, j)] = x;
      row[j] = x;
    }
    if (tid == 0) {
      pk[pidx(i, i)] = inv;
      row[i] = inv;
    }
    __syncthreads();
    // warps over the columns j >= i, lanes over the rows k < i (no index decode: a flattened
    // e -> (e % i, e / i) loop spent most of this kernel's time in integer divisions)
    for (int j = i + warp; j < n; j += nw) {
      const double xij = row[j];
      double* cj = pk + pidx(0, j);
      if (j == i) {
        for (int k = lane; k < i; k += 32) cj[k] = -tmp[k] * xij;
      } else {
        for (int k = lane; k < i; k += 32) cj[k] = fma(-tmp[k], xij, cj[k]);
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e % n, j = e / n;
    Rinv[i + (size_t)j * ldr] = (i <= j) ? pk[pidx(i, j)] : 0.0;
  }
}

// Column j of R^{-1} (R upper, n x n) by back substitution in one warp: x = e_j; for i = j .. 0:
// x_i /= R_ii (rinv_diag[i] = 1 / R_ii), x_{0:i} -= R_{0:i,i} x_i; x_k lives in lane k % 32, slot k / 32.
// The slot loop is unrolled (q static), so x[q] needs no dynamic register select and only the slots
// at or below q are updated (a dynamic-select version spent ~100 instructions per step).
// col(i) points at R(0, i) (rows 0 .. i-1 contiguous).
template <int E, typename ColFn>
__device__ __forceinline__ void inv_column_warp(int j, int n, const double* rinv_diag, ColFn col, double* out) {
  const int lane = threadIdx.x & 31;
  double x[E];
#pragma unroll
  for (int q = 0; q < E; ++q) x[q] = (lane + 32 * q == j) ? 1.0 : 0.0;
  const int qj = j >> 5;
#pragma unroll
  for (int q = E - 1; q >= 0; --q) {
    if (q > qj) continue;                                   // warp-uniform
    for (int ii = (q == qj ? (j & 31) : 31); ii >= 0; --ii) {
      const int i = 32 * q + ii;
      const double* ci = col(i);
      double wk[E];
#pragma unroll
      for (int q2 = 0; q2 <= q; ++q2)
        wk[q2] = (q2 < q || lane < ii) ? ci[lane + 32 * q2] : 0.0;
      const double xi = __shfl_sync(0xffffffffu, x[q], ii) * rinv_diag[i];
      if (lane == ii) x[q] = xi;
#pragma unroll
      for (int q2 = 0; q2 <= q; ++q2) x[q2] = fma(-wk[q2], xi, x[q2]);
    }
  }
#pragma unroll
  for (int q = 0; q < E; ++q)
    if (lane + 32 * q < n) out[lane + 32 * q] = x[q];
}

// Same contract for ell <= 128 (E = ceil(ell / 32) elements per lane; the paper's ranks up to 100 and
// CholeskyQR3 passes at them) with one block barrier per elimination step instead of two: the lane
// that updates row k+1 of a trailing column also publishes it into a double-buffered row, which is
// step k+1's pivot row.  R^{-1} is then formed one column per warp with no block barrier at all:
// x = e_j; for i = j..0: x_i /= R_ii, x_{0:i} -= R_{0:i,i} x_i (x held E elements per lane, x_i
// broadcast by a shuffle).  W (ell x ell, ld ell) in dynamic shared memory (128 KB at ell = 128).
template <int E>
__global__ void __launch_bounds__(1024) chol_inv_small_kernel(int ell, double* G, int ldg, double* Rinv, int ldr,
                                                             int shift_mode, double* sc) {
  extern __shared__ double W[];
  __shared__ double rowb[2][32 * E];
  __shared__ double rsq[32 * E];
  __shared__ double shift;
  const int n = ell, tid = threadIdx.x, warp = warp_uniform_id(), lane = tid & 31, nw = blockDim.x >> 5;
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e % n, j = e / n;
    W[i + j * n] = 0.5 * (G[i + (size_t)j * ldg] + G[j + (size_t)i * ldg]);
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    if (shift_mode == 1) {
      double tr = 0.0;
      for (int i = 0; i < n; ++i) tr += W[i + i * n];
      s = 11.0 * (sc[S_SHIFT] * n + (double)n * (n + 1)) * 0x1p-53 * tr;
    }
    shift = s;
  }
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) W[i + i * n] += shift;
  __syncthreads();
  for (int j = tid; j < n; j += blockDim.x) rowb[0][j] = W[j * n];
  __syncthreads();
  for (int k = 0; k < n; ++k) {  // right-looking, unscaled row k (as chol_inv_kernel)
    const double* rk = rowb[k & 1];
    double* rn = rowb[(k + 1) & 1];
    const double piv = rk[k];
    if (!(piv > 0.0) || !isfinite(piv)) {  // uniform
      if (tid == 0) sc[S_CHOLFAIL] = 1.0;
      return;
    }
    const double inv = 1.0 / piv;
    for (int j = k + 1 + warp; j < n; j += nw) {
      const double akj = rk[j] * inv;
      for (int i = k + 1 + lane; i <= j; i += 32) {
        const double v = fma(-rk[i], akj, W[i + j * n]);
        W[i + j * n] = v;
        if (i == k + 1) rn[j] = v;
      }
    }
    __syncthreads();
  }
  for (int i = tid; i < n; i += blockDim.x) rsq[i] = 1.0 / sqrt(W[i + i * n]);
  __syncthreads();
  for (int e = tid; e < n * n; e += blockDim.x) {  // R = diag(rsq) W (upper), out to G
    const int i = e % n, j = e / n;
    const double r = (i <= j) ? W[e] * rsq[i] : 0.0;
    W[e] = r;
    G[i + (size_t)j * ldg] = r;
  }
  __syncthreads();
  for (int j = warp; j < n; j += nw)
    inv_column_warp<E>(j, n, rsq, [&](int i) { return W + (size_t)i * n; }, Rinv + (size_t)j * ldr);
}

// Same contract as chol_inv_kernel for ell > 226 (no single-CTA shared-memory layout fits): the
// same right-looking unblocked Cholesky and the same parallel back substitution for R^{-1}, spread
// over a cooperative grid with a grid barrier between the steps (W, X, the pivot row in global memory,
// L2-resident: 10 MB at ell = 800).  One CTA of 256 threads took 205 ms at ell = 800.
__device__ __forceinline__ void cgrid_barrier(unsigned int* bar, unsigned int nblocks, unsigned int& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned int target = epoch * nblocks;
    red_add_release_gpu(bar, 1u);
    while (ld_relaxed_gpu(bar) < target) {
    }
    fence_acquire_gpu();
  }
  __syncthreads();
}
__global__ void __launch_bounds__(1024) chol_inv_grid_kernel(int n, double* G, int ldg, double* Rinv, int ldr,
                                                             int shift_mode, double* sc, double* W, double* X,
                                                             double* rowk, double* rsq, double* shiftp,
                                                             unsigned int* bar) {
  const int lx = n | 1;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, GT = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int64_t gw = gt >> 5, GW = GT >> 5;
  unsigned int epoch = 0;
  for (int64_t e = gt; e < (int64_t)n * n; e += GT) {
    const int i = (int)(e % n), j = (int)(e / n);
    W[i + (size_t)j * n] = 0.5 * (G[i + (size_t)j * ldg] + G[j + (size_t)i * ldg]);
  }
  for (int64_t e = gt; e < (int64_t)n * lx; e += GT) X[e] = 0.0;
  cgrid_barrier(bar, gridDim.x, epoch);
  if (gt == 0) {
    double s = 0.0;
    if (shift_mode == 1) {
      double tr = 0.0;
      for (int i = 0; i < n; ++i) tr += W[i + (size_t)i * n];
      s = 11.0 * (sc[S_SHIFT] * n + (double)n * (n + 1)) * 0x1p-53 * tr;
    }
    *shiftp = s;
  }
  cgrid_barrier(bar, gridDim.x, epoch);
  if (shift_mode == 1) {
    const double sh = __ldcg(shiftp);
    for (int64_t i = gt; i < n; i += GT) W[i + (size_t)i * n] += sh;
    cgrid_barrier(bar, gridDim.x, epoch);
  }
  for (int k = 0; k < n; ++k) {
    const double piv = __ldcg(W + k + (size_t)k * n);
    if (!(piv > 0.0) || !isfinite(piv)) {        // grid-uniform: every thread read the same pivot
      if (gt == 0) sc[S_CHOLFAIL] = 1.0;
      return;
    }
    for (int64_t i = k + 1 + gt; i < n; i += GT) rowk[i] = __ldcg(W + k + (size_t)i * n);
    cgrid_barrier(bar, gridDim.x, epoch);
    const double inv = 1.0 / piv;
    for (int64_t j = k + 1 + gw; j < n; j += GW) {
      const double akj = __ldcg(rowk + j) * inv;
      for (int64_t i = k + 1 + lane; i <= j; i += 32)
        W[i + (size_t)j * n] = fma(-__ldcg(rowk + i), akj, __ldcg(W + i + (size_t)j * n));
    }
    cgrid_barrier(bar, gridDim.x, epoch);
  }
  for (int64_t i = gt; i < n; i += GT) rsq[i] = 1.0 / sqrt(__ldcg(W + i + (size_t)i * n));
  cgrid_barrier(bar, gridDim.x, epoch);
  for (int64_t e = gt; e < (int64_t)n * n; e += GT) {
    const int i = (int)(e % n), j = (int)(e / n);
    const double w = __ldcg(W + i + (size_t)j * n);
    W[i + (size_t)j * n] = (i <= j) ? w * __ldcg(rsq + i) : 0.0;
  }
  for (int64_t j = gt; j < n; j += GT) X[j + (size_t)j * lx] = 1.0;
  cgrid_barrier(bar, gridDim.x, epoch);
  for (int i = n - 1; i >= 0; --i) {
    const double inv = 1.0 / __ldcg(W + i + (size_t)i * n);
    for (int64_t j = i + gt; j < n; j += GT) X[i + (size_t)j * lx] *= inv;
    cgrid_barrier(bar, gridDim.x, epoch);
    for (int64_t j = i + gw; j < n; j += GW) {   // warps over columns, lanes over rows (no index decode)
      const double xij = __ldcg(X + i + (size_t)j * lx);
      for (int k = lane; k < i; k += 32)
        X[k + (size_t)j * lx] = fma(-__ldcg(W + k + (size_t)i * n), xij, __ldcg(X + k + (size_t)j * lx));
    }
    cgrid_barrier(bar, gridDim.x, epoch);
  }
  for (int64_t e = gt; e < (int64_t)n * n; e += GT) {
    const int i = (int)(e % n), j = (int)(e / n);
    G[i + (size_t)j * ldg] = __ldcg(W + i + (size_t)j * n);
    Rinv[i + (size_t)j * ldr] = __ldcg(X + i + (size_t)j * lx);
  }
}

// Same contract as chol_inv_kernel, blocked, for ell <= 226 in ONE CTA (packed upper storage as
// chol_inv_packed_kernel).  The unblocked kernels spend a block barrier and a full trailing sweep
// (LDS + LDS + FMA + STS per element) on every elimination step.  Here:
//   * a panel of PB = 8 rows: step k updates only the panel rows (k, k0 + PB), one column per
//     thread (a single warp took longer: ~40 dependent shared-memory round trips per step);
//   * then the rows below the panel take the panel's PB rank-1 updates at once,
//     W_ij -= sum_k R_ki R_kj with R_k = W_k / sqrt(W_kk), in 4 x 4 register tiles of the upper
//     triangle (one 16-byte load per four FMAs);
//   * R^{-1} one column per warp by back substitution with shuffles (as chol_inv_small_kernel).
// The same unscaled right-looking recurrence (rows scaled by 1/sqrt(W_kk) at the end) in a different
// summation order.  Failure (non-positive / non-finite pivot) sets sc[S_CHOLFAIL] = 1.
template <int E>
__global__ void __launch_bounds__(1024) chol_inv_blk_kernel(int ell, double* G, int ldg, double* Rinv, int ldr,
                                                           int shift_mode, double* sc, long long* tr) {
  long long t0 = clock64(), tpanel = 0, ttrail = 0;
  constexpr int PB = 8;
  extern __shared__ double pk[];
  __shared__ double dinv[256];   // 1 / W_kk of the unscaled pivots; later 1 / sqrt(W_kk)
  __shared__ __align__(16) double prow[PB * 256];   // the current panel's rows of R, row-major
  __shared__ double shift;
  const int n = ell;
  const int tid = threadIdx.x, warp = warp_uniform_id(), lane = tid & 31, nw = blockDim.x >> 5;
  for (int j = warp; j < n; j += nw)
    for (int i = lane; i <= j; i += 32) pk[pidx(i, j)] = 0.5 * (G[i + (size_t)j * ldg] + G[j + (size_t)i * ldg]);
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    if (shift_mode == 1) {
      double tr = 0.0;
      for (int i = 0; i < n; ++i) tr += pk[pidx(i, i)];
      s = 11.0 * (sc[S_SHIFT] * n + (double)n * (n + 1)) * 0x1p-53 * tr;
    }
    shift = s;
  }
  __syncthreads();
  if (shift_mode == 1) {
    for (int i = tid; i < n; i += blockDim.x) pk[pidx(i, i)] += shift;
    __syncthreads();
  }
  for (int k0 = 0; k0 < n; k0 += PB) {
    const int kend = min(k0 + PB, n);
    long long ta = clock64();
    for (int k = k0; k < kend; ++k) {   // the panel: one column per thread, <= PB - 1 rows each
      const double piv = pk[pidx(k, k)];
      if (!(piv > 0.0) || !isfinite(piv)) {   // block-uniform: every thread read the same pivot
        if (tid == 0) sc[S_CHOLFAIL] = 1.0;
        return;
      }
      const double inv = 1.0 / piv;
      if (tid == 0) dinv[k] = inv;
      const int j = k + 1 + tid;             // blockDim.x >= n
      if (j < n) {
        const double akj = pk[pidx(k, j)] * inv;
        double* cj = pk + pidx(0, j);
#pragma unroll
        for (int u = 1; u < PB; ++u) {
          const int i = k + u;
          if (i < kend && i <= j) cj[i] = fma(-pk[pidx(k, i)], akj, cj[i]);
        }
      }
      __syncthreads();
    }
    long long tb = clock64();
    tpanel += tb - ta;
    const int m2 = n - kend;   // trailing rows / columns [kend, n), upper part, 4 x 4 tiles
    if (m2 > 0) {
      // the panel rows, unscaled, into a row-major buffer (contiguous 4-wide loads below; rows past
      // the panel are zero)
      // scaled by 1 / sqrt(W_kk): these are rows of R, and the update is the plain product
      // W_ij -= sum_r R_ri R_rj (no per-term pivot multiply)
      for (int e = tid; e < PB * m2; e += blockDim.x) {
        const int r = e / m2, j = kend + e % m2;
        prow[r * 256 + j] = (k0 + r < kend) ? pk[pidx(k0 + r, j)] * sqrt(dinv[k0 + r]) : 0.0;
      }
      __syncthreads();
      // upper-triangle tiles only (linear index -> (ti, tj), tj = floor((sqrt(8t + 1) - 1) / 2)): a
      // square tile loop with the lower half skipped left half of every warp idle
      const int nt = (m2 + 3) >> 2;
      const int ntri = nt * (nt + 1) / 2;
      for (int t = tid; t < ntri; t += blockDim.x) {
        int tj = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
        while (tj * (tj + 1) / 2 > t) --tj;
        while ((tj + 1) * (tj + 2) / 2 <= t) ++tj;
        const int ti = t - tj * (tj + 1) / 2;
        const int i0 = kend + 4 * ti, j0 = kend + 4 * tj;
        double acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
#pragma unroll
        for (int r = 0; r < PB; ++r) {
          const double2 a01 = *reinterpret_cast<const double2*>(prow + r * 256 + i0);
          const double2 a23 = *reinterpret_cast<const double2*>(prow + r * 256 + i0 + 2);
          const double2 b01 = *reinterpret_cast<const double2*>(prow + r * 256 + j0);
          const double2 b23 = *reinterpret_cast<const double2*>(prow + r * 256 + j0 + 2);
          const double ai[4] = {a01.x, a01.y, a23.x, a23.y};
          const double bj[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = fma(ai[u], bj[v], acc[u][v]);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int j = j0 + v;
          if (j >= n) continue;
          double* cj = pk + pidx(0, j);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (i0 + u <= j) cj[i0 + u] -= acc[u][v];
        }
      }
    }
    __syncthreads();
    ttrail += clock64() - tb;
  }
  const long long tc = clock64();
  for (int i = tid; i < n; i += blockDim.x) dinv[i] = 1.0 / sqrt(pk[pidx(i, i)]);
  __syncthreads();
  for (int j = warp; j < n; j += nw)
    for (int i = lane; i <= j; i += 32) pk[pidx(i, j)] *= dinv[i];
  __syncthreads();
  for (int e = tid; e < n * n; e += blockDim.x) {  // R out (lower zeroed)
    const int i = e % n, j = e / n;
    G[i + (size_t)j * ldg] = (i <= j) ? pk[pidx(i, j)] : 0.0;
  }
  // R^{-1}: column j by back substitution, x = e_j; for i = j .. 0: x_i /= R_ii, x_{0:i} -= R_{0:i,i} x_i
  const long long td = clock64();
  for (int j = warp; j < n; j += nw)
    inv_column_warp<E>(j, n, dinv, [&](int i) { return pk + pidx(0, i); }, Rinv + (size_t)j * ldr);
  if (tr != nullptr) {
    __syncthreads();
    if (tid == 0) { tr[0] = tc - t0; tr[1] = tpanel; tr[2] = ttrail; tr[3] = td - tc; tr[4] = clock64() - td; }
  }
}

int launch_chol_inv(nys_ctx* ctx, int ell, double* G, int ldg, double* Rinv, int ldr, int shift_mode) {
  const size_t need = ((size_t)ell * ell + (size_t)ell * (ell | 1)) * sizeof(double);
  const size_t need_packed = (size_t)ell * (ell + 1) / 2 * sizeof(double);
  static const int small_max = [] {
    const char* s = getenv("NYS_CHOL_SMALL_MAX");  // tuning / A-B override (default 128; 0 disables)
    return s ? atoi(s) : 128;
  }();
  // blocked kernel from blk_min (tuning override NYS_CHOL_BLK_MIN; NYS_CHOL_UNBLOCKED=1: never)
  static const int blk_min = getenv("NYS_CHOL_UNBLOCKED") ? 1 << 30
                             : getenv("NYS_CHOL_BLK_MIN") ? atoi(getenv("NYS_CHOL_BLK_MIN")) : 129;
  if (ell >= blk_min && ell <= 226) {
    const size_t smp = need_packed > 48 * 1024 ? need_packed : 48 * 1024;
    auto launch = [&](auto kern) -> int {
      NYS_TRY(ensure_max_smem(ctx, (const void*)kern, smp));
      long long* tr = getenv("NYS_CHOL_TRACE") ? (long long*)ctx->ws("chol_trace", 64) : nullptr;
      kern<<<1, 1024, need_packed, ctx->stream>>>(ell, G, ldg, Rinv, ldr, shift_mode, ctx->sc, tr);
      if (tr) {
        long long h[5];
        cudaMemcpyAsync(h, tr, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        fprintf(stderr, "[choltrace] ell=%d cholesky %lld (panels %lld, trailing %lld) scale+R %lld inverse %lld cycles\n", ell,
                h[0], h[1], h[2], h[3], h[4]);
      }
      return NYS_OK;
    };
    if (ell <= 64) NYS_TRY(launch(chol_inv_blk_kernel<2>));
    else if (ell <= 128) NYS_TRY(launch(chol_inv_blk_kernel<4>));
    else NYS_TRY(launch(chol_inv_blk_kernel<8>));
  } else if (ell <= small_max && ell <= 128) {
    const size_t sm = (size_t)ell * ell * sizeof(double);
    static const int thr = getenv("NYS_CHOL_THREADS") ? atoi(getenv("NYS_CHOL_THREADS")) : 1024;   // tuning
    if (ell <= 64) {
      chol_inv_small_kernel<2><<<1, thr, sm, ctx->stream>>>(ell, G, ldg, Rinv, ldr, shift_mode, ctx->sc);
    } else {
      NYS_TRY(ensure_max_smem(ctx, (const void*)chol_inv_small_kernel<4>, 128 * 1024));
      chol_inv_small_kernel<4><<<1, thr, sm, ctx->stream>>>(ell, G, ldg, Rinv, ldr, shift_mode, ctx->sc);
    }
  } else if (need > 200 * 1024 && need_packed <= 208 * 1024) {
    NYS_TRY(ensure_max_smem(ctx, (const void*)chol_inv_packed_kernel, 208 * 1024));
    chol_inv_packed_kernel<<<1, 1024, need_packed, ctx->stream>>>(ell, G, ldg, Rinv, ldr, shift_mode, ctx->sc);
  } else if (need <= 200 * 1024) {
    NYS_TRY(ensure_max_smem(ctx, (const void*)chol_inv_kernel<true>, 200 * 1024));
    chol_inv_kernel<true><<<1, 256, need, ctx->stream>>>(ell, G, ldg, Rinv, ldr, shift_mode, ctx->sc, nullptr);
  } else if (getenv("NYS_CHOL_1CTA") != nullptr) {
    double* gws = ctx->wsd("chol_ws", (size_t)ell * ell + (size_t)ell * (ell | 1) + 2 * (size_t)ell);
    chol_inv_kernel<false><<<1, 256, 0, ctx->stream>>>(ell, G, ldg, Rinv, ldr, shift_mode, ctx->sc, gws);
  } else {
    double* W = ctx->wsd("cg_W", (size_t)ell * ell);
    double* X = ctx->wsd("cg_X", (size_t)ell * (ell | 1));
    double* rowk = ctx->wsd("cg_rowk", (size_t)ell);
    double* rsq = ctx->wsd("cg_rsq", (size_t)ell);
    double* shiftp = ctx->wsd("cg_shift", 1);
    unsigned int* bar = (unsigned int*)ctx->ws("cg_bar", 64);
    NYS_CUDA_TRY(ctx, cudaMemsetAsync(bar, 0, 64, ctx->stream));
    int blocks = (int)(((int64_t)ell * ell / 2 + 1023) / 1024);   // ~one element of the first update per thread
    int occ = 0;
    NYS_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chol_inv_grid_kernel, 1024, 0));
    if (blocks > occ * ctx->num_sms) blocks = occ * ctx->num_sms;
    if (blocks > 64) blocks = 64;                  // grid barriers get slower with more CTAs
    if (blocks < 1) blocks = 1;
    double* scp = ctx->sc;
    void* args[] = {&ell, &G, &ldg, &Rinv, &ldr, &shift_mode, &scp, &W, &X, &rowk, &rsq, &shiftp, &bar};
    NYS_CUDA_TRY(ctx, cudaLaunchCooperativeKernel((const void*)chol_inv_grid_kernel, dim3(blocks), dim3(1024), args, 0,
                                                 ctx->stream));
  }
  ctx->launches++;
  return ctx->check_launch("chol_inv");
}

// Out = R1 * R2 for upper-triangular ell x ell (all with leading dimension ld)
__global__ void trmm_upper_kernel(int n, int ld, const double* R1, const double* R2, double* Out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int i = e % n, j = e / n;
    double s = 0.0;
    if (i <= j)
      for (int k = i; k <= j; ++k) s = fma(R1[i + k * ld], R2[k + j * ld], s);
    Out[i + j * ld] = s;
  }
}
int launch_trmm_upper(nys_ctx* ctx, int ell, int ld, const double* R1, const double* R2, double* Out) {
  int g = (ell * ell + 255) / 256;
  trmm_upper_kernel<<<g, 256, 0, ctx->stream>>>(ell, ld, R1, R2, Out);
  ctx->launches++;
  return ctx->check_launch("trmm_upper");
}

// ------------------------------------------------------------------------------------------
// one-sided Jacobi on X = R^T (ell x ell): X V = U_X Sigma; then R = V Sigma U_X^T, so the LEFT
// singular vectors of R are the accumulated rotations V (orthonormal to rounding).
// Round-robin (circle) ordering: ell/2 disjoint pairs per round, one warp per pair; column norms
// are recomputed exactly each sweep and updated incrementally within it (alpha' = alpha - t gamma,
// beta' = beta + t gamma), so each pair needs a single dot product.  The rotation angle uses
// fast reciprocal / square-root approximations refined by Newton steps: only c needs full
// accuracy (c^2 + s^2 = 1 keeps V orthogonal); t only steers convergence.
// Output: V (ell x ell, ld ldv) and sigma sorted descending (columns of V permuted to match).
// ------------------------------------------------------------------------------------------
// One warp per column pair (E = NMAX / 32 elements per lane, fully unrolled and predicated): a
// round costs one dot product (5 shuffle levels), one rotation and the two column updates.
// Rotation (symmetric Schur, fp64): zeta = (beta - alpha) / (2 gamma),
// t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), c = (1 + t^2)^{-1/2}, s = c t; the reciprocal and
// rsqrt come from fp32 seeds refined by Newton steps.  Only c needs full fp64 accuracy given t
// (c^2 (1 + t^2) = 1 keeps V orthogonal whatever t is): the rsqrts take two Newton steps from the
// ~2^-22 fp32 seed (error ~2^-44 -> below 2^-53).  zeta and t steer the rotation and the incremental
// norm update alpha - t gamma, beta + t gamma (norms are recomputed exactly every sweep): one step
// each (relative error ~2^-44, a residual coupling ~1e-13 gamma that the next sweep removes).
// seeds straight from the fp64 MUFU approximations (rcp / rsqrt .approx.ftz.f64, ~2^-22 relative):
// no fp64 <-> fp32 conversions on the rotation's dependency chain
__device__ __forceinline__ double rcp_seed(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ double rsqrt_seed(double y) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  return r;
}
__device__ __forceinline__ double fast_rcp1(double x) {
  const double ax = fabs(x);
  if (!(ax > 1e-30 && ax < 1e30)) return 1.0 / x;
  const double r = rcp_seed(x);
  return r * fma(-x, r, 2.0);
}
__device__ __forceinline__ double fast_rsqrt2(double y) {  // y in [1, 1e30)
  double r = rsqrt_seed(y);
  const double hy = -0.5 * y;
  r = r * fma(hy * r, r, 1.5);
  r = r * fma(hy * r, r, 1.5);
  return r;
}
__device__ __forceinline__ void jacobi_rotation(double al, double be, double ga, double& c, double& s, double& t) {
  const double zeta = (be - al) * 0.5 * fast_rcp1(ga);
  const double az = fabs(zeta);
  if (az > 1e8) {
    t = 0.5 * fast_rcp1(zeta);
  } else {
    const double y = fma(zeta, zeta, 1.0);
    t = copysign(fast_rcp1(az + y * fast_rsqrt2(y)), zeta);
  }
  c = fast_rsqrt2(fma(t, t, 1.0));
  s = c * t;
}

// Rotation of the pair (x_p, x_q), al = ||x_p||^2, be = ||x_q||^2, ga = x_p^T x_q, d = al - be:
// x_p' = c x_p - s x_q, x_q' = s x_p + c x_q with x_p'^T x_q' = (1/2) sin 2t d + cos 2t ga = 0, |t| <= pi/4:
//   ir = (d^2 + 4 ga^2)^{-1/2}, cos 2t = |d| ir, c^2 = (1 + cos 2t) / 2, c = c^2 (c^2)^{-1/2},
//   s = sin 2t / (2c) = -sgn(d) ga ir (c^2)^{-1/2}, tan t = s / c = s (c^2)^{-1/2};
// c^2 + s^2 = 1 up to the two rsqrt roundings (each refined to full fp64 precision), and the norms
// update as al - tan(t) ga, be + tan(t) ga (jacobi_kernel's incremental update).
__device__ __forceinline__ bool jacobi_rotation_rsqrt(double al, double be, double ga, double& c, double& sn,
                                                      double& t) {
  const double d = al - be;
  const double q = fma(d, d, 4.0 * ga * ga);
  const bool ok = q >= 1e-290 && q <= 1e290;
  const double ir = fast_rsqrt2(ok ? q : 1.0);
  const double c2 = fma(0.5, fabs(d) * ir, 0.5);
  const double rc = fast_rsqrt2(c2);                    // c2 in [1/2, 1]
  const double g = (d < 0.0 ? ga : -ga) * ir;           // -sgn(d) ga ir  (sgn(0) = +1)
  c = c2 * rc;
  sn = g * rc;
  t = sn * rc;
  return ok;
}

// rsqrt form, with the zeta / t form for out-of-range inputs (warp-uniform in the one-warp-per-pair kernels)
__device__ __forceinline__ void jacobi_rot(double al, double be, double ga, double& c, double& sn, double& t) {
  if (!jacobi_rotation_rsqrt(al, be, ga, c, sn, t)) jacobi_rotation(al, be, ga, c, sn, t);
}

template <int NMAX, bool SM>
__global__ void __launch_bounds__(1024) jacobi_kernel(int n, const double* R, int ldr, double* Vout, int ldv,
                                                      double* sigma, double* gws, double* jsweeps, long long* jdbg) {
  constexpr int E = NMAX / 32;
  extern __shared__ double jsm[];
  double* X = SM ? jsm : gws;
  double* V = X + (size_t)n * n;
  __shared__ int rotated;
  __shared__ double abs_floor;
  __shared__ double sv[NMAX];
  __shared__ int order[NMAX];
  __shared__ double nrm[NMAX];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e % n, j = e / n;
    X[i + j * n] = R[j + i * ldr];  // X = R^T
    V[i + j * n] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int P = (n % 2 == 0) ? n : n + 1;
  const int nwarp = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double tol = fmax(1e-15, (double)n * 0x1p-53);
  const double tol2 = tol * tol;
  auto wsum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    for (int j = warp; j < n; j += nwarp) {    // exact column norms
      double a = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = lane + 32 * e;
        if (i < n) a = fma(X[i + j * n], X[i + j * n], a);
      }
      a = wsum(a);
      if (lane == 0) nrm[j] = a;
    }
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    // absolute floor of the rotation test: a coupling |x_p^T x_q| below eps^2-level of the largest
    // column norm^2 changes X^T X = R R^T by far less than the Nystrom shift nu (~eps ||Y||) that
    // Alg. 1 line 8 subtracts anyway, so such pairs are left alone (pairs of noise-level columns
    // otherwise keep rotating on rounding for the full sweep cap)
    if (warp == 0) {
      double mx = 0.0;
      for (int j = lane; j < n; j += 32) mx = fmax(mx, nrm[j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) abs_floor = 1e-2 * 0x1p-52 * mx;
    }
    __syncthreads();
    const double floor_g = abs_floor;
    for (int r = 0; r < P - 1; ++r) {
      for (int pi = warp; pi < P / 2; pi += nwarp) {
        int a, b;
        if (pi == 0) { a = r; b = P - 1; }
        else {
          a = r + pi; if (a >= P - 1) a -= P - 1;
          b = r - pi; if (b < 0) b += P - 1;
        }
        if (a >= n || b >= n) continue;         // the dummy column of odd n (warp-uniform)
        const int p = a < b ? a : b, q = a < b ? b : a;
        // X and V columns loaded together up front (the V loads would otherwise wait behind the
        // X stores of the rotation: same shared array, possible aliasing)
        long long tj0 = 0, tj1 = 0, tj2 = 0, tj3 = 0;
        const bool jtr = jdbg != nullptr && warp == 0 && lane == 0 && sweep == 1 && r < 8;
        if (jtr) tj0 = clock64();
        double xp[E], xq[E], vp[E], vq[E];
        double ga = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = lane + 32 * e;
          xp[e] = (i < n) ? X[i + p * n] : 0.0;
          xq[e] = (i < n) ? X[i + q * n] : 0.0;
          vp[e] = (i < n) ? V[i + p * n] : 0.0;
          vq[e] = (i < n) ? V[i + q * n] : 0.0;
          ga = fma(xp[e], xq[e], ga);
        }
        ga = wsum(ga);
        if (jtr) tj1 = clock64();
        const double al = nrm[p], be = nrm[q];
        if (ga * ga > tol2 * al * be && fabs(ga) > floor_g) {   // warp-uniform
          double c, sn, t;
          jacobi_rot(al, be, ga, c, sn, t);
          if (jtr) tj2 = clock64();
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = lane + 32 * e;
            if (i < n) {
              X[i + p * n] = c * xp[e] - sn * xq[e];
              X[i + q * n] = sn * xp[e] + c * xq[e];
              V[i + p * n] = c * vp[e] - sn * vq[e];
              V[i + q * n] = sn * vp[e] + c * vq[e];
            }
          }
          if (jtr) {
            tj3 = clock64();
            jdbg[4 * r + 0] = tj1 - tj0;
            jdbg[4 * r + 1] = tj2 - tj1;
            jdbg[4 * r + 2] = tj3 - tj2;
          }
          if (lane == 0) {
            nrm[p] = fmax(al - t * ga, 0.0);
            nrm[q] = be + t * ga;
            rotated = 1;
          }
        }
      }
      __syncthreads();
      if (jdbg != nullptr && threadIdx.x == 0 && sweep == 1 && r < 8) {
        __shared__ long long jt_prev;
        const long long now = clock64();
        if (r > 0) jdbg[4 * r + 3] = now - jt_prev;
        jt_prev = now;
      }
    }
    if (!rotated) break;
    __syncthreads();
  }
  if (threadIdx.x == 0) jsweeps[0] = (double)(sweep + 1);
  // sigma_j = ||x_j||, then sort descending (rank sort, ties by index)
  for (int j = warp; j < n; j += nwarp) {
    double a = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = lane + 32 * e;
      if (i < n) a = fma(X[i + j * n], X[i + j * n], a);
    }
    a = wsum(a);
    if (lane == 0) sv[j] = sqrt(a);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    int rk = 0;
    for (int k = 0; k < n; ++k) rk += (sv[k] > sv[j]) || (sv[k] == sv[j] && k < j);
    order[rk] = j;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) sigma[j] = sv[order[j]];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e % n, j = e / n;
    Vout[i + j * ldv] = V[i + order[j] * n];
  }
}

// The same one-sided Jacobi with G lanes per column pair (32 / G pairs per warp) for small ell.  A round
// is a dependent chain (loads, dot, G-lane shuffle sum, rotation, update, barrier) with few warps to
// hide it, so this variant is written for a short chain and few instructions:
//   * X and V are stored with a padded leading dimension LD = G * E (rows n .. LD-1 stay zero: a
//     rotation of zeros is zero), so the loads and stores need no predicates or zero-fills;
//   * the rotation comes from two reciprocal square roots and no division (below), ~170 cycles of
//     dependent fp64 latency instead of ~400 for the zeta / t form; out-of-range inputs (never seen
//     in the Nystrom factor, whose column norms lie between nu and ||N||) take the zeta / t form for
//     the whole warp;
//   * a warp issues the rotation once for all its pairs.
// Measured at ell = 50 with one warp per pair: ~2700 cycles per round.  Same circle ordering,
// incremental norms, absolute floor, convergence test and output as jacobi_kernel.
//
template <int G, int E>
__global__ void __launch_bounds__(32 * ((G * E / 2 + 32 / G - 1) / (32 / G))) jacobi_packed_kernel(
    int n, const double* R, int ldr, double* Vout, int ldv, double* sigma, double* jsweeps, double kpred) {
  constexpr int PPW = 32 / G;
  constexpr int LD = G * E;
  extern __shared__ double jsm[];
  double* X = jsm;                    // [n][LD]  X = R^T, zero rows n .. LD-1
  double* V = X + (size_t)n * LD;     // [n][LD]
  __shared__ int rotated, big_rot;
  __shared__ double abs_floor;
  __shared__ double sv[LD];
  __shared__ int order[LD];
  __shared__ double nrm[LD];
  for (int e = threadIdx.x; e < n * LD; e += blockDim.x) {
    const int i = e % LD, j = e / LD;
    X[e] = (i < n) ? R[j + i * ldr] : 0.0;
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int P = (n % 2 == 0) ? n : n + 1;
  const int nwarp = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int pi = warp * PPW + lane / G;     // this group's pair slot (nwarp * PPW >= P / 2)
  const int ngroups = nwarp * PPW;
  const double tol = fmax(1e-15, (double)n * 0x1p-53);
  const double tol2 = tol * tol;
  auto gsum = [&](double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  auto colnorm2 = [&](int j) {
    const double* xj = X + (size_t)j * LD + gl;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & 1) a1 = fma(xj[G * e], xj[G * e], a1);
      else a0 = fma(xj[G * e], xj[G * e], a0);
    }
    return gsum(a0 + a1);
  };
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    for (int j0 = 0; j0 < n; j0 += ngroups) {   // exact column norms (group-uniform trip count)
      const int j = j0 + pi;
      const double a = colnorm2(j < n ? j : 0);
      if (gl == 0 && j < n) nrm[j] = a;
    }
    if (threadIdx.x == 0) { rotated = 0; big_rot = 0; }
    __syncthreads();
    if (warp == 0) {   // absolute floor of the rotation test (as jacobi_kernel)
      double mx = 0.0;
      for (int j = lane; j < n; j += 32) mx = fmax(mx, nrm[j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) abs_floor = 1e-2 * 0x1p-52 * mx;
    }
    __syncthreads();
    const double floor_g = abs_floor;
    for (int r = 0; r < P - 1; ++r) {
      int a, b;
      if (pi == 0) { a = r; b = P - 1; }
      else {
        a = r + pi; if (a >= P - 1) a -= P - 1;
        b = r - pi; if (b < 0) b += P - 1;
      }
      const bool valid = pi < P / 2 && a < n && b < n;   // group-uniform (the dummy column of odd n)
      const int p = valid ? (a < b ? a : b) : 0, q = valid ? (a < b ? b : a) : 0;
      double* xp_ = X + (size_t)p * LD + gl;
      double* xq_ = X + (size_t)q * LD + gl;
      double* vp_ = V + (size_t)p * LD + gl;
      double* vq_ = V + (size_t)q * LD + gl;
      const double al0 = nrm[p], be0 = nrm[q];
      double xp[E], xq[E], vp[E], vq[E];
      double g0 = 0.0, g1 = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        xp[e] = xp_[G * e];
        xq[e] = xq_[G * e];
        vp[e] = vp_[G * e];
        vq[e] = vq_[G * e];
        if (e & 1) g1 = fma(xp[e], xq[e], g1);
        else g0 = fma(xp[e], xq[e], g0);
      }
      const double ga = gsum(g0 + g1);
      const double al = valid ? al0 : 1.0, be = valid ? be0 : 1.0;
      const bool rot = valid && ga * ga > tol2 * al * be && fabs(ga) > floor_g;   // group-uniform
      double c, sn, t;
      const bool ok = jacobi_rotation_rsqrt(al, be, rot ? ga : 1.0, c, sn, t);   // once for all groups
      if (__any_sync(0xffffffffu, rot && !ok)) jacobi_rotation(al, be, rot ? ga : 1.0, c, sn, t);
      if (rot) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          xp_[G * e] = c * xp[e] - sn * xq[e];
          xq_[G * e] = sn * xp[e] + c * xq[e];
          vp_[G * e] = c * vp[e] - sn * vq[e];
          vq_[G * e] = sn * vp[e] + c * vq[e];
        }
        if (gl == 0) {
          nrm[p] = fmax(al - t * ga, 0.0);
          nrm[q] = be + t * ga;
          rotated = 1;
          if (kpred == 0.0 || ga * ga * kpred > tol * al * be) big_rot = 1;   // eta^2 > tol / kpred (jacobi_kpred)
        }
      }
      __syncthreads();
    }
    if (!rotated || !big_rot) break;
    __syncthreads();
  }
  if (threadIdx.x == 0) jsweeps[0] = (double)(sweep + 1);
  for (int j0 = 0; j0 < n; j0 += ngroups) {   // sigma_j = ||x_j||
    const int j = j0 + pi;
    const double a = colnorm2(j < n ? j : 0);
    if (gl == 0 && j < n) sv[j] = sqrt(a);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {   // rank sort descending, ties by index
    int rk = 0;
    for (int k = 0; k < n; ++k) rk += (sv[k] > sv[j]) || (sv[k] == sv[j] && k < j);
    order[rk] = j;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) sigma[j] = sv[order[j]];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e % n, j = e / n;
    Vout[i + j * ldv] = V[i + (size_t)order[j] * LD];
  }
}

// Early exit of the packed and block Jacobi: cyclic Jacobi converges
// quadratically, the largest relative coupling eta = |x_p^T x_q| / (||x_p|| ||x_q||) of a sweep being
// about the square of the previous sweep's.  A sweep that rotates only pairs with eta^2 <= tol / kpred
// (kpred = 1e4: eta <= 7.5e-10 at ell = 50) is the last working one: the next sweep would find every
// eta near eta^2 << tol and rotate nothing, so it is skipped (tools/jacobi_conv_sim.py: ell = 50 / 64
// histories 5e-4, 7e-7, 5e-13, 0).  If a near-tie of singular values slowed that last step, the residual
// coupling eta' ~ eta^2 / gap enters R R^T = V (X^T X) V^T as an O(eta') relative error of N_hat, below
// the operator parity bound.  NYS_JACOBI_VERIFY=1: always run the verifying sweep (kpred = 0).
static double jacobi_kpred() {
  static const double k = (getenv("NYS_JACOBI_VERIFY") && atoi(getenv("NYS_JACOBI_VERIFY")) != 0) ? 0.0 : 1e4;
  return k;
}

template <int G, int E>
static int launch_jacobi_packed(nys_ctx* ctx, int ell, const double* R, int ldr, double* V, int ldv, double* sigma) {
  constexpr int PPW = 32 / G;
  const size_t need = 2 * (size_t)ell * G * E * sizeof(double);
  const int pairs = (ell + 1) / 2;
  const int warps = (pairs + PPW - 1) / PPW;
  auto k = jacobi_packed_kernel<G, E>;
  NYS_TRY(ensure_max_smem(ctx, (const void*)k, need > 48 * 1024 ? need : 48 * 1024));
  k<<<1, 32 * warps, need, ctx->stream>>>(ell, R, ldr, V, ldv, sigma, ctx->sc + S_JSWEEPS, jacobi_kpred());
  ctx->launches++;
  return ctx->check_launch("jacobi_packed");
}

// The same one-sided Jacobi for ell > 113 (X and V no longer fit one CTA's shared memory): a
// thread-block CLUSTER of C CTAs holds the columns cyclically (column j in CTA j % C, slot j / C) and
// every pair reads / writes its four columns and two norms through distributed shared memory; a
// cluster barrier separates the rounds.  Same ordering, rotation, convergence test and output.
template <int NMAX, int C>
__global__ void __launch_bounds__(1024) jacobi_cluster_kernel(int n, const double* R, int ldr, double* Vout, int ldv,
                                                              double* sigma, double* jsweeps) {
  constexpr int E = NMAX / 32;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  extern __shared__ double jsm[];
  const int ncl = (n + C - 1) / C;
  double* Xl = jsm;                       // local slot t = global column rank + C t, ld n
  double* Vl = jsm + (size_t)ncl * n;
  __shared__ double nrm_l[NMAX / C + 1];
  __shared__ double flag_l[2];            // [0] max column norm^2 of this CTA, [1] rotated in this sweep
  __shared__ double sv_all[NMAX];
  __shared__ int order[NMAX];
  auto xcol = [&](int j) { return cl.map_shared_rank(Xl + (size_t)(j / C) * n, j % C); };
  auto vcol = [&](int j) { return cl.map_shared_rank(Vl + (size_t)(j / C) * n, j % C); };
  auto nrmp = [&](int j) { return cl.map_shared_rank(nrm_l + j / C, j % C); };
  for (int e = threadIdx.x; e < ncl * n; e += blockDim.x) {
    const int t = e / n, i = e % n, j = rank + C * t;
    Xl[e] = (j < n) ? R[j + (size_t)i * ldr] : 0.0;  // X = R^T
    Vl[e] = (j < n && i == j) ? 1.0 : 0.0;
  }
  const int P = (n % 2 == 0) ? n : n + 1;
  const int nwarp = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double tol = fmax(1e-15, (double)n * 0x1p-53);
  const double tol2 = tol * tol;
  auto wsum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  __syncthreads();
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    for (int t = warp; t < ncl; t += nwarp) {  // exact norms of the local columns
      double a = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = lane + 32 * e;
        if (i < n) a = fma(Xl[i + (size_t)t * n], Xl[i + (size_t)t * n], a);
      }
      a = wsum(a);
      if (lane == 0) nrm_l[t] = (rank + C * t < n) ? a : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double mx = 0.0;
      for (int t = 0; t < ncl; ++t) mx = fmax(mx, nrm_l[t]);
      flag_l[0] = mx;
      flag_l[1] = 0.0;
    }
    cl.sync();
    double mxall = 0.0;
    for (int r = 0; r < C; ++r) mxall = fmax(mxall, *cl.map_shared_rank(&flag_l[0], r));
    const double floor_g = 1e-2 * 0x1p-52 * mxall;   // as jacobi_kernel
    for (int r = 0; r < P - 1; ++r) {
      for (int pi = rank + C * warp; pi < P / 2; pi += C * nwarp) {
        int a, b;
        if (pi == 0) { a = r; b = P - 1; }
        else {
          a = r + pi; if (a >= P - 1) a -= P - 1;
          b = r - pi; if (b < 0) b += P - 1;
        }
        if (a >= n || b >= n) continue;
        const int p = a < b ? a : b, q = a < b ? b : a;
        double* Xp = xcol(p);
        double* Xq = xcol(q);
        double* Vp = vcol(p);
        double* Vq = vcol(q);
        double xp[E], xq[E], vp[E], vq[E];
        double ga = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = lane + 32 * e;
          xp[e] = (i < n) ? Xp[i] : 0.0;
          xq[e] = (i < n) ? Xq[i] : 0.0;
          vp[e] = (i < n) ? Vp[i] : 0.0;
          vq[e] = (i < n) ? Vq[i] : 0.0;
          ga = fma(xp[e], xq[e], ga);
        }
        ga = wsum(ga);
        double* np_ = nrmp(p);
        double* nq_ = nrmp(q);
        const double al = *np_, be = *nq_;
        if (ga * ga > tol2 * al * be && fabs(ga) > floor_g) {
          double c, sn, t;
          jacobi_rot(al, be, ga, c, sn, t);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = lane + 32 * e;
            if (i < n) {
              Xp[i] = c * xp[e] - sn * xq[e];
              Xq[i] = sn * xp[e] + c * xq[e];
              Vp[i] = c * vp[e] - sn * vq[e];
              Vq[i] = sn * vp[e] + c * vq[e];
            }
          }
          if (lane == 0) {
            *np_ = fmax(al - t * ga, 0.0);
            *nq_ = be + t * ga;
            flag_l[1] = 1.0;
          }
        }
      }
      cl.sync();
    }
    bool any = false;
    for (int r = 0; r < C; ++r) any = any || (*cl.map_shared_rank(&flag_l[1], r) != 0.0);
    cl.sync();  // every CTA has read the flags before the next sweep resets them
    if (!any) break;
  }
  if (rank == 0 && threadIdx.x == 0) jsweeps[0] = (double)(sweep + 1);
  for (int t = warp; t < ncl; t += nwarp) {  // sigma of the local columns
    double a = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = lane + 32 * e;
      if (i < n) a = fma(Xl[i + (size_t)t * n], Xl[i + (size_t)t * n], a);
    }
    a = wsum(a);
    if (lane == 0) nrm_l[t] = sqrt(a);
  }
  cl.sync();
  for (int j = threadIdx.x; j < n; j += blockDim.x) sv_all[j] = *nrmp(j);
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {  // rank sort, ties by index (every CTA the same)
    int rk = 0;
    for (int k = 0; k < n; ++k) rk += (sv_all[k] > sv_all[j]) || (sv_all[k] == sv_all[j] && k < j);
    order[rk] = j;
  }
  __syncthreads();
  for (int jo = rank; jo < n; jo += C) {
    const double* src = vcol(order[jo]);
    if (threadIdx.x == 0) sigma[jo] = sv_all[order[jo]];
    for (int i = threadIdx.x; i < n; i += blockDim.x) Vout[i + (size_t)jo * ldv] = src[i];
  }
  cl.sync();  // no CTA leaves while a peer still reads its shared memory
}

// Block one-sided Jacobi over a cluster of C CTAs (ell > 112): the columns form 2C blocks of
// bs = ceil(ell / 2C); each CTA holds two blocks (a "top" and a "bottom" slot, plus a spare) in its
// OWN shared memory and processes their column pairs locally (one warp per pair, a CTA barrier per
// local round); between block rounds the blocks move one position along the round-robin ring
// (t_1 .. t_{C-1}, b_{C-1} .. b_0; t_0 fixed) through two DSMEM pushes into free slots.  Block round 0
// of a sweep pairs every column of the two blocks (the within-block pairs), the other 2C - 2 rounds
// the cross pairs only, so each pair of columns meets once per sweep (a cyclic ordering).  Same
// rotation, incremental norms, convergence test and output as jacobi_kernel.  Shared memory is read
// remotely only by the block moves, never per pair (per-pair DSMEM traffic made the column-cyclic
// cluster kernel ~11 us per round).
template <int G, int E, int C>
__global__ void __launch_bounds__(512 * G / 32) jacobi_block_kernel(int n, int bs, const double* R, int ldr, double* Vout,
                                                            int ldv, double* sigma, double* jsweeps, double kpred) {
  // Columns are stored with a padded stride LDc = 32 E (rows n .. LDc-1 zero: a rotation of zeros is
  // zero), so a pair's loads and stores need no predicates; every slot access is an offset into the
  // CTA's own shared array (LDS / STS, not generic loads); the roles of a pair (which column plays "p")
  // are resolved once per pair, not per element.  (Measured on B200 at ell = 200 before these changes:
  // ~650 instructions and ~5000 cycles per local round, mostly integer address arithmetic and selects.)
  // G lanes per column pair (32 / G pairs per warp, as jacobi_packed_kernel): E = ceil(n / G)
  constexpr int LDc = G * E;
  constexpr int PPW = 32 / G;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  extern __shared__ double jsm[];
  // slot layout (offsets into jsm): X (bs columns x LDc), V (bs x LDc), nrm (bs), block id (1), pad
  const int slot = (2 * bs * LDc + bs + 2 + 1) & ~1;   // even: 16-byte aligned slots
  __shared__ int smap[3];             // this CTA's slot indices of (top, bottom, spare); read by peers
  __shared__ double flag_l[3];          // [0] max column norm^2, [1] rotated, [2] rotated with eta^2 > tol / kpred
  __shared__ double sv_all[256];
  __shared__ int order[256];
  if (threadIdx.x == 0) { smap[0] = 0; smap[1] = 1; smap[2] = 2; }
  int top = 0, bot = 1, spare = 2;
  const int nwarp = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gl = lane % G, gslot = warp * PPW + lane / G, ngs = nwarp * PPW;   // pair slot of this lane group
  auto Xo = [&](int s, int j) { return s * slot + j * LDc; };
  auto Vo = [&](int s, int j) { return s * slot + (bs + j) * LDc; };
  auto No = [&](int s) { return s * slot + 2 * bs * LDc; };
  auto Bo = [&](int s) { return s * slot + 2 * bs * LDc + bs; };
  auto cnt = [&](int b) { const int c0 = b * bs; return c0 >= n ? 0 : (n - c0 < bs ? n - c0 : bs); };
  // initial blocks: t_c = block c, b_c = block 2C - 1 - c
  for (int w = 0; w < 2; ++w) {
    const int b = (w == 0) ? rank : 2 * C - 1 - rank;
    for (int e = threadIdx.x; e < bs * LDc; e += blockDim.x) {
      const int j = e / LDc, i = e % LDc, gj = b * bs + j;
      jsm[Xo(w, j) + i] = (j < cnt(b) && i < n) ? R[gj + (size_t)i * ldr] : 0.0;   // X = R^T
      jsm[Vo(w, j) + i] = (j < cnt(b) && i == gj) ? 1.0 : 0.0;
    }
    if (threadIdx.x == 0) jsm[Bo(w)] = (double)b;
  }
  const double tol = fmax(1e-15, (double)n * 0x1p-53);
  const double tol2 = tol * tol;
  auto gsum = [&](double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  auto colnorm2 = [&](int off) {   // a whole warp per column
    double a0 = 0.0;
    for (int i = lane; i < LDc; i += 32) a0 = fma(jsm[off + i], jsm[off + i], a0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    return a0;
  };
  __syncthreads();
  // one pair (p, q) of LOCAL columns: p, q in [0, 2 bs) (< bs: top slot, else bottom slot); bt / bb:
  // the block ids in the top / bottom slots
  // (valid: group-uniform; every lane of the warp runs the shuffles)
  auto do_pair = [&](int p, int q, bool valid, double floor_g, int bt, int bb) {
    const int sp = p < bs ? top : bot, sq = q < bs ? top : bot;
    const int jp = p < bs ? p : p - bs, jq = q < bs ? q : q - bs;
    const int bp = p < bs ? bt : bb, bq = q < bs ? bt : bb;
    valid = valid && jp < cnt(bp) && jq < cnt(bq);
    // the global column with the smaller index plays "p" (as in the column-cyclic kernels)
    const bool swp = (bp * bs + jp) > (bq * bs + jq);
    const int s0 = swp ? sq : sp, j0 = swp ? jq : jp, s1 = swp ? sp : sq, j1 = swp ? jp : jq;
    const int x0 = valid ? Xo(s0, j0) : 0, x1 = valid ? Xo(s1, j1) : 0, v0 = valid ? Vo(s0, j0) : 0,
              v1 = valid ? Vo(s1, j1) : 0;
    const int n0 = No(s0) + j0, n1 = No(s1) + j1;
    const double al = valid ? jsm[n0] : 1.0, be = valid ? jsm[n1] : 1.0;
    double a0[E], a1[E], w0[E], w1[E];
    double g0 = 0.0, g1 = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = gl + G * e;
      a0[e] = jsm[x0 + i];
      a1[e] = jsm[x1 + i];
      w0[e] = jsm[v0 + i];
      w1[e] = jsm[v1 + i];
      if (e & 1) g1 = fma(a0[e], a1[e], g1);
      else g0 = fma(a0[e], a1[e], g0);
    }
    const double ga = gsum(g0 + g1);
    const bool rot = valid && ga * ga > tol2 * al * be && fabs(ga) > floor_g;   // group-uniform
    double c, sn, t;
    const bool ok = jacobi_rotation_rsqrt(al, be, rot ? ga : 1.0, c, sn, t);   // once for all groups
    if (__any_sync(0xffffffffu, rot && !ok)) jacobi_rotation(al, be, rot ? ga : 1.0, c, sn, t);
    if (rot) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = gl + G * e;
        jsm[x0 + i] = c * a0[e] - sn * a1[e];
        jsm[x1 + i] = sn * a0[e] + c * a1[e];
        jsm[v0 + i] = c * w0[e] - sn * w1[e];
        jsm[v1 + i] = sn * w0[e] + c * w1[e];
      }
      if (gl == 0) {
        jsm[n0] = fmax(al - t * ga, 0.0);
        jsm[n1] = be + t * ga;
        flag_l[1] = 1.0;
        if (kpred == 0.0 || ga * ga * kpred > tol * al * be) flag_l[2] = 1.0;   // jacobi_kpred
      }
    }
  };
  // move a slot's contents (X, V, nrm, id) into a peer's slot (DSMEM, 16-byte stores)
  auto push = [&](int src_slot, int dst_rank, int dst_slot_idx) {
    double* dst = cl.map_shared_rank(jsm + (size_t)dst_slot_idx * slot, dst_rank);
    const int nv = slot / 2;
    const double2* s2 = reinterpret_cast<const double2*>(jsm + (size_t)src_slot * slot);
    double2* d2 = reinterpret_cast<double2*>(dst);
    for (int e = threadIdx.x; e < nv; e += blockDim.x) d2[e] = s2[e];
  };
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    for (int w = 0; w < 2; ++w) {  // exact norms of the local columns
      const int S = w == 0 ? top : bot;
      for (int j = warp; j < bs; j += nwarp) {
        const double a = colnorm2(Xo(S, j));
        if (lane == 0) jsm[No(S) + j] = a;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double mx = 0.0;
      for (int j = 0; j < bs; ++j) mx = fmax(mx, fmax(jsm[No(top) + j], jsm[No(bot) + j]));
      flag_l[0] = mx;
      flag_l[1] = 0.0;
      flag_l[2] = 0.0;
    }
    cl.sync();
    double mxall = 0.0;
    for (int r = 0; r < C; ++r) mxall = fmax(mxall, *cl.map_shared_rank(&flag_l[0], r));
    const double floor_g = 1e-2 * 0x1p-52 * mxall;
    for (int br = 0; br < 2 * C - 1; ++br) {
      const int bt = (int)jsm[Bo(top)], bb = (int)jsm[Bo(bot)];
      if (br == 0) {                                   // all pairs of the 2 bs local columns
        const int P2 = 2 * bs;                         // even
        for (int r = 0; r < P2 - 1; ++r) {
          for (int base = 0; base < P2 / 2; base += ngs) {   // warp-uniform trip count
            const int pi = base + gslot;
            int a, b;
            if (pi == 0) { a = r; b = P2 - 1; }
            else {
              a = r + pi; if (a >= P2 - 1) a -= P2 - 1;
              b = r - pi; if (b < 0) b += P2 - 1;
            }
            const bool v = pi < P2 / 2;
            do_pair(v ? (a < b ? a : b) : 0, v ? (a < b ? b : a) : 1, v, floor_g, bt, bb);
          }
          __syncthreads();
        }
      } else {                                         // cross pairs (top i, bottom (i + r) mod bs)
        for (int r = 0; r < bs; ++r) {
          for (int base = 0; base < bs; base += ngs) {
            const int i = base + gslot;
            int k = i + r;
            if (k >= bs) k -= bs;
            const bool v = i < bs;
            do_pair(v ? i : 0, v ? bs + k : bs, v, floor_g, bt, bb);
          }
          __syncthreads();
        }
      }
      // ---- move the blocks one position along the ring -----------------------------------------
      cl.sync();                                       // every CTA finished with its blocks
      // phase A: t_c -> t_{c+1} (c = 1 .. C-2), b_0 -> t_1; t_{C-1} becomes b_{C-1} locally (below)
      if (rank >= 1 && rank <= C - 2) push(top, rank + 1, *cl.map_shared_rank(&smap[2], rank + 1));
      if (rank == 0) push(bot, 1, *cl.map_shared_rank(&smap[2], 1));
      cl.sync();
      // phase B: b_c -> b_{c-1} (c = 1 .. C-1) into the slot freed in phase A
      //   (CTA c - 1 >= 1: its old top slot; CTA 0: its old bottom slot)
      if (rank >= 1) push(bot, rank - 1, *cl.map_shared_rank(&smap[rank - 1 >= 1 ? 0 : 1], rank - 1));
      cl.sync();
      // slot renaming: CTA 0 keeps its slots (its bottom slot was refilled in phase B); the others take
      // the spare (filled in phase A) as top, the old top (refilled in B, or relabelled at C - 1) as
      // bottom, and the old bottom (sent in B) as spare
      if (rank != 0) {
        const int nt = spare, nb = top, ns = bot;
        top = nt; bot = nb; spare = ns;
      }
      if (threadIdx.x == 0) { smap[0] = top; smap[1] = bot; smap[2] = spare; }
      cl.sync();                                       // peers read smap only after this
    }
    bool any = false, big = false;
    for (int r = 0; r < C; ++r) {
      any = any || (*cl.map_shared_rank(&flag_l[1], r) != 0.0);
      big = big || (*cl.map_shared_rank(&flag_l[2], r) != 0.0);
    }
    cl.sync();
    if (!any || !big) break;
  }
  if (rank == 0 && threadIdx.x == 0) jsweeps[0] = (double)(sweep + 1);
  // sigma of the local columns
  for (int w = 0; w < 2; ++w) {
    const int S = w == 0 ? top : bot;
    for (int j = warp; j < bs; j += nwarp) {
      const double a = colnorm2(Xo(S, j));
      if (lane == 0) jsm[No(S) + j] = sqrt(a);
    }
  }
  __syncthreads();
  // every CTA publishes (global index -> sigma) of its two live blocks into sv_all of every peer
  for (int w = 0; w < 2; ++w) {
    const int S = w == 0 ? top : bot;
    const int b = (int)jsm[Bo(S)];
    for (int j = threadIdx.x; j < cnt(b); j += blockDim.x)
      for (int r = 0; r < C; ++r) *cl.map_shared_rank(&sv_all[b * bs + j], r) = jsm[No(S) + j];
  }
  cl.sync();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {  // rank sort, ties by index (the same in every CTA)
    int rk = 0;
    for (int k = 0; k < n; ++k) rk += (sv_all[k] > sv_all[j]) || (sv_all[k] == sv_all[j] && k < j);
    order[rk] = j;
  }
  __syncthreads();
  // each CTA writes the output columns whose source column it holds
  for (int w = 0; w < 2; ++w) {
    const int S = w == 0 ? top : bot;
    const int b = (int)jsm[Bo(S)];
    for (int jo = 0; jo < n; ++jo) {
      const int src = order[jo];
      if (src / bs != b || src - b * bs >= cnt(b)) continue;
      const int vo = Vo(S, src - b * bs);
      if (threadIdx.x == 0) sigma[jo] = sv_all[src];
      for (int i = threadIdx.x; i < n; i += blockDim.x) Vout[i + (size_t)jo * ldv] = jsm[vo + i];
    }
  }
  cl.sync();
}

template <int C>
static int launch_jacobi_cluster(nys_ctx* ctx, int ell, const double* R, int ldr, double* V, int ldv, double* sigma,
                                 size_t smem) {
  auto k = jacobi_cluster_kernel<256, C>;
  NYS_TRY(ensure_max_smem(ctx, (const void*)k, smem));
  int warps = ((ell + 1) / 2 + C - 1) / C;
  if (warps > 32) warps = 32;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(32 * warps);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  NYS_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, k, ell, R, ldr, V, ldv, sigma, ctx->sc + S_JSWEEPS));
  return NYS_OK;
}

template <int G, int E, int C>
static int launch_jacobi_block_ec(nys_ctx* ctx, int ell, const double* R, int ldr, double* V, int ldv, double* sigma) {
  const int bs = (ell + 2 * C - 1) / (2 * C);
  const size_t slot = ((size_t)2 * bs * G * E + bs + 2 + 1) & ~(size_t)1;
  const size_t smem = 3 * slot * sizeof(double);
  if (smem > 220 * 1024) { ctx->set_error("jacobi_block: blocks do not fit shared memory"); return NYS_EINVAL; }
  auto k = jacobi_block_kernel<G, E, C>;
  NYS_TRY(ensure_max_smem(ctx, (const void*)k, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(32 * ((bs < 1 ? 1 : bs) + 32 / G - 1) / (32 / G));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  NYS_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, k, ell, bs, R, ldr, V, ldv, sigma, ctx->sc + S_JSWEEPS, jacobi_kpred()));
  return NYS_OK;
}
template <int C>
static int launch_jacobi_block_c(nys_ctx* ctx, int ell, const double* R, int ldr, double* V, int ldv, double* sigma) {
  // (16 lanes per pair measured at ell = 200: 2.81 vs 3.06 ms but one more sweep on other inputs, and
  //  no gain at ell = 80 / 100: one warp per pair here)
  switch ((ell + 31) / 32) {   // E = elements per lane (padded column stride 32 E)
    case 1: case 2: case 3: return launch_jacobi_block_ec<32, 3, C>(ctx, ell, R, ldr, V, ldv, sigma);
    case 4: return launch_jacobi_block_ec<32, 4, C>(ctx, ell, R, ldr, V, ldv, sigma);
    case 5: return launch_jacobi_block_ec<32, 5, C>(ctx, ell, R, ldr, V, ldv, sigma);
    case 6: return launch_jacobi_block_ec<32, 6, C>(ctx, ell, R, ldr, V, ldv, sigma);
    case 7: return launch_jacobi_block_ec<32, 7, C>(ctx, ell, R, ldr, V, ldv, sigma);
    default: return launch_jacobi_block_ec<32, 8, C>(ctx, ell, R, ldr, V, ldv, sigma);
  }
}
// cluster size 8 (measured best or equal from ell = 64 to 200 against clusters of 2 and 4); the
// override must keep bs = ceil(ell / 2C) <= 16 (one warp per pair, 512 threads)
static int launch_jacobi_block(nys_ctx* ctx, int ell, const double* R, int ldr, double* V, int ldv, double* sigma) {
  int C = 8;
  if (const char* e = getenv("NYS_JACOBI_C")) C = atoi(e);
  if ((ell + 2 * C - 1) / (2 * C) > 16) C = 8;
  if (C == 2) return launch_jacobi_block_c<2>(ctx, ell, R, ldr, V, ldv, sigma);
  if (C == 4) return launch_jacobi_block_c<4>(ctx, ell, R, ldr, V, ldv, sigma);
  return launch_jacobi_block_c<8>(ctx, ell, R, ldr, V, ldv, sigma);
}

template <int NMAX>
static int launch_jacobi_t(nys_ctx* ctx, int ell, const double* R, int ldr, double* V, int ldv, double* sigma) {
  const size_t need = 2 * (size_t)ell * ell * sizeof(double);
  const int pairs = (ell + 1) / 2;
  int nthr = 32 * pairs;
  if (nthr > 1024) nthr = 1024;
  if (need <= 200 * 1024) {
    NYS_TRY(ensure_max_smem(ctx, (const void*)jacobi_kernel<NMAX, true>, 200 * 1024));
    long long* jdbg = getenv("NYS_JACOBI_TRACE") ? (long long*)ctx->ws("jac_dbg", 32 * 8) : nullptr;
    jacobi_kernel<NMAX, true><<<1, nthr, need, ctx->stream>>>(ell, R, ldr, V, ldv, sigma, nullptr, ctx->sc + S_JSWEEPS, jdbg);
    if (jdbg) {
      long long h[32];
      cudaMemcpyAsync(h, jdbg, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream);
      cudaStreamSynchronize(ctx->stream);
      for (int r = 1; r < 8; ++r)
        fprintf(stderr, "[jactrace] ell=%d round=%d dot=%lld rot=%lld upd=%lld round_total=%lld cycles\n", ell, r, h[4 * r],
                h[4 * r + 1], h[4 * r + 2], h[4 * r + 3]);
    }
  } else {
    // cluster of C CTAs: the smallest C whose per-CTA share of X and V fits 208 KB
    int C = 2;
    while (C < 8 && 2 * (size_t)((ell + C - 1) / C) * ell * sizeof(double) > 208 * 1024) C *= 2;
    const size_t smem = 2 * (size_t)((ell + C - 1) / C) * ell * sizeof(double);
    if (NMAX == 256 && getenv("NYS_JACOBI_CYCLIC") == nullptr && getenv("NYS_JACOBI_GLOBAL") == nullptr) {
      NYS_TRY(launch_jacobi_block(ctx, ell, R, ldr, V, ldv, sigma));   // block Jacobi over 8 CTAs
    } else if (NMAX == 256 && smem <= 208 * 1024 && getenv("NYS_JACOBI_GLOBAL") == nullptr) {
      if (C == 2) NYS_TRY(launch_jacobi_cluster<2>(ctx, ell, R, ldr, V, ldv, sigma, smem));
      else if (C == 4) NYS_TRY(launch_jacobi_cluster<4>(ctx, ell, R, ldr, V, ldv, sigma, smem));
      else NYS_TRY(launch_jacobi_cluster<8>(ctx, ell, R, ldr, V, ldv, sigma, smem));
    } else {
      double* gws = ctx->wsd("jacobi_ws", 2 * (size_t)ell * ell);
      jacobi_kernel<NMAX, false><<<1, nthr, 0, ctx->stream>>>(ell, R, ldr, V, ldv, sigma, gws, ctx->sc + S_JSWEEPS, nullptr);
    }
  }
  ctx->launches++;
  return ctx->check_launch("jacobi");
}

// ------------------------------------------------------------------------------------------
// The same one-sided Jacobi for ell > 256 (the paper's ell = 800 on STL-10): X (= R^T) and V
// no longer fit any CTA or cluster's shared memory, so they live in global memory (L2-resident: 10 MB
// at ell = 800) and the ell / 2 pairs of a round go to ell / 2 warps spread over a cooperative grid,
// one pair per warp, columns streamed in 32-element chunks; a grid barrier (monotonic counter)
// separates the rounds.  Same circle ordering, the same fp64 rotation, exact norms recomputed each
// sweep and updated within it, the same absolute floor and convergence test as jacobi_kernel.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void jgrid_barrier(unsigned int* bar, unsigned int nblocks, unsigned int& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned int target = epoch * nblocks;
    red_add_release_gpu(bar, 1u);
    while (ld_relaxed_gpu(bar) < target) {
    }
    fence_acquire_gpu();
  }
  __syncthreads();
}

template <int E>
__global__ void __launch_bounds__(256) jacobi_grid_kernel(int n, const double* R, int ldr, double* Vout, int ldv,
                                                           double* sigma, double* X, double* V, double* nrm,
                                                           double* cmax, unsigned int* bar, double* jsweeps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + warp;                  // global warp id
  const int W = gridDim.x * nw;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, GT = gridDim.x * blockDim.x;
  unsigned int epoch = 0;
  for (int64_t e = gt; e < (int64_t)n * n; e += GT) {
    const int i = (int)(e % n), j = (int)(e / n);
    X[e] = R[j + (size_t)i * ldr];                        // X = R^T
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  jgrid_barrier(bar, gridDim.x, epoch);
  const int P = (n % 2 == 0) ? n : n + 1;
  const double tol = fmax(1e-15, (double)n * 0x1p-53);
  const double tol2 = tol * tol;
  __shared__ double smax[32];   // <= 8 warps (256 threads)
  __shared__ int srot;
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    double mx = 0.0;
    for (int j = gw; j < n; j += W) {                     // exact column norms
      double a = 0.0;
      for (int i = lane; i < n; i += 32) a = fma(X[i + (size_t)j * n], X[i + (size_t)j * n], a);
      a = warp_sum(a);
      if (lane == 0) nrm[j] = a;
      mx = fmax(mx, a);
    }
    if (lane == 0) smax[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = 0.0;
      for (int q = 0; q < nw; ++q) b = fmax(b, smax[q]);
      cmax[blockIdx.x] = b;
      srot = 0;
    }
    jgrid_barrier(bar, gridDim.x, epoch);
    double gmax = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) gmax = fmax(gmax, __ldcg(cmax + b));
    const double floor_g = 1e-2 * 0x1p-52 * gmax;
    for (int r = 0; r < P - 1; ++r) {
      for (int pi = gw; pi < P / 2; pi += W) {
        int a, b;
        if (pi == 0) { a = r; b = P - 1; }
        else {
          a = r + pi; if (a >= P - 1) a -= P - 1;
          b = r - pi; if (b < 0) b += P - 1;
        }
        if (a >= n || b >= n) continue;
        const int p = a < b ? a : b, q = a < b ? b : a;
        double* xp = X + (size_t)p * n;
        double* xq = X + (size_t)q * n;
        // the two columns in registers (E elements per lane, every load in flight at once), one dot
        double a0[E], a1[E];
        double ga = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = lane + 32 * e;
          a0[e] = (i < n) ? __ldcg(xp + i) : 0.0;
          a1[e] = (i < n) ? __ldcg(xq + i) : 0.0;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) ga = fma(a0[e], a1[e], ga);
        ga = warp_sum(ga);
        const double al = __ldcg(nrm + p), be = __ldcg(nrm + q);
        if (ga * ga > tol2 * al * be && fabs(ga) > floor_g) {
          double c, sn, t;
          jacobi_rot(al, be, ga, c, sn, t);
          double* vp = V + (size_t)p * n;
          double* vq = V + (size_t)q * n;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = lane + 32 * e;
            if (i < n) {
              xp[i] = c * a0[e] - sn * a1[e];
              xq[i] = sn * a0[e] + c * a1[e];
            }
          }
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = lane + 32 * e;
            a0[e] = (i < n) ? __ldcg(vp + i) : 0.0;
            a1[e] = (i < n) ? __ldcg(vq + i) : 0.0;
          }
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = lane + 32 * e;
            if (i < n) {
              vp[i] = c * a0[e] - sn * a1[e];
              vq[i] = sn * a0[e] + c * a1[e];
            }
          }
          if (lane == 0) {
            nrm[p] = fmax(al - t * ga, 0.0);
            nrm[q] = be + t * ga;
            srot = 1;
          }
        }
      }
      jgrid_barrier(bar, gridDim.x, epoch);
    }
    // any rotation in the sweep, anywhere: per-CTA flags through cmax (reused), one more barrier
    if (threadIdx.x == 0) cmax[gridDim.x + blockIdx.x] = (double)srot;
    jgrid_barrier(bar, gridDim.x, epoch);
    bool any = false;
    for (int b = 0; b < (int)gridDim.x; ++b) any = any || (__ldcg(cmax + gridDim.x + b) != 0.0);
    if (!any) break;
  }
  if (gt == 0) jsweeps[0] = (double)(sweep + 1);
  // sigma_j = ||x_j||, rank sort descending (ties by index), V permuted
  for (int j = gw; j < n; j += W) {
    double a = 0.0;
    for (int i = lane; i < n; i += 32) a = fma(__ldcg(X + i + (size_t)j * n), __ldcg(X + i + (size_t)j * n), a);
    a = warp_sum(a);
    if (lane == 0) nrm[j] = sqrt(a);
  }
  jgrid_barrier(bar, gridDim.x, epoch);
  for (int j = gt; j < n; j += GT) {
    const double sj = __ldcg(nrm + j);
    int rk = 0;
    for (int k = 0; k < n; ++k) {
      const double sk = __ldcg(nrm + k);
      rk += (sk > sj) || (sk == sj && k < j);
    }
    sigma[rk] = sj;
    for (int i = 0; i < n; ++i) Vout[i + (size_t)rk * ldv] = __ldcg(V + i + (size_t)j * n);
  }
}

static int launch_jacobi_grid(nys_ctx* ctx, int ell, const double* R, int ldr, double* V, int ldv, double* sigma) {
  const int pairs = (ell + 1) / 2;
  const int blocks = (pairs + 7) / 8;                     // one warp per pair, 256-thread CTAs
  double* X = ctx->wsd("jg_X", (size_t)ell * ell);
  double* Vw = ctx->wsd("jg_V", (size_t)ell * ell);
  double* nrm = ctx->wsd("jg_nrm", (size_t)ell);
  double* cmax = ctx->wsd("jg_cmax", (size_t)2 * blocks);
  unsigned int* bar = (unsigned int*)ctx->ws("jg_bar", 64);
  NYS_CUDA_TRY(ctx, cudaMemsetAsync(bar, 0, 64, ctx->stream));
  double* js = ctx->sc + S_JSWEEPS;
  void* args[] = {&ell, &R, &ldr, &V, &ldv, &sigma, &X, &Vw, &nrm, &cmax, &bar, &js};
  // E = 32 elements per lane: ell <= 1024 (kMaxEll)
  NYS_CUDA_TRY(ctx, cudaLaunchCooperativeKernel((const void*)jacobi_grid_kernel<32>, dim3(blocks), dim3(256), args, 0,
                                               ctx->stream));
  ctx->launches++;
  return ctx->check_launch("jacobi_grid");
}

int launch_jacobi_svd(nys_ctx* ctx, int ell, const double* R, int ldr, double* V, int ldv, double* sigma) {
  if (ell > 256) return launch_jacobi_grid(ctx, ell, R, ldr, V, ldv, sigma);
  // block Jacobi over an 8-CTA cluster from ell = block_min on (tuning override NYS_JACOBI_BLOCK_MIN)
  int block_min = 72;   // measured crossover (sketch at m = 20532): 64 equal, 80 2.65 vs 3.59 ms, 112 3.99 vs 6.21 ms
  if (const char* e = getenv("NYS_JACOBI_BLOCK_MIN")) block_min = atoi(e);
  // packed single-CTA kernel up to packed_max (<= 112: X and V in 200 KB of shared memory)
  static const int packed_max =
      std::min(112, getenv("NYS_JACOBI_PACKED_MAX") ? atoi(getenv("NYS_JACOBI_PACKED_MAX")) : 64);
  if (ell > packed_max && ell >= block_min && ell >= 16 && ell <= 256 && getenv("NYS_JACOBI_CYCLIC") == nullptr) {
    NYS_TRY(launch_jacobi_block(ctx, ell, R, ldr, V, ldv, sigma));
    ctx->launches++;
    return ctx->check_launch("jacobi_block");
  }
  // G lanes per pair (NYS_JACOBI_WARP=1: one warp per pair)
  static const bool warp_pairs = getenv("NYS_JACOBI_WARP") != nullptr;
  // lanes per pair: 8 up to ell = 56, 16 above (measured on B200 per sweep: ell = 50 37.9 vs 39.1 us,
  // ell = 64 (G = 8 needs E = 8) 74 vs 55 us); NYS_JACOBI_G forces one (tuning)
  static const int jg = getenv("NYS_JACOBI_G") ? atoi(getenv("NYS_JACOBI_G")) : 0;
  const int G = jg ? jg : (ell <= 56 ? 8 : 16);
  if (!warp_pairs && ell <= packed_max) {
    if (G == 16) {
      if (ell <= 32) return launch_jacobi_packed<16, 2>(ctx, ell, R, ldr, V, ldv, sigma);
      if (ell <= 64) return launch_jacobi_packed<16, 4>(ctx, ell, R, ldr, V, ldv, sigma);
      return launch_jacobi_packed<16, 7>(ctx, ell, R, ldr, V, ldv, sigma);
    }
    if (ell <= 24) return launch_jacobi_packed<8, 3>(ctx, ell, R, ldr, V, ldv, sigma);
    if (ell <= 56) return launch_jacobi_packed<8, 7>(ctx, ell, R, ldr, V, ldv, sigma);
    if (ell <= 64) return launch_jacobi_packed<8, 8>(ctx, ell, R, ldr, V, ldv, sigma);
    return launch_jacobi_packed<16, 7>(ctx, ell, R, ldr, V, ldv, sigma);
  }
  if (ell <= 64) return launch_jacobi_t<64>(ctx, ell, R, ldr, V, ldv, sigma);
  if (ell <= 112) return launch_jacobi_t<128>(ctx, ell, R, ldr, V, ldv, sigma);   // above: cluster path
  return launch_jacobi_t<256>(ctx, ell, R, ldr, V, ldv, sigma);
}

// lambda_hat = max{0, sigma^2 - nu}
__global__ void lambda_kernel(int ell, const double* sigma, double* lam, const double* sc) {
  const double nu = sc[S_NU];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ell) lam[i] = fmax(0.0, sigma[i] * sigma[i] - nu);
}
int launch_lambda_from_sigma(nys_ctx* ctx, int ell, const double* sigma, double* lam) {
  lambda_kernel<<<(ell + 127) / 128, 128, 0, ctx->stream>>>(ell, sigma, lam, ctx->sc);
  ctx->launches++;
  return ctx->check_launch("lambda");
}

// ||U^T U - I||_F from a Gram matrix already computed into G (ell x ell)
__global__ void orth_err_kernel(int ell, const double* G, int ldg, double* sc, int slot) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int e = threadIdx.x; e < ell * ell; e += blockDim.x) {
    const int i = e % ell, j = e / ell;
    const double v = G[i + j * ldg] - (i == j ? 1.0 : 0.0);
    acc = fma(v, v, acc);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    sc[slot] = sqrt(s);
  }
}
int launch_orth_err(nys_ctx* ctx, int64_t m, int ell, const double* U, int64_t ldu, int slot) {
  double* G = ctx->wsd("orth_gram", (size_t)ell * ell);
  GemmCall g;
  g.M = ell; g.N = ell; g.K = m; g.A = U; g.lda = ldu; g.a_kmajor = true; g.B = U; g.ldb = ldu; g.C = G; g.ldc = ell;
  NYS_TRY(launch_gemm(ctx, g));
  orth_err_kernel<<<1, 256, 0, ctx->stream>>>(ell, G, ell, ctx->sc, slot);
  ctx->launches++;
  return ctx->check_launch("orth_err");
}

}  // namespace nys
