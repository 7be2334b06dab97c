// Partial Cholesky preconditioner of Chol-IP-PMM (the paper's comparison arm, P:250-349;
// SURVEY §8(f) f2): pivot selection, factor post-processing and the P^{-1} application.
//
//   diag(N_delta) -> the ell largest entries = pivots P (reading C1: original diagonal, ties -> smaller
//   index, sorted by value descending) ; Y = N_delta E_P (the sketch GEMMs with a selection "Omega") ;
//   N11 = Y[P, :] = R^T R (chol_inv gives R and R^{-1}) ; Z = Y R^{-1}: rows P = L11 = R^T, rows Q = L21 ;
//   diag(S)_i = diag(N_delta)_i - ||Z_i||^2 (i in Q).
//   P^{-1} v (eq. P:309-322): u1 = R^{-T} v[P] ; w_i = (v_i - Z_i u1) / S_ii (i in Q) ;
//   g = sum_{i in Q} Z_i^T w_i ; w1 = R^{-1} (u1 - g) ; out[P] = w1, out[Q] = w.
// Z is kept ROW-major (Zt[i][k], row stride ell) for the row kernels.
#include "k_vec.cuh"

namespace nys {

// ---- top-ell selection: 8-bit radix select on the (non-negative) fp64 bit patterns, one CTA ----
__global__ void __launch_bounds__(1024) topl_select_kernel(const double* v, int64_t m, int ell, int64_t* piv,
                                                           int* pivpos) {
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix, s_mask;
  __shared__ int s_need;
  __shared__ unsigned int s_cnt_gt, s_cnt_eq;
  __shared__ int64_t sel[256];
  __shared__ double selv[256];
  __shared__ unsigned int warp_cnt[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t i = tid; i < m; i += nt) pivpos[i] = -1;
  if (tid == 0) { s_prefix = 0ull; s_mask = 0ull; s_need = ell; }
  __syncthreads();
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = tid; b < 256; b += nt) hist[b] = 0u;
    __syncthreads();
    const unsigned long long pre = s_prefix, msk = s_mask;
    for (int64_t i = tid; i < m; i += nt) {
      const unsigned long long key = (unsigned long long)__double_as_longlong(v[i]);
      if ((key & msk) == pre) atomicAdd(&hist[(key >> shift) & 255ull], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      int need = s_need;
      int b = 255;
      for (; b > 0; --b) {
        if ((int)hist[b] >= need) break;
        need -= (int)hist[b];
      }
      s_need = need;
      s_prefix = pre | ((unsigned long long)b << shift);
      s_mask = msk | (255ull << shift);
    }
    __syncthreads();
  }
  // threshold key T = s_prefix; take every key > T and the s_need smallest indices with key == T
  const unsigned long long T = s_prefix;
  const int need_eq = s_need;
  if (tid == 0) { s_cnt_gt = 0u; s_cnt_eq = 0u; }
  __syncthreads();
  for (int64_t i = tid; i < m; i += nt) {
    const unsigned long long key = (unsigned long long)__double_as_longlong(v[i]);
    if (key > T) {
      const unsigned int pos = atomicAdd(&s_cnt_gt, 1u);
      sel[pos] = i;
      selv[pos] = v[i];
    }
  }
  __syncthreads();
  const int base = (int)s_cnt_gt;
  // equal keys in index order: chunked block scan
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int64_t c0 = 0; c0 < m; c0 += nt) {
    const int64_t i = c0 + tid;
    const bool eq = (i < m) && ((unsigned long long)__double_as_longlong(v[i]) == T);
    const unsigned int bal = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) warp_cnt[warp] = __popc(bal);
    __syncthreads();
    unsigned int before = 0, total = 0;
    for (int w = 0; w < nw; ++w) {
      if (w < warp) before += warp_cnt[w];
      total += warp_cnt[w];
    }
    const unsigned int rank = s_cnt_eq + before + __popc(bal & ((1u << lane) - 1u));
    if (eq && (int)rank < need_eq) {
      sel[base + rank] = i;
      selv[base + rank] = v[i];
    }
    __syncthreads();
    if (tid == 0) s_cnt_eq += total;
    __syncthreads();
  }
  // order the ell selected by (value desc, index asc)
  for (int k = tid; k < ell; k += nt) {
    int rk = 0;
    for (int j = 0; j < ell; ++j)
      rk += (selv[j] > selv[k]) || (selv[j] == selv[k] && sel[j] < sel[k]);
    piv[rk] = sel[k];
  }
  __syncthreads();
  for (int k = tid; k < ell; k += nt) pivpos[piv[k]] = k;
}

// Om = E_P (m x ell, ld ldo): Om[piv_k, k] = 1
__global__ void selection_kernel(int64_t m, int ell, const int64_t* piv, double* Om, int64_t ldo) {
  const int64_t tot = (int64_t)ell * ldo;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % ldo, k = e / ldo;
    Om[e] = (i < m && piv[k] == i) ? 1.0 : 0.0;
  }
}

// Y[piv_k, k] += delta ; N11[j][k] = Y[piv_j, k]  (ell x ell, column-major ld ell)
__global__ void pivot_block_kernel(double* Y, int64_t ldy, const int64_t* piv, int ell, double delta, double* N11) {
  const int k = blockIdx.x;
  for (int j = threadIdx.x; j < ell; j += blockDim.x) {
    double v = Y[piv[j] + k * ldy];
    if (j == k) {
      v += delta;
      Y[piv[j] + k * ldy] = v;
    }
    N11[j + (size_t)k * ell] = v;
  }
}

// dS_i = diag_i - ||Zt_i||^2 for i in Q, 0 at pivot rows.  One warp per row.
__global__ void chol_ds_kernel(int64_t m, int ell, const double* Zt, const double* dg, const int* pivpos, double* dS) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += nw) {
    double s = 0.0;
    for (int k = lane; k < ell; k += 32) {
      const double z = Zt[(size_t)i * ell + k];
      s = fma(z, z, s);
    }
    s = warp_sum(s);
    if (lane == 0) dS[i] = (pivpos[i] >= 0) ? 0.0 : dg[i] - s;
  }
}

// ---- P^{-1} application ------------------------------------------------------------------
// k1: u1 = R^{-T} v[P]   (R^{-1} upper, ld ldr): u1_k = sum_{j <= k} Rinv[j][k] v[piv_j]
__global__ void chol_u1_kernel(const double* v, const int64_t* piv, const double* Rinv, int ldr, int ell, double* u1,
                               const double* done) {
  if (done != nullptr && *done != 0.0) return;
  __shared__ double vp[256];
  for (int j = threadIdx.x; j < ell; j += blockDim.x) vp[j] = v[piv[j]];
  __syncthreads();
  for (int k = threadIdx.x; k < ell; k += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j <= k; ++j) s = fma(Rinv[j + (size_t)k * ldr], vp[j], s);
    u1[k] = s;
  }
}

// k2: w_i = (v_i - Zt_i u1) / dS_i (0 at pivot rows); block partials of g = sum_i Zt_i w_i.
// One warp per row (lanes over the ell columns); per-lane accumulation of g, warp rows reduced in
// shared memory in a fixed order; part[(c) * G + block], c < ell.
__global__ void __launch_bounds__(256) chol_rows_kernel(int64_t m, int ell, const double* v, const double* Zt,
                                                        const double* dS, const int* pivpos, const double* u1,
                                                        double* w, double* part, const double* done) {
  if (done != nullptr && *done != 0.0) return;
  __shared__ double us[256];
  __shared__ double wred[8][257];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int k = tid; k < ell; k += 256) us[k] = u1[k];
  for (int k = lane; k < ell; k += 32) wred[warp][k] = 0.0;
  __syncthreads();
  double ul[8], gl[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    ul[q] = (lane + 32 * q < ell) ? us[lane + 32 * q] : 0.0;
    gl[q] = 0.0;
  }
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < m; i += nw) {
    double zr[8];
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = lane + 32 * q;
      zr[q] = (k < ell) ? Zt[(size_t)i * ell + k] : 0.0;
      s = fma(zr[q], ul[q], s);
    }
    s = warp_sum(s);
    const bool pv = pivpos[i] >= 0;
    const double wi = pv ? 0.0 : (v[i] - s) / dS[i];
    if (lane == 0) w[i] = wi;
#pragma unroll
    for (int q = 0; q < 8; ++q) gl[q] = fma(zr[q], wi, gl[q]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (lane + 32 * q < ell) wred[warp][lane + 32 * q] = gl[q];
  __syncthreads();
  for (int c = tid; c < ell; c += 256) {
    const double t = ((wred[0][c] + wred[1][c]) + (wred[2][c] + wred[3][c])) + ((wred[4][c] + wred[5][c]) + (wred[6][c] + wred[7][c]));
    part[(size_t)c * gridDim.x + blockIdx.x] = t;
  }
}

// g_c = sum_b part[c][b]  (one block per column, fixed order)
__global__ void __launch_bounds__(256) chol_gred_kernel(const double* part, int G, double* g, const double* done) {
  if (done != nullptr && *done != 0.0) return;
  __shared__ double ws[8];
  const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double acc = 0.0;
  for (int k = tid; k < G; k += 256) acc += part[(size_t)c * G + k];
  acc = warp_sum(acc);
  if (lane == 0) ws[warp] = acc;
  __syncthreads();
  if (tid == 0) g[c] = ((ws[0] + ws[1]) + (ws[2] + ws[3])) + ((ws[4] + ws[5]) + (ws[6] + ws[7]));
}

// k4: w1 = R^{-1} (u1 - g) (redundantly per block, ell^2 work), out_i = w_i (i in Q), out[piv_j] = w1_j;
// optional PCG: rz = r^T out partials, last block -> beta, rz (as pcg_precond_kernel)
__global__ void __launch_bounds__(256) chol_out_kernel(int64_t m, int ell, const double* u1, const double* g,
                                                       const double* Rinv, int ldr, const int* pivpos, const double* w,
                                                       double* out, const double* r, double* part, unsigned int* counter,
                                                       double* sc, int init, int pcg) {
  if (pcg && sc[S_DONE] != 0.0) return;
  __shared__ double t[256];
  __shared__ double w1[256];
  const int tid = threadIdx.x;
  for (int k = tid; k < ell; k += 256) t[k] = u1[k] - g[k];
  __syncthreads();
  for (int j = tid; j < ell; j += 256) {
    double s = 0.0;
    for (int k = j; k < ell; ++k) s = fma(Rinv[j + (size_t)k * ldr], t[k], s);
    w1[j] = s;
  }
  __syncthreads();
  double rz = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * 256 + tid; i < m; i += (int64_t)gridDim.x * 256) {
    const int pp = pivpos[i];
    const double zi = (pp >= 0) ? w1[pp] : w[i];
    out[i] = zi;
    if (pcg) rz = fma(r[i], zi, rz);
  }
  if (!pcg) return;
  double v[1] = {rz};
  block_sum_to_part<1>(v, part, gridDim.x);
  if (last_block_arrive(counter) && warp_uniform_id() == 0) {
    const double rzn = warp_sum_array(part, gridDim.x);
    if (threadIdx.x != 0) return;
    const double rzo = sc[S_RZ];
    sc[S_BETA] = init ? 0.0 : rzn / rzo;
    sc[S_RZ] = rzn;
    if (!(rzn > 0.0) || !isfinite(rzn)) { sc[S_STATUS] = (double)NYS_EBREAKDOWN; sc[S_DONE] = 1.0; }
    *counter = 0u;
  }
}

// ------------------------------------------------------------------------------------------
int launch_topl_select(nys_ctx* ctx, const double* v, int64_t m, int ell, int64_t* piv, int* pivpos) {
  topl_select_kernel<<<1, 1024, 0, ctx->stream>>>(v, m, ell, piv, pivpos);
  ctx->launches++;
  return ctx->check_launch("topl_select");
}

int launch_selection(nys_ctx* ctx, int64_t m, int ell, const int64_t* piv, double* Om, int64_t ldo) {
  int64_t tot = (int64_t)ell * ldo;
  int g = (int)((tot + 255) / 256);
  if (g > 4 * ctx->num_sms) g = 4 * ctx->num_sms;
  selection_kernel<<<g, 256, 0, ctx->stream>>>(m, ell, piv, Om, ldo);
  ctx->launches++;
  return ctx->check_launch("selection");
}

int launch_pivot_block(nys_ctx* ctx, double* Y, int64_t ldy, const int64_t* piv, int ell, double delta, double* N11) {
  pivot_block_kernel<<<ell, 128, 0, ctx->stream>>>(Y, ldy, piv, ell, delta, N11);
  ctx->launches++;
  return ctx->check_launch("pivot_block");
}

int launch_chol_ds(nys_ctx* ctx, int64_t m, int ell, const double* Zt, const double* dg, const int* pivpos, double* dS) {
  int64_t g = (m + 7) / 8;
  if (g > 4 * ctx->num_sms) g = 4 * ctx->num_sms;
  chol_ds_kernel<<<(unsigned)g, 256, 0, ctx->stream>>>(m, ell, Zt, dg, pivpos, dS);
  ctx->launches++;
  return ctx->check_launch("chol_ds");
}

// P^{-1} v -> out.  pcg = 1: the PCG preconditioning step (r = v, rz / beta into the scalar slots,
// early exit when sc[S_DONE] is set).  `ws` holds u1 (ell), g (ell), w (m), partials.
int launch_chol_apply(nys_ctx* ctx, const CholFactors& F, const double* v, double* out, int pcg, int init) {
  const int64_t m = F.m;
  const int ell = F.ell;
  const double* done = pcg ? ctx->sc + S_DONE : nullptr;
  double* u1 = ctx->wsd("chol_u1", (size_t)ell);
  double* g = ctx->wsd("chol_g", (size_t)ell);
  double* w = ctx->wsd("chol_w", (size_t)m);
  int64_t G = (m + 7) / 8;
  if (G > 2 * ctx->num_sms) G = 2 * ctx->num_sms;
  double* part = ctx->wsd("chol_part", (size_t)ell * G);
  if (ell > 0) chol_u1_kernel<<<1, 256, 0, ctx->stream>>>(v, F.piv, F.Rinv, F.ldr, ell, u1, done);
  chol_rows_kernel<<<(unsigned)G, 256, 0, ctx->stream>>>(m, ell, v, F.Zt, F.dS, F.pivpos, u1, w, part, done);
  if (ell > 0) chol_gred_kernel<<<ell, 256, 0, ctx->stream>>>(part, (int)G, g, done);
  int64_t G2 = (m + 255) / 256;
  if (G2 > 4 * ctx->num_sms) G2 = 4 * ctx->num_sms;
  double* part2 = ctx->wsd("chol_part2", (size_t)G2);
  chol_out_kernel<<<(unsigned)G2, 256, 0, ctx->stream>>>(m, ell, u1, g, F.Rinv, F.ldr, F.pivpos, w, out, v, part2,
                                                         ctx->counters + 3, ctx->sc, init, pcg);
  ctx->launches += 4;
  return ctx->check_launch("chol_apply");
}

}  // namespace nys
