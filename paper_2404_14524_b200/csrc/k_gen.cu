// Elementwise kernels of Nys-IP-PMM for FREE and BOX-CONSTRAINED variables, (P~)/(D~)
// (Alg. 5, App. B.2-B.3).  vt[j]: 0 = I (x >= 0),
// 1 = F (free), 2 = J (0 <= x <= u).  w, s (and their directions) are 0 off J; z is 0 on F.
// The K1-K3 kernels (matvec, sketch, PCG) are unchanged: only D and the right-hand sides change.
#include "k_vec.cuh"

namespace nys {

#define GRID_STRIDE(j, n) for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < (n); j += (int64_t)gridDim.x * blockDim.x)

// d = (Q + Theta^{-1} + rho I)^{-1},  Theta^{-1} = z/x on IJ (+ s/w on J), 0 on F
__global__ void gen_scaling_kernel(int64_t n, const int8_t* vt, const double* q, const double* x, const double* z,
                                   const double* w, const double* s, double rho, double* d) {
  GRID_STRIDE(j, n) {
    const int t = vt[j];
    double th = (t == 1) ? 0.0 : z[j] / x[j];
    if (t == 2) th += s[j] / w[j];
    d[j] = 1.0 / (q[j] + th + rho);
  }
}

// predictor RHS (eq. P:867-876) and Alg. 4 line 1:
//   r_d = rD + rho (x - zeta)   [rD = c + Qx - A^T y - z + s]
//   r_u = u - x - w (J) ; r_xz = -x z (IJ) ; r_ws = -w s (J)
//   xi_au = -r_xz / x (IJ) + (r_ws - s r_u) / w (J) ; t = d (r_d + xi_au)
__global__ void gen_pred_rhs_kernel(int64_t n, const int8_t* vt, const double* ub, const double* x, const double* z,
                                    const double* w, const double* s, const double* zeta, const double* rD, double rho,
                                    const double* d, double* rd, double* rxz, double* ru, double* rws, double* xiau,
                                    double* t) {
  GRID_STRIDE(j, n) {
    const int ty = vt[j];
    const double xj = x[j];
    const double r = rD[j] + rho * (xj - zeta[j]);
    const double rx = (ty == 1) ? 0.0 : -xj * z[j];
    double u_ = 0.0, rw = 0.0, xa = (ty == 1) ? 0.0 : -rx / xj;
    if (ty == 2) {
      u_ = ub[j] - xj - w[j];
      rw = -w[j] * s[j];
      xa += (rw - s[j] * u_) / w[j];
    }
    rd[j] = r;
    rxz[j] = rx;
    ru[j] = u_;
    rws[j] = rw;
    xiau[j] = xa;
    t[j] = d[j] * (r + xa);
  }
}

// corrector RHS (eq. P:894-897): r_d = r_p = r_u = 0 ; r_xz = mu~ - dxp dzp (IJ) ; r_ws = mu~ - dwp dsp (J)
__global__ void gen_corr_rhs_kernel(int64_t n, const int8_t* vt, const double* x, const double* w, const double* dxp,
                                    const double* dzp, const double* dwp, const double* dsp, const double* sc,
                                    const double* d, double* rxz, double* ru, double* rws, double* xiau, double* t) {
  const double mut = sc[S_MUT];
  GRID_STRIDE(j, n) {
    const int ty = vt[j];
    const double rx = (ty == 1) ? 0.0 : mut - dxp[j] * dzp[j];
    double rw = 0.0, xa = (ty == 1) ? 0.0 : -rx / x[j];
    if (ty == 2) {
      rw = mut - dwp[j] * dsp[j];
      xa += rw / w[j];
    }
    rxz[j] = rx;
    ru[j] = 0.0;
    rws[j] = rw;
    xiau[j] = xa;
    t[j] = d[j] * xa;
  }
}

// Alg. 4 line 3 after dx: dz = X^{-1}(r_xz - Z dx) (IJ), 0 (F) ; dw = r_u - dx (J) ; ds = W^{-1}(r_ws - S dw) (J)
__global__ void gen_recover_kernel(int64_t n, const int8_t* vt, const double* x, const double* z, const double* w,
                                   const double* s, const double* dx, const double* rxz, const double* ru,
                                   const double* rws, double* dz, double* dw, double* ds) {
  GRID_STRIDE(j, n) {
    const int ty = vt[j];
    dz[j] = (ty == 1) ? 0.0 : (rxz[j] - z[j] * dx[j]) / x[j];
    if (ty == 2) {
      const double dwj = ru[j] - dx[j];
      dw[j] = dwj;
      ds[j] = (rws[j] - s[j] * dwj) / w[j];
    } else {
      dw[j] = 0.0;
      ds[j] = 0.0;
    }
  }
}

// stepsizes (eq. P:1493-1497): min over I_x (IJ, dx < 0) of -x/dx and I_w (J, dw < 0) of -w/dw; dual with
// z (IJ) and s (J).  Optional combination dx = dx1 + dx2 etc. (final direction).  -> sc[S_TMP0], sc[S_TMP1]
struct GenRatioArgs {
  int64_t n;
  const int8_t* vt;
  const double *x, *z, *w, *s;
  double *dx, *dz, *dw, *ds;
  const double *dx1, *dx2, *dz1, *dz2, *dw1, *dw2, *ds1, *ds2;
  double* sc;
  double* part;
  unsigned int* counter;
};
__global__ void __launch_bounds__(256) gen_ratio_kernel(const GenRatioArgs R) {
  double mp = 1.0e300, md = 1.0e300;
  GRID_STRIDE(i, R.n) {
    double dx, dz, dw, ds;
    if (R.dx1) {
      dx = R.dx1[i] + R.dx2[i]; R.dx[i] = dx;
      dz = R.dz1[i] + R.dz2[i]; R.dz[i] = dz;
      dw = R.dw1[i] + R.dw2[i]; R.dw[i] = dw;
      ds = R.ds1[i] + R.ds2[i]; R.ds[i] = ds;
    } else {
      dx = R.dx[i]; dz = R.dz[i]; dw = R.dw[i]; ds = R.ds[i];
    }
    const int ty = R.vt[i];
    if (ty != 1) {
      if (dx < 0.0) mp = fmin(mp, -R.x[i] / dx);
      if (dz < 0.0) md = fmin(md, -R.z[i] / dz);
    }
    if (ty == 2) {
      if (dw < 0.0) mp = fmin(mp, -R.w[i] / dw);
      if (ds < 0.0) md = fmin(md, -R.s[i] / ds);
    }
  }
  __shared__ double sh[2][32];
  mp = warp_min(mp);
  md = warp_min(md);
  const int wi = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sh[0][wi] = mp; sh[1][wi] = md; }
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

// r_U = u - x - w on J (0 elsewhere)
__global__ void gen_ru_kernel(int64_t n, const int8_t* vt, const double* ub, const double* x, const double* w, double* ru) {
  GRID_STRIDE(j, n) ru[j] = (vt[j] == 2) ? ub[j] - x[j] - w[j] : 0.0;
}

// initial point (App. B.2): from x~ (in x) and g = c - A^T y~ + Q x~ (in z):
//   z~_J = g/2, z~_I = g, z~_F = 0 ; s~_J = -z~_J ; w~_J = u - x~ ; masked statistics -> st[0..11]:
//   0 min x~_IJ, 1 min w~_J, 2 min z~_IJ, 3 min s~_J, 4 sum x~_IJ, 5 sum w~_J, 6 sum z~_IJ, 7 sum s~_J,
//   8 x~^T z~ (IJ), 9 w~^T s~ (J), 10 |IJ|, 11 |J|   (per block -> part, last block -> st)
__global__ void __launch_bounds__(256) gen_init_stats_kernel(int64_t n, const int8_t* vt, const double* ub, double* x,
                                                            double* z, double* w, double* s, double* part,
                                                            unsigned int* counter, double* st) {
  double mn[4] = {1.0e300, 1.0e300, 1.0e300, 1.0e300};
  double sm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  GRID_STRIDE(j, n) {
    const int ty = vt[j];
    const double xj = x[j], g = z[j];
    double zj = 0.0, sj = 0.0, wj = 0.0;
    if (ty == 0) zj = g;
    if (ty == 2) {
      zj = 0.5 * g;
      sj = -zj;
      wj = ub[j] - xj;
    }
    z[j] = zj;
    s[j] = sj;
    w[j] = wj;
    if (ty != 1) {
      mn[0] = fmin(mn[0], xj);
      mn[2] = fmin(mn[2], zj);
      sm[0] += xj;
      sm[2] += zj;
      sm[4] += xj * zj;
      sm[6] += 1.0;
    }
    if (ty == 2) {
      mn[1] = fmin(mn[1], wj);
      mn[3] = fmin(mn[3], sj);
      sm[1] += wj;
      sm[3] += sj;
      sm[5] += wj * sj;
      sm[7] += 1.0;
    }
  }
  __shared__ double shm[4][32], shs[8][32];
#pragma unroll
  for (int k = 0; k < 4; ++k) mn[k] = warp_min(mn[k]);
#pragma unroll
  for (int k = 0; k < 8; ++k) sm[k] = warp_sum(sm[k]);
  const int wi = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) shm[k][wi] = mn[k];
#pragma unroll
    for (int k = 0; k < 8; ++k) shs[k][wi] = sm[k];
  }
  __syncthreads();
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int k = 0; k < 4; ++k) {
      double a = 1.0e300;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a = fmin(a, shm[k][i]);
      part[(size_t)k * G + blockIdx.x] = a;
    }
    for (int k = 0; k < 8; ++k) {
      double a = 0.0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) a += shs[k][i];
      part[(size_t)(4 + k) * G + blockIdx.x] = a;
    }
  }
  if (last_block_arrive(counter) && warp_uniform_id() == 0) {
    // order: 0 min x, 1 min w, 2 min z, 3 min s ; sums (4 + k): x, w? -> map to the documented slots
    const double mx = warp_min_array(part + 0 * (size_t)G, G), mw = warp_min_array(part + 1 * (size_t)G, G);
    const double mz = warp_min_array(part + 2 * (size_t)G, G), ms = warp_min_array(part + 3 * (size_t)G, G);
    const double sx = warp_sum_array(part + 4 * (size_t)G, G), sw = warp_sum_array(part + 5 * (size_t)G, G);
    const double sz = warp_sum_array(part + 6 * (size_t)G, G), ss = warp_sum_array(part + 7 * (size_t)G, G);
    const double xz = warp_sum_array(part + 8 * (size_t)G, G), ws = warp_sum_array(part + 9 * (size_t)G, G);
    const double nij = warp_sum_array(part + 10 * (size_t)G, G), nj = warp_sum_array(part + 11 * (size_t)G, G);
    if (threadIdx.x != 0) return;
    *counter = 0u;
    st[0] = mx; st[1] = mw; st[2] = mz; st[3] = ms;
    st[4] = sx; st[5] = sw; st[6] = sz; st[7] = ss;
    st[8] = xz; st[9] = ws; st[10] = nij; st[11] = nj;
  }
}

// x0_IJ = x~ + dpt (x0_F = x~) ; w0_J = w~ + dpt ; z0_IJ = z~ + ddt (z_F = 0) ; s0_J = s~ + ddt
__global__ void gen_init_apply_kernel(int64_t n, const int8_t* vt, double* x, double* z, double* w, double* s,
                                      double dpt, double ddt) {
  GRID_STRIDE(j, n) {
    const int ty = vt[j];
    if (ty != 1) {
      x[j] += dpt;
      z[j] += ddt;
    }
    if (ty == 2) {
      w[j] += dpt;
      s[j] += ddt;
    }
  }
}

// v = scale * u with u_IF = 0 (ub is read on J only)
__global__ void gen_half_u_kernel(int64_t n, const int8_t* vt, const double* ub, double scale, double* v) {
  GRID_STRIDE(j, n) v[j] = (vt[j] == 2) ? scale * ub[j] : 0.0;
}

// argument check: vt in {0, 1, 2}; ub_J finite and > 0 (ub == NULL allowed when no entry is 2)
__global__ void gen_check_kernel(int64_t n, const int8_t* vt, const double* ub, unsigned long long* bad) {
  GRID_STRIDE(j, n) {
    const int t = vt[j];
    bool ok = t >= 0 && t <= 2;
    if (t == 2) ok = ub != nullptr && ub[j] > 0.0 && ub[j] < 1.0e300;
    if (!ok) atomicAdd(bad, 1ull);
  }
}

// ------------------------------------------------------------------------------------------
// structure 2: A = [B, S_0, ..., S_{K-1}], S_k = scale_k [e_{row0_k} ... e_{row0_k + count_k - 1}]
// (never materialised).  u_unit / d_unit / atv_unit point at the unit part of the n-vectors.
// ------------------------------------------------------------------------------------------
// atv_unit[j] = scale_k y[row0_k + j - off_k]  (A^T y on the unit columns)
__global__ void unit_expand_kernel(UnitBlocks U, const double* y, double* atv_unit) {
  GRID_STRIDE(j, U.total) {
    int k = 0;
    while (k + 1 < U.nb && j >= U.off[k + 1]) ++k;
    atv_unit[j] = U.scale[k] * y[U.row0[k] + (j - U.off[k])];
  }
}
// out_i = add_i + sum_k [i in block k] scale_k u_unit[off_k + i - row0_k]   (fixed block order)
// diag mode: out_i = sum_k [i in block k] scale_k^2 d_unit[...]             (the e term)
__global__ void unit_fold_kernel(UnitBlocks U, int64_t m, const double* u_unit, const double* add, int diag,
                                 double* out) {
  GRID_STRIDE(i, m) {
    double s = add ? add[i] : 0.0;
    for (int k = 0; k < U.nb; ++k) {
      const int64_t r = i - U.row0[k];
      if (r >= 0 && r < U.count[k]) {
        const double v = u_unit[U.off[k] + r];
        s += diag ? U.scale[k] * U.scale[k] * v : U.scale[k] * v;
      }
    }
    out[i] = s;
  }
}

static int ggrid(nys_ctx* ctx, int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 4 * ctx->num_sms) g = 4 * ctx->num_sms;
  return g < 1 ? 1 : (int)g;
}

int launch_gen_scaling(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* q, const double* x, const double* z,
                       const double* w, const double* s, double rho, double* d) {
  if (n <= 0) return NYS_OK;
  gen_scaling_kernel<<<ggrid(ctx, n), 256, 0, ctx->stream>>>(n, vt, q, x, z, w, s, rho, d);
  ctx->launches++;
  return ctx->check_launch("gen_scaling");
}
int launch_gen_pred_rhs(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* ub, const double* x, const double* z,
                        const double* w, const double* s, const double* zeta, const double* rD, double rho,
                        const double* d, double* rd, double* rxz, double* ru, double* rws, double* xiau, double* t) {
  if (n <= 0) return NYS_OK;
  gen_pred_rhs_kernel<<<ggrid(ctx, n), 256, 0, ctx->stream>>>(n, vt, ub, x, z, w, s, zeta, rD, rho, d, rd, rxz, ru,
                                                              rws, xiau, t);
  ctx->launches++;
  return ctx->check_launch("gen_pred_rhs");
}
int launch_gen_corr_rhs(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* x, const double* w, const double* dxp,
                        const double* dzp, const double* dwp, const double* dsp, const double* d, double* rxz,
                        double* ru, double* rws, double* xiau, double* t) {
  if (n <= 0) return NYS_OK;
  gen_corr_rhs_kernel<<<ggrid(ctx, n), 256, 0, ctx->stream>>>(n, vt, x, w, dxp, dzp, dwp, dsp, ctx->sc, d, rxz, ru,
                                                              rws, xiau, t);
  ctx->launches++;
  return ctx->check_launch("gen_corr_rhs");
}
int launch_gen_recover(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* x, const double* z, const double* w,
                       const double* s, const double* dx, const double* rxz, const double* ru, const double* rws,
                       double* dz, double* dw, double* ds) {
  if (n <= 0) return NYS_OK;
  gen_recover_kernel<<<ggrid(ctx, n), 256, 0, ctx->stream>>>(n, vt, x, z, w, s, dx, rxz, ru, rws, dz, dw, ds);
  ctx->launches++;
  return ctx->check_launch("gen_recover");
}
int launch_gen_ratio(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* x, const double* z, const double* w,
                     const double* s, double* dx, double* dz, double* dw, double* ds, const double* dx1,
                     const double* dx2, const double* dz1, const double* dz2, const double* dw1, const double* dw2,
                     const double* ds1, const double* ds2, int counter_slot) {
  GenRatioArgs R{};
  R.n = n; R.vt = vt; R.x = x; R.z = z; R.w = w; R.s = s; R.dx = dx; R.dz = dz; R.dw = dw; R.ds = ds;
  R.dx1 = dx1; R.dx2 = dx2; R.dz1 = dz1; R.dz2 = dz2; R.dw1 = dw1; R.dw2 = dw2; R.ds1 = ds1; R.ds2 = ds2;
  R.sc = ctx->sc;
  int g = ggrid(ctx, n);
  R.part = ctx->wsd("gen_ratio_part", (size_t)2 * g);
  R.counter = ctx->counters + counter_slot;
  gen_ratio_kernel<<<g, 256, 0, ctx->stream>>>(R);
  ctx->launches++;
  return ctx->check_launch("gen_ratio");
}
int launch_gen_ru(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* ub, const double* x, const double* w,
                  double* ru) {
  if (n <= 0) return NYS_OK;
  gen_ru_kernel<<<ggrid(ctx, n), 256, 0, ctx->stream>>>(n, vt, ub, x, w, ru);
  ctx->launches++;
  return ctx->check_launch("gen_ru");
}
int launch_gen_init_stats(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* ub, double* x, double* z, double* w,
                          double* s, double* st) {
  int g = ggrid(ctx, n);
  double* part = ctx->wsd("gen_init_part", (size_t)12 * g);
  gen_init_stats_kernel<<<g, 256, 0, ctx->stream>>>(n, vt, ub, x, z, w, s, part, ctx->counters + 12, st);
  ctx->launches++;
  return ctx->check_launch("gen_init_stats");
}
int launch_gen_init_apply(nys_ctx* ctx, int64_t n, const int8_t* vt, double* x, double* z, double* w, double* s,
                          double dpt, double ddt) {
  if (n <= 0) return NYS_OK;
  gen_init_apply_kernel<<<ggrid(ctx, n), 256, 0, ctx->stream>>>(n, vt, x, z, w, s, dpt, ddt);
  ctx->launches++;
  return ctx->check_launch("gen_init_apply");
}
int launch_gen_half_u(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* ub, double scale, double* v) {
  if (n <= 0) return NYS_OK;
  gen_half_u_kernel<<<ggrid(ctx, n), 256, 0, ctx->stream>>>(n, vt, ub, scale, v);
  ctx->launches++;
  return ctx->check_launch("gen_half_u");
}
int launch_unit_expand(nys_ctx* ctx, const UnitBlocks& U, const double* y, double* atv_unit) {
  if (U.total <= 0) return NYS_OK;
  unit_expand_kernel<<<ggrid(ctx, U.total), 256, 0, ctx->stream>>>(U, y, atv_unit);
  ctx->launches++;
  return ctx->check_launch("unit_expand");
}
int launch_unit_fold(nys_ctx* ctx, const UnitBlocks& U, int64_t m, const double* u_unit, const double* add, int diag,
                     double* out) {
  unit_fold_kernel<<<ggrid(ctx, m), 256, 0, ctx->stream>>>(U, m, u_unit, add, diag, out);
  ctx->launches++;
  return ctx->check_launch("unit_fold");
}
int launch_gen_check(nys_ctx* ctx, int64_t n, const int8_t* vt, const double* ub, unsigned long long* bad) {
  if (n <= 0) return NYS_OK;
  gen_check_kernel<<<ggrid(ctx, n), 256, 0, ctx->stream>>>(n, vt, ub, bad);
  ctx->launches++;
  return ctx->check_launch("gen_check");
}

}  // namespace nys
