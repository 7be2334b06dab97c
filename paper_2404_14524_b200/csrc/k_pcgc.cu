// Persistent cluster PCG (P^{-1} of P:418) for m > 8192 on one GPU — ONE launch for the
// whole solve, where the graph path (k_vec.cu) pays per iteration a K1 launch with its pipeline
// ramp-up / drain, three vector kernels and their launch gaps.
//
// The matvec phase is the cluster path of K1 (k_matvec.cu): a thread-block cluster of cl CTAs owns
// panels (single columns) of A, CTA rank q the row slice [q rs, (q + 1) rs); per panel the CTA dot
// partials are pushed to every peer with st.async (complete_tx on the peer's ring mbarrier) and the
// rank-1 update of the previous panel runs while they travel (lag-1 pipeline), so every CTA of the
// cluster forms the same t_j = d_j (a_j^T p).  The producer warp streams the CTA's column segments
// through the S-stage cp.async.bulk ring CONTINUOUSLY across iterations (A does not depend on the
// iterate), so HBM keeps streaming through the barrier phases.  Per iteration k:
//   P1  p_k slice (registers); partial w of the cluster's columns -> Wp[cluster][slice]; p^T N p
//       partial (d_j (a_j^T p)^2 summed by rank 0, the (delta + e) p^2 rows by cluster 0) -> pwp
//                                                                           -> grid barrier
//   P2  alpha = rz / p^T N p (every CTA sums pwp in one order); own rows (a contiguous range of
//       the m rows): w = sum of the cluster partial rows + (delta + e) p, x += alpha p,
//       r -= alpha w; ||r||^2 and U^T r partial row                         -> grid barrier
//   P3  every CTA sums the partial rows in one fixed order (identical decisions): converged?
//       h = s o (U^T r), r^T z = ||r||^2 + (U^T r)^T h, beta; own rows p_{k+1} = r + U h + beta p_k
//                                                                           -> grid barrier
// Same recurrence and stopping rule as the persistent kernel (k_pcg.cu) and the oracle's textbook
// PCG: zero start, alpha = r^T z / p^T w, absolute stop ||r|| <= tol, breakdown on p^T w <= 0.
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "k_vec.cuh"

namespace nys {

struct PcgCParams {
  const double* A;
  int64_t lda, m, n;
  const double* d;
  const double* e;
  const double* U;       // m x ell column-major, ld ldu
  int64_t ldu;
  int ell;
  const double* s;       // ell coefficients (lam_l + mu)/(lam_i + mu) - 1
  const double* rhs;
  double* x;
  double* r;
  double* P0;            // p double buffer
  double* P1;
  double* Wp;            // [clusters][wp_ld] partial w rows
  int64_t wp_ld;
  double* pwp;           // [G] CTA partials of sum_j d_j (a_j^T p)^2
  double* pwrow;         // [G] CTA partials of the row part p^T (delta I + diag e) p (own rows, formed with p)
  double* part1;         // [G][1 + ell]
  double* sc;
  unsigned int* bar;     // grid barrier counter (zeroed before the launch)
  int max_iter;
  int stages;
  int cl;
  int64_t rs;            // rows per cluster rank (even)
  int64_t rpc;           // rows per CTA in the vector phases
  unsigned long long* trace;   // debug (NYS_PCG_TRACE): [2 CTAs][16 iterations][8] globaltimer stamps
  unsigned long long* trace_mv;  // debug: [G] matvec-phase duration of every CTA at iteration 9
  int acq_spin;                  // grid barrier: acquire-load spin (1) or relaxed spin + acq_rel fence (0)
};

constexpr int PC_T = 480;              // consumer threads (15 warps) + 1 producer warp
constexpr int PC_W = PC_T / 32;
constexpr int PC_DB = 4;               // dot-exchange ring depth (lag-1 argument of k_matvec.cu)
constexpr int PC_LMAX = 256;

__device__ __forceinline__ void pcgc_grid_barrier(unsigned int* bar, unsigned int nblocks, unsigned int& epoch,
                                                  bool bar_acquire_spin) {
  named_bar_sync(9, PC_T);
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned int target = epoch * nblocks;
    red_add_release_gpu(bar, 1u);
    if (bar_acquire_spin) {
      while (ld_acquire_gpu(bar) < target) {
      }
    } else {
      while (ld_relaxed_gpu(bar) < target) {
      }
      fence_acquire_gpu();
    }
  }
  named_bar_sync(9, PC_T);
}

template <int RPT>
__global__ void __launch_bounds__(PC_T + 32, 1) pcg_cluster_kernel(const PcgCParams P) {
  constexpr int SS = PC_T * RPT;       // stage slot rows (>= rs): rows past the copy stay zero
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int S = P.stages;
  const int cl = P.cl;
  double* stage = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(stage + (size_t)S * SS);
  uint64_t* empty = full + S;
  uint64_t* dotbar = empty + S;
  double* red = reinterpret_cast<double*>(dotbar + PC_DB);   // [2][PC_W]
  double* slots = red + 2 * PC_W;                             // [PC_DB][cl]
  __shared__ double rsh[PC_T];
  __shared__ double gpart[PC_LMAX];
  __shared__ double hsh[PC_LMAX + 32];
  __shared__ double gsh[PC_LMAX];
  __shared__ double colred[PC_T];
  __shared__ double wsh[32];
  __shared__ double s_scal[4];
  __shared__ volatile int s_stop;
  __shared__ volatile long long s_issued;

  const int tid = threadIdx.x, warp = warp_uniform_id(), lane = tid & 31;
  const unsigned int G = gridDim.x;
  const unsigned int bid = blockIdx.x;
  const uint32_t crank = cluster_ctarank();
  const uint32_t cid = cluster_id_x();
  const uint32_t ncl = ncluster_x();
  const int64_t r0 = (int64_t)crank * P.rs;
  int64_t rows_valid = P.m - r0;
  rows_valid = rows_valid < 0 ? 0 : (rows_valid > P.rs ? P.rs : rows_valid);
  const uint32_t copy_bytes = (uint32_t)(((rows_valid + 1) & ~int64_t(1)) * 8);
  // columns c = ccol + i ncl (ccol = the cluster ids in reverse: cluster 0, which takes the first share
  // of the vector phases' rows, gets the shorter column list when n is not a multiple of the clusters)
  const uint32_t ccol = ncl - 1 - cid;
  const int64_t niter = ((int64_t)ccol < P.n) ? (P.n - ccol + ncl - 1) / ncl : 0;
  const int ell = P.ell;
  int64_t v_lo = (int64_t)bid * P.rpc;
  v_lo = v_lo > P.m ? P.m : v_lo;
  int64_t v_hi = v_lo + P.rpc;
  v_hi = v_hi > P.m ? P.m : v_hi;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], PC_W);
    }
    for (int s = 0; s < PC_DB; ++s) mbar_init(&dotbar[s], 1);   // own arrive.expect_tx; peers complete_tx
    fence_mbar_init();
    s_stop = 0;
    s_issued = 0;
  }
  for (int c = tid; c < PC_LMAX + 32; c += PC_T + 32) hsh[c] = 0.0;   // zero tail: the U h loop reads past ell
  {
    // zero the pad rows of every stage slot once (disjoint from what the bulk copies write)
    const int64_t crow = (rows_valid + 1) & ~int64_t(1);
    const int64_t npad = SS - crow;
    if (npad > 0)
      for (int64_t e = tid; e < (int64_t)S * npad; e += PC_T + 32) stage[(e / npad) * SS + crow + (e % npad)] = 0.0;
  }
  cluster_sync_all();

  if (warp == PC_W) {
    // ---------------- producer warp: this CTA's column segments, iteration after iteration -------
    if (lane == 0 && niter > 0) {
      const uint64_t pol = l2_evict_first_policy();
      long long q = 0;
      int s = 0;
      uint32_t eph = 1u;      // parity of the empty-barrier phase to wait for (first pass: none)
      int64_t itp = 0;        // panel index within the CTA's set (q mod niter, kept incrementally)
      for (;; ++s, ++q) {
        if (s == S) { s = 0; eph ^= 1u; }
        if (q >= S) {
          bool stop = false;
          for (;;) {
            uint32_t ok;
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(ok)
                : "r"(smem_u32(&empty[s])), "r"(eph)
                : "memory");
            if (ok) break;
            if (s_stop) { stop = true; break; }
          }
          if (stop) break;
        }
        if (s_stop) break;
        const int64_t col = (int64_t)ccol + itp * ncl;
        if (++itp == niter) itp = 0;
        if (copy_bytes > 0) {
          mbar_arrive_expect_tx(&full[s], copy_bytes);
          bulk_g2s(stage + (size_t)s * SS, P.A + col * P.lda + r0, copy_bytes, &full[s], pol);
        } else {
          mbar_arrive(&full[s]);
        }
      }
      s_issued = q;
    }
    __syncwarp();
    named_bar_sync(10, PC_T + 32);   // exit handshake with the consumers
    cluster_sync_all();              // the consumers' final cluster barrier
    return;
  }

  // ======================= consumers =========================================================
  // an odd slice length copies one row past the slice (16-byte bulk sizes): its owner zeroes it in
  // every stage it reads and fences that write against the next bulk copy into the stage
  const bool odd_owner = (rows_valid & 1) && (rows_valid % PC_T) == tid && rows_valid < SS;
  long long qc = 0;        // panels consumed
  int cs = 0;              // stage ring position of the next panel, and its full-barrier parity
  uint32_t cph = 0u;
  long long qd = 0;        // panels exchanged (dot ring position)
  unsigned int bar_epoch = 0;
  double rz = 0.0;
  int iters = 0;
  int status = 0;
  const double delta = P.sc[S_DELTA];
  const int ncol = 1 + ell;
  int trace_k = -1;
  auto stamp = [&](int slot) {
    if (P.trace != nullptr && tid == 0 && (bid == 0 || bid == G - 1) && trace_k >= 0 && trace_k < 16) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      P.trace[((bid == 0 ? 0 : 1) * 16 + trace_k) * 8 + slot] = t;
    }
  };

  // ---- the CTA's own rows: (init) x = 0, r = rhs | x += alpha p_k, r -= alpha w; rr, U^T r row -------
  // alpha = rz / p^T N p is formed by warp 0 from the pwp partials while the row operands (p, e, x, r
  // and the cluster partial rows of w) are in flight; returns false on a p^T N p breakdown (uniform)
  auto rows_phase = [&](bool init, const double* pk) -> bool {
    double rr = 0.0;
    double alpha = 0.0;
    for (int c = tid; c < ell; c += PC_T) gpart[c] = 0.0;
    for (int64_t i0 = v_lo; i0 < v_hi || (!init && i0 == v_lo); i0 += PC_T) {
      const int64_t i = i0 + tid;
      const bool own = i < v_hi;
      double ri = 0.0, pi = 0.0, wi = 0.0, xi = 0.0;
      if (own) {
        if (init) {
          ri = P.rhs[i];
        } else {
          pi = __ldcg(pk + i);
          xi = P.x[i];
          ri = P.r[i];
          const double ei = P.e ? P.e[i] : 0.0;
          double acc = 0.0;
          for (uint32_t k0 = 0; k0 < ncl; k0 += 24) {   // the cluster partial rows, in cluster order
            double v[24];
#pragma unroll
            for (int u = 0; u < 24; ++u) v[u] = (k0 + u < ncl) ? __ldcg(P.Wp + (size_t)(k0 + u) * P.wp_ld + i) : 0.0;
#pragma unroll
            for (int w = 16; w > 0; w >>= 1)
#pragma unroll
              for (int u = 0; u < w; ++u)
                if (u + w < 24) v[u] += v[u + w];
            acc += v[0];
          }
          wi = acc + (delta + ei) * pi;
        }
      }
      if (!init && i0 == v_lo) {
        if (warp == 0) {
          const double pw = warp_sum_array(P.pwp, (int)G) + warp_sum_array(P.pwrow, (int)G);
          if (lane == 0) s_scal[2] = pw;
        }
        named_bar_sync(9, PC_T);
        const double pw = s_scal[2];
        if (!(pw > 0.0) || !isfinite(pw)) return false;
        alpha = rz / pw;
      }
      if (own) {
        if (init) {
          P.x[i] = 0.0;
        } else {
          P.x[i] = fma(alpha, pi, xi);
          ri = fma(-alpha, wi, ri);
        }
        P.r[i] = ri;
      }
      if (i0 >= v_hi) break;   // (a CTA without rows only formed alpha)
      rr = fma(ri, ri, rr);
      rsh[tid] = ri;
      named_bar_sync(9, PC_T);
      // U^T r over this chunk: warp w takes columns 4w .. 4w+3, 4w + 60 ..; lane L rows L, L + 32, ..
      // (coalesced 256-B column reads), 4 columns x 8 row blocks of loads in flight
      const int nrow = (int)((v_hi - i0) < PC_T ? (v_hi - i0) : PC_T);
      for (int c0 = 4 * warp; c0 < ell; c0 += 4 * PC_W) {
        double a[4] = {0.0, 0.0, 0.0, 0.0};
        for (int q0 = 0; q0 < nrow; q0 += 256) {
          double v[4][8];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int q = q0 + lane + 32 * k;
              v[cc][k] = (c0 + cc < ell && q < nrow) ? __ldg(P.U + (size_t)(c0 + cc) * P.ldu + i0 + q) : 0.0;
            }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int q = q0 + lane + 32 * k;
            const double rv = (q < nrow) ? rsh[q] : 0.0;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) a[cc] = fma(v[cc][k], rv, a[cc]);
          }
        }
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const double t = warp_sum(a[cc]);
          if (lane == 0 && c0 + cc < ell) gpart[c0 + cc] += t;
        }
      }
      named_bar_sync(9, PC_T);
    }
    const double rrw = warp_sum(rr);
    if (lane == 0) wsh[warp] = rrw;
    named_bar_sync(9, PC_T);
    double* row = P.part1 + (size_t)bid * ncol;
    if (tid == 0) {
      double b = 0.0;
      for (int w = 0; w < PC_W; ++w) b += wsh[w];
      row[0] = b;
    }
    for (int c = tid; c < ell; c += PC_T) row[1 + c] = gpart[c];
    return true;
  };

  // ---- grid barrier, then every CTA sums the G partial rows itself in one fixed order ----------------
  // thread (slice sl, column c) sums rows g = sl, sl + NS, ... (LB loads in flight, pairwise tree), then
  // the NS slice sums are added in order: s_scal[0] = ||r||^2, gsh = U^T r, hsh = s o U^T r,
  // s_scal[1] = r^T z = ||r||^2 + (U^T r)^T h
  auto reduce_rows = [&]() {
    pcgc_grid_barrier(P.bar, G, bar_epoch, P.acq_spin != 0);
    const int CP = ncol <= 120 ? 120 : (ncol <= 240 ? 240 : 480);
    const int NS = PC_T / CP;
    const int sl = tid / CP, c = tid % CP;
    if (c < ncol) {
      constexpr int LB = 40;
      double tot = 0.0;
#pragma unroll 1
      for (int g0 = sl; g0 < (int)G; g0 += NS * LB) {
        double v[LB];
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const int gg = g0 + NS * u;
          v[u] = (gg < (int)G) ? __ldcg(P.part1 + (size_t)gg * ncol + c) : 0.0;
        }
#pragma unroll
        for (int w = 32; w > 0; w >>= 1)
#pragma unroll
          for (int u = 0; u < w; ++u)
            if (u + w < LB) v[u] += v[u + w];
        tot += v[0];
      }
      colred[sl * CP + c] = tot;
    }
    named_bar_sync(9, PC_T);
    for (int cc = tid; cc < ncol; cc += PC_T) {
      double sum = 0.0;
      for (int q = 0; q < NS; ++q) sum += colred[q * CP + cc];
      if (cc == 0) s_scal[0] = sum;
      else {
        gsh[cc - 1] = sum;
        hsh[cc - 1] = P.s[cc - 1] * sum;
      }
    }
    named_bar_sync(9, PC_T);
    if (warp == 0) {
      double acc = 0.0;
      for (int cc = lane; cc < ell; cc += 32) acc = fma(gsh[cc], hsh[cc], acc);
      acc = warp_sum(acc);
      if (lane == 0) s_scal[1] = s_scal[0] + acc;
    }
    named_bar_sync(9, PC_T);
  };

  // ---- own rows: p_next = r + U h + beta p_cur (U h: 20 column loads in flight per row) -------------
  // (with the row part of the next p^T N p: (delta + e_i) p_i^2 over the own rows -> pwrow[bid])
  auto prec_rows = [&](bool init, double beta, const double* pcur, double* pnext) {
    double prow = 0.0;
    for (int64_t i0 = v_lo; i0 < v_hi; i0 += PC_T) {
      const int64_t i = i0 + tid;
      if (i >= v_hi) continue;
      const double ei = P.e ? P.e[i] : 0.0;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int c0 = 0; c0 < ell; c0 += 20) {
        double v[20];
#pragma unroll
        for (int k = 0; k < 20; ++k) v[k] = (c0 + k < ell) ? __ldg(P.U + (size_t)(c0 + k) * P.ldu + i) : 0.0;
#pragma unroll
        for (int k = 0; k < 20; ++k) acc[k & 3] = fma(v[k], hsh[c0 + k], acc[k & 3]);
      }
      const double zi = __ldcg(P.r + i) + ((acc[0] + acc[1]) + (acc[2] + acc[3]));
      const double pi = init ? zi : fma(beta, __ldcg(pcur + i), zi);
      pnext[i] = pi;
      prow = fma((delta + ei) * pi, pi, prow);
    }
    const double pw_w = warp_sum(prow);
    if (lane == 0) wsh[warp] = pw_w;
    named_bar_sync(9, PC_T);
    if (tid == 0) {
      double b = 0.0;
      for (int w = 0; w < PC_W; ++w) b += wsh[w];
      P.pwrow[bid] = b;
    }
  };

  // ---- the stop test after a reduction (identical in every CTA) ------------------------------------
  auto converged = [&](bool init) -> bool {
    const double rrt = s_scal[0];
    bool cv = sqrt(rrt) <= P.sc[S_TOL];
    if (!isfinite(rrt)) { status = NYS_EBREAKDOWN; cv = true; }
    if (!init) ++iters;
    if (cv || iters >= P.max_iter) {
      if (bid == 0 && tid == 0) P.sc[S_RR] = rrt;
      return true;
    }
    return false;
  };

  // initialisation (k = -1): x = 0, r = rhs, p_0 = z_0 -> P1
  rows_phase(true, nullptr);
  reduce_rows();
  bool stop = converged(true);
  if (!stop) {
    const double rzn = s_scal[1];
    if (!(rzn > 0.0) || !isfinite(rzn)) {
      status = NYS_EBREAKDOWN;
      stop = true;
    } else {
      rz = rzn;
      prec_rows(true, 0.0, nullptr, P.P1);
      pcgc_grid_barrier(P.bar, G, bar_epoch, P.acq_spin != 0);
    }
  }
  for (int k = 0; !stop; ++k) {
    const double* pk = (k & 1) ? P.P0 : P.P1;   // p_k
    double* pn = (k & 1) ? P.P1 : P.P0;         // receives p_{k+1}
    trace_k = k;
    stamp(0);
    unsigned long long t_mv0 = 0;
    if (P.trace_mv != nullptr && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_mv0));
    // ---- P1: p_k slice; fused matvec over this cluster's panels (lag-1 dot exchange) --------------
    double vreg[RPT], wacc[RPT];
    double pwacc = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int64_t rl = tid + (int64_t)PC_T * i;
      vreg[i] = (rl < rows_valid) ? __ldcg(pk + r0 + rl) : 0.0;
      wacc[i] = 0.0;
    }
    double dprev = 0.0;
    int sp = 0;
    for (int64_t it = 0; it <= niter; ++it) {
      double dcur = 0.0;
      if (it < niter) {
        mbar_wait(&full[cs], cph);
        double* sb = stage + (size_t)cs * SS;
        if (odd_owner) sb[rows_valid] = 0.0;
        dcur = __ldg(P.d + (int64_t)ccol + it * ncl);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < RPT; ++i) acc[i & 3] = fma(sb[tid + PC_T * i], vreg[i], acc[i & 3]);
        const double pd = warp_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
        const long long jd = qd + it;
        const int db = (int)(jd & (PC_DB - 1));
        double* rb = red + (size_t)(jd & 1) * PC_W;
        if (lane == 0) rb[warp] = pd;
        if (tid == 0) mbar_arrive_expect_tx(&dotbar[db], (uint32_t)(cl * 8));
        named_bar_sync(1, PC_T);
        if (warp == 0) {
          double xs = (lane < PC_W) ? rb[lane] : 0.0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
          if (lane < cl) {
            const uint32_t my_slot = smem_u32(&slots[(size_t)db * cl + crank]);
            st_async_f64(mapa_shared(my_slot, (uint32_t)lane), xs, mapa_shared(smem_u32(&dotbar[db]), (uint32_t)lane));
          }
        }
      }
      if (it >= 1) {
        const long long jd = qd + it - 1;
        const int db = (int)(jd & (PC_DB - 1));
        mbar_wait(&dotbar[db], (uint32_t)((jd / PC_DB) & 1));
        // the cl CTA partials summed by a 16-wide xor butterfly: the same bits on every CTA
        double xs = ((lane & 15) < cl) ? slots[(size_t)db * cl + (lane & 15)] : 0.0;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
        const double t = dprev * xs;
        if (tid == 0 && crank == 0) pwacc = fma(t, xs, pwacc);   // d_j (a_j^T p)^2
        const double* sb = stage + (size_t)sp * SS;
#pragma unroll
        for (int i = 0; i < RPT; ++i) wacc[i] = fma(sb[tid + PC_T * i], t, wacc[i]);
        if (odd_owner) fence_proxy_async_shared();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sp]);
      }
      if (it < niter) {
        dprev = dcur;
        sp = cs;
        ++qc;
        if (++cs == S) { cs = 0; cph ^= 1u; }
      }
    }
    qd += niter;
    {
      double* outp = P.Wp + (size_t)cid * P.wp_ld + r0;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int64_t rl = tid + (int64_t)PC_T * i;
        if (rl < rows_valid) outp[rl] = wacc[i];
      }
      const double wsum = warp_sum(pwacc);
      if (lane == 0) wsh[warp] = wsum;
      named_bar_sync(9, PC_T);
      if (tid == 0) {
        double b = 0.0;
        for (int w = 0; w < PC_W; ++w) b += wsh[w];
        P.pwp[bid] = b;
      }
    }
    stamp(1);
    if (P.trace_mv != nullptr && tid == 0 && k == 9) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      P.trace_mv[bid] = t - t_mv0;
    }
    pcgc_grid_barrier(P.bar, G, bar_epoch, P.acq_spin != 0);
    stamp(2);
    // ---- P2: alpha, own rows, partial rows -------------------------------------------------------
    if (!rows_phase(false, pk)) { status = NYS_EBREAKDOWN; break; }
    stamp(3);
    // ---- P3: reduction, stop test, p_{k+1} -------------------------------------------------------
    reduce_rows();
    stamp(4);
    if (converged(false)) break;
    const double rzn = s_scal[1];
    if (!(rzn > 0.0) || !isfinite(rzn)) { status = NYS_EBREAKDOWN; break; }
    const double beta = rzn / rz;
    rz = rzn;
    prec_rows(false, beta, pk, pn);
    stamp(5);
    pcgc_grid_barrier(P.bar, G, bar_epoch, P.acq_spin != 0);
    stamp(6);
  }

  // ---- exit: stop the producer, drain in-flight bulk copies, publish the scalars ------------------
  if (tid == 0) s_stop = 1;
  named_bar_sync(10, PC_T + 32);
  const long long issued = s_issued;
  for (; qc < issued; ++qc) {
    mbar_wait(&full[cs], cph);
    if (++cs == S) { cs = 0; cph ^= 1u; }
  }
  if (bid == 0 && tid == 0) {
    P.sc[S_ITERS] = (double)iters;
    P.sc[S_STATUS] = (double)status;
    P.sc[S_DONE] = 1.0;
    P.sc[S_RZ] = rz;
  }
  __syncwarp();
  cluster_sync_all();   // no CTA leaves while a peer may still address its shared memory
}

// ------------------------------------------------------------------------------------------
bool pcg_cluster_supported(nys_ctx* ctx, int64_t m, int64_t n, int ell) {
  return !ctx->multi() && m > 8192 && m <= 16LL * 8640 && n > 0 && ell <= PC_LMAX &&
         getenv("NYS_NO_PCG_CLUSTER") == nullptr && getenv("NYS_NO_PERSISTENT") == nullptr;
}

int launch_pcg_cluster(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d,
                       const double* e, const double* U, int64_t ldu, int ell, const double* s, const double* rhs,
                       double* x, int max_iter) {
  constexpr int RPT = 18;
  constexpr int SS = PC_T * RPT;
  auto k = pcg_cluster_kernel<RPT>;
  struct Plan {
    int cl = 0, stages = 0, ncl = 0;
    size_t smem = 0;
  };
  static std::mutex mu;
  static std::map<std::pair<int, int64_t>, Plan> plans;
  Plan pl;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = plans.find({ctx->device, m});
    if (it != plans.end()) pl = it->second;
  }
  if (pl.cl == 0) {
    const size_t fixed = (size_t)2 * PC_W * 8 + (size_t)PC_DB * 8 + (size_t)PC_DB * 16 * 8;
    int stages = (int)((212 * 1024 - fixed) / ((size_t)SS * 8 + 16));
    if (stages > 8) stages = 8;
    if (stages < 2) stages = 2;
    const size_t smem = (size_t)stages * SS * 8 + 2 * (size_t)stages * 8 + fixed;
    NYS_TRY(ensure_max_smem(ctx, (const void*)k, smem));
    NYS_CUDA_TRY(ctx, cudaFuncSetAttribute((const void*)k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    // smallest cluster whose resident CTA count is within 5 % of the best (as the K1 planner)
    int clmin = (int)((m + SS - 1) / SS);
    if (clmin < 2) clmin = 2;
    int res[17] = {0}, ncls[17] = {0}, best = 0;
    for (int c = clmin; c <= 16; ++c) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(c * ctx->num_sms));
      cfg.blockDim = dim3(PC_T + 32);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = 0;
      if (cudaOccupancyMaxActiveClusters(&nc, (const void*)k, &cfg) != cudaSuccess) { cudaGetLastError(); nc = 0; }
      ncls[c] = nc;
      res[c] = nc * c;
      if (res[c] > best) best = res[c];
    }
    if (best == 0) { ctx->set_error("cluster PCG: no cluster configuration fits on the device"); return NYS_ECUDA; }
    for (int c = clmin; c <= 16; ++c)
      if (res[c] > 0 && res[c] * 20 >= best * 19) { pl.cl = c; break; }
    if (const char* oc = getenv("NYS_PCG_CL")) {   // tuning override
      const int o = atoi(oc);
      if (o >= clmin && o <= 16 && res[o] > 0) pl.cl = o;
    }
    pl.ncl = ncls[pl.cl];
    pl.stages = stages;
    pl.smem = smem;
    std::lock_guard<std::mutex> lk(mu);
    plans[{ctx->device, m}] = pl;
  }
  int64_t ncl = pl.ncl;
  if (ncl > n) ncl = n;
  if (ncl < 1) ncl = 1;
  const int G = (int)(ncl * pl.cl);
  const int64_t mp = (m + 1) & ~int64_t(1);
  PcgCParams P{};
  P.A = A; P.lda = lda; P.m = m; P.n = n; P.d = d; P.e = e; P.U = U; P.ldu = ldu; P.ell = ell; P.s = s;
  P.rhs = rhs; P.x = x;
  P.r = ctx->wsd("pc_r", (size_t)mp);
  P.P0 = ctx->wsd("pc_p0", (size_t)mp);
  P.P1 = ctx->wsd("pc_p1", (size_t)mp);
  P.wp_ld = mp;
  P.Wp = ctx->wsd("pc_Wp", (size_t)ncl * mp);
  P.pwp = ctx->wsd("pc_pwp", (size_t)G);
  P.pwrow = ctx->wsd("pc_pwrow", (size_t)G);
  P.part1 = ctx->wsd("pc_part1", (size_t)G * (1 + ell));
  P.bar = (unsigned int*)ctx->ws("pc_bar", 64);
  P.sc = ctx->sc;
  P.max_iter = max_iter;
  P.stages = pl.stages;
  P.cl = pl.cl;
  P.rs = (((m + pl.cl - 1) / pl.cl) + 1) & ~int64_t(1);
  P.rpc = (m + G - 1) / G;
  P.acq_spin = getenv("NYS_BAR_FENCE") ? 0 : 1;
  NYS_CUDA_TRY(ctx, cudaMemsetAsync(P.bar, 0, 64, ctx->stream));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)G);
  cfg.blockDim = dim3(PC_T + 32);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = pl.cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  // grid-wide barriers need every CTA resident: G = the device's max active clusters x cl, launched
  // cooperatively (the launch fails rather than deadlocks if they do not fit)
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  // NYS_PCG_NOCOOP=1: a plain cluster launch of the same grid (Nsight Compute cannot launch cooperative
  // cluster kernels; it serialises kernels, so the occupancy-sized grid is co-resident there)
  cfg.numAttrs = getenv("NYS_PCG_NOCOOP") ? 1 : 2;
  if (getenv("NYS_DEBUG"))
    fprintf(stderr, "[nys] cluster PCG m=%lld n=%lld ell=%d: cl=%d clusters=%lld G=%d rs=%lld rpc=%lld stages=%d smem=%zu\n",
            (long long)m, (long long)n, ell, pl.cl, (long long)ncl, G, (long long)P.rs, (long long)P.rpc, pl.stages,
            pl.smem);
  const bool trace = getenv("NYS_PCG_TRACE") != nullptr;
  if (trace) {
    P.trace = (unsigned long long*)ctx->ws("pc_trace", 2 * 16 * 8 * 8);
    NYS_CUDA_TRY(ctx, cudaMemsetAsync(P.trace, 0, 2 * 16 * 8 * 8, ctx->stream));
    P.trace_mv = (unsigned long long*)ctx->ws("pc_trace_mv", (size_t)G * 8);
    NYS_CUDA_TRY(ctx, cudaMemsetAsync(P.trace_mv, 0, (size_t)G * 8, ctx->stream));
  }
  // if fewer clusters can be co-resident than the occupancy query promised (a profiler's reserved
  // resources, another context on the GPU), the cooperative launch is refused: retry with fewer clusters
  // (the vector-phase row ranges follow G; every workspace above is sized for the largest grid)
  for (;;) {
    const cudaError_t le = cudaLaunchKernelEx(&cfg, k, P);
    if (le == cudaSuccess) break;
    if ((le == cudaErrorCooperativeLaunchTooLarge || le == cudaErrorInvalidConfiguration ||
         le == cudaErrorLaunchOutOfResources) && ncl > 1) {
      cudaGetLastError();
      --ncl;
      const int Gr = (int)(ncl * pl.cl);
      cfg.gridDim = dim3((unsigned)Gr);
      P.rpc = (m + Gr - 1) / Gr;
      continue;
    }
    ctx->set_error(std::string("pcg_cluster launch: ") + cudaGetErrorString(le));
    return NYS_ECUDA;
  }
  ctx->launches++;
  if (trace) {
    unsigned long long h[2 * 16 * 8];
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(h, P.trace, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    NYS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    {
      std::vector<unsigned long long> mvt((size_t)G);
      NYS_CUDA_TRY(ctx, cudaMemcpy(mvt.data(), P.trace_mv, (size_t)G * 8, cudaMemcpyDeviceToHost));
      std::string line;
      for (int q = 0; q < G; q += pl.cl) {   // per cluster: the slowest CTA's matvec phase (us)
        unsigned long long mx = 0;
        for (int r = 0; r < pl.cl && q + r < G; ++r) mx = mvt[q + r] > mx ? mvt[q + r] : mx;
        char b[32];
        snprintf(b, sizeof(b), " %.1f", mx * 1e-3);
        line += b;
      }
      fprintf(stderr, "[pcgctrace] it=9 matvec phase per cluster (us):%s\n", line.c_str());
    }
    for (int c = 0; c < 2; ++c)
      for (int it = 8; it < 12; ++it) {
        const unsigned long long* r = h + (c * 16 + it) * 8;
        if (r[0] == 0 || r[6] == 0) continue;
        fprintf(stderr, "[pcgctrace] cta=%s it=%d matvec=%.2f bar1=%.2f rows=%.2f reduce=%.2f prec=%.2f bar3=%.2f total=%.2f us\n",
                c ? "last" : "0", it, (r[1] - r[0]) * 1e-3, (r[2] - r[1]) * 1e-3, (r[3] - r[2]) * 1e-3,
                (r[4] - r[3]) * 1e-3, (r[5] - r[4]) * 1e-3, (r[6] - r[5]) * 1e-3, (r[6] - r[0]) * 1e-3);
      }
  }
  return ctx->check_launch("pcg_cluster");
}

}  // namespace nys
