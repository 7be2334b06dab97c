// K1 — fused fp64 normal-equation matvec  w = A diag(d) A^T v (+ e o v + delta v)
// (PAPER.md:201 N_k = A (Q + Theta^{-1} + rho I)^{-1} A^T, P:835 the PCG operator).
//
// ONE pass over A.  A is column-major; a "panel" is BN consecutive columns.  A CTA (or a
// thread-block cluster of CL CTAs splitting the rows, for m > 8192) owns whole panels:
//   1. a producer warp streams each column segment (contiguous in memory) into a shared
//      memory stage with 1-D bulk async copies (cp.async.bulk, L2 evict_first) completing on
//      an mbarrier; S stages are in flight;
//   2. consumer threads copy their rows of the stage into registers and release the stage;
//   3. column dots (A^T v)_j: FMA in registers, warp shuffles, a per-group shared reduction
//      and (CL > 1) a DSMEM exchange of the CTA partials through remote mbarrier arrives;
//      every CTA sums the CL partials in rank order, so t_j = d_j (A^T v)_j is identical on
//      all CTAs of the cluster;
//   4. the same registers are reused for the rank-BN update  w_acc += A_panel t_panel.
// Each cluster writes its m-slice partial w to a workspace row; `mv_finalize` sums the
// partials in a fixed order (deterministic) and applies (delta + e) v, additive terms and
// the optional PCG dot p^T w / alpha = rz / p^T w.
//
// The same kernel also provides the T-only pass (A^T v with IPM epilogues), the N-only
// pass (A u) that Alg. 4 needs, and both at once on independent operands
// (MV_BOTH: A^T y with an epilogue and A x from the same read of A — the residuals).
#include <cstdlib>
#include <mutex>

#include "nys_common.cuh"

namespace nys {

// ------------------------------------------------------------------------------------------
// finalize: out_i = sgn * sum_k Wp[k][i] + (delta + e_i) v_i + add_i ; optional PCG dot
// ------------------------------------------------------------------------------------------
struct FinParams {
  const double* Wp;
  int64_t wp_ld;
  int nparts;
  int64_t m;
  double sgn;
  double delta;
  int use_delta;
  const double* e;
  const double* v;      // operand vector (p for PCG)
  const double* add;
  double* out;
  int pcg_alpha;
  double* sc;           // scalar slots
  double* part;         // per-block partials (pcg dot)
  unsigned int* counter;
  const double* done;
};

// 16 rows x 16 partial groups per 256 threads (tid < 256); fixed summation order (deterministic).
// Row blocks b, b + nb, ... of 16 rows; the partial rows are read through L2 (they may have been
// written by other CTAs of the same launch).  Then the optional PCG dot (last-block pattern).
__device__ __forceinline__ void fin_rows(const FinParams& F, int b, int nb, double (*red)[17], double* sred,
                                         bool* am_last) {
  const int tid = threadIdx.x, row = tid & 15, grp = (tid >> 4) & 15;
  const bool act = tid < 256;
  double dot = 0.0;
  for (int64_t i0 = (int64_t)b * 16; i0 < F.m; i0 += (int64_t)nb * 16) {
    const int64_t i = i0 + row;
    if (act) {
      double acc = 0.0;
      if (i < F.m) {
        for (int k0 = grp; k0 < F.nparts; k0 += 128) {  // 8 independent L2 loads per round
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int k = k0 + 16 * u;
            v[u] = (k < F.nparts) ? __ldcg(F.Wp + (size_t)k * F.wp_ld + i) : 0.0;
          }
          acc += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
        }
      }
      red[row][grp] = acc;
    }
    __syncthreads();
    if (tid < 16 && i < F.m) {
      const double* v = red[row];
      double s = (((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]))) +
                 (((v[8] + v[9]) + (v[10] + v[11])) + ((v[12] + v[13]) + (v[14] + v[15])));
      s *= F.sgn;
      const double vi = (F.use_delta || F.pcg_alpha) ? __ldcg(F.v + i) : 0.0;  // may be p_out of this launch
      if (F.use_delta) s += (F.delta + (F.e ? F.e[i] : 0.0)) * vi;
      if (F.add) s += F.add[i];
      F.out[i] = s;
      if (F.pcg_alpha) dot = fma(vi, s, dot);
    }
    __syncthreads();
  }
  if (!F.pcg_alpha) return;
  dot = warp_sum(dot);
  if (act && (tid & 31) == 0) sred[tid >> 5] = dot;
  __syncthreads();
  if (tid == 0) {
    double bs = 0.0;
    for (int w = 0; w < 8; ++w) bs += sred[w];
    F.part[b] = bs;
    __threadfence();
    const unsigned prev = atomicAdd(F.counter, 1u);
    *am_last = (prev == (unsigned)nb - 1);
  }
  __syncthreads();
  if (*am_last && warp_uniform_id() == 0) {
    __threadfence();
    const double pw = warp_sum_array(F.part, nb);
    if (tid != 0) return;
    *F.counter = 0u;
    F.sc[S_PW] = pw;
    if (!(pw > 0.0) || !isfinite(pw)) {
      F.sc[S_STATUS] = (double)NYS_EBREAKDOWN;
      F.sc[S_DONE] = 1.0;
      F.sc[S_ALPHA] = 0.0;
    } else {
      F.sc[S_ALPHA] = F.sc[S_RZ] / pw;
    }
  }
}

__global__ void __launch_bounds__(256) mv_finalize(const FinParams F) {
  if (F.done != nullptr && *F.done != 0.0) return;
  __shared__ double red[16][17];
  __shared__ double sred[8];
  __shared__ bool am_last;
  fin_rows(F, blockIdx.x, gridDim.x, red, sred, &am_last);
}

// self-resetting grid barrier (count, generation); the launch is cooperative (all CTAs resident)
__device__ __forceinline__ void mv_grid_sync(unsigned int* bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = bar + 1;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicExch(bar + 1, g + 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

struct MatvecParams {
  const double* A;
  int64_t lda, m, n;
  const double* z;
  const double* p;
  const double* beta;
  double* p_out;
  const double* d;
  const double* u;
  double* Wp;
  int64_t wp_ld;
  int tep;
  double* t1;
  double* t2;
  const double *ta, *tb, *tc, *td, *tx, *tdd;
  const double* done;
  int64_t rs;
  int64_t npanels;
  int stages;
  int l2pf;             // producer: L2 prefetch this many panels beyond the shared-memory ring
  int cl;
  int rc;               // reduction cluster size (cl == 1 only): CTAs of a cluster sum their w partials via DSMEM
  const double* delta_slot;  // if set, delta = *delta_slot
  double* pwp;          // FUSED: per-CTA partial of v^T (A D A^T + delta I + diag e) v  (or null)
  double delta;
  const double* e;
  double* tbuf;         // TONLY: raw column dots (A^T v)_j, epilogue applied after the loop
  int fuse_fin;         // cl == 1, rc == 1: finalize in-kernel after a grid barrier (cooperative launch)
  FinParams fin;
  unsigned int* gbar;   // [2] grid barrier (count, generation)
};

__device__ __forceinline__ void t_epilogue(const MatvecParams& P, int64_t j, double s) {
  if (P.tep == TE_PLAIN) {
    P.t1[j] = s;
  } else if (P.tep == TE_DX) {
    // Alg. 4 (P:840, P:842 / A15): dx = d (A^T dy - r_d - xi_au);  dz = (r_xz - z dx) / x
    double rd = P.ta ? P.ta[j] : 0.0;
    double dx = P.tdd[j] * (s - rd - P.tb[j]);
    P.t1[j] = dx;
    P.t2[j] = (P.tc[j] - P.td[j] * dx) / P.tx[j];
  } else {  // TE_RD: r_D = c + q x - A^T y - z
    double zz = P.td ? P.td[j] : 0.0;
    P.t1[j] = P.ta[j] + P.tb[j] * P.tc[j] - s - zz;
  }
}

template <int T, int GT, int RPT, int CPG, int MODE, bool VS, bool CLU>
__global__ void __launch_bounds__(T + 32, 1) matvec_kernel(const MatvecParams P) {
  constexpr int NG = T / GT;
  constexpr int WPG = GT / 32;
  constexpr int BN = NG * CPG;
  constexpr int DB = 4;  // depth of the cluster dot-exchange ring (>= 4: see the lag-1 argument below)
  extern __shared__ __align__(128) unsigned char smem_raw[];

  if (P.done != nullptr && *P.done != 0.0) return;  // grid-uniform early exit (PCG converged)

  const int S = P.stages;
  const int64_t rs = P.rs;
  // stage column stride: the cluster path pads each column slot to GT * RPT rows (>= rs), the rows a
  // thread block covers, so the inner loops read every slot row without bounds checks (the pad rows
  // are zero-filled once below and never written by the bulk copies)
  const int64_t ss = CLU ? (int64_t)GT * RPT : rs;
  const int cl = CLU ? P.cl : 1;
  double* stage = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(stage + (size_t)S * BN * ss);
  uint64_t* empty = full + S;
  uint64_t* dotbar = empty + S;                       // DB barriers (CLU)
  double* red = reinterpret_cast<double*>(dotbar + DB);
  double* slots = red + 2 * NG * WPG * CPG;           // [DB][cl][CPG] (CLU)
  double* vsm = slots + (size_t)DB * cl * CPG;        // VS: the operand slice v (rs doubles)

  const int tid = threadIdx.x;
  const int warp = warp_uniform_id(), lane = tid & 31;
  const int rc = P.rc;
  const uint32_t crank = CLU ? cluster_ctarank() : 0u;
  const uint32_t cid = CLU ? cluster_id_x() : blockIdx.x;
  const uint32_t ncl = CLU ? ncluster_x() : gridDim.x;
  const int64_t r0 = (int64_t)crank * rs;
  int64_t rows_valid = P.m - r0;
  rows_valid = rows_valid < 0 ? 0 : (rows_valid > rs ? rs : rows_valid);
  const uint32_t copy_bytes = (uint32_t)(((rows_valid + 1) & ~int64_t(1)) * 8);
  const int64_t niter = (cid < P.npanels) ? (P.npanels - cid + ncl - 1) / ncl : 0;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], T / 32);
    }
    if (CLU)
      for (int s = 0; s < DB; ++s) mbar_init(&dotbar[s], 1);  // own arrive.expect_tx; peers complete_tx
    fence_mbar_init();
  }
  if (CLU) {
    // zero the pad rows [copy rows, GT * RPT) of every stage slot once: disjoint from what the bulk
    // copies write, so no proxy fence is needed (the cluster barrier below orders them before use)
    const int64_t crow = (rows_valid + 1) & ~int64_t(1);
    const int64_t npad = ss - crow;
    if (npad > 0)
      for (int64_t e = tid; e < (int64_t)S * BN * npad; e += T + 32)
        stage[(e / npad) * ss + crow + (e % npad)] = 0.0;
  }
  if (CLU) cluster_sync_all(); else __syncthreads();

  const int g = tid / GT;
  const int lig = tid % GT;
  double vreg[VS ? 1 : RPT];
  double wacc[RPT];
  double pwacc = 0.0;
#pragma unroll
  for (int i = 0; i < RPT; ++i) { if (!VS) vreg[i] = 0.0; wacc[i] = 0.0; }

  if (warp == T / 32) {
    // ------------------------------ producer warp ------------------------------------------
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      // contiguous panels (no cluster split, column stride == smem stride): one copy per stage
      const bool contig = !CLU && P.lda == rs;
      int s = 0;
      uint32_t eph = 1u;  // parity of the empty-barrier phase to wait for (first pass: none)
      const int PF = P.l2pf;
      for (int64_t it = 0; it < niter; ++it, ++s) {
        if (s == S) { s = 0; eph ^= 1u; }
        // L2 prefetch of the panel PF stages beyond the ring: more bytes in flight per SM than the
        // shared-memory stages hold (the bulk copies then hit L2)
        if (PF > 0) {
          const int64_t itp = (it == 0) ? -1 : it + S - 1 + PF;   // the first call covers S..S+PF-1 below
          for (int64_t q = (it == 0 ? S : itp); q <= (it == 0 ? S + PF - 1 : itp); ++q) {
            if (q >= niter) break;
            const int64_t c0 = (int64_t)(cid + q * ncl) * BN;
            int64_t nc = P.n - c0;
            nc = nc > BN ? BN : nc;
            if (nc <= 0) break;
            if (contig) {
              bulk_prefetch_l2(P.A + c0 * P.lda, (uint32_t)((nc - 1) * rs * 8) + copy_bytes);
            } else {
              for (int c = 0; c < nc; ++c) bulk_prefetch_l2(P.A + (c0 + c) * P.lda + r0, copy_bytes);
            }
          }
        }
        if (it >= S) mbar_wait(&empty[s], eph);
        const int64_t col0 = (int64_t)(cid + it * ncl) * BN;
        int64_t ncols = P.n - col0;
        ncols = ncols > BN ? BN : ncols;
        if (ncols <= 0) {
          mbar_arrive(&full[s]);
        } else if (contig) {
          const uint32_t bytes = (uint32_t)((ncols - 1) * rs * 8) + copy_bytes;  // lda even: 16-B multiple
          mbar_arrive_expect_tx(&full[s], bytes);
          bulk_g2s(stage + (size_t)s * BN * rs, P.A + col0 * P.lda, bytes, &full[s], pol);
        } else {
          mbar_arrive_expect_tx(&full[s], (uint32_t)ncols * copy_bytes);
          for (int c = 0; c < ncols; ++c)
            bulk_g2s(stage + ((size_t)s * BN + c) * ss, P.A + (col0 + c) * P.lda + r0, copy_bytes, &full[s], pol);
        }
      }
    }
  } else {
    // ------------------------------ consumers ----------------------------------------------
    if (MODE != MV_NONLY && MODE != MV_DIAG) {
      const double bval = (P.beta != nullptr) ? *P.beta : 0.0;
      // every operand load first, then the p_out stores: a store that may alias z / p would
      // otherwise serialise the following loads (one L2 round trip per row)
      double zr[RPT], pr[RPT];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int64_t rl = lig + (int64_t)GT * i;
        const bool ok = rl < rs && rl < rows_valid;
        zr[i] = ok ? P.z[r0 + rl] : 0.0;
        pr[i] = (ok && P.p != nullptr) ? P.p[r0 + rl] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int64_t rl = lig + (int64_t)GT * i;
        if (rl < rs) {
          double v = 0.0;
          if (rl < rows_valid) {
            v = (P.p != nullptr) ? zr[i] + bval * pr[i] : zr[i];
            if (P.p_out != nullptr && cid == 0 && g == 0) P.p_out[r0 + rl] = v;
          }
          if (VS) { if (g == 0) vsm[rl] = v; } else vreg[i] = v;
        }
      }
    }
    if (VS) named_bar_sync(1, T);  // vsm complete (NG == 1 for VS)

    if (CLU && MODE != MV_NONLY && MODE != MV_DIAG) {
      // ---- cluster path (rows split over cl CTAs; NG == 1; v in registers).  Lag-1 software
      // pipeline: the CTA partial dots of panel `it` are pushed to every peer with st.async
      // (completing bytes on the peer's dotbar), and the rank-CPG update of panel it-1 runs
      // while they travel, so no CTA waits a DSMEM round trip on the critical path.  The dot and
      // the update both read the panel from its shared-memory stage (no panel registers: the
      // 512-thread CTA has ~120 registers per thread); a stage is released after its update.
      // Per-panel critical path kept short: 4 independent FMA chains, xor-tree reductions
      // (warp, then CTA by warp 0), one peer per lane for the publish.
      // Ring safety: a peer publishes panel j+DB only after consuming j+DB-2, which needs our
      // publish of j+DB-2, issued after our consume of j+DB-3 >= j for DB >= 3 (DB = 4 here).
      static_assert(WPG <= 32, "one lane per warp partial");
      // an odd slice length copies one row past the slice (bulk sizes are 16-byte multiples): the
      // thread owning that row zeroes it in every stage it reads (then fences the generic write
      // against the next bulk copy into the stage), so garbage there can never reach a dot
      const bool odd_owner = (rows_valid & 1) && (rows_valid % GT) == lig && rows_valid < ss;
      const int ssi = (int)ss;
      double dprev[CPG];
      int64_t cprev = 0;
#pragma unroll
      for (int c = 0; c < CPG; ++c) dprev[c] = 0.0;
      int s = 0, sp = 0;
      uint32_t ph = 0;
      for (int64_t it = 0; it <= niter; ++it) {
        double dcur[CPG];
        const int64_t col0 = (int64_t)(cid + it * ncl) * BN;
        if (it < niter) {
          mbar_wait(&full[s], ph);
          double* sb = stage + (size_t)s * BN * ss;
          if (odd_owner) {
#pragma unroll
            for (int c = 0; c < CPG; ++c) sb[c * ss + rows_valid] = 0.0;
          }
#pragma unroll
          for (int c = 0; c < CPG; ++c)   // FUSED: d_j;  BOTH: the N-part coefficient u_j
            dcur[c] = (col0 + c < P.n) ? (MODE == MV_FUSED ? __ldg(P.d + col0 + c) : MODE == MV_BOTH ? __ldg(P.u + col0 + c) : 0.0) : 0.0;
          double pd[CPG];
#pragma unroll
          for (int c = 0; c < CPG; ++c) {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (col0 + c < P.n) {      // warp-uniform; rows past the slice read the zero pad / vreg = 0
#pragma unroll
              for (int i = 0; i < RPT; ++i)
                acc[i & 3] = fma(sb[c * ssi + lig + GT * i], vreg[VS ? 0 : i], acc[i & 3]);
            }
            pd[c] = warp_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
          }
          const int db = (int)(it & (DB - 1));
          double* rb = red + (size_t)(it & 1) * WPG * CPG;
          if (lane == 0) {
#pragma unroll
            for (int c = 0; c < CPG; ++c) rb[c * WPG + warp] = pd[c];
          }
          if (tid == 0) mbar_arrive_expect_tx(&dotbar[db], (uint32_t)(cl * CPG * 8));
          named_bar_sync(1, T);
          if (warp == 0) {
            const uint32_t my_bar = smem_u32(&dotbar[db]);
#pragma unroll
            for (int c = 0; c < CPG; ++c) {
              double x = (lane < WPG) ? rb[c * WPG + lane] : 0.0;
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
              if (lane < cl) {
                const uint32_t my_slot = smem_u32(&slots[((size_t)db * cl + crank) * CPG + c]);
                st_async_f64(mapa_shared(my_slot, (uint32_t)lane), x, mapa_shared(my_bar, (uint32_t)lane));
              }
            }
          }
        }
        if (it >= 1) {
          const int64_t j = it - 1;
          const int db = (int)(j & (DB - 1));
          mbar_wait(&dotbar[db], (uint32_t)((j / DB) & 1));
          double pd[CPG];
#pragma unroll
          for (int c = 0; c < CPG; ++c) {
            // the cl (<= 16) CTA partials, lane r holding rank r's, summed by a 16-wide xor butterfly:
            // fp addition is commutative, so every lane of every CTA of the cluster gets the same bits
            // (the same t_j), at 1 load + 4 shuffle-adds per warp instead of cl loads + adds per thread
            double x = ((lane & 15) < cl) ? slots[((size_t)db * cl + (lane & 15)) * CPG + c] : 0.0;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            pd[c] = x;
          }
          if (MODE == MV_TONLY || MODE == MV_BOTH) {  // raw dot to global; epilogue after the loop
            if (crank == 0) {
#pragma unroll
              for (int c = 0; c < CPG; ++c)
                if (lig == c && cprev + c < P.n) P.tbuf[cprev + c] = pd[c];
            }
          }
          if (MODE == MV_FUSED || MODE == MV_BOTH) {
            double t[CPG];
#pragma unroll
            for (int c = 0; c < CPG; ++c) t[c] = MODE == MV_FUSED ? dprev[c] * pd[c] : dprev[c];
            if (MODE == MV_FUSED && lig == 0 && crank == 0) {
#pragma unroll
              for (int c = 0; c < CPG; ++c) pwacc = fma(t[c], pd[c], pwacc);  // d_j (a_j^T v)^2
            }
            const double* sb = stage + (size_t)sp * BN * ss;
#pragma unroll
            for (int c = 0; c < CPG; ++c) {
              if (cprev + c < P.n) {   // warp-uniform
#pragma unroll
                for (int i = 0; i < RPT; ++i) wacc[i] = fma(sb[c * ssi + lig + GT * i], t[c], wacc[i]);
              }
            }
          }
          if (odd_owner) fence_proxy_async_shared();
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[sp]);
        }
        if (it < niter) {
#pragma unroll
          for (int c = 0; c < CPG; ++c) dprev[c] = dcur[c];
          cprev = col0;
          sp = s;
          if (++s == S) { s = 0; ph ^= 1u; }
        }
      }
    } else {
    int s = -1;
    uint32_t par = 1u;
    for (int64_t it = 0; it < niter; ++it) {
      if (++s == S) s = 0;
      if (s == 0) par ^= 1u;
      const int64_t col0 = (int64_t)(cid + it * ncl) * BN + (int64_t)g * CPG;
      mbar_wait(&full[s], par);
      double a[CPG][RPT];
      const double* sb = stage + ((size_t)s * BN + (size_t)g * CPG) * ss;
#pragma unroll
      for (int c = 0; c < CPG; ++c) {
        const bool cv = (col0 + c) < P.n;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int64_t rl = lig + (int64_t)GT * i;
          a[c][i] = (cv && rl < rows_valid) ? sb[(size_t)c * ss + rl] : 0.0;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);

      double dpre[CPG];  // scaling of this group's columns, loaded before the dot (hides L2 latency)
#pragma unroll
      for (int c = 0; c < CPG; ++c)
        dpre[c] = (col0 + c < P.n) ? ((MODE == MV_FUSED || MODE == MV_DIAG) ? __ldg(P.d + col0 + c)
                                       : MODE == MV_BOTH ? __ldg(P.u + col0 + c) : 0.0) : 0.0;
      double t[CPG];
      if (MODE != MV_NONLY && MODE != MV_DIAG) {
        double pd[CPG];
#pragma unroll
        for (int c = 0; c < CPG; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            const int64_t rl = lig + (int64_t)GT * i;
            const double vv = VS ? ((rl < rs) ? vsm[rl] : 0.0) : vreg[VS ? 0 : i];
            acc = fma(a[c][i], vv, acc);
          }
          pd[c] = warp_sum(acc);
        }
        if (WPG > 1) {
          double* rb = red + ((size_t)(it & 1) * NG + g) * WPG * CPG;
          if (lane == 0) {
#pragma unroll
            for (int c = 0; c < CPG; ++c) rb[(warp % WPG) * CPG + c] = pd[c];
          }
          named_bar_sync(1 + g, GT);
#pragma unroll
          for (int c = 0; c < CPG; ++c) {
            double tot = 0.0;
#pragma unroll
            for (int w = 0; w < WPG; ++w) tot += rb[w * CPG + c];
            pd[c] = tot;
          }
        }
        if (MODE == MV_FUSED) {
#pragma unroll
          for (int c = 0; c < CPG; ++c) t[c] = dpre[c] * pd[c];
          if (lig == 0 && crank == 0) {
#pragma unroll
            for (int c = 0; c < CPG; ++c) pwacc = fma(t[c], pd[c], pwacc);  // d_j (a_j^T v)^2
          }
        } else {  // MV_TONLY / MV_BOTH: raw dot to global; the epilogue runs after the loop (no stall here)
          if (crank == 0) {
#pragma unroll
            for (int c = 0; c < CPG; ++c)
              if (lig == c && col0 + c < P.n) P.tbuf[col0 + c] = pd[c];
          }
          if (MODE == MV_BOTH) {
#pragma unroll
            for (int c = 0; c < CPG; ++c) t[c] = dpre[c];
          }
        }
      } else if (MODE == MV_DIAG) {
#pragma unroll
        for (int c = 0; c < CPG; ++c) t[c] = dpre[c];
      } else {
#pragma unroll
        for (int c = 0; c < CPG; ++c) t[c] = (col0 + c < P.n) ? P.u[col0 + c] : 0.0;
      }
      if (MODE != MV_TONLY) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          double acc = wacc[i];
#pragma unroll
          for (int c = 0; c < CPG; ++c) acc = fma(MODE == MV_DIAG ? a[c][i] * a[c][i] : a[c][i], t[c], acc);
          wacc[i] = acc;
        }
      }
    }
    }
  }
  if (MODE == MV_TONLY || MODE == MV_BOTH) {
    __syncthreads();  // this CTA's raw dots are visible to all its threads
    if (crank == 0) {
      for (int64_t e = tid; e < niter * BN; e += T + 32) {
        const int64_t j = (int64_t)(cid + (e / BN) * ncl) * BN + (e % BN);
        if (j < P.n) t_epilogue(P, j, P.tbuf[j]);
      }
    }
  }
  if (MODE == MV_FUSED && P.pwp != nullptr) {
    // row part of v^T (delta I + diag e) v, once (cluster 0, group 0), then CTA partial
    if (cid == 0 && g == 0 && tid < T) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int64_t rl = lig + (int64_t)GT * i;
        if (rl < rows_valid) {
          const double v = VS ? vsm[rl] : vreg[VS ? 0 : i];
          const double dl = P.delta_slot ? *P.delta_slot : P.delta;
          pwacc = fma((dl + (P.e ? P.e[r0 + rl] : 0.0)) * v, v, pwacc);
        }
      }
    }
    __shared__ double pws[32];
    const double wsum = warp_sum(pwacc);
    __syncthreads();
    if (lane == 0) pws[warp] = wsum;
    __syncthreads();
    if (tid == 0) {
      double b = 0.0;
      for (int w = 0; w < (T + 32) / 32; ++w) b += pws[w];
      P.pwp[blockIdx.x] = b;
    }
  }
  if (MODE != MV_TONLY && rc > 1) {
    // CTA total into smem, then the rc CTAs of the cluster each reduce a row range over all
    // rc CTAs through DSMEM (rank order: deterministic) -> one partial row per cluster
    __syncthreads();
    double* wsum = stage;
    if (tid < T) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int64_t rl = lig + (int64_t)GT * i;
        if (rl < rows_valid) wsum[(size_t)g * rs + rl] = wacc[i];
      }
    }
    __syncthreads();
    double* tot = stage + (size_t)NG * rs;
    if (NG > 1) {
      for (int64_t r = tid; r < rows_valid; r += T + 32) {
        double sacc = 0.0;
#pragma unroll
        for (int gg = 0; gg < NG; ++gg) sacc += wsum[(size_t)gg * rs + r];
        tot[r] = sacc;
      }
    } else {
      tot = wsum;
    }
    __syncwarp();
    cluster_sync_all();
    const uint32_t rr_ = cluster_ctarank();
    const int64_t chunk = (rows_valid + rc - 1) / rc;
    const int64_t lo = (int64_t)rr_ * chunk;
    int64_t hi = lo + chunk;
    if (hi > rows_valid) hi = rows_valid;
    double* outp = P.Wp + (size_t)cluster_id_x() * P.wp_ld;
    const uint32_t tbase = smem_u32(tot);
    for (int64_t r = lo + tid; r < hi; r += T + 32) {
      double sacc = 0.0;
      for (int q = 0; q < rc; ++q) sacc += ld_cluster_f64(mapa_shared(tbase + (uint32_t)(r * 8), (uint32_t)q));
      outp[r] = sacc;
    }
    __syncwarp();
    cluster_sync_all();
  } else if (MODE != MV_TONLY) {
    __syncthreads();  // all bulk copies consumed: the stage memory is free for the group sum
    double* outp = P.Wp + (size_t)cid * P.wp_ld + r0;
    if (NG == 1) {
      if (tid < T) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int64_t rl = lig + (int64_t)GT * i;
          if (rl < rows_valid) outp[rl] = wacc[i];
        }
      }
    } else {
      double* wsum = stage;
      if (tid < T) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int64_t rl = lig + (int64_t)GT * i;
          if (rl < rows_valid) wsum[(size_t)g * rs + rl] = wacc[i];
        }
      }
      __syncthreads();
      for (int64_t r = tid; r < rows_valid; r += T + 32) {
        double sacc = 0.0;
#pragma unroll
        for (int gg = 0; gg < NG; ++gg) sacc += wsum[(size_t)gg * rs + r];
        outp[r] = sacc;
      }
    }
  }
  if (!CLU && MODE != MV_TONLY && P.fuse_fin) {
    // every partial row is complete after the grid barrier; this CTA finalizes its row blocks
    __shared__ double fred[16][17];
    __shared__ double fsred[8];
    __shared__ bool fam_last;
    mv_grid_sync(P.gbar, gridDim.x);
    fin_rows(P.fin, blockIdx.x, gridDim.x, fred, fsred, &fam_last);
  }
  if (cl > 1) {
    __syncwarp();
    cluster_sync_all();
  }
}

// ------------------------------------------------------------------------------------------
// host dispatch
// ------------------------------------------------------------------------------------------
struct MvCfg {
  int T, GT, RPT, CPG;
};

static MvCfg pick_cfg(int64_t rs, bool clu) {
  if (clu) {  // cluster path: rows split over the cluster, one group of 480 consumer threads: with the
              // producer warp 16 warps, 4 per SM sub-partition -> 128 registers per thread (measured on
              // B200, m = 50000: 512 threads / 96 registers spill, 256 threads / 34 rows are DFMA-latency
              // bound at 4.9 TB/s; 480 / 18 rows: 6.8 TB/s at full clock)
    if (rs <= 3840) return {480, 480, 8, 2};
    if (rs <= 6720) return {480, 480, 14, 1};
    return {480, 480, 18, 1};
  }
  if (rs <= 64) return {256, 32, 2, 4};
  if (rs <= 128) return {256, 32, 4, 2};
  if (rs <= 256) return {256, 64, 4, 2};
  if (rs <= 1024) return {256, 128, 8, 2};
  if (rs <= 2048) return {256, 256, 8, 4};
  if (rs <= 4096) return {512, 512, 8, 2};
  return {512, 512, 16, 1};
}

typedef void (*MvKernel)(const MatvecParams);

template <int MODE>
static MvKernel kernel_for(const MvCfg& c, bool clu) {
  if (clu) {
    if (c.RPT == 8 && c.CPG == 2) return matvec_kernel<480, 480, 8, 2, MODE, false, true>;
    if (c.RPT == 14) return matvec_kernel<480, 480, 14, 1, MODE, false, true>;
    return matvec_kernel<480, 480, 18, 1, MODE, false, true>;
  }
  if (c.T == 256 && c.GT == 32 && c.RPT == 2 && c.CPG == 4) return matvec_kernel<256, 32, 2, 4, MODE, false, false>;
  if (c.T == 256 && c.GT == 32 && c.RPT == 4 && c.CPG == 2) return matvec_kernel<256, 32, 4, 2, MODE, false, false>;
  if (c.T == 256 && c.GT == 64 && c.RPT == 4 && c.CPG == 2) return matvec_kernel<256, 64, 4, 2, MODE, false, false>;
  if (c.T == 256 && c.GT == 128 && c.RPT == 8 && c.CPG == 2) return matvec_kernel<256, 128, 8, 2, MODE, false, false>;
  if (c.T == 256 && c.GT == 256 && c.RPT == 8 && c.CPG == 4) return matvec_kernel<256, 256, 8, 4, MODE, false, false>;
  if (c.T == 256 && c.GT == 256 && c.RPT == 8 && c.CPG == 2) return matvec_kernel<256, 256, 8, 2, MODE, false, false>;
  if (c.T == 512 && c.GT == 512 && c.RPT == 4 && c.CPG == 4) return matvec_kernel<512, 512, 4, 4, MODE, false, false>;
  if (c.T == 512 && c.GT == 512 && c.RPT == 4 && c.CPG == 2) return matvec_kernel<512, 512, 4, 2, MODE, false, false>;
  if (c.T == 512 && c.GT == 512 && c.RPT == 8 && c.CPG == 2) return matvec_kernel<512, 512, 8, 2, MODE, false, false>;
  return matvec_kernel<512, 512, 16, 1, MODE, true, false>;
}

static MvKernel kernel_for_mode(int mode, const MvCfg& c, bool clu) {
  switch (mode) {
    case MV_FUSED: return kernel_for<MV_FUSED>(c, clu);
    case MV_TONLY: return kernel_for<MV_TONLY>(c, clu);
    case MV_NONLY: return kernel_for<MV_NONLY>(c, clu);
    case MV_BOTH: return kernel_for<MV_BOTH>(c, clu);
    default: return kernel_for<MV_DIAG>(c, clu);
  }
}

struct MvPlan {
  MvCfg cfg;
  int cl = 1;
  int64_t rs = 0;
  int stages = 2;
  size_t smem = 0;
  int64_t npanels = 0;
  int grid = 0;       // CTAs
  int nparts = 0;     // clusters (= partial rows)
  int rc = 1;         // reduction cluster (cl == 1)
  int cdim = 1;       // launch cluster dimension (cl or rc)
};

static bool cfg_vs(const MvCfg& c, bool clu) { return !clu && c.RPT >= 16; }

static size_t mv_smem_bytes(const MvCfg& c, int64_t rs, int stages, int cl, bool clu) {
  const int NG = c.T / c.GT, WPG = c.GT / 32, BN = NG * c.CPG;
  constexpr int DB = 4;
  const int64_t ss = clu ? (int64_t)c.GT * c.RPT : rs;   // stage column stride (kernel: `ss`)
  size_t b = (size_t)stages * BN * ss * 8;
  b += (size_t)2 * stages * 8 + (size_t)DB * 8;
  b += (size_t)2 * NG * WPG * c.CPG * 8;
  b += (size_t)DB * cl * c.CPG * 8;
  if (cfg_vs(c, clu)) b += (size_t)rs * 8;
  return b;
}

// process-wide caches, shared by every context: contexts may be driven from several host threads
// at once (the loopback ranks of one process), so every access holds the lock
static std::map<std::tuple<int, int, int64_t, int64_t, int64_t>, MvPlan> g_plans;
static std::mutex g_plans_mu;

static int make_plan(nys_ctx* ctx, int mode, int64_t m, int64_t n, int64_t lda, MvPlan& pl) {
  auto key = std::make_tuple(ctx->device, mode, m, n, lda);
  {
    std::lock_guard<std::mutex> lk(g_plans_mu);
    auto itp = g_plans.find(key);
    if (itp != g_plans.end()) { pl = itp->second; return NYS_OK; }
  }
  // Geometry for a cluster split cl: rows per CTA rs, thread config, stages, smem, kernel.
  struct Geo {
    int64_t rs;
    MvCfg c;
    int stages;
    size_t smem;
    MvKernel k;
  };
  auto derive = [&](int cl_, Geo& G) -> int {
    int64_t rs_ = (m + cl_ - 1) / cl_;
    rs_ = (rs_ + 1) & ~int64_t(1);
    // whole-column CTAs with a near-tight lda: stride the stage by lda so a panel (BN consecutive
    // columns) is ONE contiguous bulk copy (the padding rows are masked off in the kernel)
    if (cl_ == 1 && lda >= rs_ && lda <= rs_ + 32) rs_ = lda;
    const bool clu_ = cl_ > 1;
    MvCfg c_ = pick_cfg(rs_, clu_);
    if (const char* ov = getenv("NYS_MV_CFG")) {  // debug/tuning override "T,GT,RPT,CPG" (must be instantiated)
      MvCfg o;
      if (sscanf(ov, "%d,%d,%d,%d", &o.T, &o.GT, &o.RPT, &o.CPG) == 4 && (int64_t)o.GT * o.RPT >= rs_) c_ = o;
    }
    const int BN_ = (c_.T / c_.GT) * c_.CPG;
    const size_t stage_bytes = (size_t)BN_ * (clu_ ? (int64_t)c_.GT * c_.RPT : rs_) * 8;
    size_t budget = clu_ ? 212 * 1024 : (rs_ <= 1024) ? 96 * 1024 : 200 * 1024;
    if (const char* sb = getenv("NYS_MV_SMEM_KB")) budget = (size_t)atoi(sb) * 1024;
    if (cfg_vs(c_, clu_)) budget -= (size_t)rs_ * 8;
    int st = (int)(budget / stage_bytes);
    st = st > 8 ? 8 : st;
    if (st < 2) st = 2;
    G.rs = rs_; G.c = c_; G.stages = st;
    G.smem = mv_smem_bytes(c_, rs_, st, cl_, clu_);
    G.k = kernel_for_mode(mode, c_, clu_);
    NYS_TRY(ensure_max_smem(ctx, (const void*)G.k, G.smem));
    if (cl_ > 8) NYS_CUDA_TRY(ctx, cudaFuncSetAttribute(G.k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    return NYS_OK;
  };
  auto resident_ctas = [&](int cl_, const Geo& G) -> int {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(cl_ * ctx->num_sms));
    cfg.blockDim = dim3((unsigned)(G.c.T + 32));
    cfg.dynamicSmemBytes = G.smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl_;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl_ = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl_, G.k, &cfg) != cudaSuccess) { cudaGetLastError(); ncl_ = 0; }
    return ncl_ * cl_;
  };
  // m <= 8192: whole columns per CTA.  Larger m: split the rows over a cluster of cl CTAs with
  // <= 8640 rows each (18 rows per thread: the register budget of the pipelined cluster path).
  // Cluster sizes need not be powers of two; GPCs do not hold equal numbers of clusters of every
  // size, so pick the SMALLEST cl (largest row slice: per-panel overheads amortised over more
  // bytes) whose resident CTA count is within 5% of the best over all admissible cl
  // (measured on B200, m = 50000: cl = 6 -> 132 CTAs, 6.68 TB/s; cl = 8 -> 120 CTAs, 5.59 TB/s).
  int cl = 1;
  Geo geo;
  if (m > 8192) {
    int clmin = (int)((m + 8639) / 8640);
    if (clmin < 2) clmin = 2;
    if (clmin > 16) { ctx->set_error("matvec: m too large for the cluster split (m <= 16 * 8640)"); return NYS_EINVAL; }
    int forced = 0;
    if (const char* oc = getenv("NYS_MV_CL")) {  // tuning override of the cluster split
      const int o = atoi(oc);
      if (o >= clmin && o <= 16) forced = o;
    }
    int res[17] = {0};
    int best = 0;
    for (int k = clmin; k <= 16; ++k) {
      if (forced && k != forced) continue;
      Geo G;
      NYS_TRY(derive(k, G));
      res[k] = resident_ctas(k, G);
      if (res[k] > best) best = res[k];
    }
    if (best == 0) { ctx->set_error("matvec: no cluster configuration fits on the device"); return NYS_ECUDA; }
    for (int k = clmin; k <= 16; ++k)
      if (res[k] > 0 && res[k] * 20 >= best * 19) { cl = k; break; }
  }
  NYS_TRY(derive(cl, geo));
  const bool clu = cl > 1;
  const int64_t rs = geo.rs;
  const MvCfg c = geo.c;
  const int stages = geo.stages;
  const size_t smem = geo.smem;
  MvKernel k = geo.k;
  const int NG = c.T / c.GT, BN = NG * c.CPG;
  (void)clu;
  const int64_t npanels = (n + BN - 1) / BN;
  int grid = 0;
  int rc = 1;
  auto max_clusters = [&](int csize, int& out) -> int {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(csize * ctx->num_sms));
    cfg.blockDim = dim3((unsigned)(c.T + 32));
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    out = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&out, k, &cfg);
    if (e != cudaSuccess) { cudaGetLastError(); out = 0; }
    return NYS_OK;
  };
  if (cl == 1) {
    int occ = 0;
    NYS_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, c.T + 32, smem));
    if (occ < 1) occ = 1;
    int64_t g = (int64_t)ctx->num_sms * occ;
    grid = (int)(npanels < g ? npanels : g);
    // reduction clusters: pick the cluster size (8 or 4) that keeps >= 95% of the CTAs resident
    // measured on B200 (config 1): DSMEM reduction clusters cost more than the partial rows they
    // save (rc=2: +8%, rc=4/8: fewer resident CTAs), so they are opt-in (NYS_MV_RC) only
    if (mode != MV_TONLY && grid >= 16 && getenv("NYS_MV_RC")) {
      const char* frc = getenv("NYS_MV_RC");
      const double keep = frc ? 0.0 : 0.95;
      for (int cs : {8, 4, 2}) {
        if (frc && atoi(frc) != cs) continue;
        int ncs = 0;
        max_clusters(cs, ncs);
        int64_t gc = (int64_t)ncs * cs;
        int64_t need = (npanels + cs - 1) / cs * cs;
        if (gc > need) gc = need;
        if (getenv("NYS_DEBUG")) fprintf(stderr, "[nys] reduction cluster %d: max active clusters %d -> %lld CTAs (grid %d)\n", cs, ncs, (long long)gc, grid);
        if (gc >= (int64_t)(keep * grid) && gc >= cs) { rc = cs; grid = (int)gc; break; }
      }
    }
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(cl * ctx->num_sms));
    cfg.blockDim = dim3((unsigned)(c.T + 32));
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    NYS_CUDA_TRY(ctx, cudaOccupancyMaxActiveClusters(&ncl, k, &cfg));
    if (ncl < 1) { ctx->set_error("matvec: cluster configuration does not fit on the device"); return NYS_ECUDA; }
    int64_t g = ncl;
    g = npanels < g ? npanels : g;
    grid = (int)(g * cl);
  }
  if (grid < cl) grid = cl;
  pl.cfg = c; pl.cl = cl; pl.rs = rs; pl.stages = stages; pl.smem = smem; pl.npanels = npanels;
  pl.grid = grid; pl.rc = rc; pl.cdim = cl > 1 ? cl : rc; pl.nparts = grid / pl.cdim;
  {
    std::lock_guard<std::mutex> lk(g_plans_mu);
    g_plans[key] = pl;
  }
  if (getenv("NYS_DEBUG"))
    fprintf(stderr, "[nys] matvec plan mode=%d m=%lld n=%lld: T=%d GT=%d RPT=%d CPG=%d cl=%d rc=%d rs=%lld stages=%d smem=%zu grid=%d nparts=%d npanels=%lld\n",
            mode, (long long)m, (long long)n, c.T, c.GT, c.RPT, c.CPG, cl, rc, (long long)rs, stages, smem, grid, pl.nparts,
            (long long)npanels);
  return NYS_OK;
}

// a rank with no columns still forms the PCG direction p = z + beta p (replicated m-space state)
__global__ void empty_shard_prologue_kernel(int64_t m, const double* z, const double* p, const double* beta,
                                            double* p_out, const double* done) {
  if (done != nullptr && *done != 0.0) return;
  const double b = (beta != nullptr) ? *beta : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    p_out[i] = (p != nullptr) ? z[i] + b * p[i] : z[i];
}

int ensure_max_smem(nys_ctx* ctx, const void* fn, size_t bytes) {
  static std::map<std::pair<int, const void*>, size_t> set;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(ctx->device, fn);
  auto it = set.find(key);
  if (it != set.end() && it->second >= bytes) return NYS_OK;
  NYS_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  set[key] = bytes;
  return NYS_OK;
}

int launch_matvec(nys_ctx* ctx, const MatvecCall& c) {
  if (c.m <= 0) return NYS_OK;
  MvPlan pl;
  NYS_TRY(make_plan(ctx, c.mode, c.m, c.n, c.lda, pl));
  const int64_t wp_ld = (c.m + 1) & ~int64_t(1);
  double* Wp = nullptr;
  if (c.mode != MV_TONLY) Wp = ctx->wsd("mv_partials", (size_t)pl.nparts * wp_ld);
  double* pwp = nullptr;
  if (c.mode == MV_FUSED && c.pcg_fused) pwp = ctx->wsd("mv_pwp", (size_t)pl.grid);
  double* tbuf = (c.mode == MV_TONLY || c.mode == MV_BOTH) ? ctx->wsd("mv_tbuf", (size_t)(c.n > 0 ? c.n : 1)) : nullptr;
  // finalize parameters (used in-kernel when fusable, else by mv_finalize)
  FinParams F{};
  int fgrid = (int)((c.m + 15) / 16);
  if (fgrid > 2 * ctx->num_sms) fgrid = 2 * ctx->num_sms;
  const bool want_fin = c.mode != MV_TONLY && !c.pcg_fused && c.out != nullptr;
  const bool fuse = want_fin && c.n > 0 && pl.cl == 1 && pl.rc == 1 && getenv("NYS_FUSED_FIN") != nullptr;
  // (measured on B200, m = 2000: the in-kernel grid barrier costs what the separate finalize
  //  launch does inside a CUDA graph, so the fused variant is opt-in)
  if (want_fin) {
    F.Wp = Wp; F.wp_ld = wp_ld; F.nparts = pl.nparts; F.m = c.m; F.sgn = c.sgn;
    F.delta = c.delta; F.use_delta = c.use_delta ? 1 : 0; F.e = c.e;
    F.v = (c.p_out != nullptr) ? c.p_out : c.z;
    F.add = c.add; F.out = c.out; F.pcg_alpha = c.pcg_alpha ? 1 : 0; F.sc = ctx->sc;
    F.counter = ctx->counters + 0;
    F.done = c.done;
    F.part = ctx->wsd("fin_part", (size_t)(fuse ? pl.grid : fgrid));
  }
  unsigned int* gbar = nullptr;
  if (fuse) {
    const bool fresh = ctx->bufs.find("mv_gbar") == ctx->bufs.end();
    gbar = (unsigned int*)ctx->ws("mv_gbar", 64);
    if (fresh) NYS_CUDA_TRY(ctx, cudaMemsetAsync(gbar, 0, 64, ctx->stream));
  }
  if (c.n > 0 || c.mode == MV_TONLY) {
    MatvecParams P{};
    P.A = c.A; P.lda = c.lda; P.m = c.m; P.n = c.n;
    P.z = c.z; P.p = c.p; P.beta = c.beta; P.p_out = c.p_out; P.d = c.d; P.u = c.u;
    P.Wp = Wp; P.wp_ld = wp_ld;
    P.tep = c.tep; P.t1 = c.t1; P.t2 = c.t2; P.ta = c.ta; P.tb = c.tb; P.tc = c.tc; P.td = c.td; P.tx = c.tx; P.tdd = c.tdd;
    P.done = c.done; P.rs = pl.rs; P.npanels = pl.npanels; P.stages = pl.stages; P.cl = pl.cl;
    static const int l2pf = getenv("NYS_MV_PF") ? atoi(getenv("NYS_MV_PF")) : 0;
    P.l2pf = l2pf;
    P.pwp = pwp; P.delta = c.delta; P.e = c.e; P.tbuf = tbuf; P.rc = pl.rc;
    P.delta_slot = c.delta_from_slot ? ctx->sc + S_DELTA : nullptr;
    P.fuse_fin = fuse ? 1 : 0;
    P.fin = F;
    P.gbar = gbar;
    MvKernel k = kernel_for_mode(c.mode, pl.cfg, pl.cl > 1);
    if (c.n > 0) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)pl.grid);
      cfg.blockDim = dim3((unsigned)(pl.cfg.T + 32));
      cfg.dynamicSmemBytes = pl.smem;
      cfg.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      if (fuse) {  // grid barrier inside: all CTAs must be co-resident
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
      } else {
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = pl.cdim;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
      }
      cfg.attrs = at;
      cfg.numAttrs = 1;
      NYS_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, k, P));
      ctx->launches++;
      if (c.mode == MV_FUSED) ctx->matvecs++;
    }
  }
  if (c.mode == MV_TONLY) return NYS_OK;
  if (c.n <= 0) {  // empty shard: zero partials, and the operand prologue the kernel would have done
    NYS_CUDA_TRY(ctx, cudaMemsetAsync(Wp, 0, sizeof(double) * (size_t)pl.nparts * wp_ld, ctx->stream));
    if (pwp) NYS_CUDA_TRY(ctx, cudaMemsetAsync(pwp, 0, sizeof(double) * (size_t)pl.grid, ctx->stream));
    if (c.mode == MV_FUSED && c.p_out != nullptr) {   // v = z + beta p is still this rank's p (PCG)
      empty_shard_prologue_kernel<<<(unsigned)((c.m + 255) / 256), 256, 0, ctx->stream>>>(c.m, c.z, c.p, c.beta,
                                                                                          c.p_out, c.done);
      ctx->launches++;
      NYS_TRY(ctx->check_launch("empty_shard_prologue"));
    }
  }
  if (c.pcg_fused) {  // the PCG update kernel consumes the partials directly (no finalize)
    if (c.fused_out) {
      c.fused_out->Wp = Wp; c.fused_out->wp_ld = wp_ld; c.fused_out->nparts = pl.nparts;
      c.fused_out->pwp = pwp; c.fused_out->npw = pl.grid;
    }
    return NYS_OK;
  }
  if (!want_fin || fuse) return NYS_OK;
  mv_finalize<<<fgrid, 256, 0, ctx->stream>>>(F);
  ctx->launches++;
  return ctx->check_launch("mv_finalize");
}

}  // namespace nys
