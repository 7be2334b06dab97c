// Persistent PCG on (A D A^T + diag(e) + delta I) x = rhs with the Nystrom P^{-1}
// — ONE cooperative launch for the whole solve (single GPU, m <= 8192 so that a CTA
// holds the full column height).
//
// Every CTA owns a contiguous, balanced range of columns of A (streamed in panels, as in the fused
// matvec, k_matvec.cu) and a fixed chunk of rows of the m-space vectors.  Per iteration k:
//   P1  load p_k (all rows); w_partial = A_cols (d o (A_cols^T p_k)), p^T N p partial
//                                                                          -> grid barrier
//   P2  alpha = rz / p^T N p; own rows: w = sum of the partials + (delta + e) p; x += alpha p;
//       r -= alpha w; ||r||^2 and U^T r partial rows                       -> grid barrier
//   P3  every CTA sums all partial rows itself in one fixed order (identical decisions):
//       converged? h = s o (U^T r); r^T z = ||r||^2 + (U^T r)^T h (no extra reduction);
//       beta; own rows: z = r + U h, p_{k+1} = z + beta p_k              -> grid barrier
// The producer warp streams A panels through the S-stage cp.async.bulk ring CONTINUOUSLY across
// iterations (A does not depend on the iterate) and prefetches further panels into L2, so HBM keeps
// streaming through the barrier phases.  Grid barriers involve the consumer threads only; the
// producer polls a stop flag so it can never block the exit.
#include <cooperative_groups.h>

#include <chrono>
#include <cstdlib>
#include <vector>

#include "k_vec.cuh"

namespace cg = cooperative_groups;

namespace nys {

struct PcgPParams {
  const double* A;
  int64_t lda, m, n;
  const double* d;
  const double* e;
  const double* U;
  int64_t ldu;
  int ell;
  const double* s;       // ell coefficients (lam_l + mu)/(lam_i + mu) - 1
  const double* rhs;
  double* x;
  double* r;
  double* z;             // == r when ell == 0
  double* P0;            // p double buffer
  double* P1;
  double* Wp;            // [G][wp_ld] partial w
  int64_t wp_ld;
  double* pwp;           // [G]
  double* part1;         // [G][(1 + ell)]   (rr, U^T r) partial row per CTA
  double* gtot;          // [ceil(G/RG)][1 + ell] group totals of part1
  double* tot;           // [1 + ell] grand totals
  unsigned int* rbar;    // [66]: group arrival counters [0, 64), top counter [64], publish flag [65]
  double* sc;
  unsigned int* bar;     // [2]: count, generation
  int max_iter;
  int stages;
  int l2_prefetch;            // panels prefetched into L2 ahead of the smem ring
  int l2_keep;                // panels per CTA copied with evict_last (L2-resident across iterations)
  unsigned long long* trace;  // debug (NYS_PCG_TRACE): [2 CTAs][32 iters][8] globaltimer stamps
  unsigned long long* trace_arr;
  int flat_red;               // 1: grid barrier + every CTA reduces all partial rows; 0: two-level last-arriver tree  // debug: [3][G] arrival stamps of every CTA at the 3 syncs of iteration 14
  int64_t npanels;
  int64_t rows_per_cta;
  int64_t ss;                 // stage row stride (lda when near-tight, else even(m))
  int acq_spin;               // grid barrier: acquire-load spin (1) or relaxed spin + acq_rel fence (0)
};

// Grid barrier on a monotonically increasing arrival counter (zeroed before the launch): each CTA
// adds 1 (fire-and-forget reduction) and polls until the counter reaches epoch * G.  No "last
// arriver" reset round trip, no sleep granularity on the release.
__device__ __forceinline__ void pcg_grid_barrier(unsigned int* bar, unsigned int nblocks, int nthreads,
                                                 unsigned int& epoch, bool bar_acquire_spin) {
  named_bar_sync(9, nthreads);
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
  named_bar_sync(9, nthreads);
}

constexpr int RG = 16;  // CTAs per first-level reduction group (G <= 64 * RG)


template <int T, int GT, int RPT, int CPG>
__global__ void __launch_bounds__(T + 32, 1) pcg_persistent_kernel(const PcgPParams P) {
  constexpr int NG = T / GT;
  constexpr int WPG = GT / 32;
  constexpr int BN = NG * CPG;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int S = P.stages;
  // stage row stride: lda when it is near-tight (a panel of BN consecutive columns is then ONE bulk
  // copy; the padding rows are read but masked off), else the even column height with one copy per column
  const int64_t rs = P.ss;
  const bool contig = (P.ss == P.lda);
  double* stage = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(stage + (size_t)S * BN * rs);
  uint64_t* empty = full + S;
  double* red = reinterpret_cast<double*>(empty + S);  // 2 * NG * WPG * CPG
  __shared__ double hsh[256];
  __shared__ double gsh[256];
  __shared__ double colred[512];
  __shared__ int s_role;
  __shared__ double chunk_red[16][17];
  __shared__ double s_scal[8];
  __shared__ volatile int s_stop;
  __shared__ volatile long long s_issued;

  const int tid = threadIdx.x, warp = warp_uniform_id(), lane = tid & 31;
  const unsigned int G = gridDim.x;
  const unsigned int cid = blockIdx.x;
  // this CTA's contiguous column range [c_lo, c_hi) (balanced to one column), streamed in panels of
  // BN columns with a ragged last panel
  const int64_t c_lo = (P.n * (int64_t)cid) / G, c_hi = (P.n * ((int64_t)cid + 1)) / G;
  const int64_t niter = (c_hi - c_lo + BN - 1) / BN;
  const uint32_t copy_bytes = (uint32_t)(((P.m + 1) & ~int64_t(1)) * 8);
  const int64_t r_lo = (int64_t)cid * P.rows_per_cta;
  int64_t r_hi = r_lo + P.rows_per_cta;
  if (r_hi > P.m) r_hi = P.m;
  const int ell = P.ell;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], T / 32);
    }
    fence_mbar_init();
    s_stop = 0;
    s_issued = 0;
  }
  __syncthreads();

  if (warp == T / 32) {
    // ---------------- producer warp: stream this CTA's panels, iteration after iteration ------
    long long q = 0;
    if (lane == 0 && niter > 0) {
      const uint64_t pol_stream = l2_evict_first_policy();
      // the first `l2_keep` panels of this CTA's set are re-read every iteration from L2: they are
      // copied with evict_last so that they stay resident across iterations (A is about L2-sized
      // at the small configs); the rest streams with evict_first
      const uint64_t pol_keep = l2_evict_last_policy();
      // L2 prefetch runs PF panels ahead of the smem ring: the reduction / barrier phases of an
      // iteration leave HBM idle, so the next matvec's panels are pulled into L2 meanwhile
      long long pf = 0;
      int64_t pfi = 0;        // pf mod niter, kept incrementally (no 64-bit division per panel)
      const int PF = P.l2_prefetch;
      int s = -1;
      uint32_t par = 1u;      // parity of the empty-barrier phase to wait for (first pass: none)
      int64_t it = 0;         // q mod niter
      for (;; ++q) {
        if (++s == S) { s = 0; par ^= 1u; }
        for (; pf < q + S + PF; ++pf) {
          const int64_t c0 = c_lo + pfi * BN;
          if (++pfi == niter) pfi = 0;
          int64_t nc = c_hi - c0;
          nc = nc > BN ? BN : nc;
          if (pf >= q + S) bulk_prefetch_l2(P.A + c0 * P.lda, (uint32_t)(((nc - 1) * P.lda) * 8) + copy_bytes);
        }
        if (q >= S) {
          bool stop = false;
          for (;;) {
            uint32_t ok;
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(ok)
                : "r"(smem_u32(&empty[s])), "r"(par)
                : "memory");
            if (ok) break;
            if (s_stop) { stop = true; break; }
          }
          if (stop) break;
        }
        if (s_stop) break;
        const int64_t col0 = c_lo + it * BN;
        int64_t ncols = c_hi - col0;
        ncols = ncols > BN ? BN : ncols;
        if (contig) {
          const uint32_t bytes = (uint32_t)((ncols - 1) * rs * 8) + copy_bytes;
          mbar_arrive_expect_tx(&full[s], bytes);
          bulk_g2s(stage + (size_t)s * BN * rs, P.A + col0 * P.lda, bytes, &full[s],
                   it < P.l2_keep ? pol_keep : pol_stream);
        } else {
          mbar_arrive_expect_tx(&full[s], (uint32_t)ncols * copy_bytes);
          for (int c = 0; c < ncols; ++c)
            bulk_g2s(stage + ((size_t)s * BN + c) * rs, P.A + (col0 + c) * P.lda, copy_bytes, &full[s],
                     it < P.l2_keep ? pol_keep : pol_stream);
        }
        if (++it == niter) it = 0;
      }
      s_issued = q;
    }
    __syncwarp();
    named_bar_sync(10, T + 32);  // exit handshake with the consumers
    return;
  }

  // ======================= consumers =========================================================
  const int g = tid / GT;
  const int lig = tid % GT;
  const int row16 = tid & 15, grp16 = (tid >> 4) & 15;  // first 256 threads: 16 rows x 16 groups
  const int hrow = lane & 15, hw = 2 * warp + (lane >> 4);
  long long qc = 0;  // consumed stage counter
  int cs = 0;        // its stage index and full-barrier parity (kept incrementally)
  uint32_t cph = 0u;
  unsigned int bar_epoch = 0;  // grid barriers passed (thread 0)
  unsigned int red_epoch = 0;  // column reductions done (thread 0)
  int trace_k = 0;
  auto arrive_stamp = [&](int which) {
    if (P.trace_arr != nullptr && tid == 0 && trace_k == 14) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      P.trace_arr[(size_t)which * G + cid] = t;
    }
  };
  auto stamp = [&](int slot) {
    if (P.trace != nullptr && tid == 0 && (cid == 0 || cid == G - 1) && trace_k < 32) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      P.trace[((cid == 0 ? 0 : 1) * 32 + trace_k) * 16 + slot] = t;
    }
  };
  double rz = 0.0, beta = 0.0;
  int iters = 0;
  int status = 0;
  bool conv = false;

  // ---- init: x = 0, r = rhs, rr, U^T r  ------------------------------------------------------
  auto rows_phase_rr_ut = [&](bool init, double alpha, const double* pnew, const double* Wp, double delta) -> bool {
    // own rows in chunks of 16: (init) x = 0, r = rhs | x += alpha p, r -= alpha w ; partials.
    // (!init) alpha = rz / p^T N p is formed here by warp 0 from the pwp partials while the first
    // chunk's row operands and partial-row sums are in flight; false on a p^T N p breakdown (no update)
    double rr = 0.0;
    bool first = true;
    double gacc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) gacc[k] = 0.0;
    for (int64_t i0 = r_lo; i0 < r_hi; i0 += 16) {
      const int64_t i = i0 + row16;
      // everything that does not depend on the partial sums is loaded up front (one round trip
      // overlapped with the partial-row reduction instead of two more after it)
      double pre_p = 0.0, pre_e = 0.0, pre_x = 0.0, pre_r = 0.0;
      if (tid < 16 && i < r_hi) {
        if (init) {
          pre_r = P.rhs[i];
        } else {
          pre_p = __ldcg(pnew + i);
          pre_e = P.e ? P.e[i] : 0.0;
          pre_x = P.x[i];
          pre_r = P.r[i];
        }
      }
      // (the 512-thread configurations keep the U loads after the barrier: register budget)
      constexpr bool PRE_U = (T == 256);
      double uval[PRE_U ? 16 : 1];
#pragma unroll
      for (int k = 0; k < (PRE_U ? 16 : 1); ++k) {
        const int c = hw + 16 * k;
        uval[k] = (PRE_U && warp < 8 && c < ell && i0 + hrow < r_hi) ? P.U[(size_t)c * P.ldu + i0 + hrow] : 0.0;
      }
      if (!init && warp < 8) {
        double acc = 0.0;
        if (i < r_hi) {
          for (int c0 = grp16; c0 < (int)G; c0 += 160) {  // 10 independent L2 loads: one round at G <= 160
            double v[10];
#pragma unroll
            for (int u = 0; u < 10; ++u) {
              const int c = c0 + 16 * u;
              v[u] = (c < (int)G) ? __ldcg(Wp + (size_t)c * P.wp_ld + i) : 0.0;
            }
            acc += (((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]))) + (v[8] + v[9]);
          }
        }
        chunk_red[row16][grp16] = acc;
      }
      if (!init && first && warp == 0) {
        const double pw = warp_sum_array(P.pwp, G);
        if (lane == 0) s_scal[2] = pw;
      }
      named_bar_sync(9, T);
      if (!init && first) {
        first = false;
        const double pw = s_scal[2];
        if (!(pw > 0.0) || !isfinite(pw)) return false;
        alpha = rz / pw;
      }
      if (tid < 16) {
        double ri = 0.0;
        if (i < r_hi) {
          if (init) {
            ri = pre_r;
            P.x[i] = 0.0;
          } else {
            const double* v = chunk_red[row16];
            const double wsum = (((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]))) +
                                (((v[8] + v[9]) + (v[10] + v[11])) + ((v[12] + v[13]) + (v[14] + v[15])));
            const double wi = wsum + (delta + pre_e) * pre_p;
            P.x[i] = fma(alpha, pre_p, pre_x);
            ri = fma(-alpha, wi, pre_r);
          }
          P.r[i] = ri;
        }
        hsh[row16] = ri;
        rr = fma(ri, ri, rr);
      }
      named_bar_sync(9, T);
      if (warp < 8) {
        const double hr = hsh[hrow];
        if constexpr (PRE_U) {
#pragma unroll
          for (int k = 0; k < 16; ++k) gacc[k] = fma(uval[k], hr, gacc[k]);
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int c = hw + 16 * k;
            if (c < ell && i0 + hrow < r_hi) gacc[k] = fma(P.U[(size_t)c * P.ldu + i0 + hrow], hr, gacc[k]);
          }
        }
      }
      named_bar_sync(9, T);
    }
    if (!init && first) {   // a CTA without rows takes the same breakdown decision
      if (warp == 0) {
        const double pw = warp_sum_array(P.pwp, G);
        if (lane == 0) s_scal[2] = pw;
      }
      named_bar_sync(9, T);
      const double pw = s_scal[2];
      if (!(pw > 0.0) || !isfinite(pw)) return false;
    }
    // write partials: rr (threads < 16 hold pieces) and U^T r (half-warps)
    double rrw = warp_sum(rr);
    if (tid == 0) P.part1[(size_t)cid * (1 + ell)] = rrw;
    if (warp < 8) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (16 * k < ell) {
          double gsum = gacc[k];
          gsum += __shfl_xor_sync(0xffffffffu, gsum, 8);
          gsum += __shfl_xor_sync(0xffffffffu, gsum, 4);
          gsum += __shfl_xor_sync(0xffffffffu, gsum, 2);
          gsum += __shfl_xor_sync(0xffffffffu, gsum, 1);
          const int c = hw + 16 * k;
          if (hrow == 0 && c < ell) P.part1[(size_t)cid * (1 + ell) + 1 + c] = gsum;
        }
      }
    }
    return true;
  };

  // P3: converged? then h = s o (U^T r), r^T z = r^T r + (U^T r)^T h (no extra reduction), beta, and
  // own rows: z = r + U h, p_next = z + beta p_cur
  auto phase_prec = [&](bool init, const double* pcur, double* pnext) -> bool {
    // all 1 + ell sums of the CTA partial rows part1[cid][.] (||r||^2, U^T r): a grid barrier, then
    // EVERY CTA reduces the G partial rows itself in one fixed order (identical totals and decisions
    // in every CTA).  Thread (s, c) sums column c over the slice g = s, s + NS, ... with LB loads in
    // flight (one L2 round trip at G = 148), then the NS slice sums are added in order.  Measured:
    // the previous two-level "last arriver reduces" chain released CTAs 6.7 us after the last
    // arrival, this 1.5 us barrier + the flat read about half of that.
    // the first own-row chunk's z-row operands (U rows, r, p_k: none depends on the reduction) are
    // loaded BEFORE the grid barrier, so their L2 latency hides behind it
    // (T = 256 only: the 512-thread variants have no registers to spare)
    constexpr bool PRE_Z = (T == 256);
    constexpr int UZ = 4;   // columns per group preloaded (ell <= 64 entirely; the rest loads after)
    double uz[UZ];
    double zr0 = 0.0, zp0 = 0.0;
    if constexpr (PRE_Z) {
      const int64_t i = r_lo + row16;
#pragma unroll
      for (int k = 0; k < UZ; ++k) {
        const int c = grp16 + 16 * k;
        uz[k] = (warp < 8 && c < ell && i < r_hi) ? __ldg(P.U + (size_t)c * P.ldu + i) : 0.0;
      }
      if (tid < 16 && i < r_hi) {
        zr0 = P.r[i];
        zp0 = init ? 0.0 : __ldcg(pcur + i);
      }
    }
    {
      const int ncol = 1 + ell;
      if (P.flat_red) {
      named_bar_sync(9, T);  // this CTA's partial row is written
      if (!init) arrive_stamp(1);
      pcg_grid_barrier(P.bar, G, T, bar_epoch, P.acq_spin != 0);
      constexpr int LB = 38;
      const int CP = (ncol <= 32) ? 32 : (ncol <= 64) ? 64 : (ncol <= 128 || T <= 128) ? 128 : (T <= 256 ? 256 : 512);
      const int NS = T / CP;
      const int sl = tid / CP, cix = tid % CP;
#pragma unroll 1
      for (int c = cix; c < ncol; c += CP) {
        double tot = 0.0;
#pragma unroll 1
        for (int g0 = sl; g0 < (int)G; g0 += NS * LB) {
          double v[LB];
#pragma unroll
          for (int u = 0; u < LB; ++u) {
            const int gg = g0 + NS * u;
            v[u] = (gg < (int)G) ? __ldcg(P.part1 + (size_t)gg * ncol + c) : 0.0;
          }
          static_assert(LB <= 64, "pairwise tree below covers 64 terms");
#pragma unroll
          for (int w = 32; w > 0; w >>= 1)
#pragma unroll
            for (int u = 0; u < w; ++u)
              if (u + w < LB) v[u] += v[u + w];
          tot += v[0];
        }
        colred[sl * ncol + c] = tot;
      }
      } else {
      const unsigned int ngr = (G + RG - 1) / RG;
      const unsigned int grp = cid / RG;
      const unsigned int gsz = (grp + 1 == ngr) ? G - grp * RG : RG;
      named_bar_sync(9, T);  // this CTA's partial row is written
      if (!init) arrive_stamp(1);
      if (tid == 0) {
        ++red_epoch;
        const unsigned int old = atom_add_acqrel_gpu(P.rbar + grp, 1u);
        s_role = (old + 1 == red_epoch * gsz) ? 1 : 0;
      }
      named_bar_sync(9, T);
      if (s_role) {  // last CTA of its group: group totals
        for (int c = tid; c < ncol; c += T) {
          double v[RG];
#pragma unroll
          for (int u = 0; u < RG; ++u)
            v[u] = (u < (int)gsz) ? __ldcg(P.part1 + (size_t)(grp * RG + u) * ncol + c) : 0.0;
#pragma unroll
          for (int w = RG / 2; w > 0; w >>= 1)
#pragma unroll
            for (int u = 0; u < w; ++u) v[u] += v[u + w];
          P.gtot[(size_t)grp * ncol + c] = v[0];
        }
        named_bar_sync(9, T);
        if (tid == 0) {
          const unsigned int old = atom_add_acqrel_gpu(P.rbar + 64, 1u);
          s_role = (old + 1 == red_epoch * ngr) ? 2 : 1;
        }
        named_bar_sync(9, T);
        if (s_role == 2) {  // last group: grand totals, then publish
          for (int c = tid; c < ncol; c += T) {
            double acc = 0.0;
            for (unsigned int g0 = 0; g0 < ngr; g0 += 8) {
              double v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) v[u] = (g0 + u < ngr) ? __ldcg(P.gtot + (size_t)(g0 + u) * ncol + c) : 0.0;
              acc += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
            }
            P.tot[c] = acc;
          }
          named_bar_sync(9, T);
          if (tid == 0) st_release_gpu(P.rbar + 65, red_epoch);
        }
      }
      if (tid == 0) {
        while (ld_relaxed_gpu(P.rbar + 65) < red_epoch) {
        }
        fence_acquire_gpu();
      }
      named_bar_sync(9, T);
      for (int c = tid; c < ncol; c += T) colred[c] = __ldcg(P.tot + c);
      }
      named_bar_sync(9, T);
      const int NSf = P.flat_red ? T / ((ncol <= 32) ? 32 : (ncol <= 64) ? 64 : (ncol <= 128 || T <= 128) ? 128 : (T <= 256 ? 256 : 512)) : 1;
      for (int c = tid; c < ncol; c += T) {
        double sum = 0.0;
        for (int q = 0; q < NSf; ++q) sum += colred[q * ncol + c];
        if (c == 0) s_scal[0] = sum;
        else {
          gsh[c - 1] = sum;
          hsh[c - 1] = P.s[c - 1] * sum;
        }
      }
      named_bar_sync(9, T);
      if (warp == 0 && ell > 0) {  // r^T z = r^T r + sum_c g_c h_c : the same fixed order in every CTA
        double acc = 0.0;
        for (int c = lane; c < ell; c += 32) acc = fma(gsh[c], hsh[c], acc);
        acc = warp_sum(acc);
        if (lane == 0) s_scal[1] = s_scal[0] + acc;
      }
      named_bar_sync(9, T);
    }
    if (!init) stamp(6);
    const double rrt = s_scal[0];
    const double tol = P.sc[S_TOL];
    bool cv = sqrt(rrt) <= tol;
    if (!isfinite(rrt)) { status = NYS_EBREAKDOWN; cv = true; }
    if (!init) ++iters;
    if (cv || iters >= P.max_iter) {
      if (cid == 0 && tid == 0) { P.sc[S_RR] = rrt; }
      conv = cv;
      return true;
    }
    if (ell > 0) {
      const double rzn = s_scal[1];
      if (!(rzn > 0.0) || !isfinite(rzn)) { status = NYS_EBREAKDOWN; return true; }
      beta = init ? 0.0 : rzn / rz;
      rz = rzn;
      for (int64_t i0 = r_lo; i0 < r_hi; i0 += 16) {
        const int64_t i = i0 + row16;
        const bool first = PRE_Z && i0 == r_lo;
        double pre_r = 0.0, pre_p = 0.0;
        if (tid < 16 && i < r_hi) {
          pre_r = first ? zr0 : P.r[i];
          pre_p = first ? zp0 : (init ? 0.0 : __ldcg(pcur + i));
        }
        if (warp < 8) {
          double acc = 0.0;
          if (i < r_hi) {
            if (first) {
#pragma unroll
              for (int k = 0; k < UZ; ++k)
                if (grp16 + 16 * k < ell) acc = fma(uz[k], hsh[grp16 + 16 * k], acc);
              for (int c = grp16 + 16 * UZ; c < ell; c += 16) acc = fma(P.U[(size_t)c * P.ldu + i], hsh[c], acc);
            } else {
              for (int c = grp16; c < ell; c += 16) acc = fma(P.U[(size_t)c * P.ldu + i], hsh[c], acc);
            }
          }
          chunk_red[row16][grp16] = acc;
        }
        named_bar_sync(9, T);
        if (tid < 16 && i < r_hi) {
          const double* v = chunk_red[row16];
          const double us = (((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]))) +
                            (((v[8] + v[9]) + (v[10] + v[11])) + ((v[12] + v[13]) + (v[14] + v[15])));
          const double zi = pre_r + us;
          P.z[i] = zi;
          pnext[i] = init ? zi : fma(beta, pre_p, zi);
        }
        named_bar_sync(9, T);
      }
      if (!init) stamp(7);
      if (!init) arrive_stamp(2);
      pcg_grid_barrier(P.bar, G, T, bar_epoch, P.acq_spin != 0);   // p_next complete on every row
    } else {
      beta = init ? 0.0 : rrt / rz;
      rz = rrt;
    }
    return false;
  };

  const double delta = P.sc[S_DELTA];
  // one call site per phase (k = -1 is the initialisation: x = 0, r = rhs, first reduction, p_0):
  // the phase lambdas inline, so their state stays in registers
  int k = -1;
  double alpha = 0.0;
  for (;;) {
    const bool init = k < 0;
    double* pold = (k & 1) ? P.P1 : P.P0;   // p_{k-1}; receives p_{k+1} at the end of iteration k
    double* pnew = (k & 1) ? P.P0 : P.P1;   // p_k
    if (!init) {
    trace_k = k;
    stamp(0);
    // ---- P1: v = z + beta p ; fused matvec over this CTA's panels ----------------------------
    double vreg[RPT];
    double wacc[RPT];
    // all loads first (z, p are written by other CTAs in this launch: read through L2), then the
    // stores: interleaving them would serialise the loads behind possibly-aliasing stores
    if (ell > 0) {  // p_k was formed row-wise at the end of the previous phase_prec
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int64_t rl = lig + (int64_t)GT * i;
        vreg[i] = (rl < P.m) ? __ldcg(pnew + rl) : 0.0;
        wacc[i] = 0.0;
      }
    } else {
      double zr[RPT], pr[RPT];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int64_t rl = lig + (int64_t)GT * i;
        zr[i] = (rl < P.m) ? __ldcg(P.z + rl) : 0.0;
        pr[i] = (rl < P.m && k > 0) ? __ldcg(pold + rl) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int64_t rl = lig + (int64_t)GT * i;
        const double v = (k > 0) ? fma(beta, pr[i], zr[i]) : zr[i];
        if (rl < P.m && cid == 0 && g == 0) pnew[rl] = v;
        vreg[i] = (rl < P.m) ? v : 0.0;
        wacc[i] = 0.0;
      }
    }
    double pwacc = 0.0;
    stamp(8);
    // d of the next panel is loaded one panel ahead (its L2 latency would otherwise sit on every
    // panel's critical path: short columns make that dominant)
    double dnext[CPG];
#pragma unroll
    for (int c = 0; c < CPG; ++c) {
      const int64_t col = c_lo + (int64_t)g * CPG + c;
      dnext[c] = (niter > 0 && col < c_hi) ? __ldg(P.d + col) : 0.0;
    }
    for (int64_t it = 0; it < niter; ++it, ++qc) {
      const int s = cs;
      const uint32_t par = cph;
      if (++cs == S) { cs = 0; cph ^= 1u; }
      const int64_t col0 = c_lo + it * BN + (int64_t)g * CPG;
      double dpre[CPG];
#pragma unroll
      for (int c = 0; c < CPG; ++c) {
        dpre[c] = dnext[c];
        const int64_t coln = col0 + BN + c;
        dnext[c] = (it + 1 < niter && coln < c_hi) ? __ldg(P.d + coln) : 0.0;
      }
      mbar_wait(&full[s], par);
      if (it == 0) stamp(9);
      if (it == niter / 2) stamp(10);
      if (it == niter - 1) stamp(11);
      double a[CPG][RPT];
      const double* sb = stage + ((size_t)s * BN + (size_t)g * CPG) * rs;
#pragma unroll
      for (int c = 0; c < CPG; ++c) {
        const bool cv = (col0 + c) < c_hi;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int64_t rl = lig + (int64_t)GT * i;
          a[c][i] = (cv && rl < P.m) ? sb[(size_t)c * rs + rl] : 0.0;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      double pd[CPG];
#pragma unroll
      for (int c = 0; c < CPG; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) acc = fma(a[c][i], vreg[i], acc);
        pd[c] = warp_sum(acc);
      }
      if (WPG > 1) {
        double* rb = red + ((size_t)(qc & 1) * NG + g) * WPG * CPG;
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
      double t[CPG];
#pragma unroll
      for (int c = 0; c < CPG; ++c) t[c] = dpre[c] * pd[c];
      if (lig == 0) {
#pragma unroll
        for (int c = 0; c < CPG; ++c) pwacc = fma(t[c], pd[c], pwacc);
      }
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        double acc = wacc[i];
#pragma unroll
        for (int c = 0; c < CPG; ++c) acc = fma(a[c][i], t[c], acc);
        wacc[i] = acc;
      }
    }
    // p^T (delta I + diag e) p : CTA 0, group 0
    if (cid == 0 && g == 0) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int64_t rl = lig + (int64_t)GT * i;
        if (rl < P.m) pwacc = fma((delta + (P.e ? P.e[rl] : 0.0)) * vreg[i], vreg[i], pwacc);
      }
    }
    // CTA partials: w (group-summed through global atomics-free path) and p^T N p
    {
      double* outp = P.Wp + (size_t)cid * P.wp_ld;
      if (NG == 1) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int64_t rl = lig + (int64_t)GT * i;
          if (rl < P.m) outp[rl] = wacc[i];
        }
      } else {
        // groups write in turn (fixed order) through the partial row itself
        for (int gg = 0; gg < NG; ++gg) {
          if (g == gg) {
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
              const int64_t rl = lig + (int64_t)GT * i;
              if (rl < P.m) outp[rl] = (gg == 0) ? wacc[i] : outp[rl] + wacc[i];
            }
          }
          named_bar_sync(9, T);
        }
      }
      const double wsum = warp_sum(pwacc);
      if (lane == 0) chunk_red[0][warp] = wsum;  // <= 16 consumer warps
      named_bar_sync(9, T);
      if (tid == 0) {
        double b = 0.0;
        for (int w = 0; w < T / 32; ++w) b += chunk_red[0][w];
        P.pwp[cid] = b;
      }
    }
    stamp(1);
    arrive_stamp(0);
    pcg_grid_barrier(P.bar, G, T, bar_epoch, P.acq_spin != 0);
    stamp(2);
    }  // !init
    // ---- P2: alpha, own-row updates, partials --------------------------------------------------
    if (!rows_phase_rr_ut(init, alpha, init ? nullptr : pnew, init ? nullptr : P.Wp, delta)) {
      status = NYS_EBREAKDOWN;
      break;
    }
    if (!init) {
      stamp(3);
      stamp(4);
    }
    // ---- P3 / P4 -------------------------------------------------------------------------------
    // k = -1: p_0 -> P1 (= pnew of k = 0); else p_{k+1} -> pold (= pnew of k + 1)
    const bool stop = phase_prec(init, init ? nullptr : pnew, init ? P.P1 : pold);
    if (!init) stamp(5);
    if (stop) break;
    ++k;
  }

  // ---- exit: stop the producer, drain in-flight bulk copies, publish the scalars --------------
  if (tid == 0) s_stop = 1;
  named_bar_sync(10, T + 32);
  const long long issued = s_issued;
  for (; qc < issued; ++qc) {
    mbar_wait(&full[cs], cph);
    if (++cs == S) { cs = 0; cph ^= 1u; }
  }
  if (cid == 0 && tid == 0) {
    P.sc[S_ITERS] = (double)iters;
    P.sc[S_STATUS] = (double)status;
    P.sc[S_DONE] = 1.0;
    P.sc[S_RZ] = rz;
  }
}

// ------------------------------------------------------------------------------------------
// Small problems (m <= 256, A <= ~1 MB, e.g. BASELINE config 0: m = 100, n = 400): the whole PCG solve
// in ONE CTA of 1024 threads.  The persistent grid kernel above pays three grid barriers per
// iteration (~13.6 us at config 0: pure synchronisation latency); here every synchronisation is a
// __syncthreads and A (L2-resident after the first iteration) is read by 32 warps, one column per
// warp per step: the dot a_j^T p (lanes over rows, a shuffle sum), t_j = d_j a_j^T p, and the rank-1
// update of the warp's row accumulators — the fused one-pass matvec of k_matvec.cu in miniature.
// Same recurrence as the oracle's textbook PCG: zero start, alpha = r^T z / p^T w with
// p^T w formed from w, the absolute stop ||r|| <= tol checked before the first iteration and after
// every update, breakdown on p^T w <= 0; r^T z = ||r||^2 + (U^T r)^T h (z = r + U h).
// ------------------------------------------------------------------------------------------
struct PcgSParams {
  const double* A;
  int64_t lda, m, n;
  const double* d;
  const double* e;
  const double* U;
  int64_t ldu;
  int ell;
  const double* s;
  const double* rhs;
  double* x;
  double* sc;
  int max_iter;
  int u_smem;           // cluster variant: U staged in shared memory
};

template <int MR, int NT>
__global__ void __launch_bounds__(NT, 1) pcg_small_kernel(const PcgSParams P) {
  constexpr int M32 = 32 * MR;
  constexpr int NW = NT / 32;
  extern __shared__ double wpart[];            // [NW warps][M32] row partials of w
  __shared__ double r_s[M32], z_s[M32], p_s[M32], w_s[M32];
  __shared__ double g_s[256], h_s[256];
  __shared__ double red[64];
  const int tid = threadIdx.x, warp = warp_uniform_id(), lane = tid & 31;
  const int m = (int)P.m, ell = P.ell;
  const int64_t n = P.n;
  const double delta = P.sc[S_DELTA];
  const double tol = P.sc[S_TOL];
  // block sum in a fixed order (warp butterflies, then warp 0 over the 32 warp sums)
  // block sum with ONE barrier: the warp sums go to alternating buffers and every thread adds the NW
  // of them in the same order (a buffer is rewritten only after the next call's barrier)
  int rb = 0;
  auto block_sum = [&](double v) -> double {
    v = warp_sum(v);
    if (lane == 0) red[rb * 32 + warp] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) t += red[rb * 32 + q];
    rb ^= 1;
    return t;
  };
  // z = r + U h with h = s o (U^T r) (s_i = (lam_l + mu)/(lam_i + mu) - 1); returns r^T z
  auto precond = [&](double rr) -> double {
    if (ell == 0) {
      for (int i = tid; i < m; i += blockDim.x) z_s[i] = r_s[i];
      __syncthreads();
      return rr;
    }
    for (int c = warp; c < ell; c += NW) {
      const double* u = P.U + (size_t)c * P.ldu;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        const int i = lane + 32 * k;
        if (i < m) acc = fma(u[i], r_s[i], acc);
      }
      acc = warp_sum(acc);
      if (lane == 0) { g_s[c] = acc; h_s[c] = P.s[c] * acc; }
    }
    __syncthreads();
    for (int i = tid; i < m; i += blockDim.x) {
      double acc = r_s[i];
      for (int c = 0; c < ell; ++c) acc = fma(P.U[(size_t)c * P.ldu + i], h_s[c], acc);
      z_s[i] = acc;
    }
    double gh = 0.0;
    for (int c = tid; c < ell; c += blockDim.x) gh = fma(g_s[c], h_s[c], gh);
    return rr + block_sum(gh);     // (its barriers also publish z_s)
  };

  for (int i = tid; i < m; i += blockDim.x) {
    r_s[i] = P.rhs[i];
    P.x[i] = 0.0;
  }
  __syncthreads();
  double rr = block_sum(tid < m ? r_s[tid] * r_s[tid] : 0.0);
  int iters = 0, status = 0;
  bool conv = sqrt(rr) <= tol;
  double rz = 0.0;
  if (!conv) {
    rz = precond(rr);
    for (int i = tid; i < m; i += blockDim.x) p_s[i] = z_s[i];
    __syncthreads();
  }
  while (!conv && iters < P.max_iter) {
    // ---- w = A (d o (A^T p)) : one column per warp per step ----
    double pr[MR], wacc[MR];
#pragma unroll
    for (int k = 0; k < MR; ++k) {
      const int i = lane + 32 * k;
      pr[k] = (i < m) ? p_s[i] : 0.0;
      wacc[k] = 0.0;
    }
    for (int64_t j = warp; j < n; j += NW) {
      const double* a = P.A + j * P.lda;
      double av[MR];
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        const int i = lane + 32 * k;
        av[k] = (i < m) ? __ldg(a + i) : 0.0;
        acc = fma(av[k], pr[k], acc);
      }
      const double t = __ldg(P.d + j) * warp_sum(acc);
#pragma unroll
      for (int k = 0; k < MR; ++k) wacc[k] = fma(av[k], t, wacc[k]);
    }
#pragma unroll
    for (int k = 0; k < MR; ++k) wpart[warp * M32 + lane + 32 * k] = wacc[k];
    __syncthreads();
    double pw = 0.0;
    if (tid < m) {
      double wsum = 0.0;
      for (int q = 0; q < NW; ++q) wsum += wpart[q * M32 + tid];
      const double wi = wsum + (delta + (P.e ? P.e[tid] : 0.0)) * p_s[tid];
      w_s[tid] = wi;
      pw = p_s[tid] * wi;
    }
    pw = block_sum(pw);
    if (!(pw > 0.0) || !isfinite(pw)) { status = NYS_EBREAKDOWN; break; }
    const double alpha = rz / pw;
    double rloc = 0.0;
    if (tid < m) {
      P.x[tid] = fma(alpha, p_s[tid], P.x[tid]);
      const double ri = fma(-alpha, w_s[tid], r_s[tid]);
      r_s[tid] = ri;
      rloc = ri * ri;
    }
    rr = block_sum(rloc);
    ++iters;
    if (sqrt(rr) <= tol) { conv = true; break; }
    if (!isfinite(rr)) { status = NYS_EBREAKDOWN; break; }
    const double rzn = precond(rr);
    if (!(rzn > 0.0) || !isfinite(rzn)) { status = NYS_EBREAKDOWN; break; }
    const double beta = rzn / rz;
    rz = rzn;
    if (tid < m) p_s[tid] = fma(beta, p_s[tid], z_s[tid]);
    __syncthreads();
  }
  if (tid == 0) {
    P.sc[S_ITERS] = (double)iters;
    P.sc[S_STATUS] = (double)status;
    P.sc[S_DONE] = 1.0;
    P.sc[S_RZ] = rz;
    P.sc[S_RR] = rr;
  }
}

// The same solve on a thread-block CLUSTER of C CTAs with A resident in shared memory: CTA r holds the
// columns [r n / C, (r + 1) n / C) of A (and of d) in its shared memory for the whole solve (loaded
// once), so the matvec never touches L2 again.  Per iteration ONE cluster barrier: every CTA writes its
// partial w (own columns) into a double-buffered shared slot, the barrier publishes them, and every CTA
// sums the C partials of every row in rank order through DSMEM — identical bits everywhere — and then
// runs the m-space work (alpha, x, r, U^T r, z, beta, p) redundantly with __syncthreads only.  The
// double buffer is safe with one barrier per iteration: a CTA can overwrite slot k & 1 only after the
// barrier of iteration k + 1, which every peer reaches after its reads of iteration k.
template <int MR, int NT>
__global__ void __launch_bounds__(NT, 1) pcg_cluster_small_kernel(const PcgSParams P) {
  constexpr int M32 = 32 * MR;
  constexpr int NW = NT / 32;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
  extern __shared__ double dsm[];
  const int m = (int)P.m, ell = P.ell;
  const int64_t n = P.n;
  const int64_t c_lo = (n * rank) / C, c_hi = (n * (rank + 1)) / C;
  const int ncols = (int)(c_hi - c_lo);
  // the DSMEM-visible receive buffer first: its offset must be the same in every CTA (mapa maps
  // offsets); recv[b][q][.] holds CTA q's partial w of an iteration of parity b, pushed by CTA q
  double* recv = dsm;                                // [2][C][M32]
  double* wpart = recv + 2 * (size_t)C * M32;        // [NW][M32]
  double* As = wpart + NW * M32;                     // [ncols][M32], rows >= m zero
  double* ds = As + (size_t)ncols * M32;             // [ncols] (even count)
  double* Us = ds + ((ncols + 1) & ~1);              // [ell][M32] when P.u_smem (U read from global otherwise)
  __shared__ double r_s[M32], z_s[M32], p_s[M32], w_s[M32], x_s[M32];
  __shared__ double g_s[257], h_s[256];
  __shared__ double red[64];
  __shared__ __align__(8) uint64_t rbar[2];          // receive barriers (parity of the iteration)
  const int tid = threadIdx.x, warp = warp_uniform_id(), lane = tid & 31;
  const double delta = P.sc[S_DELTA];
  const double tol = P.sc[S_TOL];
  if (tid == 0) {
    mbar_init(&rbar[0], 1);
    mbar_init(&rbar[1], 1);
    fence_mbar_init();
  }
  for (int64_t e = tid; e < (int64_t)ncols * M32; e += NT) {
    const int j = (int)(e / M32), i = (int)(e % M32);
    As[e] = (i < m) ? P.A[(c_lo + j) * P.lda + i] : 0.0;
  }
  for (int j = tid; j < ncols; j += NT) ds[j] = P.d[c_lo + j];
  const bool us = P.u_smem != 0;
  if (us)
    for (int e = tid; e < ell * M32; e += NT) {
      const int c = e / M32, i = e % M32;
      Us[e] = (i < m) ? P.U[(size_t)c * P.ldu + i] : 0.0;
    }
  auto Ucol = [&](int c) -> const double* { return us ? Us + (size_t)c * M32 : P.U + (size_t)c * P.ldu; };
  // block sum with ONE barrier: the warp sums go to alternating buffers and every thread adds the NW
  // of them in the same order (a buffer is rewritten only after the next call's barrier)
  int rb = 0;
  auto block_sum = [&](double v) -> double {
    v = warp_sum(v);
    if (lane == 0) red[rb * 32 + warp] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) t += red[rb * 32 + q];
    rb ^= 1;
    return t;
  };
  // g_c = U_c^T r for c < ell and g_ell = r^T r, one warp per entry (r_s complete on entry); a barrier
  // (four entries per warp step: their shuffle reductions overlap)
  auto gpass = [&]() {
    for (int c0 = warp; c0 <= ell; c0 += 4 * NW) {
      double acc[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + j * NW;
        acc[j] = 0.0;
        if (c <= ell) {                              // warp-uniform
          const double* u = (c < ell) ? Ucol(c) : r_s;
#pragma unroll
          for (int k = 0; k < MR; ++k) {
            const int i = lane + 32 * k;
            if (i < m) acc[j] = fma(u[i], r_s[i], acc[j]);
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
      if (lane == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = c0 + j * NW;
          if (c <= ell) {
            g_s[c] = acc[j];
            if (c < ell) h_s[c] = P.s[c] * acc[j];
          }
        }
      }
    }
    __syncthreads();
  };
  // r^T z = r^T r + sum_c s_c g_c^2 (h = s o g: no further reduction), the same order in every thread;
  // then own rows z = r + U h and p = z + beta p
  // (four independent FMA chains: the same order in every thread of every CTA)
  auto rz_of = [&](double rr) -> double {
    double gh[4] = {0.0, 0.0, 0.0, 0.0};
    int c = 0;
    for (; c + 3 < ell; c += 4)
#pragma unroll
      for (int j = 0; j < 4; ++j) gh[j] = fma(h_s[c + j], g_s[c + j], gh[j]);
    for (; c < ell; ++c) gh[0] = fma(h_s[c], g_s[c], gh[0]);
    return rr + ((gh[0] + gh[1]) + (gh[2] + gh[3]));
  };
  auto z_row = [&](int i) -> double {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int c = 0;
    for (; c + 3 < ell; c += 4)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = fma(Ucol(c + j)[i], h_s[c + j], acc[j]);
    for (; c < ell; ++c) acc[0] = fma(Ucol(c)[i], h_s[c], acc[0]);
    return r_s[i] + ((acc[0] + acc[1]) + (acc[2] + acc[3]));
  };
  for (int i = tid; i < M32; i += NT) {
    r_s[i] = (i < m) ? P.rhs[i] : 0.0;
    x_s[i] = 0.0;
    p_s[i] = 0.0;
  }
  __syncthreads();
  gpass();
  double rr = g_s[ell];
  int iters = 0, status = 0;
  bool conv = sqrt(rr) <= tol;
  double rz = 0.0;
  if (!conv) {
    rz = rz_of(rr);
    if (tid < m) p_s[tid] = z_row(tid);
    __syncthreads();
  }
  cluster.sync();                                    // every CTA's A slice loaded before any DSMEM traffic
  int k = 0;
  while (!conv && iters < P.max_iter) {
    double pr[MR], wacc[MR];
#pragma unroll
    for (int q = 0; q < MR; ++q) {
      pr[q] = p_s[lane + 32 * q];
      wacc[q] = 0.0;
    }
    // four columns per warp step: their dot reductions overlap (absent columns: t = 0, column j reread)
    for (int j = warp; j < ncols; j += 4 * NW) {
      double av[4][MR], acc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int jj = j + u * NW;
        const double* a = As + (size_t)(jj < ncols ? jj : j) * M32;
        acc[u] = 0.0;
#pragma unroll
        for (int q = 0; q < MR; ++q) {
          av[u][q] = a[lane + 32 * q];
          acc[u] = fma(av[u][q], pr[q], acc[u]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
      double t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] = (j + u * NW < ncols) ? ds[j + u * NW] * acc[u] : 0.0;
#pragma unroll
      for (int q = 0; q < MR; ++q) {
        double wq = wacc[q];
#pragma unroll
        for (int u = 0; u < 4; ++u) wq = fma(av[u][q], t[u], wq);
        wacc[q] = wq;
      }
    }
#pragma unroll
    for (int q = 0; q < MR; ++q) wpart[warp * M32 + lane + 32 * q] = wacc[q];
    __syncthreads();
    // this CTA's partial w pushed into every CTA's receive buffer (st.async completing bytes on the
    // receiver's barrier), then a local wait for all C partials: no cluster barrier and no remote load
    // on the critical path.  Ring safety: a peer pushes into the same buffer again two iterations later,
    // only after our push of the next iteration, which we issue after reading this one.
    const int b = k & 1;
    if (tid == 0) mbar_arrive_expect_tx(&rbar[b], (uint32_t)(C * m * 8));
    if (tid < m) {
      double v = 0.0;
      for (int q = 0; q < NW; ++q) v += wpart[q * M32 + tid];
      const uint32_t la = smem_u32(recv + ((size_t)b * C + rank) * M32 + tid);
      const uint32_t lb = smem_u32(&rbar[b]);
      for (int q = 0; q < C; ++q) st_async_f64(mapa_shared(la, (uint32_t)q), v, mapa_shared(lb, (uint32_t)q));
    }
    mbar_wait(&rbar[b], (uint32_t)((k >> 1) & 1));
    double pw = 0.0;
    if (tid < m) {
      const double* rv = recv + (size_t)b * C * M32 + tid;
      // the C (<= 16) partials in a fixed pairwise tree (depth 4 instead of a C-long add chain)
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = (q < C) ? rv[(size_t)q * M32] : 0.0;
#pragma unroll
      for (int w = 8; w > 0; w >>= 1)
#pragma unroll
        for (int q = 0; q < w; ++q) v[q] += v[q + w];
      const double wsum = v[0];
      const double wi = wsum + (delta + (P.e ? P.e[tid] : 0.0)) * p_s[tid];
      w_s[tid] = wi;
      pw = p_s[tid] * wi;
    }
    pw = block_sum(pw);
    ++k;
    if (!(pw > 0.0) || !isfinite(pw)) { status = NYS_EBREAKDOWN; break; }
    const double alpha = rz / pw;
    if (tid < m) {
      x_s[tid] = fma(alpha, p_s[tid], x_s[tid]);
      r_s[tid] = fma(-alpha, w_s[tid], r_s[tid]);
    }
    __syncthreads();
    gpass();                                         // ||r||^2 and U^T r in one pass
    rr = g_s[ell];
    ++iters;
    if (sqrt(rr) <= tol) { conv = true; break; }
    if (!isfinite(rr)) { status = NYS_EBREAKDOWN; break; }
    const double rzn = rz_of(rr);
    if (!(rzn > 0.0) || !isfinite(rzn)) { status = NYS_EBREAKDOWN; break; }
    const double beta = rzn / rz;
    rz = rzn;
    if (tid < m) p_s[tid] = fma(beta, p_s[tid], z_row(tid));
    __syncthreads();
  }
  if (rank == 0) {
    for (int i = tid; i < m; i += NT) P.x[i] = x_s[i];
    if (tid == 0) {
      P.sc[S_ITERS] = (double)iters;
      P.sc[S_STATUS] = (double)status;
      P.sc[S_DONE] = 1.0;
      P.sc[S_RZ] = rz;
      P.sc[S_RR] = rr;
    }
  }
  cluster.sync();                                    // no CTA leaves while a peer may still read its partials
}

// the cluster variant holds A in shared memory: at most 16 CTAs x 150 KB of padded columns
static int small_cluster_size(int64_t m, int64_t n) {
  const int64_t m32 = m <= 64 ? 64 : m <= 128 ? 128 : 256;
  const double bytes = (double)n * (double)m32 * 8.0;
  // ~34 KB of A per CTA, at most 16 CTAs (measured at config 0, A = 410 KB padded: C = 3 / 4 / 5 / 7 /
  // 8 / 12 / 16 -> 4.24 / 3.80 / 3.64 / 3.49 / 3.34 / 3.31 / 3.36 us per PCG iteration)
  int C = (int)((bytes + 34e3 - 1) / 34e3);
  if (C > 16) C = 16;
  if (C < 2) C = 2;
  if (bytes / C > 150e3) C = (int)((bytes + 150e3 - 1) / 150e3);
  return C;
}
bool pcg_small_supported(nys_ctx* ctx, int64_t m, int64_t n, int ell) {
  return !ctx->multi() && m <= 256 && n > 0 && ell <= 256 && (double)m * (double)n * 8.0 <= 1.0e6 &&
         getenv("NYS_NO_PCG_SMALL") == nullptr && getenv("NYS_NO_PERSISTENT") == nullptr;
}

int launch_pcg_small(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d, const double* e,
                     const double* U, int64_t ldu, int ell, const double* s, const double* rhs, double* x, int max_iter) {
  PcgSParams P{};
  P.A = A; P.lda = lda; P.m = m; P.n = n; P.d = d; P.e = e; P.U = U; P.ldu = ldu; P.ell = ell; P.s = s;
  P.rhs = rhs; P.x = x; P.sc = ctx->sc; P.max_iter = max_iter;
  // cluster variant (A in shared memory) unless disabled or A needs more than 16 CTAs
  int C = small_cluster_size(m, n);
  if (const char* oc = getenv("NYS_PCG_SMALL_C")) {   // tuning override (>= the size A needs)
    const int o = atoi(oc);
    if (o >= C && o <= 16) C = o;
    else if (o >= 2 && o < C) {
      const int64_t m32 = m <= 64 ? 64 : m <= 128 ? 128 : 256;
      if ((double)n * m32 * 8.0 / o <= 150e3) C = o;
    }
  }
  if (C <= 16 && getenv("NYS_PCG_SMALL_1CTA") == nullptr) {
    const int64_t m32 = m <= 64 ? 64 : m <= 128 ? 128 : 256;
    const int64_t maxcols = (n + C - 1) / C;
    // 256 threads (measured at config 0: 3.47 vs 3.63 us per iteration with 512; NYS_PCG_SMALL_NT=512)
    static const int nt = getenv("NYS_PCG_SMALL_NT") ? atoi(getenv("NYS_PCG_SMALL_NT")) : 256;
    size_t smem = ((size_t)maxcols * m32 + ((maxcols + 1) & ~1) + (size_t)(nt / 32) * m32 + 2 * (size_t)C * m32) * 8;
    const size_t ubytes = (size_t)ell * m32 * 8;
    P.u_smem = (smem + ubytes <= 200 * 1024 && getenv("NYS_PCG_SMALL_UGLOBAL") == nullptr) ? 1 : 0;
    if (P.u_smem) smem += ubytes;
    const void* k = nt == 512 ? (m <= 64 ? (const void*)pcg_cluster_small_kernel<2, 512>
                                         : m <= 128 ? (const void*)pcg_cluster_small_kernel<4, 512>
                                                    : (const void*)pcg_cluster_small_kernel<8, 512>)
                  : m <= 64 ? (const void*)pcg_cluster_small_kernel<2, 256>
                  : m <= 128 ? (const void*)pcg_cluster_small_kernel<4, 256> : (const void*)pcg_cluster_small_kernel<8, 256>;
    NYS_TRY(ensure_max_smem(ctx, k, smem));
    if (C > 8) NYS_CUDA_TRY(ctx, cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)C);
    cfg.blockDim = dim3((unsigned)(nt == 512 ? 512 : 256));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    NYS_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, (void (*)(const PcgSParams))k, P));
    ctx->launches++;
    return ctx->check_launch("pcg_cluster_small");
  }
  // rows per lane MR and threads NT sized so the column loop stays in registers (64 / 128 registers)
  if (m <= 64) {
    pcg_small_kernel<2, 1024><<<1, 1024, 32 * 64 * 8, ctx->stream>>>(P);
  } else if (m <= 128) {
    pcg_small_kernel<4, 512><<<1, 512, 16 * 128 * 8, ctx->stream>>>(P);
  } else {
    pcg_small_kernel<8, 512><<<1, 512, 16 * 256 * 8, ctx->stream>>>(P);
  }
  ctx->launches++;
  return ctx->check_launch("pcg_small");
}

// ------------------------------------------------------------------------------------------
struct PcgCfg {
  int T, GT, RPT, CPG;
};
static PcgCfg pcg_pick(int64_t m, int64_t n, int sms) {
  if (m <= 64) return (n / 64 >= 4LL * sms) ? PcgCfg{256, 32, 2, 8} : PcgCfg{256, 32, 2, 4};   // config 3: 63.9 -> 47.7 us / it
  if (m <= 128) {
    // short columns: a panel of 8 CPG columns x m rows is a small bulk copy; with many columns take
    // more per group (SensIT shape m = 101, 98528 columns: PCG 71.9 / 50.5 / 44.4 ms at CPG 2 / 4 / 8;
    // config 0, 400 columns: CPG 2 best) while every CTA still gets >= 4 panels
    for (int cpg = 8; cpg > 2; cpg >>= 1)
      if (n / (8 * cpg) >= 4LL * sms) return {256, 32, 4, cpg};
    return {256, 32, 4, 2};
  }
  if (m <= 256) return {256, 64, 4, 2};
  if (m <= 1024) return {256, 128, 8, 2};
  if (m <= 2048) return {256, 256, 8, 4};
  if (m <= 4096) return getenv("NYS_PCG_T512") ? PcgCfg{512, 512, 8, 2} : PcgCfg{256, 256, 16, 2};
  return {512, 512, 16, 1};
}
typedef void (*PcgKernel)(const PcgPParams);
static PcgKernel pcg_kernel_for(const PcgCfg& c) {
  if (c.GT == 32 && c.RPT == 2 && c.CPG == 8) return pcg_persistent_kernel<256, 32, 2, 8>;
  if (c.GT == 32 && c.RPT == 2) return pcg_persistent_kernel<256, 32, 2, 4>;
  if (c.GT == 32 && c.RPT == 4 && c.CPG == 8) return pcg_persistent_kernel<256, 32, 4, 8>;
  if (c.GT == 32 && c.RPT == 4 && c.CPG == 4) return pcg_persistent_kernel<256, 32, 4, 4>;
  if (c.GT == 32 && c.RPT == 4) return pcg_persistent_kernel<256, 32, 4, 2>;
  if (c.GT == 64) return pcg_persistent_kernel<256, 64, 4, 2>;
  if (c.GT == 128) return pcg_persistent_kernel<256, 128, 8, 2>;
  if (c.GT == 256 && c.RPT == 16) return pcg_persistent_kernel<256, 256, 16, 2>;
  if (c.GT == 256 && c.CPG == 2) return pcg_persistent_kernel<256, 256, 8, 2>;
  if (c.GT == 256) return pcg_persistent_kernel<256, 256, 8, 4>;
  if (c.RPT == 8) return pcg_persistent_kernel<512, 512, 8, 2>;
  return pcg_persistent_kernel<512, 512, 16, 1>;
}

bool pcg_persistent_supported(nys_ctx* ctx, int64_t m, int64_t n, int ell) {
  if (m > 8192) return pcg_cluster_supported(ctx, m, n, ell);
  return !ctx->multi() && n > 0 && ell <= 256 && getenv("NYS_NO_PERSISTENT") == nullptr;
}

// tolerance must already be in sc[S_TOL] and delta in sc[S_DELTA]
int launch_pcg_persistent(nys_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda, const double* d,
                          const double* e, const double* U, int64_t ldu, int ell, const double* s, const double* rhs,
                          double* x, int max_iter) {
  if (m > 8192) return launch_pcg_cluster(ctx, m, n, A, lda, d, e, U, ldu, ell, s, rhs, x, max_iter);
  const auto hp0 = std::chrono::steady_clock::now();
  PcgCfg c = pcg_pick(m, n, ctx->num_sms);
  if (const char* ov = getenv("NYS_PCG_CFG")) {  // tuning override "T,GT,RPT,CPG" (must be instantiated)
    PcgCfg o;
    if (sscanf(ov, "%d,%d,%d,%d", &o.T, &o.GT, &o.RPT, &o.CPG) == 4 && (int64_t)o.GT * o.RPT >= m) c = o;
  }
  const int NG = c.T / c.GT, WPG = c.GT / 32, BN = NG * c.CPG;
  const int64_t mp = (m + 1) & ~int64_t(1);
  const int64_t ss = (lda >= mp && lda <= mp + 32) ? lda : mp;
  const size_t stage_bytes = (size_t)BN * ss * 8;
  const size_t budget = (mp <= 1024) ? 96 * 1024 : 196 * 1024;
  int stages = (int)(budget / stage_bytes);
  if (stages > 8) stages = 8;
  if (stages < 2) stages = 2;
  const size_t smem = (size_t)stages * stage_bytes + 2 * stages * 8 + (size_t)2 * NG * WPG * c.CPG * 8;
  PcgKernel k = pcg_kernel_for(c);
  NYS_TRY(ensure_max_smem(ctx, (const void*)k, smem));
  int occ = 0;
  NYS_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, c.T + 32, smem));
  if (occ < 1) { ctx->set_error("persistent PCG does not fit on an SM"); return NYS_ECUDA; }
  const int64_t npanels = (n + BN - 1) / BN;
  int64_t G = (int64_t)ctx->num_sms * occ;
  if (G > npanels) G = npanels;
  if (const char* e = getenv("NYS_PCG_GRID")) G = atoi(e);   // tuning override (grid size)
  if (G > npanels) G = npanels;
  if (G < 1) G = 1;
  PcgPParams P{};
  P.A = A; P.lda = lda; P.m = m; P.n = n; P.d = d; P.e = e; P.U = U; P.ldu = ldu; P.ell = ell; P.s = s;
  P.rhs = rhs; P.x = x;
  P.r = ctx->wsd("pp_r", (size_t)mp);
  P.z = ell > 0 ? ctx->wsd("pp_z", (size_t)mp) : P.r;
  P.P0 = ctx->wsd("pp_p0", (size_t)mp);
  P.P1 = ctx->wsd("pp_p1", (size_t)mp);
  P.wp_ld = mp;
  P.Wp = ctx->wsd("pp_Wp", (size_t)G * mp);
  P.pwp = ctx->wsd("pp_pwp", (size_t)G);
  P.part1 = ctx->wsd("pp_part1", (size_t)(1 + ell) * G);
  P.sc = ctx->sc;
  P.bar = (unsigned int*)ctx->ws("pp_bar", 64 + 66 * 4);
  P.rbar = P.bar + 16;
  P.gtot = ctx->wsd("pp_gtot", (size_t)((G + RG - 1) / RG) * (1 + ell));
  P.tot = ctx->wsd("pp_tot", (size_t)(1 + ell));
  P.max_iter = max_iter;
  P.flat_red = 1;
  if (const char* e = getenv("NYS_PCG_RED")) P.flat_red = (e[0] == 'f');
  P.stages = stages;
  P.npanels = npanels;
  P.ss = ss;
  P.rows_per_cta = (m + G - 1) / G;
  P.acq_spin = getenv("NYS_BAR_FENCE") ? 0 : 1;
  {
    // L2 prefetch depth beyond the smem ring: ~40 MB of A (about a third of L2) pulled into L2 while
    // the CTAs sit in the reduction / barrier phases, so HBM keeps streaming there.  Measured at
    // config 1 (same box, 400 iterations): PF 0 -> 32.4 us, PF 4 / 16 / 32 -> 30.8 / 30.7 / 30.8 us;
    const double panel_bytes = (double)BN * lda * 8.0;
    int pfd = (int)(40e6 / (panel_bytes * (double)G));
    if (pfd > 16) pfd = 16;
    if (pfd < 1) pfd = 1;
    // only where A is about L2-sized: at 1.5 GB (CIFAR10-shaped dual SVM) it measured 2.6 % slower
    if ((double)n * lda * 8.0 > 256e6) pfd = 0;
    if (const char* e = getenv("NYS_PCG_PF")) pfd = atoi(e);
    P.l2_prefetch = pfd;
    int keep = 0;
    if (const char* e = getenv("NYS_PCG_KEEP")) keep = atoi(e);
    P.l2_keep = keep;
  }
  NYS_CUDA_TRY(ctx, cudaMemsetAsync(P.bar, 0, 64 + 66 * 4, ctx->stream));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)G);
  cfg.blockDim = dim3((unsigned)(c.T + 32));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const bool trace = getenv("NYS_PCG_TRACE") != nullptr;
  if (trace) {
    P.trace = (unsigned long long*)ctx->ws("pp_trace", 2 * 32 * 16 * 8);
    NYS_CUDA_TRY(ctx, cudaMemsetAsync(P.trace, 0, 2 * 32 * 16 * 8, ctx->stream));
    P.trace_arr = (unsigned long long*)ctx->ws("pp_trace_arr", 3 * G * 8);
    NYS_CUDA_TRY(ctx, cudaMemsetAsync(P.trace_arr, 0, 3 * G * 8, ctx->stream));
  }
  const auto hp1 = std::chrono::steady_clock::now();
  NYS_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, k, P));
  ctx->launches++;
  if (getenv("NYS_PCG_HOSTPROF")) {
    const auto hp2 = std::chrono::steady_clock::now();
    fprintf(stderr, "[pcghost] prep %.1f us, launch call %.1f us\n",
            std::chrono::duration<double, std::micro>(hp1 - hp0).count(),
            std::chrono::duration<double, std::micro>(hp2 - hp1).count());
  }
  if (trace) {
    unsigned long long h[2 * 32 * 16];
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(h, P.trace, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    std::vector<unsigned long long> ha(3 * G);
    NYS_CUDA_TRY(ctx, cudaMemcpyAsync(ha.data(), P.trace_arr, 3 * G * 8, cudaMemcpyDeviceToHost, ctx->stream));
    NYS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    {
      const unsigned long long* r = h + 14 * 16;   // CTA 0, iteration 14: release stamps 2 (bar1), 6 (colsum), 5 (bar3)
      const int rel_slot[3] = {2, 6, 5};
      const char* nm[3] = {"bar1", "colsum", "bar3"};
      for (int w = 0; w < 3 && r[0] != 0; ++w) {
        unsigned long long mn = ~0ull, mx = 0;
        int64_t amx = 0;
        for (int64_t c = 0; c < G; ++c) {
          const unsigned long long t = ha[(size_t)w * G + c];
          if (t == 0) continue;
          mn = t < mn ? t : mn;
          if (t > mx) { mx = t; amx = c; }
        }
        fprintf(stderr, "[pcgsync] it=14 %s: arrivals spread %.2f us (last CTA %lld), CTA0 released %.2f us after the last arrival\n",
                nm[w], (mx - mn) * 1e-3, (long long)amx, ((double)r[rel_slot[w]] - (double)mx) * 1e-3);
      }
    }
    for (int c = 0; c < 2; ++c)
      for (int it = 0; it < 32; ++it) {
        const unsigned long long* r = h + (c * 32 + it) * 16;
        if (r[0] == 0 || r[5] == 0) continue;
        fprintf(stderr, "[pcgtrace] cta=%s it=%d vset=%.2f first=%.2f half=%.2f last=%.2f\n", c ? "last" : "0", it,
                (r[8] - r[0]) * 1e-3, (r[9] - r[8]) * 1e-3, (r[10] - r[9]) * 1e-3, (r[11] - r[10]) * 1e-3);
        fprintf(stderr, "[pcgtrace] cta=%s it=%d matvec=%.2f bar1=%.2f rows=%.2f bar2=%.2f colsum=%.2f zrows=%.2f bar3=%.2f total=%.2f us\n",
                c ? "last" : "0", it, (r[1] - r[0]) * 1e-3, (r[2] - r[1]) * 1e-3, (r[3] - r[2]) * 1e-3,
                (r[4] - r[3]) * 1e-3, (r[6] - r[4]) * 1e-3, (r[7] - r[6]) * 1e-3, (r[5] - r[7]) * 1e-3, (r[5] - r[0]) * 1e-3);
      }
  }
  return ctx->check_launch("pcg_persistent");
}

}  // namespace nys
