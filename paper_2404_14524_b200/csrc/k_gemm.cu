// fp64 tensor-core GEMM for the Nystrom sketch (Alg. 1 line 2: Y = N Omega computed as
// A (d o (A^T Omega))) and the O(m l^2) products of the factorisation (Gram, triangular
// solves by the inverse factor, U = Q W).
//
// B200 has no tcgen05 kind::f64 (ptxas rejects it): fp64 tensor-core math is
// warp-level DMMA, `mma.sync.aligned.m16n8k4.row.col.f64`.  CTA tile 64x64x16, 4 warps with
// 32x32 warp tiles (2 x 4 MMAs per k4 step), 3-stage cp.async (16 B, zero-fill at the
// ragged edges) shared-memory pipeline, padded layouts so every fragment load is
// bank-conflict free.  Long K (the n-direction of Y = A T) is split across CTAs; partial
// tiles are summed in a fixed order by gemm_reduce (deterministic).
#include <cuda.h>   // CUtensorMap (the encode entry point is fetched through cudaGetDriverEntryPoint)

#include <algorithm>
#include <mutex>

#include "k_vec.cuh"

namespace nys {

constexpr int GBM = 64, GBN = 64, GBK = 16, GST = 3;
constexpr int LDA_K = GBK + 4;  // smem [BM][LDA_K] when A is K-major
constexpr int LDA_M = GBM + 4;  // smem [BK][LDA_M] when A is M-major
constexpr int LDB_K = GBK + 4;  // smem [BN][LDB_K]
constexpr int A_STAGE = (GBM * LDA_K > GBK * LDA_M) ? GBM * LDA_K : GBK * LDA_M;
constexpr int B_STAGE = GBN * LDB_K;

struct GemmParams {
  int64_t M, N, K;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  const double* row_scale;
  const double* addv;
  const double* addm;
  int64_t ldadd;
  int64_t kchunk;
  int partial;    // 1: write raw tile to C + split*M*N (ld = M)
};

__device__ __forceinline__ void cp_async16(void* smem, const void* g, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(g), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ int clamp_bytes(int64_t remaining_elems) {
  if (remaining_elems <= 0) return 0;
  return remaining_elems >= 2 ? 16 : 8;
}

template <bool AK>
__device__ __forceinline__ void load_stage(const GemmParams& G, double* As, double* Bs, int64_t i0, int64_t j0,
                                           int64_t k0, int64_t kend) {
  const int tid = threadIdx.x;
  // A tile: 512 chunks of 16 B
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int ch = tid + q * 128;
    if (AK) {
      const int r = ch >> 3, kc = ch & 7;
      const int64_t gi = i0 + r, gk = k0 + 2 * kc;
      const int nb = (gi < G.M) ? clamp_bytes(kend - gk) : 0;
      const double* src = nb ? (G.A + gi * G.lda + gk) : G.A;
      cp_async16(As + r * LDA_K + 2 * kc, src, nb);
    } else {
      const int k = ch >> 5, ic = ch & 31;
      const int64_t gi = i0 + 2 * ic, gk = k0 + k;
      const int nb = (gk < kend) ? clamp_bytes(G.M - gi) : 0;
      const double* src = nb ? (G.A + gi + gk * G.lda) : G.A;
      cp_async16(As + k * LDA_M + 2 * ic, src, nb);
    }
  }
  // B tile: BN x BK, K contiguous
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int ch = tid + q * 128;
    const int j = ch >> 3, kc = ch & 7;
    const int64_t gj = j0 + j, gk = k0 + 2 * kc;
    const int nb = (gj < G.N) ? clamp_bytes(kend - gk) : 0;
    const double* src = nb ? (G.B + gk + gj * G.ldb) : G.B;
    cp_async16(Bs + j * LDB_K + 2 * kc, src, nb);
  }
}

template <bool AK>
__global__ void __launch_bounds__(128) dgemm_kernel(const GemmParams G) {
  extern __shared__ __align__(128) double gsm[];
  double* Asm = gsm;
  double* Bsm = gsm + GST * A_STAGE;
  // N-tiles vary fastest across the grid: the CTAs that share an A tile (the ceil(N/64) <= 4
  // column blocks of a sketch with l <= 256) run together, so A streams from HBM once and the
  // other reads hit L2
  const int64_t i0 = (int64_t)blockIdx.y * GBM;
  const int64_t j0 = (int64_t)blockIdx.x * GBN;
  const int64_t kbeg = (int64_t)blockIdx.z * G.kchunk;
  int64_t kend = kbeg + G.kchunk;
  if (kend > G.K) kend = G.K;
  const int nk = (kend > kbeg) ? (int)((kend - kbeg + GBK - 1) / GBK) : 0;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp & 1, wn = warp >> 1;
  const int gq = lane >> 2, tq = lane & 3;

  double acc[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

#pragma unroll
  for (int s = 0; s < GST - 1; ++s) {
    if (s < nk) load_stage<AK>(G, Asm + s * A_STAGE, Bsm + s * B_STAGE, i0, j0, kbeg + (int64_t)s * GBK, kend);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<GST - 2>();
    __syncthreads();
    const int nxt = kt + GST - 1;
    if (nxt < nk)
      load_stage<AK>(G, Asm + (nxt % GST) * A_STAGE, Bsm + (nxt % GST) * B_STAGE, i0, j0, kbeg + (int64_t)nxt * GBK, kend);
    cp_async_commit();
    const double* As = Asm + (kt % GST) * A_STAGE;
    const double* Bs = Bsm + (kt % GST) * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < GBK / 4; ++kk) {
      const int k = 4 * kk + tq;
      double af[2][2], bf[4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int r = 32 * wm + 16 * mt + gq;
        if (AK) {
          af[mt][0] = As[r * LDA_K + k];
          af[mt][1] = As[(r + 8) * LDA_K + k];
        } else {
          af[mt][0] = As[k * LDA_M + r];
          af[mt][1] = As[k * LDA_M + r + 8];
        }
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = Bs[(32 * wn + 8 * nt + gq) * LDB_K + k];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_16x8x4(acc[mt][nt], af[mt][0], af[mt][1], bf[nt]);
    }
  }
  cp_async_wait<0>();

  // epilogue
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int64_t row = i0 + 32 * wm + 16 * mt + gq + 8 * (c >> 1);
        const int64_t col = j0 + 32 * wn + 8 * nt + 2 * tq + (c & 1);
        if (row < G.M && col < G.N) {
          double v = acc[mt][nt][c];
          if (G.partial) {
            G.C[(size_t)blockIdx.z * G.M * G.N + row + col * G.M] = v;
          } else {
            if (G.row_scale) v *= G.row_scale[row];
            if (G.addv) v += G.addv[row] * G.addm[row + col * G.ldadd];
            G.C[row + col * G.ldc] = v;
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// N-adaptive DMMA GEMM: CTA tile 128 x (8 NT), 4 warps x 32 rows, m16n8k8 f64 MMAs (A fragment
// rows g, g+8 / cols t, t+4; B fragment k = t, t+4, n = g; layouts checked on B200 by
// scratch/dmma_probe.cu).  NT is picked per call so that 8 NT tiles the sketch width l with the
// least padding (l = 200 -> NT = 5 exactly; a 64-wide tile would compute 256 columns), BK = 16,
// 3-stage cp.async ring.  Padded smem rows: K-major leading dimension = 20 doubles (row stride 4
// banks-of-8B mod 16 -> the minimum 2 wavefronts per fragment load), M-major = BM + 8.
// ------------------------------------------------------------------------------------------
constexpr int HBM_ = 128, HBK = 16, HST = 3;
constexpr int HLD_K = HBK + 4;      // [rows][HLD_K] for K-major tiles (A when AK, and B)
constexpr int HLD_M = HBM_ + 8;     // [HBK][HLD_M] for M-major A
constexpr int HA_STAGE = (HBM_ * HLD_K > HBK * HLD_M) ? HBM_ * HLD_K : HBK * HLD_M;

__device__ __forceinline__ void dmma_16x8x8(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

template <int NT, bool AK>
__device__ __forceinline__ void hload_stage(const GemmParams& G, double* As, double* Bs, int64_t i0, int64_t j0,
                                            int64_t k0, int64_t kend) {
  const int tid = threadIdx.x;
  // A: 128 x 16 doubles = 1024 chunks of 16 B, 8 per thread
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int ch = tid + q * 128;
    if (AK) {
      const int r = ch >> 3, kc = ch & 7;
      const int64_t gi = i0 + r, gk = k0 + 2 * kc;
      const int nb = (gi < G.M) ? clamp_bytes(kend - gk) : 0;
      const double* src = nb ? (G.A + gi * G.lda + gk) : G.A;
      cp_async16(As + r * HLD_K + 2 * kc, src, nb);
    } else {
      const int k = ch >> 6, ic = ch & 63;
      const int64_t gi = i0 + 2 * ic, gk = k0 + k;
      const int nb = (gk < kend) ? clamp_bytes(G.M - gi) : 0;
      const double* src = nb ? (G.A + gi + gk * G.lda) : G.A;
      cp_async16(As + k * HLD_M + 2 * ic, src, nb);
    }
  }
  // B: (8 NT) x 16 doubles, K contiguous = 64 NT chunks
#pragma unroll
  for (int q = 0; q < (64 * NT + 127) / 128; ++q) {
    const int ch = tid + q * 128;
    if (ch < 64 * NT) {
      const int j = ch >> 3, kc = ch & 7;
      const int64_t gj = j0 + j, gk = k0 + 2 * kc;
      const int nb = (gj < G.N) ? clamp_bytes(kend - gk) : 0;
      const double* src = nb ? (G.B + gk + gj * G.ldb) : G.B;
      cp_async16(Bs + j * HLD_K + 2 * kc, src, nb);
    }
  }
}

template <int NT, bool AK>
__global__ void __launch_bounds__(128) dgemm_nt_kernel(const GemmParams G) {
  constexpr int BN = 8 * NT;
  constexpr int B_ST = BN * HLD_K;
  extern __shared__ __align__(128) double gsm[];
  double* Asm = gsm;
  double* Bsm = gsm + HST * HA_STAGE;
  const int64_t j0 = (int64_t)blockIdx.x * BN;      // N-tiles fastest: CTAs sharing an A tile run together
  const int64_t i0 = (int64_t)blockIdx.y * HBM_;
  const int64_t kbeg = (int64_t)blockIdx.z * G.kchunk;
  int64_t kend = kbeg + G.kchunk;
  if (kend > G.K) kend = G.K;
  const int nk = (kend > kbeg) ? (int)((kend - kbeg + HBK - 1) / HBK) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;

  double acc[2][NT][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

#pragma unroll
  for (int st = 0; st < HST - 1; ++st) {
    if (st < nk) hload_stage<NT, AK>(G, Asm + st * HA_STAGE, Bsm + st * B_ST, i0, j0, kbeg + (int64_t)st * HBK, kend);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<HST - 2>();
    __syncthreads();
    const int nxt = kt + HST - 1;
    if (nxt < nk)
      hload_stage<NT, AK>(G, Asm + (nxt % HST) * HA_STAGE, Bsm + (nxt % HST) * B_ST, i0, j0, kbeg + (int64_t)nxt * HBK,
                          kend);
    cp_async_commit();
    const double* As = Asm + (kt % HST) * HA_STAGE;
    const double* Bs = Bsm + (kt % HST) * B_ST;
#pragma unroll
    for (int kk = 0; kk < HBK / 8; ++kk) {
      const int k = 8 * kk + tq;
      double af[2][4], bf[NT][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int r = 32 * warp + 16 * mt + gq;
        if (AK) {
          af[mt][0] = As[r * HLD_K + k];
          af[mt][1] = As[(r + 8) * HLD_K + k];
          af[mt][2] = As[r * HLD_K + k + 4];
          af[mt][3] = As[(r + 8) * HLD_K + k + 4];
        } else {
          af[mt][0] = As[k * HLD_M + r];
          af[mt][1] = As[k * HLD_M + r + 8];
          af[mt][2] = As[(k + 4) * HLD_M + r];
          af[mt][3] = As[(k + 4) * HLD_M + r + 8];
        }
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        bf[nt][0] = Bs[(8 * nt + gq) * HLD_K + k];
        bf[nt][1] = Bs[(8 * nt + gq) * HLD_K + k + 4];
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_16x8x8(acc[mt][nt], af[mt], bf[nt]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int64_t row = i0 + 32 * warp + 16 * mt + gq + 8 * (c >> 1);
        const int64_t col = j0 + 8 * nt + 2 * tq + (c & 1);
        if (row < G.M && col < G.N) {
          double v = acc[mt][nt][c];
          if (G.partial) {
            G.C[(size_t)blockIdx.z * G.M * G.N + row + col * G.M] = v;
          } else {
            if (G.row_scale) v *= G.row_scale[row];
            if (G.addv) v += G.addv[row] * G.addm[row + col * G.ldadd];
            G.C[row + col * G.ldc] = v;
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// TMA-fed, warp-specialised DMMA GEMM (the sketch products at large M and K).  CTA tile
// 128 x (8 NT), BK = 16, TS-stage mbarrier ring; warp 4 is the producer, warps 0-3 the consumers
// (32 rows each, m16n8k8 f64 MMAs exactly as dgemm_nt_kernel).
//   * K-contiguous operands (B always; A when AK, i.e. A^T of a column-major matrix) arrive by
//     cp.async.bulk.tensor.2d (UTMALDG) with the 128-byte swizzle: a 16-double row of the box is
//     one 128-B line whose 16-B chunks are XOR-permuted by (row % 8), so the fragment loads (8 rows x
//     4 k per instruction) touch every bank at most twice — the 2-wavefront minimum of 256 B.
//     Out-of-range rows / columns are zero-filled by the tensor unit.
//   * an M-contiguous A (Y = A T) arrives as 16 one-dimensional bulk copies per stage (UBLKCP), one
//     per column segment, into rows padded to 136 doubles (conflict-free, as dgemm_nt_kernel).
// The consumers release a stage with one mbarrier arrive per warp; no __syncthreads in the loop.
// ------------------------------------------------------------------------------------------
constexpr int TS = 3;                                    // stages (3 CTAs of 68 KB per SM)
constexpr int TA_K_BYTES = HBM_ * HBK * 8;               // 16384: swizzled K-major A box
constexpr int TA_M_BYTES = HBK * HLD_M * 8;              // 17408: padded M-major A rows
constexpr int TA_BYTES = TA_M_BYTES;                     // the A slot (1 KB multiple: 17 KB)

__host__ __device__ constexpr int tma_b_bytes(int nt) { return ((8 * nt * HBK * 8 + 1023) / 1024) * 1024; }
__host__ __device__ constexpr int tma_stage_bytes(int nt) { return TA_BYTES + tma_b_bytes(nt); }

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// element (row, k) of a swizzled [rows][16] fp64 box (k in 0..15)
__device__ __forceinline__ int swz(int row, int k) { return row * 16 + ((((k >> 1) ^ (row & 7)) << 1) | (k & 1)); }

template <int NT, bool AK>
__global__ void __launch_bounds__(160) dgemm_tma_kernel(const GemmParams G, const __grid_constant__ CUtensorMap mapA,
                                                        const __grid_constant__ CUtensorMap mapB) {
  constexpr int BN = 8 * NT;
  constexpr int STAGE = tma_stage_bytes(NT);
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  // the dynamic window's base is only guaranteed 16-B aligned: round up to the 1 KB the swizzle needs
  unsigned char* tsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + (size_t)TS * STAGE);
  uint64_t* empty = full + TS;
  const int64_t j0 = (int64_t)blockIdx.x * BN;
  const int64_t i0 = (int64_t)blockIdx.y * HBM_;
  const int64_t kbeg = (int64_t)blockIdx.z * G.kchunk;
  int64_t kend = kbeg + G.kchunk;
  if (kend > G.K) kend = G.K;
  const int nk = (kend > kbeg) ? (int)((kend - kbeg + HBK - 1) / HBK) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_mbar_init();
  }
  if (!AK) {   // stale-but-finite smem: padded rows / columns past K are never copied (their B is 0)
    double* z = reinterpret_cast<double*>(tsm);
    for (int e = threadIdx.x; e < TS * STAGE / 8; e += blockDim.x) z[e] = 0.0;
  }
  __syncthreads();

  if (warp == 4) {
    // ------------------------------ producer ------------------------------------------------
    const uint64_t pol = l2_evict_first_policy();
    int s = 0;
    uint32_t eph = 1u;
    for (int kt = 0; kt < nk; ++kt, ++s) {
      if (s == TS) { s = 0; eph ^= 1u; }
      if (kt >= TS) mbar_wait(&empty[s], eph);
      unsigned char* st = tsm + (size_t)s * STAGE;
      const int64_t k0 = kbeg + (int64_t)kt * HBK;
      int ncols = (int)((kend - k0) < HBK ? (kend - k0) : HBK);
      int64_t rows = G.M - i0;
      rows = rows > HBM_ ? HBM_ : rows;
      const uint32_t cbytes = (uint32_t)(((rows + 1) & ~int64_t(1)) * 8);
      const uint32_t abytes = AK ? (uint32_t)TA_K_BYTES : (uint32_t)ncols * cbytes;
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[s], abytes + (uint32_t)(BN * HBK * 8));
        if (AK) tma_load_2d(st, &mapA, (int)k0, (int)i0, &full[s]);
        tma_load_2d(st + TA_BYTES, &mapB, (int)k0, (int)j0, &full[s]);
      }
      __syncwarp();
      if (!AK && lane < ncols)
        bulk_g2s(st + (size_t)lane * HLD_M * 8, G.A + i0 + (k0 + lane) * G.lda, cbytes, &full[s], pol);
    }
    return;
  }
  // ------------------------------ consumers --------------------------------------------------
  const int gq = lane >> 2, tq = lane & 3;
  double acc[2][NT][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;
  int s = 0;
  uint32_t ph = 0;
  for (int kt = 0; kt < nk; ++kt) {
    mbar_wait(&full[s], ph);
    const double* As = reinterpret_cast<const double*>(tsm + (size_t)s * STAGE);
    const double* Bs = reinterpret_cast<const double*>(tsm + (size_t)s * STAGE + TA_BYTES);
#pragma unroll
    for (int kk = 0; kk < HBK / 8; ++kk) {
      const int k = 8 * kk + tq;
      double af[2][4], bf[NT][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int r = 32 * warp + 16 * mt + gq;
        if (AK) {
          af[mt][0] = As[swz(r, k)];
          af[mt][1] = As[swz(r + 8, k)];
          af[mt][2] = As[swz(r, k + 4)];
          af[mt][3] = As[swz(r + 8, k + 4)];
        } else {
          af[mt][0] = As[k * HLD_M + r];
          af[mt][1] = As[k * HLD_M + r + 8];
          af[mt][2] = As[(k + 4) * HLD_M + r];
          af[mt][3] = As[(k + 4) * HLD_M + r + 8];
        }
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        bf[nt][0] = Bs[swz(8 * nt + gq, k)];
        bf[nt][1] = Bs[swz(8 * nt + gq, k + 4)];
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_16x8x8(acc[mt][nt], af[mt], bf[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == TS) { s = 0; ph ^= 1u; }
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int64_t row = i0 + 32 * warp + 16 * mt + gq + 8 * (c >> 1);
        const int64_t col = j0 + 8 * nt + 2 * tq + (c & 1);
        if (row < G.M && col < G.N) {
          double v = acc[mt][nt][c];
          if (G.partial) {
            G.C[(size_t)blockIdx.z * G.M * G.N + row + col * G.M] = v;
          } else {
            if (G.row_scale) v *= G.row_scale[row];
            if (G.addv) v += G.addv[row] * G.addm[row + col * G.ldadd];
            G.C[row + col * G.ldc] = v;
          }
        }
      }
    }
  }
}

typedef void (*TmaKernel)(const GemmParams, const CUtensorMap, const CUtensorMap);
template <bool AK>
static TmaKernel tma_kernel(int nt) {
  switch (nt) {
    case 1: return dgemm_tma_kernel<1, AK>;
    case 2: return dgemm_tma_kernel<2, AK>;
    case 3: return dgemm_tma_kernel<3, AK>;
    case 4: return dgemm_tma_kernel<4, AK>;
    case 5: return dgemm_tma_kernel<5, AK>;
    case 6: return dgemm_tma_kernel<6, AK>;
    case 7: return dgemm_tma_kernel<7, AK>;
    default: return dgemm_tma_kernel<8, AK>;
  }
}

static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}
// 2-D fp64 tensor (inner extent d0 contiguous, d1 columns of stride ld doubles), box {16, rows}, 128-B swizzle
static bool make_map(CUtensorMap* map, const double* base, int64_t d0, int64_t d1, int64_t ld, int rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)d0, (cuuint64_t)d1};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)HBK, (cuuint32_t)rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

typedef void (*DgemmKernel)(const GemmParams);
template <bool AK>
static DgemmKernel nt_kernel(int nt) {
  switch (nt) {
    case 1: return dgemm_nt_kernel<1, AK>;
    case 2: return dgemm_nt_kernel<2, AK>;
    case 3: return dgemm_nt_kernel<3, AK>;
    case 4: return dgemm_nt_kernel<4, AK>;
    case 5: return dgemm_nt_kernel<5, AK>;
    case 6: return dgemm_nt_kernel<6, AK>;
    case 7: return dgemm_nt_kernel<7, AK>;
    default: return dgemm_nt_kernel<8, AK>;
  }
}
// pick NT (1..8) minimising the padded width ceil(N / 8NT) * 8NT, ties -> larger NT
// least padded width over NT in [2, 7], ties -> the smaller NT (NT = 1 only for N <= 8).  Measured on B200
// (tools/gemm_vs_cublas.py with NYS_GEMM_NT, ms per sketch pair): NT = 1 re-reads the A tile once per
// 8-column tile and NT = 8 holds 64 accumulators per thread — both the slowest at every width tried
// (l = 100: NT 1..8 = 0.922 0.841 0.843 0.886 0.835 0.991 0.847 0.892; l = 128: NT 2 2.07, NT 8 2.61;
// l = 256: NT 3 3.41, NT 8 3.92) while the exact fits NT = 7 (l = 50) and NT = 5 (l = 200, the headline
// 61.0 ms vs 64.8-72.9 for NT 2, 3, 4, 7) stay
static int pick_nt(int64_t N) {
  if (const char* e = getenv("NYS_GEMM_NT")) {   // tuning override (1..8)
    const int o = atoi(e);
    if (o >= 1 && o <= 8) return o;
  }
  if (N <= 8) return 1;
  int best = 2;
  int64_t best_w = ((N + 15) / 16) * 16;
  for (int nt = 3; nt <= 7; ++nt) {
    const int64_t w = ((N + 8 * nt - 1) / (8 * nt)) * (8 * nt);
    if (w < best_w) { best_w = w; best = nt; }
  }
  return best;
}

__global__ void gemm_reduce_kernel(int64_t M, int64_t N, int splits, const double* P, double* C, int64_t ldc,
                                   const double* row_scale, const double* addv, const double* addm, int64_t ldadd) {
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e % M, col = e / M;
    double v = 0.0;
    for (int s = 0; s < splits; ++s) v += P[(size_t)s * total + e];
    if (row_scale) v *= row_scale[row];
    if (addv) v += addv[row] * addm[row + col * ldadd];
    C[row + col * ldc] = v;
  }
}

static int launch_gemm_old(nys_ctx* ctx, const GemmCall& g);

// K = 0 (a rank with no columns): C = the epilogue's additive term only (addv o addm, else 0)
__global__ void gemm_k0_kernel(int64_t M, int64_t N, double* C, int64_t ldc, const double* addv, const double* addm,
                               int64_t ldadd) {
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e % M, col = e / M;
    C[row + col * ldc] = addv ? addv[row] * addm[row + col * ldadd] : 0.0;
  }
}

// tuning override of the split-K count (per operand layout: K-major A, i.e. T = A^T Omega, or M-major
// A, i.e. Y = A T): NYS_GEMM_SPLITS_K / NYS_GEMM_SPLITS_M, read per call
static int split_override(const GemmCall& g) {
  const char* e = getenv(g.a_kmajor ? "NYS_GEMM_SPLITS_K" : "NYS_GEMM_SPLITS_M");
  return e ? atoi(e) : 0;
}

int launch_gemm(nys_ctx* ctx, const GemmCall& g) {
  if (g.M <= 0 || g.N <= 0) return NYS_OK;
  if (g.K <= 0) {
    int64_t blocks = (g.M * g.N + 255) / 256;
    if (blocks > 4 * ctx->num_sms) blocks = 4 * ctx->num_sms;
    gemm_k0_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(g.M, g.N, g.C, g.ldc, g.addv, g.addm, g.ldadd);
    ctx->launches++;
    return ctx->check_launch("gemm_k0");
  }
  // the 128-row kernel pays off on the sketch products once both M and K reach ~1000 (measured on
  // B200, tools/gemm_sweep.py: config-1 sketch 196 -> 165-177 us, config-2 shape 955 -> 892-912 us,
  // 20000 x 5000 x 300 4280 -> 3989-4002 us); short products (the Gram and small factorisation GEMMs,
  // config 3's K = 64 / M = 64 sketch) keep the 64 x 64 kernel.  Tuning override NYS_GEMM_NT_MIN="M,K".
  int64_t min_m = 512, min_k = 1024;
  if (const char* e = getenv("NYS_GEMM_NT_MIN")) {
    long long a = 0, b = 0;
    if (sscanf(e, "%lld,%lld", &a, &b) == 2) { min_m = a; min_k = b; }
  }
  if (g.M < min_m || g.K < min_k || getenv("NYS_GEMM_OLD")) return launch_gemm_old(ctx, g);
  const int NT = pick_nt(g.N);
  const int BN = 8 * NT;
  // TMA path (default): tensor maps over A (K-major case) and B; the cp.async kernel stays as the
  // fallback for operands the tensor unit cannot address (odd leading dimensions, misalignment) and
  // as an A/B switch (NYS_GEMM_CPASYNC)
  CUtensorMap mapA{}, mapB{};
  // the TMA kernel from M K >= 2.5e7 (config-1 sketch, M K = 1.6e7: the cp.async kernel, 165 vs 173 us)
  bool tma = getenv("NYS_GEMM_CPASYNC") == nullptr && (double)g.M * (double)g.K >= 2.5e7 &&
             (g.lda % 2) == 0 && (g.ldb % 2) == 0 &&
             aligned16(g.A) && aligned16(g.B) && g.K < (int64_t(1) << 31) && g.M < (int64_t(1) << 31);
  if (tma) {
    if (g.a_kmajor) tma = make_map(&mapA, g.A, g.K, g.M, g.lda, HBM_);
    tma = tma && make_map(&mapB, g.B, g.K, g.N, g.ldb, BN);
  }
  const size_t smem = tma ? (size_t)TS * tma_stage_bytes(NT) + 2 * TS * 8 + 1024
                          : (size_t)HST * (HA_STAGE + BN * HLD_K) * sizeof(double);
  DgemmKernel k = g.a_kmajor ? nt_kernel<true>(NT) : nt_kernel<false>(NT);
  TmaKernel kt = g.a_kmajor ? tma_kernel<true>(NT) : tma_kernel<false>(NT);
  NYS_TRY(ensure_max_smem(ctx, tma ? (const void*)kt : (const void*)k, smem));
  const int64_t mt = (g.M + HBM_ - 1) / HBM_, nt = (g.N + BN - 1) / BN;
  const int64_t kslabs = (g.K + HBK - 1) / HBK;
  int splits = g.splits > 0 ? g.splits : split_override(g);
  if (splits <= 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma ? (const void*)kt : (const void*)k, tma ? 160 : 128,
                                                      smem) != cudaSuccess) { cudaGetLastError(); occ = 0; }
    const int64_t slots = (int64_t)(occ > 0 ? occ : 2) * ctx->num_sms, tiles = mt * nt;
    const int64_t smax = kslabs / 8 > 0 ? kslabs / 8 : 1;
    int64_t sp = 1;
    if (tiles < slots) {
      // few tiles: split K so that tiles x S fits ONE wave of the resident slots (a split that spills a
      // few CTAs into a second wave nearly doubles the time: config-1 Y = A T, 16 tiles, S = 19 on 296
      // slots: 0.194 ms for the sketch pair, S = 18: 0.165), at most 16 (the S M N partials and their
      // reduce grow with S: config-2 shape T = A^T Omega, 16 tiles: S = 27 0.924 ms, 16 0.871, 8 0.886)
      sp = slots / tiles;
      if (sp > smax) sp = smax;
      if (sp > 16) sp = 16;
      if (sp < 1) sp = 1;
    } else if (!getenv("NYS_GEMM_NO_WAVE_SPLIT")) {
      // many tiles: split K only to fill the last wave.  Time ~ ceil(tiles * S / slots) / S (equal
      // tiles); the smallest S (<= 4, >= 64 K-slabs per split) within 1 % of the best, if that gains
      // >= 3 % over S = 1.  Measured on B200, the config-4 sketch (1955 tiles, 444 slots, 4.4 waves): the
      // unsplit GEMM ran 0.84 of the DMMA peak with the SM pipes 84 % busy — the last wave's idle SMs
      auto cost = [&](int64_t S) { return (double)((tiles * S + slots - 1) / slots) / (double)S; };
      double best = cost(1);
      for (int64_t S = 2; S <= 4 && kslabs / S >= 64; ++S) best = std::min(best, cost(S));
      if (cost(1) > best * 1.03)   // a split costs partials (S M N doubles) and a reduce: only for >= 3 %
        for (int64_t S = 2; S <= 4 && kslabs / S >= 64; ++S)
          if (cost(S) <= best * 1.01) { sp = S; break; }
    }
    splits = (int)sp;
  }
  int64_t kchunk = (g.K + splits - 1) / splits;
  kchunk = ((kchunk + HBK - 1) / HBK) * HBK;
  if (kchunk < HBK) kchunk = HBK;
  splits = (int)((g.K + kchunk - 1) / kchunk);
  if (splits < 1) splits = 1;
  GemmParams P{};
  P.M = g.M; P.N = g.N; P.K = g.K; P.A = g.A; P.lda = g.lda; P.B = g.B; P.ldb = g.ldb;
  P.row_scale = g.row_scale; P.addv = g.addv; P.addm = g.addm; P.ldadd = g.ldadd; P.kchunk = kchunk;
  double* part = nullptr;
  if (splits > 1) {
    part = ctx->wsd("gemm_part", (size_t)splits * g.M * g.N);
    P.C = part; P.ldc = g.M; P.partial = 1;
  } else {
    P.C = g.C; P.ldc = g.ldc; P.partial = 0;
  }
  if (mt > 65535) { ctx->set_error("dgemm: M too large for the grid"); return NYS_EINVAL; }
  dim3 grid((unsigned)nt, (unsigned)mt, (unsigned)splits);
  if (tma) kt<<<grid, 160, smem, ctx->stream>>>(P, mapA, mapB);
  else k<<<grid, 128, smem, ctx->stream>>>(P);
  ctx->launches++;
  NYS_TRY(ctx->check_launch("dgemm"));
  if (splits > 1) {
    int64_t tot = g.M * g.N;
    int rg = (int)((tot + 255) / 256);
    if (rg > 4 * ctx->num_sms) rg = 4 * ctx->num_sms;
    gemm_reduce_kernel<<<rg, 256, 0, ctx->stream>>>(g.M, g.N, splits, part, g.C, g.ldc, g.row_scale, g.addv, g.addm,
                                                     g.ldadd);
    ctx->launches++;
    NYS_TRY(ctx->check_launch("gemm_reduce"));
  }
  return NYS_OK;
}

static int launch_gemm_old(nys_ctx* ctx, const GemmCall& g) {
  const size_t smem = (size_t)GST * (A_STAGE + B_STAGE) * sizeof(double);
  if (g.a_kmajor) NYS_TRY(ensure_max_smem(ctx, (const void*)dgemm_kernel<true>, smem));
  else NYS_TRY(ensure_max_smem(ctx, (const void*)dgemm_kernel<false>, smem));
  const int64_t mt = (g.M + GBM - 1) / GBM, nt = (g.N + GBN - 1) / GBN;
  const int64_t kslabs = (g.K + GBK - 1) / GBK;
  int splits = g.splits > 0 ? g.splits : split_override(g);
  if (splits <= 0) {
    const int64_t target = 3LL * ctx->num_sms;
    int64_t s = (target + mt * nt - 1) / (mt * nt);
    const int64_t smax = kslabs / 8 > 0 ? kslabs / 8 : 1;
    if (s > smax) s = smax;
    if (s < 1) s = 1;
    if (s > 256) s = 256;
    splits = (int)s;
  }
  int64_t kchunk = (g.K + splits - 1) / splits;
  kchunk = ((kchunk + GBK - 1) / GBK) * GBK;
  if (kchunk < GBK) kchunk = GBK;
  splits = (int)((g.K + kchunk - 1) / kchunk);
  if (splits < 1) splits = 1;
  GemmParams P{};
  P.M = g.M; P.N = g.N; P.K = g.K; P.A = g.A; P.lda = g.lda; P.B = g.B; P.ldb = g.ldb;
  P.row_scale = g.row_scale; P.addv = g.addv; P.addm = g.addm; P.ldadd = g.ldadd; P.kchunk = kchunk;
  double* part = nullptr;
  if (splits > 1) {
    part = ctx->wsd("gemm_part", (size_t)splits * g.M * g.N);
    P.C = part; P.ldc = g.M; P.partial = 1;
  } else {
    P.C = g.C; P.ldc = g.ldc; P.partial = 0;
  }
  if (mt > 65535) { ctx->set_error("dgemm: M too large for the grid"); return NYS_EINVAL; }
  dim3 grid((unsigned)nt, (unsigned)mt, (unsigned)splits);
  if (g.K <= 0) {
    // empty contraction: C = 0 (+ add)
    NYS_CUDA_TRY(ctx, cudaMemsetAsync(part ? part : g.C, 0, 0, ctx->stream));
  }
  if (g.a_kmajor)
    dgemm_kernel<true><<<grid, 128, smem, ctx->stream>>>(P);
  else
    dgemm_kernel<false><<<grid, 128, smem, ctx->stream>>>(P);
  ctx->launches++;
  NYS_TRY(ctx->check_launch("dgemm"));
  if (splits > 1) {
    int64_t tot = g.M * g.N;
    int rg = (int)((tot + 255) / 256);
    if (rg > 4 * ctx->num_sms) rg = 4 * ctx->num_sms;
    gemm_reduce_kernel<<<rg, 256, 0, ctx->stream>>>(g.M, g.N, splits, part, g.C, g.ldc, g.row_scale, g.addv, g.addm,
                                                     g.ldadd);
    ctx->launches++;
    NYS_TRY(ctx->check_launch("gemm_reduce"));
  }
  return NYS_OK;
}

}  // namespace nys
