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
static int pick_nt(int64_t N) {
  int best = 8;
  int64_t best_w = ((N + 63) / 64) * 64;
  for (int nt = 7; nt >= 1; --nt) {
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

int launch_gemm(nys_ctx* ctx, const GemmCall& g) {
  if (g.M <= 0 || g.N <= 0) return NYS_OK;
  if (g.K <= 0) {
    int64_t blocks = (g.M * g.N + 255) / 256;
    if (blocks > 4 * ctx->num_sms) blocks = 4 * ctx->num_sms;
    gemm_k0_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(g.M, g.N, g.C, g.ldc, g.addv, g.addm, g.ldadd);
    ctx->launches++;
    return ctx->check_launch("gemm_k0");
  }
  // the 128-row kernel pays off on tall products (the sketch at large n or m); short-M products
  // (split-K Gram / Y = A T at small m) keep the 64 x 64 kernel (measured on B200)
  int64_t min_m = 16384, min_k = 4096;   // tuning overrides: NYS_GEMM_NT_MIN="M,K"
  if (const char* e = getenv("NYS_GEMM_NT_MIN")) {
    long long a = 0, b = 0;
    if (sscanf(e, "%lld,%lld", &a, &b) == 2) { min_m = a; min_k = b; }
  }
  if (g.M < min_m || g.K < min_k || getenv("NYS_GEMM_OLD")) return launch_gemm_old(ctx, g);
  const int NT = pick_nt(g.N);
  const int BN = 8 * NT;
  const size_t smem = (size_t)HST * (HA_STAGE + BN * HLD_K) * sizeof(double);
  DgemmKernel k = g.a_kmajor ? nt_kernel<true>(NT) : nt_kernel<false>(NT);
  NYS_TRY(ensure_max_smem(ctx, (const void*)k, smem));
  const int64_t mt = (g.M + HBM_ - 1) / HBM_, nt = (g.N + BN - 1) / BN;
  const int64_t kslabs = (g.K + HBK - 1) / HBK;
  int splits = g.splits;
  if (splits <= 0) {
    const int64_t target = 2LL * ctx->num_sms;
    int64_t sp = (target + mt * nt - 1) / (mt * nt);
    const int64_t smax = kslabs / 8 > 0 ? kslabs / 8 : 1;
    if (sp > smax) sp = smax;
    if (sp < 1) sp = 1;
    if (sp > 256) sp = 256;
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
  k<<<grid, 128, smem, ctx->stream>>>(P);
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
  int splits = g.splits;
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
