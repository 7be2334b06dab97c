// DMMA shape probe: fragment layout check + throughput for mma.sync f64 m16n8k{4,8,16} on sm_100a
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int K>
__device__ __forceinline__ void mma(double (&c)[4], const double (&a)[K / 2], const double (&b)[K / 4]);

template <>
__device__ __forceinline__ void mma<4>(double (&c)[4], const double (&a)[2], const double (&b)[1]) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
template <>
__device__ __forceinline__ void mma<8>(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]),
                 "d"(b[0]), "d"(b[1]));
}
template <>
__device__ __forceinline__ void mma<16>(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, "
      "{%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]),
        "d"(b[2]), "d"(b[3]));
}

// hypothesised layouts: A element i: row = g + 8*(i&1), col = t + 4*(i>>1);  B element i: k = t + 4*i, n = g
// (for K=4: A i in {0,1}: row g / g+8, col t; B: k = t, n = g)
template <int K>
__global__ void check(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[K / 2], b[K / 4], c[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < K / 2; ++i) a[i] = A[(g + 8 * (i & 1)) * K + t + 4 * (i >> 1)];
#pragma unroll
  for (int i = 0; i < K / 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  mma<K>(c, a, b);
  // C: c0,c1 row g cols 2t,2t+1 ; c2,c3 row g+8
  C[g * 8 + 2 * t] = c[0];
  C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2];
  C[(g + 8) * 8 + 2 * t + 1] = c[3];
}

template <int K>
__global__ void bench(double* out, int iters) {
  double a[K / 2], b[K / 4];
#pragma unroll
  for (int i = 0; i < K / 2; ++i) a[i] = 1e-3 * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < K / 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  double c[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) c[j][q] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) mma<K>(c[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) s += c[j][q];
  if (s == 12345.678) out[0] = s;
}

template <int K>
void run() {
  double hA[16 * K], hB[K * 8], hC[128], ref[128];
  for (int i = 0; i < 16 * K; ++i) hA[i] = (double)(rand() % 17 - 8);
  for (int i = 0; i < K * 8; ++i) hB[i] = (double)(rand() % 13 - 6);
  for (int r = 0; r < 16; ++r)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += hA[r * K + k] * hB[k * 8 + n];
      ref[r * 8 + n] = s;
    }
  double *dA, *dB, *dC;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dC, sizeof(hC));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  check<K><<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, sizeof(hC), cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 128; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    bench<K><<<148 * 2, 32 * warps>>>(dC, 100);
    cudaEventRecord(e0);
    bench<K><<<148 * 2, 32 * warps>>>(dC, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16 * 8 * K * 8.0 * iters * 32.0 * warps * 148 * 2 / 32.0;
    printf("K=%d layout_err=%g warps/CTA=%d (2 CTA/SM): %.2f TFLOP/s\n", K, err, warps, flops / (ms * 1e-3) / 1e12);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<4>();
  run<8>();
  run<16>();
  return 0;
}
