// FP64 FMA throughput of ONE SM on the CUDA cores (no tensor pipe): 1 CTA, T threads, 8 independent
// chains per thread.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_rate dfma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int iters) {
  double a[8];
  for (int u = 0; u < 8; ++u) a[u] = threadIdx.x * 1e-3 + u;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = fma(a[u], 0.9999999, 1e-7);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int u = 0; u < 8; ++u) s += a[u];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
  for (int T : {128, 256, 512, 1024}) {
    const int iters = 4096;
    k<<<1, T>>>(o, c, iters); k<<<1, T>>>(o, c, iters);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("T=%4d: %.1f DFMA per clock per SM\n", T, (double)T * 8 * iters / h);
  }
  return 0;
}
