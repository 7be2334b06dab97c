// Dependent-chain latencies on the GPU (one warp): DFMA, DADD, MUFU rsqrt/rcp f64 seeds, SHFL f64,
// LDS f64, and one fast_rsqrt2 / jacobi rotation.  nvcc -arch=sm_100a -o lat_probe lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, double x0) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = x0 + lane; sm[lane + 32] = x0;
  __syncwarp();
  double x = x0 + lane * 1e-3;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 16; ++i) {
#pragma unroll
 for (int u = 0; u < 16; ++u) x = fma(x, 0.999999, 1e-9); }
  t1 = clock64(); if (lane == 0) cyc[0] = (t1 - t0); out[lane] = x;
  // DADD chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 16; ++i) {
#pragma unroll
 for (int u = 0; u < 16; ++u) x = x + 1e-9 * u; }
  t1 = clock64(); if (lane == 0) cyc[1] = (t1 - t0); out[lane] += x;
  // MUFU rsqrt f64 chain
  double y = 1.5 + lane;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 16; ++i) {
#pragma unroll
 for (int u = 0; u < 16; ++u) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y)); y = r + 1.0; } }
  t1 = clock64(); if (lane == 0) cyc[2] = (t1 - t0); out[lane] += y;
  // MUFU rcp f64 chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 16; ++i) {
#pragma unroll
 for (int u = 0; u < 16; ++u) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y)); y = r + 1.0; } }
  t1 = clock64(); if (lane == 0) cyc[3] = (t1 - t0); out[lane] += y;
  // SHFL f64 + add chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 16; ++i) {
#pragma unroll
 for (int u = 0; u < 16; ++u) y += __shfl_xor_sync(0xffffffffu, y, 1 + u); }
  t1 = clock64(); if (lane == 0) cyc[4] = (t1 - t0); out[lane] += y;
  // LDS f64 pointer-chase-like chain (index depends on loaded value)
  int idx = lane;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 16; ++i) {
#pragma unroll
 for (int u = 0; u < 16; ++u) { double v = sm[idx]; idx = ((int)v + u) & 63; } }
  t1 = clock64(); if (lane == 0) cyc[5] = (t1 - t0); out[lane] += idx;
  // FP32 FMA chain
  float f = (float)x0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 16; ++i) {
#pragma unroll
 for (int u = 0; u < 16; ++u) f = fmaf(f, 0.999f, 1e-6f); }
  t1 = clock64(); if (lane == 0) cyc[6] = (t1 - t0); out[lane] += f;
  // double sqrt (IEEE) chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
#pragma unroll
 for (int u = 0; u < 16; ++u) y = sqrt(y) + 1.0; }
  t1 = clock64(); if (lane == 0) cyc[7] = (t1 - t0) * 4; out[lane] += y;
  // double division chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
#pragma unroll
 for (int u = 0; u < 16; ++u) y = 1.0 / y + 1.0; }
  t1 = clock64(); if (lane == 0) cyc[8] = (t1 - t0) * 4; out[lane] += y;
  // __syncthreads alone (1 warp)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 16; ++i) {
#pragma unroll
 for (int u = 0; u < 16; ++u) __syncthreads(); }
  t1 = clock64(); if (lane == 0) cyc[9] = (t1 - t0);
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 16 * 8);
  probe<<<1, 32>>>(o, c, 1.25);
  probe<<<1, 32>>>(o, c, 1.25);
  long long h[16];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[] = {"DFMA", "DADD", "MUFU.RSQ64(+DADD)", "MUFU.RCP64(+DADD)", "SHFL+DADD", "LDS(+cvt,iadd)", "FFMA32",
                      "sqrt f64 (+DADD)", "div f64 (+DADD)", "__syncthreads 1 warp"};
  for (int i = 0; i < 10; ++i) printf("%-24s %.1f cycles per dependent step\n", nm[i], h[i] / 256.0);
  return 0;
}
