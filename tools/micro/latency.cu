// Dependent-chain latencies of the scalar operations on the CPQR's critical
// path (one warp, clock64), to size the skeleton kernels' per-step latency.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  double x = x0 + threadIdx.x * 1e-12;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + 1e-9;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
  // division chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0000001 / x;
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / n;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / n;
  // hypot chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = hypot(x, 0.5) * 0.5;
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
  // shuffle + add chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1) * 1e-9;
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / n;
  // dependent LDS chain (pointer chasing via value)
  int idx = threadIdx.x & 7;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = ((int)(v * 1e9) + i) & 1023; x += v; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / n;
  // rsqrt-based (MUFU) reciprocal sqrt approx chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 2.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0) / n;
  // __syncthreads cost (one warp)
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) cyc[8] = (t1 - t0) / n;
  // float FMA chain for comparison
  float f = (float)x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = fmaf(f, 0.999f, 1e-3f);
  t1 = clock64(); if (threadIdx.x == 0) cyc[9] = (t1 - t0) / n;
  out[threadIdx.x] = x + f;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 16 * 8);
  for (int nt : {32, 128, 512}) {
    lat<<<1, nt>>>(out, cyc, 1.5, 4096);
    cudaDeviceSynchronize();
    lat<<<1, nt>>>(out, cyc, 1.5, 4096);
    cudaDeviceSynchronize();
    printf("threads %4d: dfma %lld dadd %lld ddiv %lld dsqrt %lld hypot %lld shfl+fma %lld lds-chain %lld rsqrt %lld syncthreads %lld ffma %lld (cycles)\n",
           nt, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cyc[7], cyc[8], cyc[9]);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock %d kHz\n", clk);
  return 0;
}
