// Issue-rate peak of the FP64 tensor pipe as this library uses it:
// mma.sync.aligned.m8n8k4.f64 (SASS DMMA.8x8x4) on register operands, NACC
// independent accumulator chains per warp, every SM full.  Prints JSON.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_peak dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void __launch_bounds__(256) k(double* out, int iters, double a0, double b0) {
  double c[NACC][2];
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0.0;
  const double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NACC>
double run(int nsm, int ctas_per_sm, int iters) {
  double* out;
  cudaMalloc(&out, sizeof(double) * nsm * ctas_per_sm * 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<NACC><<<nsm * ctas_per_sm, 256>>>(out, iters / 10, 1.0, 1.0);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<NACC><<<nsm * ctas_per_sm, 256>>>(out, iters, 1.0, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaFree(out);
  const double flops = 2.0 * 8 * 8 * 4 * (double)NACC * iters * 8 /*warps*/ * nsm * ctas_per_sm;
  return flops / (best * 1e-3) / 1e12;
}
int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  printf("{\"instruction\": \"mma.sync.aligned.m8n8k4.f64 (DMMA.8x8x4)\", \"sms\": %d, \"tflops\": {", nsm);
  printf("\"1 chain x 8 warps\": %.2f, ", run<1>(nsm, 1, iters));
  printf("\"4 chains x 8 warps\": %.2f, ", run<4>(nsm, 1, iters));
  printf("\"8 chains x 8 warps\": %.2f, ", run<8>(nsm, 1, iters));
  printf("\"8 chains x 16 warps\": %.2f, ", run<8>(nsm, 2, iters));
  printf("\"8 chains x 32 warps\": %.2f", run<8>(nsm, 4, iters));
  printf("}, \"how\": \"register operands, independent accumulator chains per warp, best of 5, CUDA events\"}\n");
  return 0;
}
