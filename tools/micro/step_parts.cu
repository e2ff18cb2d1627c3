// Cycle cost of the pieces of one pivoted-QR step (see cpqr_bench.cu), each
// repeated in a dependent loop by one CTA of 128 threads.
#include <cfloat>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double group_sum(double v, int G) {
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__global__ void parts(long long* cyc, double* out, int nc, int nq, int G) {
  __shared__ double vn[64];
  __shared__ int cat[64];
  __shared__ double M[40 * 100];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) { vn[i] = 1.0 + 0.001 * ((i * 37) % 64); cat[i] = (i * 5) % 64; }
  for (int i = threadIdx.x; i < 4000; i += blockDim.x) M[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int N = 1000;
  double sink = 0;
  long long t0, t1;
  // A: argmax (value, position, column) via 5 shuffle rounds
  t0 = clock64();
  for (int it = 0; it < N; ++it) {
    double bv = -1.0; int bp = nc, bc = 0;
    for (int pos = (it & 3) + lane; pos < nc; pos += 32) { const int c = cat[pos]; const double v = vn[c]; if (v > bv) { bv = v; bp = pos; bc = c; } }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; bc = oc; }
    }
    sink += bv + bc; vn[(bc + it) & 63] += 1e-12;  // keep the loop dependent
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
  // B: householder scalars
  double alpha = 0.3, xnorm = 0.7;
  t0 = clock64();
  for (int it = 0; it < N; ++it) {
    double beta = -copysign(hypot(alpha, xnorm), alpha);
    double tau = (beta - alpha) / beta;
    double scal = 1.0 / (alpha - beta);
    alpha = 0.3 + 1e-9 * (tau + scal); sink += beta;
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / N;
  // C: dot over nq rows with G lanes per column + group reduction
  const int sl = lane & (G - 1);
  const double* v = M; double* col = M + 100 * ((lane / G) + 1);
  t0 = clock64();
  for (int it = 0; it < N; ++it) {
    const int i = it & 7;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int r = i + 1 + sl;
    for (; r + 3 * G < nq; r += 4 * G) { s0 += v[r] * col[r]; s1 += v[r + G] * col[r + G]; s2 += v[r + 2 * G] * col[r + 2 * G]; s3 += v[r + 3 * G] * col[r + 3 * G]; }
    for (; r < nq; r += G) s0 += v[r] * col[r];
    const double sd = group_sum((s0 + s1) + (s2 + s3), G);
    sink += sd; col[i] += 1e-15 * sd;
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / N;
  // D: downdate: 2 divisions + sqrt chain
  double nv = 2.0, v2 = 3.0, c = 0.5;
  t0 = clock64();
  for (int it = 0; it < N; ++it) {
    double tmp = fabs(c) / nv; tmp = 1.0 - tmp * tmp; tmp = tmp > 0 ? tmp : 0;
    const double ratio = nv / v2;
    if (tmp * ratio * ratio <= 1e-8) nv = sqrt(c * c + 1.0); else nv *= sqrt(tmp);
    nv += 1.0; sink += nv;
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / N;
  // E: __syncthreads round trip
  t0 = clock64();
  for (int it = 0; it < N; ++it) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / N;
  // F: packed-key argmax (64-bit) 5 rounds
  t0 = clock64();
  for (int it = 0; it < N; ++it) {
    unsigned long long key = 0;
    for (int pos = (it & 3) + lane; pos < nc; pos += 32) {
      const double vv = vn[cat[pos]];
      const unsigned long long kk = ((unsigned long long)__double_as_longlong(vv) & ~0xFFull) | (unsigned long long)(255 - pos);
      key = kk > key ? kk : key;
    }
    for (int o = 16; o > 0; o >>= 1) { const unsigned long long ok = (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)key, o); key = ok > key ? ok : key; }
    sink += (double)(key & 0xFF); vn[(key + it) & 63] += 1e-12;
  }
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / N;
  // G: one LDS dependent pair (cat -> vn)
  int idx = lane & 15;
  t0 = clock64();
  for (int it = 0; it < N; ++it) { const int cc = cat[idx]; const double vv = vn[cc & 63]; idx = ((int)vv + it) & 15; sink += vv; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / N;
  out[threadIdx.x] = sink;
}
int main() {
  long long* cyc; double* out;
  cudaMallocManaged(&cyc, 16 * 8); cudaMalloc(&out, 1024 * 8);
  for (int G : {8, 16, 32}) {
    parts<<<1, 128>>>(cyc, out, 15, 83, G); cudaDeviceSynchronize();
    parts<<<1, 128>>>(cyc, out, 15, 83, G); cudaDeviceSynchronize();
    printf("G %2d: argmax %lld  householder %lld  dot(nq=83) %lld  downdate %lld  syncthreads %lld  key-argmax %lld  lds-pair %lld  (%s)\n",
           G, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
