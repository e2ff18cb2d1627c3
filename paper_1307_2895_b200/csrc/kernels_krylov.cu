// Device-resident preconditioned CG (the reference's pcg, src/krylov.py:48-77)
// with the GPU factor as preconditioner: CSR SpMV, deterministic two-stage
// dot products (fixed grid, fixed summation order) and fused vector updates.
// Scalars live on the device; the host reads one residual per iteration.
#include <cstdint>

#include "hifde_internal.h"

namespace hifde {

namespace {
constexpr int kDotBlocks = 296;  // 2 x 148 SMs
constexpr int kDotThreads = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[kDotThreads / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  v = 0.0;
  if (threadIdx.x < kDotThreads / 32) v = red[threadIdx.x];
  if (wid == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // valid in thread 0
}
}  // namespace

// y = A x (CSR, one thread per row)
__global__ void spmv_kernel(const int64_t* __restrict__ ip, const int32_t* __restrict__ ix,
                            const double* __restrict__ va, const double* __restrict__ x, double* __restrict__ y,
                            int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t k = ip[i]; k < ip[i + 1]; ++k) s += va[k] * x[ix[k]];
  y[i] = s;
}

// partial[b] = sum over this block's grid-stride slice of a .* c
__global__ void __launch_bounds__(kDotThreads) dot_partial_kernel(const double* __restrict__ a,
                                                                  const double* __restrict__ c, int64_t n,
                                                                  double* __restrict__ partial) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kDotThreads)
    s += a[i] * c[i];
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// out = sum(partial[0..nb)) in a fixed order
__global__ void __launch_bounds__(kDotThreads) dot_final_kernel(const double* __restrict__ partial, int nb,
                                                                double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += kDotThreads) s += partial[i];
  s = block_sum(s);
  if (threadIdx.x == 0) *out = s;
}

// sc = {rz, pAp, rr, rz_new}: alpha = rz / pAp; x += alpha p; r -= alpha ap
__global__ void cg_xr_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                             const double* __restrict__ ap, const double* __restrict__ sc, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double alpha = sc[0] / sc[1];
  x[i] += alpha * p[i];
  r[i] -= alpha * ap[i];
}

// beta = rz_new / rz; p = z + beta p; rz <- rz_new (one thread after the grid)
__global__ void cg_p_kernel(double* __restrict__ p, const double* __restrict__ z, const double* __restrict__ sc,
                            int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double beta = sc[3] / sc[0];
  p[i] = z[i] + beta * p[i];
}
__global__ void cg_shift_kernel(double* sc) { sc[0] = sc[3]; }

// z = x - y
__global__ void sub_kernel(double* __restrict__ z, const double* __restrict__ x, const double* __restrict__ y,
                           int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) z[i] = x[i] - y[i];
}
// x = y / sqrt(*nn)   (nn = ||y||^2 on the device)
__global__ void scale_kernel(double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ nn,
                             int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = y[i] / sqrt(*nn);
}

void launch_spmv(const int64_t* ip, const int32_t* ix, const double* va, const double* x, double* y, int64_t n,
                 cudaStream_t s) {
  if (n > 0) spmv_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ip, ix, va, x, y, n);
}
void launch_dot(const double* a, const double* c, int64_t n, double* partial, double* out, cudaStream_t s) {
  dot_partial_kernel<<<kDotBlocks, kDotThreads, 0, s>>>(a, c, n, partial);
  dot_final_kernel<<<1, kDotThreads, 0, s>>>(partial, kDotBlocks, out);
}
int dot_partials() { return kDotBlocks; }
void launch_cg_xr(double* x, double* r, const double* p, const double* ap, const double* sc, int64_t n,
                  cudaStream_t s) {
  if (n > 0) cg_xr_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, r, p, ap, sc, n);
}
void launch_cg_p(double* p, const double* z, double* sc, int64_t n, cudaStream_t s) {
  if (n > 0) cg_p_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, z, sc, n);
  cg_shift_kernel<<<1, 1, 0, s>>>(sc);
}

void launch_sub(double* z, const double* x, const double* y, int64_t n, cudaStream_t s) {
  if (n > 0) sub_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(z, x, y, n);
}
void launch_scale(double* x, const double* y, const double* nn, int64_t n, cudaStream_t s) {
  if (n > 0) scale_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, y, nn, n);
}

}  // namespace hifde
