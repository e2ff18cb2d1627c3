// sm_100a kernels of the HIF-DE solve sweep (apply_inverse, src/driver.py:113-129).
//
// The factor is held in Cholesky form: per elimination record C (lower,
// C C^T = A_cc) and W = C^-1 A_cq, i.e. the reference's L = C diag(C)^-1,
// D = diag(C)^2, X = diag(C)^-1 W (src/factor_ops.py:29-75).  Then
//   forward  (apply_st + solve_d): s = C^-1 v_c ; v_q -= W^T s ; v_c = s
//   backward (apply_s)           : v_c = C^-T (v_c - W v_q)
// which composes to the same F^-1 as the reference's L/D/L^T sweeps.  The
// right-hand-side block v is N x nrhs row-major.  Elimination records of one
// level share neighbour DOFs, so their v_q updates are written to a
// contribution buffer and summed per DOF in record order by a second kernel
// (deterministic, no atomics).
#include <cstdint>

#include "hifde_internal.h"

namespace hifde {

namespace {

constexpr int NT = kThreads;

// x (n x nrhs, row-major) <- C^{-1} x, C lower n x n row-major.  One barrier
// per row: row i's scaling by 1/C_ii is deferred to the next step.
__device__ void fwd_subst(const double* __restrict__ C, int n, double* x, int nrhs) {
  double prev = 0.0;
  for (int i = 0; i < n; ++i) {
    __syncthreads();
    const double cinv = 1.0 / C[(size_t)i * n + i];
    if (i > 0)
      for (int r = threadIdx.x; r < nrhs; r += NT) x[(size_t)(i - 1) * nrhs + r] *= prev;
    const int rows = n - i - 1;
    for (int e = threadIdx.x; e < rows * nrhs; e += NT) {
      const int l = i + 1 + e / nrhs, r = e - (e / nrhs) * nrhs;
      x[(size_t)l * nrhs + r] -= C[(size_t)l * n + i] * (x[(size_t)i * nrhs + r] * cinv);
    }
    prev = cinv;
  }
  __syncthreads();
  if (n > 0)
    for (int r = threadIdx.x; r < nrhs; r += NT) x[(size_t)(n - 1) * nrhs + r] *= prev;
  __syncthreads();
}

// x <- C^{-T} x (same deferred-scaling scheme, bottom-up).
__device__ void bwd_subst(const double* __restrict__ C, int n, double* x, int nrhs) {
  double prev = 0.0;
  for (int i = n - 1; i >= 0; --i) {
    __syncthreads();
    const double cinv = 1.0 / C[(size_t)i * n + i];
    if (i < n - 1)
      for (int r = threadIdx.x; r < nrhs; r += NT) x[(size_t)(i + 1) * nrhs + r] *= prev;
    for (int e = threadIdx.x; e < i * nrhs; e += NT) {
      const int l = e / nrhs, r = e - l * nrhs;
      x[(size_t)l * nrhs + r] -= C[(size_t)i * n + l] * (x[(size_t)i * nrhs + r] * cinv);
    }
    prev = cinv;
  }
  __syncthreads();
  if (n > 0)
    for (int r = threadIdx.x; r < nrhs; r += NT) x[r] *= prev;
  __syncthreads();
}

// y = P x and y = P^T x for the packed lower inverse P (n x n) and x n x nrhs.
__device__ void pinv_apply(const double* __restrict__ P, int n, const double* x, double* y, int nrhs) {
  for (int e = threadIdx.x; e < n * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    const double* row = P + (size_t)i * (i + 1) / 2;
    double s = 0.0;
    for (int l = 0; l <= i; ++l) s += row[l] * x[(size_t)l * nrhs + r];
    y[e] = s;
  }
}
__device__ void pinv_apply_t(const double* __restrict__ P, int n, const double* x, double* y, int nrhs) {
  for (int e = threadIdx.x; e < n * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    double s = 0.0;
    for (int l = i; l < n; ++l) s += P[(size_t)l * (l + 1) / 2 + i] * x[(size_t)l * nrhs + r];
    y[e] = s;
  }
}

__device__ __forceinline__ double* workspace(double* smem, double* scratch, int64_t per_rec) {
  return per_rec > 0 ? scratch + (size_t)blockIdx.x * per_rec : smem;
}

}  // namespace

__global__ void __launch_bounds__(NT) solve_elim_fwd_kernel(
    const SolveRec* __restrict__ recs, const int32_t* __restrict__ idx, const double* __restrict__ fac,
    double* __restrict__ v, int nrhs, double* __restrict__ contrib, double* scratch, int64_t per_rec) {
  extern __shared__ __align__(16) double sm[];
  const SolveRec rc = recs[blockIdx.x];
  const int nc = rc.nc, nq = rc.nq;
  double* s = workspace(sm, scratch, per_rec);
  double* s2 = s + (size_t)nc * nrhs;
  const int32_t* c = idx + rc.idx_off;
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    s[e] = v[(size_t)c[i] * nrhs + r];
  }
  if (rc.inv) {
    __syncthreads();
    pinv_apply(fac + rc.C_off, nc, s, s2, nrhs);
    __syncthreads();
    s = s2;
  } else {
    fwd_subst(fac + rc.C_off, nc, s, nrhs);
  }
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    v[(size_t)c[i] * nrhs + r] = s[e];
  }
  if (nq > 0) {
    const double* W = fac + rc.W_off;
    for (int e = threadIdx.x; e < nq * nrhs; e += NT) {
      const int a = e / nrhs, r = e - a * nrhs;
      double g = 0.0;
      for (int k = 0; k < nc; ++k) g += W[(size_t)k * nq + a] * s[(size_t)k * nrhs + r];
      contrib[(size_t)(rc.contrib_off + a) * nrhs + r] = g;
    }
  }
}

__global__ void solve_reduce_kernel(const int32_t* __restrict__ targets, const int64_t* __restrict__ ptr,
                                    const int64_t* __restrict__ ent, int ntargets,
                                    const double* __restrict__ contrib, double* __restrict__ v,
                                    int nrhs) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ntargets * nrhs) return;
  const int t = (int)(e / nrhs), r = (int)(e % nrhs);
  double acc = 0.0;
  for (int64_t p = ptr[t]; p < ptr[t + 1]; ++p) acc += contrib[(size_t)ent[p] * nrhs + r];
  v[(size_t)targets[t] * nrhs + r] -= acc;
}

__global__ void __launch_bounds__(NT) solve_elim_bwd_kernel(
    const SolveRec* __restrict__ recs, const int32_t* __restrict__ idx, const double* __restrict__ fac,
    double* __restrict__ v, int nrhs, double* scratch, int64_t per_rec) {
  extern __shared__ __align__(16) double sm[];
  const SolveRec rc = recs[blockIdx.x];
  const int nc = rc.nc, nq = rc.nq;
  double* t = workspace(sm, scratch, per_rec);
  const int32_t* c = idx + rc.idx_off;
  const int32_t* q = c + nc;
  const double* W = fac + rc.W_off;
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    double a = v[(size_t)c[i] * nrhs + r];
    for (int b = 0; b < nq; ++b) a -= W[(size_t)i * nq + b] * v[(size_t)q[b] * nrhs + r];
    t[e] = a;
  }
  if (rc.inv) {
    double* t2 = t + (size_t)nc * nrhs;
    __syncthreads();
    pinv_apply_t(fac + rc.C_off, nc, t, t2, nrhs);
    __syncthreads();
    t = t2;
  } else {
    bwd_subst(fac + rc.C_off, nc, t, nrhs);
  }
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    v[(size_t)c[i] * nrhs + r] = t[e];
  }
}

// Skeleton record: idx = sk[k] then rd[r]; T (k x r), C (r x r), W (r x k).
//   forward  (apply_ut): v_rd -= T^T v_sk ; s = C^-1 v_rd ; v_sk -= W^T s ; v_rd = s
//   backward (apply_u) : v_rd = C^-T (v_rd - W v_sk) ; v_sk -= T v_rd
__global__ void __launch_bounds__(NT) solve_skel_kernel(
    const SolveRec* __restrict__ recs, const int32_t* __restrict__ idx, const double* __restrict__ fac,
    double* __restrict__ v, int nrhs, int forward, double* scratch, int64_t per_rec) {
  extern __shared__ __align__(16) double sm[];
  const SolveRec rc = recs[blockIdx.x];
  const int r = rc.nc, k = rc.nq;
  double* xs = workspace(sm, scratch, per_rec);
  double* xr = xs + (size_t)k * nrhs;
  double* x2 = xr + (size_t)r * nrhs;
  const int32_t* sk = idx + rc.idx_off;
  const int32_t* rd = sk + k;
  const double* T = fac + rc.T_off;
  const double* C = fac + rc.C_off;
  const double* W = fac + rc.W_off;
  for (int e = threadIdx.x; e < k * nrhs; e += NT) {
    const int a = e / nrhs, j = e - a * nrhs;
    xs[e] = v[(size_t)sk[a] * nrhs + j];
  }
  for (int e = threadIdx.x; e < r * nrhs; e += NT) {
    const int b = e / nrhs, j = e - b * nrhs;
    xr[e] = v[(size_t)rd[b] * nrhs + j];
  }
  __syncthreads();
  if (forward) {
    for (int e = threadIdx.x; e < r * nrhs; e += NT) {
      const int b = e / nrhs, j = e - b * nrhs;
      double a = xr[e];
      for (int l = 0; l < k; ++l) a -= T[(size_t)l * r + b] * xs[(size_t)l * nrhs + j];
      xr[e] = a;
    }
    if (rc.inv) {
      __syncthreads();
      pinv_apply(C, r, xr, x2, nrhs);
      __syncthreads();
      for (int e = threadIdx.x; e < r * nrhs; e += NT) xr[e] = x2[e];
      __syncthreads();
    } else {
      fwd_subst(C, r, xr, nrhs);
    }
    for (int e = threadIdx.x; e < k * nrhs; e += NT) {
      const int a = e / nrhs, j = e - a * nrhs;
      double x = xs[e];
      for (int l = 0; l < r; ++l) x -= W[(size_t)l * k + a] * xr[(size_t)l * nrhs + j];
      xs[e] = x;
    }
  } else {
    for (int e = threadIdx.x; e < r * nrhs; e += NT) {
      const int b = e / nrhs, j = e - b * nrhs;
      double a = xr[e];
      for (int l = 0; l < k; ++l) a -= W[(size_t)b * k + l] * xs[(size_t)l * nrhs + j];
      xr[e] = a;
    }
    if (rc.inv) {
      __syncthreads();
      pinv_apply_t(C, r, xr, x2, nrhs);
      __syncthreads();
      for (int e = threadIdx.x; e < r * nrhs; e += NT) xr[e] = x2[e];
      __syncthreads();
    } else {
      bwd_subst(C, r, xr, nrhs);
    }
    for (int e = threadIdx.x; e < k * nrhs; e += NT) {
      const int a = e / nrhs, j = e - a * nrhs;
      double x = xs[e];
      for (int l = 0; l < r; ++l) x -= T[(size_t)a * r + l] * xr[(size_t)l * nrhs + j];
      xs[e] = x;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * nrhs; e += NT) {
    const int a = e / nrhs, j = e - a * nrhs;
    v[(size_t)sk[a] * nrhs + j] = xs[e];
  }
  for (int e = threadIdx.x; e < r * nrhs; e += NT) {
    const int b = e / nrhs, j = e - b * nrhs;
    v[(size_t)rd[b] * nrhs + j] = xr[e];
  }
}

// ---------------------------------------------------------------------------
// Tiled products for large records (see TileOp): a CTA computes 64 rows x 32
// right-hand sides, staging 32-wide K chunks of A and X in shared memory.
// ---------------------------------------------------------------------------
constexpr int kTM = 64, kTKc = 32, kRW = 32;

__device__ __forceinline__ double* op_row(int mode, int64_t off, int k, const int32_t* __restrict__ idx, double* v,
                                          double* ts, double* contrib, int nrhs) {
  if (mode == 0) return v + (size_t)idx[off + k] * nrhs;
  if (mode == 1) return ts + (size_t)(off + k) * nrhs;
  return contrib + (size_t)(off + k) * nrhs;
}

__global__ void __launch_bounds__(256) solve_tile_kernel(const TileOp* __restrict__ ops,
                                                         const int2* __restrict__ work,
                                                         const int32_t* __restrict__ idx,
                                                         const double* __restrict__ fac, double* v, int nrhs,
                                                         double* ts, double* contrib) {
  __shared__ double As[kTM][kTKc + 1];
  __shared__ double Xs[kTKc][kRW];
  const int2 w = work[blockIdx.x];
  const TileOp op = ops[w.x];
  const int i0 = w.y, r0 = blockIdx.y * kRW;
  if (r0 >= nrhs) return;
  const int nr = min(kRW, nrhs - r0);
  const int tr = threadIdx.x & 31, ti = threadIdx.x >> 5;
  const double* Am = fac + op.A_off;
  const bool trans = op.amode == 1 || op.amode == 3;
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.0;
  for (int k0 = 0; k0 < op.K; k0 += kTKc) {
    __syncthreads();
    for (int e = threadIdx.x; e < kTM * kTKc; e += 256) {
      int ii, kk;
      if (trans) { kk = e / kTM; ii = e - kk * kTM; }   // consecutive i: coalesced for A^T
      else { ii = e / kTKc; kk = e - ii * kTKc; }
      const int i = i0 + ii, k = k0 + kk;
      double a = 0.0;
      if (i < op.M && k < op.K) {
        switch (op.amode) {
          case 0: a = k <= i ? Am[(size_t)i * (i + 1) / 2 + k] : 0.0; break;
          case 1: a = k >= i ? Am[(size_t)k * (k + 1) / 2 + i] : 0.0; break;
          case 2: a = Am[(size_t)i * op.lda + k]; break;
          default: a = Am[(size_t)k * op.lda + i]; break;
        }
      }
      As[ii][kk] = a;
    }
    for (int e = threadIdx.x; e < kTKc * kRW; e += 256) {
      const int kk = e / kRW, rr = e - kk * kRW;
      const int k = k0 + kk;
      double x = 0.0;
      if (k < op.K && rr < nr) x = op_row(op.xmode, op.x_off, k, idx, v, ts, contrib, nrhs)[r0 + rr];
      Xs[kk][rr] = x;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kTKc; ++kk) {
      const double xv = Xs[kk][tr];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += As[ti + 8 * j][kk] * xv;
    }
  }
  if (tr >= nr) return;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int i = i0 + ti + 8 * j;
    if (i >= op.M) continue;
    double val = op.alpha * acc[j];
    if (op.smode >= 0) val += op_row(op.smode, op.s_off, i, idx, v, ts, contrib, nrhs)[r0 + tr];
    op_row(op.dmode, op.d_off, i, idx, v, ts, contrib, nrhs)[r0 + tr] = val;
  }
}

void launch_solve_tiles(const TileOp* ops, const int2* work, int nwork, const int32_t* idx, const double* fac,
                        double* v, int nrhs, double* tscratch, double* contrib, cudaStream_t s) {
  if (nwork <= 0) return;
  dim3 grid((unsigned)nwork, (unsigned)((nrhs + kRW - 1) / kRW));
  solve_tile_kernel<<<grid, 256, 0, s>>>(ops, work, idx, fac, v, nrhs, tscratch, contrib);
}

static void set_smem_attr(const void* fn) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

void launch_solve_elim_fwd(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac,
                           double* v, int nrhs, double* contrib, double* scratch,
                           int64_t scratch_per_rec, size_t smem, cudaStream_t s) {
  if (nrec <= 0) return;
  static bool once = (set_smem_attr((const void*)solve_elim_fwd_kernel), true);
  (void)once;
  solve_elim_fwd_kernel<<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, contrib, scratch, scratch_per_rec);
}

void launch_solve_reduce(const int32_t* targets, const int64_t* ptr, const int64_t* ent,
                         int ntargets, const double* contrib, double* v, int nrhs, cudaStream_t s) {
  if (ntargets <= 0) return;
  const int64_t total = (int64_t)ntargets * nrhs;
  const int blocks = (int)((total + 255) / 256);
  solve_reduce_kernel<<<blocks, 256, 0, s>>>(targets, ptr, ent, ntargets, contrib, v, nrhs);
}

void launch_solve_elim_bwd(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac,
                           double* v, int nrhs, double* scratch, int64_t scratch_per_rec,
                           size_t smem, cudaStream_t s) {
  if (nrec <= 0) return;
  static bool once = (set_smem_attr((const void*)solve_elim_bwd_kernel), true);
  (void)once;
  solve_elim_bwd_kernel<<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, scratch, scratch_per_rec);
}

void launch_solve_skel(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac,
                       double* v, int nrhs, int forward, double* scratch,
                       int64_t scratch_per_rec, size_t smem, cudaStream_t s) {
  if (nrec <= 0) return;
  static bool once = (set_smem_attr((const void*)solve_skel_kernel), true);
  (void)once;
  solve_skel_kernel<<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, forward, scratch, scratch_per_rec);
}

}  // namespace hifde
