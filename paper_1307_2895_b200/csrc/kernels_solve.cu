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
//
// Fine levels (records up to 96 x 192) use the single-load-phase kernels
// (solve_*_small_kernel); 48+ right-hand sides take the DMMA products in the
// general kernels; both sum in cta_gemm's order where they replace it.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "hifde_internal.h"

namespace hifde {

namespace {

constexpr int NT = kThreads;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

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

// x <- P^{-1} x and x <- P^{-T} x for the packed lower P (i.e. x <- C x and
// x <- C^T x for the Cholesky factor C = P^{-1}); column-oriented, one
// barrier per row.
__device__ void psolve_lower(const double* __restrict__ P, int n, double* x, int nrhs) {
  for (int i = 0; i < n; ++i) {
    __syncthreads();
    const double pinv = 1.0 / P[(size_t)i * (i + 1) / 2 + i];
    for (int r = threadIdx.x; r < nrhs; r += NT) x[(size_t)i * nrhs + r] *= pinv;
    __syncthreads();
    const int rows = n - i - 1;
    for (int e = threadIdx.x; e < rows * nrhs; e += NT) {
      const int l = i + 1 + e / nrhs, r = e - (e / nrhs) * nrhs;
      x[(size_t)l * nrhs + r] -= P[(size_t)l * (l + 1) / 2 + i] * x[(size_t)i * nrhs + r];
    }
  }
  __syncthreads();
}
__device__ void psolve_upper(const double* __restrict__ P, int n, double* x, int nrhs) {
  for (int i = n - 1; i >= 0; --i) {
    __syncthreads();
    const double pinv = 1.0 / P[(size_t)i * (i + 1) / 2 + i];
    for (int r = threadIdx.x; r < nrhs; r += NT) x[(size_t)i * nrhs + r] *= pinv;
    __syncthreads();
    const double* row = P + (size_t)i * (i + 1) / 2;
    for (int e = threadIdx.x; e < i * nrhs; e += NT) {
      const int l = e / nrhs, r = e - l * nrhs;
      x[(size_t)l * nrhs + r] -= row[l] * x[(size_t)i * nrhs + r];
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double* workspace(double* smem, double* scratch, int64_t per_rec) {
  return per_rec > 0 ? scratch + (size_t)blockIdx.x * per_rec : smem;
}

// One-CTA product Y (+)= alpha op(A) X, op(A) M x K, X K x nrhs and Y M x nrhs
// row-major (ld nrhs).  A is streamed from global memory in 32-wide K chunks
// staged (coalesced) in shared memory; 16 right-hand sides x 16 row groups
// per pass, 6 rows per thread.  amode: 0 packed lower P, 1 its transpose,
// 2 dense row-major (ld lda), 3 dense transposed.
constexpr int kGKC = 32, kGRB = 16, kGMI = 6;
constexpr int kGRows = (NT / kGRB) * kGMI;  // rows per pass (96)
constexpr int kMmaMinRhs = 8;               // small-record kernels: DMMA tiles from 8 right-hand sides
constexpr int kDmmaMinRhs = 48;             // right-hand sides from which products use DMMA (measured: 16 and 32
                                            // RHS have too few tiles per warp to hide DMMA latency)
// One right-hand side: a matrix-vector product read straight from global
// memory.  Row-major operands (P, dense): a warp per row, lanes along k
// (coalesced); transposed operands: lanes along 32 consecutive rows, warps
// split k, partial sums reduced through shared memory (As).
__device__ void cta_gemv(int M, int K, int amode, const double* __restrict__ A, int64_t lda, const double* x,
                         double* y, double alpha, bool accumulate, double* As) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();  // x complete
  if (amode == 0 || amode == 2) {
    for (int i = wid; i < M; i += NW) {
      const int kend = amode == 0 ? min(i + 1, K) : K;
      const double* row = amode == 0 ? A + (size_t)i * (i + 1) / 2 : A + (size_t)i * lda;
      double s0 = 0.0, s1 = 0.0;
      int k = lane;
      for (; k + 32 < kend; k += 64) {
        s0 += row[k] * x[k];
        s1 += row[k + 32] * x[k + 32];
      }
      if (k < kend) s0 += row[k] * x[k];
      const double sum = warp_sum(s0 + s1);
      if (lane == 0) y[i] = (accumulate ? y[i] : 0.0) + alpha * sum;
    }
  } else {
    for (int i0 = 0; i0 < M; i0 += 32) {
      const int i = i0 + lane;
      const int kbeg = amode == 1 ? i0 : 0;  // P^T: rows i need k >= i
      const int span = (K - kbeg + NW - 1) / NW;
      const int k0 = kbeg + wid * span, k1 = min(K, k0 + span);
      double s = 0.0;
      if (i < M)
        for (int k = k0; k < k1; ++k) {
          const double a = amode == 1 ? (k >= i ? A[(size_t)k * (k + 1) / 2 + i] : 0.0) : A[(size_t)k * lda + i];
          s += a * x[k];
        }
      As[wid * 32 + lane] = s;
      __syncthreads();
      if (wid == 0 && i < M) {
        double t = 0.0;
        for (int w = 0; w < NW; ++w) t += As[w * 32 + lane];
        y[i] = (accumulate ? y[i] : 0.0) + alpha * t;
      }
      __syncthreads();
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// The same product on the FP64 tensor cores (DMMA m8n8k4) for blocks of 8
// or more right-hand sides: per pass 96 rows x 64 right-hand sides as 8 x 8
// tiles, tile t = warp + 8 i (row tile t / ntc, column tile t % ntc), A staged
// in 32-wide K chunks as in cta_gemm, X read from shared memory.
__device__ void cta_gemm_dmma(int M, int K, int amode, const double* __restrict__ A, int64_t lda, const double* X,
                              double* Y, int nrhs, double alpha, bool accumulate, double* As) {
  constexpr int kCW = 64, kMaxT = (kGRows / 8) * (kCW / 8) / (NT / 32);  // 12 tiles per warp
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int m0 = 0; m0 < M; m0 += kGRows) {
    const int mrows = min(kGRows, M - m0);
    const int mt = (mrows + 7) / 8;
    for (int c0 = 0; c0 < nrhs; c0 += kCW) {
      const int cw = min(kCW, nrhs - c0);
      const int ntc = (cw + 7) / 8;
      const int ntiles = mt * ntc;
      double acc[kMaxT][2];
#pragma unroll
      for (int i = 0; i < kMaxT; ++i) acc[i][0] = acc[i][1] = 0.0;
      for (int k0 = 0; k0 < K; k0 += kGKC) {
        const int kc = min(kGKC, K - k0);
        __syncthreads();
        if (amode == 0 || amode == 2) {
          for (int e = threadIdx.x; e < mrows * kGKC; e += NT) {
            const int ii = e / kGKC, kk = e - ii * kGKC, i = m0 + ii, k = k0 + kk;
            double a = 0.0;
            if (kk < kc) a = amode == 0 ? (k <= i ? A[(size_t)i * (i + 1) / 2 + k] : 0.0) : A[(size_t)i * lda + k];
            As[ii * (kGKC + 1) + kk] = a;
          }
        } else {
          for (int e = threadIdx.x; e < mrows * kGKC; e += NT) {
            const int kk = e / mrows, ii = e - kk * mrows, i = m0 + ii, k = k0 + kk;
            double a = 0.0;
            if (kk < kc) a = amode == 1 ? (k >= i ? A[(size_t)k * (k + 1) / 2 + i] : 0.0) : A[(size_t)k * lda + i];
            As[ii * (kGKC + 1) + kk] = a;
          }
        }
        __syncthreads();
        // with ntc | 8 a warp's tiles share one column tile: its X fragment
        // is loaded once per k step
        const bool one_ct = (NT / 32) % ntc == 0;
        for (int ks = 0; ks < kc; ks += 4) {
          const int kl = ks + (lane & 3);  // this lane's k in the chunk
          double b0 = 0.0;
          if (one_ct) {
            const int col = c0 + (wid % ntc) * 8 + (lane >> 2);
            b0 = (kl < kc && col < nrhs) ? X[(size_t)(k0 + kl) * nrhs + col] : 0.0;
          }
#pragma unroll
          for (int i = 0; i < kMaxT; ++i) {
            const int t = wid + (NT / 32) * i;
            if (t >= ntiles) break;
            const int rt = t / ntc, ct = t - rt * ntc;
            const int row = rt * 8 + (lane >> 2);
            const double a = (kl < kc && row < mrows) ? As[row * (kGKC + 1) + kl] : 0.0;
            double b = b0;
            if (!one_ct) {
              const int col = c0 + ct * 8 + (lane >> 2);
              b = (kl < kc && col < nrhs) ? X[(size_t)(k0 + kl) * nrhs + col] : 0.0;
            }
            dmma_8x8x4(acc[i][0], acc[i][1], a, b);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < kMaxT; ++i) {
        const int t = wid + (NT / 32) * i;
        if (t >= ntiles) break;
        const int rt = t / ntc, ct = t - rt * ntc;
        const int row = m0 + rt * 8 + (lane >> 2);
        if (row >= M) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = c0 + ct * 8 + 2 * (lane & 3) + h;
          if (col >= nrhs) continue;
          double* y = Y + (size_t)row * nrhs + col;
          *y = (accumulate ? *y : 0.0) + alpha * acc[i][h];
        }
      }
    }
  }
  __syncthreads();
}

// kD: the kernel instantiation that may take the DMMA path (a separate
// instantiation, so the register budget of the DMMA tiles does not lower the
// occupancy of the CUDA-core path used for fewer right-hand sides)
template <bool kD>
__device__ void cta_gemm_t(int M, int K, int amode, const double* __restrict__ A, int64_t lda, const double* X,
                           double* Y, int nrhs, double alpha, bool accumulate, double* As) {
  if (nrhs == 1) {
    cta_gemv(M, K, amode, A, lda, X, Y, alpha, accumulate, As);
    return;
  }
  if (kD && nrhs >= kDmmaMinRhs) {
    cta_gemm_dmma(M, K, amode, A, lda, X, Y, nrhs, alpha, accumulate, As);
    return;
  }
  constexpr int RG = NT / kGRB;
  const int rr = threadIdx.x % kGRB, rg = threadIdx.x / kGRB;
  for (int m0 = 0; m0 < M; m0 += kGRows) {
    const int mrows = min(kGRows, M - m0);
    for (int r0 = 0; r0 < nrhs; r0 += kGRB) {
      double acc[kGMI];
#pragma unroll
      for (int m = 0; m < kGMI; ++m) acc[m] = 0.0;
      const int r = r0 + rr;
      for (int k0 = 0; k0 < K; k0 += kGKC) {
        const int kc = min(kGKC, K - k0);
        __syncthreads();
        if (amode == 0 || amode == 2) {
          for (int e = threadIdx.x; e < mrows * kGKC; e += NT) {
            const int ii = e / kGKC, kk = e - ii * kGKC, i = m0 + ii, k = k0 + kk;
            double a = 0.0;
            if (kk < kc) a = amode == 0 ? (k <= i ? A[(size_t)i * (i + 1) / 2 + k] : 0.0) : A[(size_t)i * lda + k];
            As[ii * (kGKC + 1) + kk] = a;
          }
        } else {
          for (int e = threadIdx.x; e < mrows * kGKC; e += NT) {
            const int kk = e / mrows, ii = e - kk * mrows, i = m0 + ii, k = k0 + kk;
            double a = 0.0;
            if (kk < kc) a = amode == 1 ? (k >= i ? A[(size_t)k * (k + 1) / 2 + i] : 0.0) : A[(size_t)k * lda + i];
            As[ii * (kGKC + 1) + kk] = a;
          }
        }
        __syncthreads();
        if (r < nrhs) {
          for (int kk = 0; kk < kc; ++kk) {
            const double x = X[(size_t)(k0 + kk) * nrhs + r];
#pragma unroll
            for (int m = 0; m < kGMI; ++m) acc[m] += As[(rg + RG * m) * (kGKC + 1) + kk] * x;
          }
        }
      }
      if (r < nrhs) {
#pragma unroll
        for (int m = 0; m < kGMI; ++m) {
          const int ii = rg + RG * m;
          if (ii >= mrows) continue;
          double* y = Y + (size_t)(m0 + ii) * nrhs + r;
          *y = (accumulate ? *y : 0.0) + alpha * acc[m];
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void cta_gemm(int M, int K, int amode, const double* __restrict__ A, int64_t lda,
                                         const double* X, double* Y, int nrhs, double alpha, bool accumulate,
                                         double* As) {
  cta_gemm_t<false>(M, K, amode, A, lda, X, Y, nrhs, alpha, accumulate, As);
}

}  // namespace

template <bool kD>
__global__ void __launch_bounds__(NT) solve_elim_fwd_kernel(
    const SolveRec* __restrict__ recs, const int32_t* __restrict__ idx, const double* __restrict__ fac,
    double* __restrict__ v, int nrhs, double* __restrict__ contrib, double* scratch, int64_t per_rec) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double As[kGRows * (kGKC + 1)];
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
    cta_gemm_t<kD>(nc, nc, 0, fac + rc.C_off, 0, s, s2, nrhs, 1.0, false, As);  // s2 = P s
    s = s2;
  } else {
    fwd_subst(fac + rc.C_off, nc, s, nrhs);
  }
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    v[(size_t)c[i] * nrhs + r] = s[e];
  }
  // contributions g = W^T s (W nc x nq row-major), summed per DOF later
  if (nq > 0) cta_gemm_t<kD>(nq, nc, 3, fac + rc.W_off, nq, s, contrib + (size_t)rc.contrib_off * nrhs, nrhs, 1.0, false, As);
}

__global__ void solve_reduce_kernel(const int32_t* __restrict__ targets, const int64_t* __restrict__ ptr,
                                    const int64_t* __restrict__ ent, int ntargets,
                                    const double* __restrict__ contrib, double* __restrict__ v,
                                    int nrhs, double sign) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ntargets * nrhs) return;
  const int t = (int)(e / nrhs), r = (int)(e % nrhs);
  double acc = 0.0;
  for (int64_t p = ptr[t]; p < ptr[t + 1]; ++p) acc += contrib[(size_t)ent[p] * nrhs + r];
  v[(size_t)targets[t] * nrhs + r] += sign * acc;
}

template <bool kD>
__global__ void __launch_bounds__(NT) solve_elim_bwd_kernel(
    const SolveRec* __restrict__ recs, const int32_t* __restrict__ idx, const double* __restrict__ fac,
    double* __restrict__ v, int nrhs, double* scratch, int64_t per_rec) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double As[kGRows * (kGKC + 1)];
  const SolveRec rc = recs[blockIdx.x];
  const int nc = rc.nc, nq = rc.nq;
  double* t = workspace(sm, scratch, per_rec);
  double* t2 = t + (size_t)nc * nrhs;
  double* xq = t2 + (size_t)nc * nrhs;
  const int32_t* c = idx + rc.idx_off;
  const int32_t* q = c + nc;
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    t[e] = v[(size_t)c[i] * nrhs + r];
  }
  for (int e = threadIdx.x; e < nq * nrhs; e += NT) {
    const int b = e / nrhs, r = e - b * nrhs;
    xq[e] = v[(size_t)q[b] * nrhs + r];
  }
  // t = v_c - W v_q  (W nc x nq row-major)
  if (nq > 0) cta_gemm_t<kD>(nc, nq, 2, fac + rc.W_off, nq, xq, t, nrhs, -1.0, true, As);
  else __syncthreads();
  if (rc.inv) {
    cta_gemm_t<kD>(nc, nc, 1, fac + rc.C_off, 0, t, t2, nrhs, 1.0, false, As);  // t2 = P^T t
    t = t2;
  } else {
    bwd_subst(fac + rc.C_off, nc, t, nrhs);
  }
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    v[(size_t)c[i] * nrhs + r] = t[e];
  }
}

// ---------------------------------------------------------------------------
// Small elimination records (nc, nq <= 64, 2..16 right-hand sides: the fine
// levels, thousands of cells).  Every load of the record -- P, W and the
// gathered rows of v -- is issued up front into shared memory with one
// barrier, so a CTA exposes one memory latency instead of one per product
// phase.  The products sum in the same order as cta_gemm (including its zero
// terms of the triangular factor), so results are bit-identical to the
// general kernels.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) solve_elim_fwd_small_kernel(const SolveRec* __restrict__ recs,
                                                                  const int32_t* __restrict__ idx,
                                                                  const double* __restrict__ fac,
                                                                  double* __restrict__ v, int nrhs,
                                                                  double* __restrict__ contrib) {
  extern __shared__ __align__(16) double sm[];
  const SolveRec rc = recs[blockIdx.x];
  const int nc = rc.nc, nq = rc.nq;
  const int np = nc * (nc + 1) / 2;
  double* sP = sm;
  double* sW = sP + np;
  double* sx = sW + (size_t)nc * nq;
  double* ss = sx + (size_t)nc * nrhs;
  const int32_t* c = idx + rc.idx_off;
  const double* P = fac + rc.C_off;
  const double* W = fac + rc.W_off;
  for (int e = threadIdx.x; e < np; e += NT) sP[e] = P[e];
  for (int e = threadIdx.x; e < nc * nq; e += NT) sW[e] = W[e];
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    sx[e] = v[(size_t)c[i] * nrhs + r];
  }
  __syncthreads();
  // s = P x_c
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    const double* Pi = sP + i * (i + 1) / 2;
    double acc = 0.0;
    for (int k = 0; k < nc; ++k) acc += (k <= i ? Pi[k] : 0.0) * sx[k * nrhs + r];
    const double y = 0.0 + 1.0 * acc;
    ss[e] = y;
    v[(size_t)c[i] * nrhs + r] = y;
  }
  __syncthreads();
  // contributions g = W^T s
  double* g = contrib + (size_t)rc.contrib_off * nrhs;
  for (int e = threadIdx.x; e < nq * nrhs; e += NT) {
    const int b = e / nrhs, r = e - b * nrhs;
    double acc = 0.0;
    for (int k = 0; k < nc; ++k) acc += sW[k * nq + b] * ss[k * nrhs + r];
    g[e] = 0.0 + 1.0 * acc;
  }
}

__global__ void __launch_bounds__(NT) solve_elim_bwd_small_kernel(const SolveRec* __restrict__ recs,
                                                                  const int32_t* __restrict__ idx,
                                                                  const double* __restrict__ fac,
                                                                  double* __restrict__ v, int nrhs) {
  extern __shared__ __align__(16) double sm[];
  const SolveRec rc = recs[blockIdx.x];
  const int nc = rc.nc, nq = rc.nq;
  const int np = nc * (nc + 1) / 2;
  double* sP = sm;
  double* sW = sP + np;
  double* st = sW + (size_t)nc * nq;
  double* sq = st + (size_t)nc * nrhs;
  const int32_t* c = idx + rc.idx_off;
  const int32_t* q = c + nc;
  const double* P = fac + rc.C_off;
  const double* W = fac + rc.W_off;
  for (int e = threadIdx.x; e < np; e += NT) sP[e] = P[e];
  for (int e = threadIdx.x; e < nc * nq; e += NT) sW[e] = W[e];
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    st[e] = v[(size_t)c[i] * nrhs + r];
  }
  for (int e = threadIdx.x; e < nq * nrhs; e += NT) {
    const int b = e / nrhs, r = e - b * nrhs;
    sq[e] = v[(size_t)q[b] * nrhs + r];
  }
  __syncthreads();
  // t = v_c - W v_q
  if (nq > 0)
    for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
      const int i = e / nrhs, r = e - i * nrhs;
      double acc = 0.0;
      for (int b = 0; b < nq; ++b) acc += sW[i * nq + b] * sq[b * nrhs + r];
      st[e] = st[e] + -1.0 * acc;
    }
  __syncthreads();
  // v_c = P^T t
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    double acc = 0.0;
    for (int k = 0; k < nc; ++k) acc += (k >= i ? sP[k * (k + 1) / 2 + i] : 0.0) * st[k * nrhs + r];
    v[(size_t)c[i] * nrhs + r] = 0.0 + 1.0 * acc;
  }
}

// ---------------------------------------------------------------------------
// Small records on the FP64 tensor cores (8+ right-hand sides): the same
// single-load phase, then every product D = op(A) X as 8 x 8 DMMA tiles
// (mma.sync m8n8k4).  Warp w owns the tile pairs p = w, w + 8, ... of
// (row tile, RHS tile); with 8, 16, 32 or 64 right-hand sides all of a warp's
// tiles share one RHS tile, so its X fragment is loaded once per k step.
// Triangular factors skip the k steps outside the triangle.  Products are
// written in place where the inputs allow (s over x_c, t over x_c), so a
// level-0 cell of config 3 needs 49 KB (forward) / 65 KB (backward).
// ---------------------------------------------------------------------------
constexpr int kMmaMaxJ = 12;  // tile pairs per warp: 96 rows x 64 RHS

__host__ __device__ inline int mma_ld(int nrhs) {  // row stride: >= nrhs, = 8 (mod 16): conflict-free B fragments
  int ld = (nrhs + 7) / 8 * 8;
  if (ld % 16 == 0) ld += 8;
  return ld;
}

// A(i, k): 0 packed lower P, 1 its transpose, 2 dense row-major, 3 dense transposed
template <int AM>
__device__ __forceinline__ double mma_a(const double* __restrict__ A, int lda, int i, int k) {
  if (AM == 0) return k <= i ? A[i * (i + 1) / 2 + k] : 0.0;
  if (AM == 1) return k >= i ? A[k * (k + 1) / 2 + i] : 0.0;
  if (AM == 2) return A[i * lda + k];
  return A[k * lda + i];
}

// kOne: the caller guarantees one batch (M <= 96 rows with 64 RHS), so the
// pair index handed to `out` is a compile-time register index
template <int AM, bool kOne = false, class Out>
__device__ __forceinline__ void warp_mma(int M, int K, const double* __restrict__ A, int lda, const double* X,
                                         int ldx, int R, Out out) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int mt = (M + 7) >> 3, ntr = (R + 7) >> 3, npair = mt * ntr;
  const int ar = lane >> 2, ak = lane & 3;
  const bool one_rt = NW % ntr == 0;  // every pair of this warp in RHS tile w % ntr
  // this warp's tile pairs p = w + NW j: with one RHS tile per warp the row
  // tile is m0 + j * dm (no division in the k loop)
  const int nj = w < npair ? (npair - 1 - w) / NW + 1 : 0;
  const int m0 = w / ntr, dm = NW / ntr, r0 = w - m0 * ntr;
  auto tmj = [&](int j) { return one_rt ? m0 + j * dm : (w + NW * j) / ntr; };
  auto trj = [&](int j) { return one_rt ? r0 : (w + NW * j) % ntr; };
  // pairs in batches of kMmaMaxJ accumulators (M up to 192 rows: 24 row tiles)
  for (int jb = 0; jb < (kOne ? min(nj, 1) : nj); jb += kMmaMaxJ) {
    const int nb = min(kMmaMaxJ, nj - jb);
    double acc[kMmaMaxJ][2];
#pragma unroll
    for (int j = 0; j < kMmaMaxJ; ++j) acc[j][0] = acc[j][1] = 0.0;
    int klo = 0, khi = K;
    if (AM == 0) khi = min(K, 8 * tmj(jb + nb - 1) + 8);
    if (AM == 1) klo = 8 * tmj(jb);
    const int cfix = 8 * r0 + ar;
    for (int k0 = klo & ~3; k0 < khi; k0 += 4) {
      const int k = k0 + ak;
      const bool kin = k < K;
      double b0 = 0.0;
      if (one_rt) b0 = (kin && cfix < R) ? X[k * ldx + cfix] : 0.0;
#pragma unroll
      for (int j = 0; j < kMmaMaxJ; ++j) {
        if (j >= nb) break;
        const int mi = tmj(jb + j);
        if (AM == 0 && k0 >= 8 * mi + 8) continue;  // above the diagonal: zero
        if (AM == 1 && k0 + 4 <= 8 * mi) continue;  // below it (transpose): zero
        const int i = 8 * mi + ar;
        const double a = (i < M && kin) ? mma_a<AM>(A, lda, i, k) : 0.0;
        double b = b0;
        if (!one_rt) {
          const int c = 8 * trj(jb + j) + ar;
          b = (kin && c < R) ? X[k * ldx + c] : 0.0;
        }
        dmma_8x8x4(acc[j][0], acc[j][1], a, b);
      }
    }
#pragma unroll
    for (int j = 0; j < kMmaMaxJ; ++j) {
      if (j >= nb) break;
      const int row = 8 * tmj(jb + j) + (lane >> 2);
      if (row >= M) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = 8 * trj(jb + j) + 2 * (lane & 3) + h;
        if (col < R) out(row, col, acc[j][h], kOne ? j : jb + j, h);
      }
    }
  }
}

// warp_mma for the pipelined kernels (registers to spare at one CTA per SM):
// the per-tile address arithmetic (packed-row bases, row strides, bounds) is
// hoisted out of the k loop; each DMMA then costs one shared load of A, a
// compare and the MMA (the loop was issue-bound on index math: ncu, config 3
// level 0, 56% issue slots busy).  Tile k steps and zero padding are as
// before, so the sums are unchanged bit for bit.
struct NoPre {
  __device__ void operator()() const {}
};
template <int AM, bool kOne = false, int MJ = kMmaMaxJ, class Out, class Pre = NoPre>
__device__ __forceinline__ void warp_mma_lean(int w, int M, int K, const double* __restrict__ A, int lda, const double* X,
                                              int ldx, int R, Out out, Pre pre = Pre{}) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31;
  const int mt = (M + 7) >> 3, ntr = (R + 7) >> 3, npair = mt * ntr;
  const int ar = lane >> 2, ak = lane & 3;
  // the pipelined kernels' RHS counts (8, 16, 32, 64) divide the warps: every
  // pair of a warp is in RHS tile w % ntr
  // this warp's tile pairs p = w + NW j: with one RHS tile per warp the row
  // tile is m0 + j * dm (no division in the k loop)
  const int nj = w < npair ? (npair - 1 - w) / NW + 1 : 0;
  const int m0 = w / ntr, dm = NW / ntr, r0 = w - m0 * ntr;
  auto tmj = [&](int j) { return m0 + j * dm; };
  // pairs in batches of MJ accumulators (M up to 192 rows: 24 row tiles)
  // kOne: exactly one pass, also for a warp without tiles, so that `pre`
  // (a group barrier between the k loops and the in-place outputs) is met by
  // every warp
  for (int jb = 0; kOne ? jb == 0 : jb < nj; jb += MJ) {
    const int nb = max(0, min(MJ, nj - jb));
    double acc[MJ][2];
    int ibase[MJ];  // per tile: the A offset of (row i, k = 0), or -1 past M
    int klim[MJ];   // per tile: the k0 bound of its nonzero A columns
    int irow[MJ];   // per tile: this lane's A row
#pragma unroll
    for (int j = 0; j < MJ; ++j) {
      acc[j][0] = acc[j][1] = 0.0;
      const int mi = j < nb ? tmj(jb + j) : 0;
      const int i = 8 * mi + ar;
      int base;
      if (AM == 0) base = i * (i + 1) / 2;
      else if (AM == 1) base = i;
      else if (AM == 2) base = i * lda;
      else base = i;
      ibase[j] = (j < nb && i < M) ? base : -1;
      irow[j] = i;
      klim[j] = AM == 0 ? 8 * mi + 8 : 8 * mi;  // AM 0: k0 < klim; AM 1: k0 + 4 > klim
    }
    int klo = 0, khi = nb > 0 ? K : 0;
    if (AM == 0 && nb > 0) khi = min(K, 8 * tmj(jb + nb - 1) + 8);
    if (AM == 1) klo = 8 * tmj(jb);
    const int cfix = 8 * r0 + ar;
    for (int k0 = klo & ~3; k0 < khi; k0 += 4) {
      const int k = k0 + ak;
      const bool kin = k < K;
      const double b = (kin && cfix < R) ? X[k * ldx + cfix] : 0.0;
      int koff;  // the k part of A's offset
      if (AM == 0) koff = k;
      else if (AM == 1) koff = k * (k + 1) / 2;
      else if (AM == 2) koff = k;
      else koff = k * lda;
#pragma unroll
      for (int j = 0; j < MJ; ++j) {
        if (j >= nb) break;
        if (AM == 0 && k0 >= klim[j]) continue;      // above the diagonal: zero
        if (AM == 1 && k0 + 4 <= klim[j]) continue;  // below it (transpose): zero
        const int i = ibase[j];
        bool nz = i >= 0 && kin;
        if (AM == 0) nz = nz && k <= irow[j];  // lower triangle
        if (AM == 1) nz = nz && k >= irow[j];  // its transpose
        const double a = nz ? A[i + koff] : 0.0;
        dmma_8x8x4(acc[j][0], acc[j][1], a, b);
      }
    }
    pre();
#pragma unroll
    for (int j = 0; j < MJ; ++j) {
      if (j >= nb) break;
      const int row = 8 * tmj(jb + j) + (lane >> 2);
      if (row >= M) continue;
      const int col = 8 * r0 + 2 * (lane & 3);
      if (col < R) out(row, col, acc[j][0], acc[j][1]);  // R even: both columns valid
    }
  }
}

// forward: s = P x_c -> v_c ; g = W^T s -> contribution rows
__global__ void __launch_bounds__(NT, 3) solve_elim_fwd_mma_kernel(const SolveRec* __restrict__ recs,
                                                                const int32_t* __restrict__ idx,
                                                                const double* __restrict__ fac,
                                                                double* __restrict__ v, int R,
                                                                double* __restrict__ contrib) {
  extern __shared__ __align__(16) double sm[];
  const SolveRec rc = recs[blockIdx.x];
  const int nc = rc.nc, nq = rc.nq, ld = mma_ld(R);
  const int np = nc * (nc + 1) / 2;
  double* sP = sm;
  double* sW = sP + np;
  double* sx = sW + nc * nq;
  const int32_t* c = idx + rc.idx_off;
  const double* P = fac + rc.C_off;
  const double* W = fac + rc.W_off;
  for (int e = threadIdx.x; e < np; e += NT) sP[e] = P[e];
  for (int e = threadIdx.x; e < nc * nq; e += NT) sW[e] = W[e];
  for (int e = threadIdx.x; e < nc * R; e += NT) {
    const int i = e / R, r = e - i * R;
    sx[i * ld + r] = v[(size_t)c[i] * R + r];
  }
  __syncthreads();
  // s = P x_c, kept in registers until every warp has read x_c, then in place
  {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ntr = (R + 7) >> 3, npair = ((nc + 7) >> 3) * ntr;
    double keep[kMmaMaxJ][2];
    warp_mma<0, true>(nc, nc, sP, 0, sx, ld, R, [&](int row, int col, double val, int j_, int h_) {
      keep[j_][h_] = val;
      v[(size_t)c[row] * R + col] = val;
    });
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kMmaMaxJ; ++j) {
      const int p = w + NW * j;
      if (p >= npair) break;
      const int mi = p / ntr, ri = p - mi * ntr, row = 8 * mi + (lane >> 2);
      if (row >= nc) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = 8 * ri + 2 * (lane & 3) + h;
        if (col < R) sx[row * ld + col] = keep[j][h];
      }
    }
  }
  __syncthreads();
  if (nq > 0) {
    double* g = contrib + (size_t)rc.contrib_off * R;
    warp_mma<3>(nq, nc, sW, nq, sx, ld, R, [&](int row, int col, double val, int j_, int h_) { g[(size_t)row * R + col] = val; });
  }
}

// backward: t = x_c - W x_q (in place) ; v_c = P^T t
__global__ void __launch_bounds__(NT, 3) solve_elim_bwd_mma_kernel(const SolveRec* __restrict__ recs,
                                                                const int32_t* __restrict__ idx,
                                                                const double* __restrict__ fac,
                                                                double* __restrict__ v, int R) {
  extern __shared__ __align__(16) double sm[];
  const SolveRec rc = recs[blockIdx.x];
  const int nc = rc.nc, nq = rc.nq, ld = mma_ld(R);
  const int np = nc * (nc + 1) / 2;
  double* sP = sm;
  double* sW = sP + np;
  double* st = sW + nc * nq;
  double* sq = st + nc * ld;
  const int32_t* c = idx + rc.idx_off;
  const int32_t* q = c + nc;
  const double* P = fac + rc.C_off;
  const double* W = fac + rc.W_off;
  for (int e = threadIdx.x; e < np; e += NT) sP[e] = P[e];
  for (int e = threadIdx.x; e < nc * nq; e += NT) sW[e] = W[e];
  for (int e = threadIdx.x; e < nc * R; e += NT) {
    const int i = e / R, r = e - i * R;
    st[i * ld + r] = v[(size_t)c[i] * R + r];
  }
  for (int e = threadIdx.x; e < nq * R; e += NT) {
    const int b = e / R, r = e - b * R;
    sq[b * ld + r] = v[(size_t)q[b] * R + r];
  }
  __syncthreads();
  if (nq > 0) {
    warp_mma<2>(nc, nq, sW, nq, sq, ld, R, [&](int row, int col, double val, int j_, int h_) { st[row * ld + col] -= val; });
    __syncthreads();
  }
  warp_mma<1>(nc, nc, sP, 0, st, ld, R, [&](int row, int col, double val, int j_, int h_) { v[(size_t)c[row] * R + col] = val; });
}

// ---------------------------------------------------------------------------
// Pipelined elimination-record solve for the fine levels (thousands of
// records of one small shape, 8+ right-hand sides): one persistent CTA per
// SM.  A producer warp streams the CTA's next records -- P, W and the
// gathered rows of v -- into a ring of S shared-memory stages with TMA bulk
// copies (cp.async.bulk, completion counted on the stage's `full` mbarrier),
// while eight consumer warps run the current record's DMMA products
// (warp_mma: the tiles and summation order of the one-record kernels above,
// so the results are bit-identical) and release the stage on its `empty`
// mbarrier.  The one-record kernels expose a load phase per record with 3
// CTAs per SM (ncu, config 3 level 0: long-scoreboard stalls on the gathers,
// 1.5 TB/s); here the loads of records k+1 .. k+S-1 overlap record k's math.
// ---------------------------------------------------------------------------
namespace pipe {
constexpr int kGroup = 256;     // consumer group: 8 warps (warp_mma's tile assignment)
constexpr int kMaxStages = 4;
constexpr int kPipeMJ = 8;      // tile pairs per warp and batch (64 rows x 64 RHS in one batch)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned tx) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok)
                 : "r"(smem_u32(b)), "r"(parity)
                 : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void group_sync(int g) { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kGroup) : "memory"); }

// Per-stage layout (doubles, every region 16-byte aligned): P (np + 2),
// W (nc nq + 2), x_c (nc ld), x_q (nq ld, backward); then ints: c (nc),
// q (nq), meta (8).
struct StageGeom {
  int offW, offX, offQ, offI, doubles;  // offsets in doubles; offI: int region
  __host__ __device__ static int even(int x) { return (x + 1) & ~1; }
  __host__ __device__ StageGeom(int max_nc, int max_nq, int ld, bool bwd) {
    const int np = max_nc * (max_nc + 1) / 2;
    offW = even(np + 2);
    offX = offW + even(max_nc * max_nq + 2);
    offQ = offX + max_nc * ld;
    offI = offQ + (bwd ? max_nq * ld : 0);
    doubles = offI + even((max_nc + max_nq + 8 + 1) / 2 + 1);
  }
};

// The byte range [src, src + bytes) rounded out to 16-byte granules, if it
// stays inside the arena; `ph` = doubles of lead-in in the staged copy.
__device__ __forceinline__ bool granules(const double* src, int n, const double* lo, const double* hi,
                                         const double*& a0, unsigned& bytes, int& ph) {
  const uintptr_t s = (uintptr_t)src, e = (uintptr_t)(src + n);
  const uintptr_t s0 = s & ~(uintptr_t)15, e0 = (e + 15) & ~(uintptr_t)15;
  a0 = (const double*)s0;
  bytes = (unsigned)(e0 - s0);
  ph = (int)((s - s0) >> 3);
  return s0 >= (uintptr_t)lo && e0 <= (uintptr_t)hi;
}

// NG consumer groups take the CTA's records in turn (record k: group k % NG).
template <bool kFwd, int NG>
__global__ void __launch_bounds__(NG * kGroup + 32, 1)
    solve_elim_pipe_kernel(const SolveRec* __restrict__ recs, int nrec, const int32_t* __restrict__ idx,
                           const double* __restrict__ fac, int64_t fac_len, double* __restrict__ v, int R,
                           double* __restrict__ contrib, int max_nc, int max_nq, int nstages) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  const int ld = mma_ld(R);
  const StageGeom sg(max_nc, max_nq, ld, !kFwd);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], kGroup / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x;
  const int nk = blockIdx.x < nrec ? (nrec - 1 - (int)blockIdx.x) / G + 1 : 0;
  if (w == NG * kGroup / 32) {
    // ---- producer warp ----
    const double* fac_end = fac + fac_len;
    for (int k = 0; k < nk; ++k) {
      const int s = k % nstages;
      if (k >= nstages) mbar_wait(&empty[s], (unsigned)((k / nstages) + 1) & 1u);
      double* st = sm + (size_t)s * sg.doubles;
      int32_t* si = reinterpret_cast<int32_t*>(st + sg.offI);
      const SolveRec rc = recs[blockIdx.x + (size_t)k * G];
      const int nc = rc.nc, nq = rc.nq, np = nc * (nc + 1) / 2;
      const double *aP, *aW;
      unsigned bP, bW;
      int pP, pW;
      const bool okP = granules(fac + rc.C_off, np, fac, fac_end, aP, bP, pP);
      const bool okW = granules(fac + rc.W_off, nc * nq, fac, fac_end, aW, bW, pW);
      const unsigned rowb = (unsigned)R * 8u;
      const unsigned tx = (okP ? bP : 0u) + (okW ? bW : 0u) + rowb * (unsigned)(nc + (kFwd ? 0 : nq));
      if (lane == 0) mbar_expect_tx(&full[s], tx);
      __syncwarp();
      if (lane == 0) {
        if (okP) bulk_g2s(st, aP, bP, &full[s]);
        if (okW) bulk_g2s(st + sg.offW, aW, bW, &full[s]);
      }
      if (!okP) for (int e = lane; e < np; e += 32) st[e] = fac[rc.C_off + e];  // arena edge: plain copies
      if (!okW) for (int e = lane; e < nc * nq; e += 32) st[sg.offW + e] = fac[rc.W_off + e];
      const int32_t* cg = idx + rc.idx_off;
      for (int i = lane; i < nc; i += 32) {
        const int g = cg[i];
        si[i] = g;
        bulk_g2s(st + sg.offX + (size_t)i * ld, v + (size_t)g * R, rowb, &full[s]);
      }
      if (!kFwd)
        for (int b = lane; b < nq; b += 32) {
          const int g = cg[nc + b];
          si[max_nc + b] = g;
          bulk_g2s(st + sg.offQ + (size_t)b * ld, v + (size_t)g * R, rowb, &full[s]);
        }
      if (lane == 0) {
        int32_t* meta = si + max_nc + max_nq;
        meta[0] = nc;
        meta[1] = nq;
        meta[2] = okP ? pP : 0;
        meta[3] = okW ? pW : 0;
        meta[4] = (int32_t)(rc.contrib_off & 0xffffffff);
        meta[5] = (int32_t)(rc.contrib_off >> 32);
      }
      __syncwarp();
      mbar_arrive(&full[s]);
    }
    return;
  }
  // ---- consumer warps ----
  // Every product keeps one RHS tile per warp (R = 8, 16, 32, 64: NW % ntr
  // == 0), so a warp reads and writes only its RHS tile's 8-column slice of
  // the staged rows.  At 64 RHS the slice is the warp's alone: results go in
  // place after its k loops, with no barrier between the products; with
  // fewer RHS the warps sharing a slice meet at a group barrier first.
  constexpr int NW = kGroup / 32;
  const int grp = w / NW;
  const int lw = w - grp * NW;  // warp within the group
  for (int k = grp; k < nk; k += NG) {
    const int s = k % nstages;
    mbar_wait(&full[s], (unsigned)(k / nstages) & 1u);
    double* st = sm + (size_t)s * sg.doubles;
    const int32_t* si = reinterpret_cast<const int32_t*>(st + sg.offI);
    const int32_t* meta = si + max_nc + max_nq;
    const int nc = meta[0], nq = meta[1];
    const double* sP = st + meta[2];
    const double* sW = st + sg.offW + meta[3];
    double* sx = st + sg.offX;
    const int32_t* c = si;
    const bool own = (R >> 3) == NW;
    auto gsync = [&]() {
      if (!own) group_sync(grp);
    };
    if (kFwd) {
      const int64_t coff = (int64_t)(uint32_t)meta[4] | ((int64_t)meta[5] << 32);
      // s = P x_c -> v_c and in place
      warp_mma_lean<0, true, kPipeMJ>(lw, nc, nc, sP, 0, sx, ld, R, [&](int row, int col, double a, double b) {
        *reinterpret_cast<double2*>(sx + row * ld + col) = make_double2(a, b);
        *reinterpret_cast<double2*>(v + (size_t)c[row] * R + col) = make_double2(a, b);
      }, gsync);
      __syncwarp();
      gsync();
      if (nq > 0) {  // g = W^T s -> contribution rows
        double* g = contrib + (size_t)coff * R;
        warp_mma_lean<3, false, kPipeMJ>(lw, nq, nc, sW, nq, sx, ld, R, [&](int row, int col, double a, double b) {
          *reinterpret_cast<double2*>(g + (size_t)row * R + col) = make_double2(a, b);
        });
      }
    } else {
      double* sq = st + sg.offQ;
      if (nq > 0) {  // t = x_c - W x_q, in place
        warp_mma_lean<2, false, kPipeMJ>(lw, nc, nq, sW, nq, sq, ld, R, [&](int row, int col, double a, double b) {
          double2* t = reinterpret_cast<double2*>(sx + row * ld + col);
          const double2 o = *t;
          *t = make_double2(o.x - a, o.y - b);
        });
        __syncwarp();
        gsync();
      }
      // v_c = P^T t
      warp_mma_lean<1, false, kPipeMJ>(lw, nc, nc, sP, 0, sx, ld, R, [&](int row, int col, double a, double b) {
        *reinterpret_cast<double2*>(v + (size_t)c[row] * R + col) = make_double2(a, b);
      });
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}
}  // namespace pipe

// skeleton record: sk[k] then rd[r]; T (k x r), P (r x r packed), W (r x k)
__global__ void __launch_bounds__(NT, 3) solve_skel_mma_kernel(const SolveRec* __restrict__ recs,
                                                            const int32_t* __restrict__ idx,
                                                            const double* __restrict__ fac,
                                                            double* __restrict__ v, int R, int forward) {
  extern __shared__ __align__(16) double sm[];
  const SolveRec rc = recs[blockIdx.x];
  const int r = rc.nc, k = rc.nq, ld = mma_ld(R);
  const int np = r * (r + 1) / 2;
  double* sT = sm;             // k x r
  double* sP = sT + k * r;     // packed r x r
  double* sW = sP + np;        // r x k
  double* xs = sW + r * k;     // k x ld
  double* xr = xs + k * ld;    // r x ld
  double* x2 = xr + r * ld;    // r x ld
  const int32_t* sk = idx + rc.idx_off;
  const int32_t* rd = sk + k;
  const double* T = fac + rc.T_off;
  const double* P = fac + rc.C_off;
  const double* W = fac + rc.W_off;
  for (int e = threadIdx.x; e < k * r; e += NT) sT[e] = T[e];
  for (int e = threadIdx.x; e < np; e += NT) sP[e] = P[e];
  for (int e = threadIdx.x; e < r * k; e += NT) sW[e] = W[e];
  for (int e = threadIdx.x; e < k * R; e += NT) {
    const int a = e / R, j = e - a * R;
    xs[a * ld + j] = v[(size_t)sk[a] * R + j];
  }
  for (int e = threadIdx.x; e < r * R; e += NT) {
    const int b = e / R, j = e - b * R;
    xr[b * ld + j] = v[(size_t)rd[b] * R + j];
  }
  __syncthreads();
  if (forward) {
    if (k > 0) {  // v_rd -= T^T v_sk
      warp_mma<3>(r, k, sT, r, xs, ld, R, [&](int row, int col, double val, int j_, int h_) { xr[row * ld + col] -= val; });
      __syncthreads();
    }
    warp_mma<0>(r, r, sP, 0, xr, ld, R, [&](int row, int col, double val, int j_, int h_) {  // s = P v_rd
      x2[row * ld + col] = val;
      v[(size_t)rd[row] * R + col] = val;
    });
    __syncthreads();
    if (k > 0)  // v_sk -= W^T s
      warp_mma<3>(k, r, sW, k, x2, ld, R, [&](int row, int col, double val, int j_, int h_) {
        v[(size_t)sk[row] * R + col] = xs[row * ld + col] - val;
      });
  } else {
    if (k > 0) {  // v_rd -= W v_sk
      warp_mma<2>(r, k, sW, k, xs, ld, R, [&](int row, int col, double val, int j_, int h_) { xr[row * ld + col] -= val; });
      __syncthreads();
    }
    warp_mma<1>(r, r, sP, 0, xr, ld, R, [&](int row, int col, double val, int j_, int h_) {  // v_rd = P^T (...)
      x2[row * ld + col] = val;
      v[(size_t)rd[row] * R + col] = val;
    });
    __syncthreads();
    if (k > 0)  // v_sk -= T v_rd
      warp_mma<2>(k, r, sT, r, x2, ld, R, [&](int row, int col, double val, int j_, int h_) {
        v[(size_t)sk[row] * R + col] = xs[row * ld + col] - val;
      });
  }
}

// Small skeleton records (r, k <= 64): the same single-load-phase scheme,
// bit-identical to solve_skel_kernel's products.
__global__ void __launch_bounds__(NT) solve_skel_small_kernel(const SolveRec* __restrict__ recs,
                                                              const int32_t* __restrict__ idx,
                                                              const double* __restrict__ fac,
                                                              double* __restrict__ v, int nrhs, int forward) {
  extern __shared__ __align__(16) double sm[];
  const SolveRec rc = recs[blockIdx.x];
  const int r = rc.nc, k = rc.nq;
  const int np = r * (r + 1) / 2;
  double* sT = sm;                          // k x r
  double* sP = sT + (size_t)k * r;          // packed r x r
  double* sW = sP + np;                     // r x k
  double* xs = sW + (size_t)r * k;          // k x nrhs
  double* xr = xs + (size_t)k * nrhs;       // r x nrhs
  double* x2 = xr + (size_t)r * nrhs;       // r x nrhs
  const int32_t* sk = idx + rc.idx_off;
  const int32_t* rd = sk + k;
  const double* T = fac + rc.T_off;
  const double* P = fac + rc.C_off;
  const double* W = fac + rc.W_off;
  for (int e = threadIdx.x; e < k * r; e += NT) sT[e] = T[e];
  for (int e = threadIdx.x; e < np; e += NT) sP[e] = P[e];
  for (int e = threadIdx.x; e < r * k; e += NT) sW[e] = W[e];
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
    if (k > 0) {  // v_rd -= T^T v_sk
      for (int e = threadIdx.x; e < r * nrhs; e += NT) {
        const int i = e / nrhs, j = e - i * nrhs;
        double acc = 0.0;
        for (int l = 0; l < k; ++l) acc += sT[l * r + i] * xs[l * nrhs + j];
        xr[e] = xr[e] + -1.0 * acc;
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < r * nrhs; e += NT) {  // s = P v_rd
      const int i = e / nrhs, j = e - i * nrhs;
      const double* Pi = sP + i * (i + 1) / 2;
      double acc = 0.0;
      for (int l = 0; l < r; ++l) acc += (l <= i ? Pi[l] : 0.0) * xr[l * nrhs + j];
      x2[e] = 0.0 + 1.0 * acc;
    }
    __syncthreads();
    if (k > 0) {  // v_sk -= W^T s
      for (int e = threadIdx.x; e < k * nrhs; e += NT) {
        const int i = e / nrhs, j = e - i * nrhs;
        double acc = 0.0;
        for (int l = 0; l < r; ++l) acc += sW[l * k + i] * x2[l * nrhs + j];
        xs[e] = xs[e] + -1.0 * acc;
      }
    }
  } else {
    if (k > 0) {  // v_rd -= W v_sk
      for (int e = threadIdx.x; e < r * nrhs; e += NT) {
        const int i = e / nrhs, j = e - i * nrhs;
        double acc = 0.0;
        for (int l = 0; l < k; ++l) acc += sW[i * k + l] * xs[l * nrhs + j];
        xr[e] = xr[e] + -1.0 * acc;
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < r * nrhs; e += NT) {  // v_rd = P^T (...)
      const int i = e / nrhs, j = e - i * nrhs;
      double acc = 0.0;
      for (int l = 0; l < r; ++l) acc += (l >= i ? sP[l * (l + 1) / 2 + i] : 0.0) * xr[l * nrhs + j];
      x2[e] = 0.0 + 1.0 * acc;
    }
    __syncthreads();
    if (k > 0) {  // v_sk -= T v_rd
      for (int e = threadIdx.x; e < k * nrhs; e += NT) {
        const int i = e / nrhs, j = e - i * nrhs;
        double acc = 0.0;
        for (int l = 0; l < r; ++l) acc += sT[i * r + l] * x2[l * nrhs + j];
        xs[e] = xs[e] + -1.0 * acc;
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * nrhs; e += NT) {
    const int a = e / nrhs, j = e - a * nrhs;
    v[(size_t)sk[a] * nrhs + j] = xs[e];
  }
  for (int e = threadIdx.x; e < r * nrhs; e += NT) {
    const int b = e / nrhs, j = e - b * nrhs;
    v[(size_t)rd[b] * nrhs + j] = x2[e];
  }
}

// Skeleton record: idx = sk[k] then rd[r]; T (k x r), C (r x r), W (r x k).
//   forward  (apply_ut): v_rd -= T^T v_sk ; s = C^-1 v_rd ; v_sk -= W^T s ; v_rd = s
//   backward (apply_u) : v_rd = C^-T (v_rd - W v_sk) ; v_sk -= T v_rd
template <bool kD>
__global__ void __launch_bounds__(NT) solve_skel_kernel(
    const SolveRec* __restrict__ recs, const int32_t* __restrict__ idx, const double* __restrict__ fac,
    double* __restrict__ v, int nrhs, int forward, double* scratch, int64_t per_rec) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double As[kGRows * (kGKC + 1)];
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
  double* xo = xr;  // final v_rd
  if (forward) {
    if (k > 0) cta_gemm_t<kD>(r, k, 3, T, r, xs, xr, nrhs, -1.0, true, As);  // v_rd -= T^T v_sk
    if (rc.inv) {
      cta_gemm_t<kD>(r, r, 0, C, 0, xr, x2, nrhs, 1.0, false, As);           // s = P v_rd
      xo = x2;
    } else {
      fwd_subst(C, r, xr, nrhs);
    }
    if (k > 0) cta_gemm_t<kD>(k, r, 3, W, k, xo, xs, nrhs, -1.0, true, As);  // v_sk -= W^T s
  } else {
    if (k > 0) cta_gemm_t<kD>(r, k, 2, W, k, xs, xr, nrhs, -1.0, true, As);  // v_rd -= W v_sk
    if (rc.inv) {
      cta_gemm_t<kD>(r, r, 1, C, 0, xr, x2, nrhs, 1.0, false, As);           // v_rd = P^T (...)
      xo = x2;
    } else {
      bwd_subst(C, r, xr, nrhs);
    }
    if (k > 0) cta_gemm_t<kD>(k, r, 2, T, r, xo, xs, nrhs, -1.0, true, As);  // v_sk -= T v_rd
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * nrhs; e += NT) {
    const int a = e / nrhs, j = e - a * nrhs;
    v[(size_t)sk[a] * nrhs + j] = xs[e];
  }
  for (int e = threadIdx.x; e < r * nrhs; e += NT) {
    const int b = e / nrhs, j = e - b * nrhs;
    v[(size_t)rd[b] * nrhs + j] = xo[e];
  }
}

// ---------------------------------------------------------------------------
// F x (GeneralizedLDL.apply, src/driver.py:95-111): the solve sweep inverted.
// apply_inverse = Fwd_0 .. Fwd_top, Bwd_top .. Bwd_0, so
// apply = BwdInv_0 .. BwdInv_top, FwdInv_top .. FwdInv_0 with, per record
// (C = P^-1 the Cholesky factor, P the stored packed inverse):
//   elimination BwdInv: v_c = C^T v_c + W v_q
//               FwdInv: v_q += W^T v_c (contributions), v_c = C v_c
//   skeleton    BwdInv: v_sk += T v_rd ; v_rd = C^T v_rd + W v_sk
//               FwdInv: v_sk += W^T v_rd ; v_rd = C v_rd + T^T v_sk
// Every record of a level (small and large) runs one CTA.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) apply_elim_kernel(
    const SolveRec* __restrict__ recs, const int32_t* __restrict__ idx, const double* __restrict__ fac,
    double* __restrict__ v, int nrhs, double* __restrict__ contrib, double* scratch, int64_t per_rec, int fwdinv) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double As[kGRows * (kGKC + 1)];
  const SolveRec rc = recs[blockIdx.x];
  const int nc = rc.nc, nq = rc.nq;
  double* t = workspace(sm, scratch, per_rec);
  double* xq = t + (size_t)nc * nrhs;
  const int32_t* c = idx + rc.idx_off;
  const int32_t* q = c + nc;
  const double* P = fac + rc.C_off;
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    t[e] = v[(size_t)c[i] * nrhs + r];
  }
  if (!fwdinv) {
    for (int e = threadIdx.x; e < nq * nrhs; e += NT) {
      const int b = e / nrhs, r = e - b * nrhs;
      xq[e] = v[(size_t)q[b] * nrhs + r];
    }
    psolve_upper(P, nc, t, nrhs);                                                   // C^T v_c
    if (nq > 0) cta_gemm(nc, nq, 2, fac + rc.W_off, nq, xq, t, nrhs, 1.0, true, As);  // + W v_q
  } else {
    __syncthreads();
    if (nq > 0) cta_gemm(nq, nc, 3, fac + rc.W_off, nq, t, contrib + (size_t)rc.contrib_off * nrhs, nrhs, 1.0, false, As);
    psolve_lower(P, nc, t, nrhs);                                                   // C v_c
  }
  for (int e = threadIdx.x; e < nc * nrhs; e += NT) {
    const int i = e / nrhs, r = e - i * nrhs;
    v[(size_t)c[i] * nrhs + r] = t[e];
  }
}

__global__ void __launch_bounds__(NT) apply_skel_kernel(
    const SolveRec* __restrict__ recs, const int32_t* __restrict__ idx, const double* __restrict__ fac,
    double* __restrict__ v, int nrhs, double* scratch, int64_t per_rec, int fwdinv) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double As[kGRows * (kGKC + 1)];
  const SolveRec rc = recs[blockIdx.x];
  const int r = rc.nc, k = rc.nq;
  double* xs = workspace(sm, scratch, per_rec);
  double* xr = xs + (size_t)k * nrhs;
  const int32_t* sk = idx + rc.idx_off;
  const int32_t* rd = sk + k;
  const double* T = fac + rc.T_off;
  const double* P = fac + rc.C_off;
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
  if (!fwdinv) {
    if (k > 0) cta_gemm(k, r, 2, T, r, xr, xs, nrhs, 1.0, true, As);   // v_sk += T v_rd
    psolve_upper(P, r, xr, nrhs);                                       // C^T v_rd
    if (k > 0) cta_gemm(r, k, 2, W, k, xs, xr, nrhs, 1.0, true, As);   // + W v_sk
  } else {
    if (k > 0) cta_gemm(k, r, 3, W, k, xr, xs, nrhs, 1.0, true, As);   // v_sk += W^T v_rd
    psolve_lower(P, r, xr, nrhs);                                       // C v_rd
    if (k > 0) cta_gemm(r, k, 3, T, r, xs, xr, nrhs, 1.0, true, As);   // + T^T v_sk
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
  if (nrhs == 1) {  // matrix-vector: stream A at full width (the 32-RHS tiling would idle 31/32 lanes)
    __shared__ double xs[1024];
    __shared__ double part[8][64];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double* Am = fac + op.A_off;
    const bool rowmaj = op.amode == 0 || op.amode == 2;
    const int mrows = min(kTM, op.M - i0);
    double acc8[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc8[q] = 0.0;
    for (int k0 = 0; k0 < op.K; k0 += 1024) {
      const int kc = min(1024, op.K - k0);
      __syncthreads();
      for (int kk = threadIdx.x; kk < kc; kk += 256) xs[kk] = op_row(op.xmode, op.x_off, k0 + kk, idx, v, ts, contrib, 1)[0];
      __syncthreads();
      if (rowmaj) {  // warp per row (8 rows each), lanes along k
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int i = i0 + wid * 8 + q;
          if (i >= op.M) continue;
          const int kend = op.amode == 0 ? min(kc, i + 1 - k0) : kc;
          const double* row = op.amode == 0 ? Am + (size_t)i * (i + 1) / 2 + k0 : Am + (size_t)i * op.lda + k0;
          double s = 0.0;
          for (int kk = lane; kk < kend; kk += 32) s += row[kk] * xs[kk];
          acc8[q] += s;
        }
      } else {  // lanes along rows (2 x 32), warps split k
        const int span = (kc + 7) / 8, ka = wid * span, kb = min(kc, ka + span);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = i0 + h * 32 + lane;
          if (i >= op.M) continue;
          double s = 0.0;
          for (int kk = ka; kk < kb; ++kk) {
            const int k = k0 + kk;
            const double a = op.amode == 1 ? (k >= i ? Am[(size_t)k * (k + 1) / 2 + i] : 0.0) : Am[(size_t)k * op.lda + i];
            s += a * xs[kk];
          }
          acc8[h] += s;
        }
      }
    }
    if (rowmaj) {
#pragma unroll
      for (int q = 0; q < 8; ++q) acc8[q] = warp_sum(acc8[q]);
      if (lane == 0)
        for (int q = 0; q < 8; ++q) part[0][wid * 8 + q] = acc8[q];
    } else {
      part[wid][lane] = acc8[0];
      part[wid][32 + lane] = acc8[1];
    }
    __syncthreads();
    for (int ii = threadIdx.x; ii < mrows; ii += 256) {
      double a = 0.0;
      if (rowmaj) a = part[0][ii];
      else
        for (int q = 0; q < 8; ++q) a += part[q][ii];
      const int i = i0 + ii;
      double val = op.alpha * a;
      if (op.smode >= 0) val += op_row(op.smode, op.s_off, i, idx, v, ts, contrib, 1)[0];
      op_row(op.dmode, op.d_off, i, idx, v, ts, contrib, 1)[0] = val;
    }
    return;
  }
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
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSolveDynSmem);
}

void launch_solve_elim_fwd(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac,
                           double* v, int nrhs, double* contrib, double* scratch,
                           int64_t scratch_per_rec, size_t smem, cudaStream_t s) {
  if (nrec <= 0) return;
  static bool once = (set_smem_attr((const void*)solve_elim_fwd_kernel<false>),
                      set_smem_attr((const void*)solve_elim_fwd_kernel<true>), true);
  (void)once;
  if (nrhs >= kDmmaMinRhs)
    solve_elim_fwd_kernel<true><<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, contrib, scratch, scratch_per_rec);
  else
    solve_elim_fwd_kernel<false><<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, contrib, scratch, scratch_per_rec);
}

size_t solve_small_smem(int max_nc, int max_nq, int nrhs) {
  if (nrhs >= kMmaMinRhs)  // DMMA kernels: x_c (forward) or x_c and x_q (backward) at stride mma_ld
    return sizeof(double) * ((size_t)max_nc * (max_nc + 1) / 2 + (size_t)max_nc * max_nq +
                             (size_t)(max_nc + max_nq) * mma_ld(nrhs));
  return sizeof(double) * ((size_t)max_nc * (max_nc + 1) / 2 + (size_t)max_nc * max_nq + 2 * (size_t)max_nc * nrhs +
                           (size_t)max_nq * nrhs);
}

// Per record of an elimination level: its smallest and largest cell DOF
// (cells ascending in the index arena), for the banded host solve.
__global__ void solve_rec_rows_kernel(const SolveRec* __restrict__ recs, int nrec, const int32_t* __restrict__ idx,
                                      int32_t* __restrict__ cmin, int32_t* __restrict__ cmax) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const SolveRec rc = recs[r];
  cmin[r] = rc.nc > 0 ? idx[rc.idx_off] : 0x7fffffff;
  cmax[r] = rc.nc > 0 ? idx[rc.idx_off + rc.nc - 1] : -1;
}
void launch_solve_rec_rows(const SolveRec* recs, int nrec, const int32_t* idx, int32_t* cmin, int32_t* cmax,
                           cudaStream_t s) {
  if (nrec > 0) solve_rec_rows_kernel<<<(nrec + 255) / 256, 256, 0, s>>>(recs, nrec, idx, cmin, cmax);
}

// Shared memory of the pipelined kernel with `stages` stages (0: the level
// does not fit two stages).
static size_t pipe_smem(int max_nc, int max_nq, int nrhs, bool fwd, int& stages) {
  const pipe::StageGeom sg(max_nc, max_nq, mma_ld(nrhs), !fwd);
  const size_t per = sizeof(double) * (size_t)sg.doubles;
  stages = (int)std::min<size_t>(pipe::kMaxStages, (kSmemCapBytes - 1024) / per);
  return stages >= 2 ? per * stages : 0;
}

void launch_solve_elim_small(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac, int64_t fac_len,
                             double* v, int nrhs, double* contrib, int max_nc, int max_nq, size_t smem, int forward,
                             cudaStream_t s) {
  if (nrec <= 0) return;
  static int nsm = [] {
    int d = 0, n = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    return n > 0 ? n : 1;
  }();
  // many records of a small shape, an even RHS count (16-byte rows): the
  // persistent pipelined kernels
  // (HIFDE_NO_SOLVE_PIPE: the one-record kernels instead -- the tests' A/B of
  // the two, which must agree bit for bit)
  static const bool no_pipe = getenv("HIFDE_NO_SOLVE_PIPE") != nullptr;
  if (!no_pipe && (nrhs == 8 || nrhs == 16 || nrhs == 32 || nrhs == 64) && max_nc <= 64 && nrec >= 4 * nsm) {
    int stages = 0;
    const size_t psm = pipe_smem(max_nc, max_nq, nrhs, forward != 0, stages);
    if (psm) {
      static bool once3 = (cudaFuncSetAttribute(pipe::solve_elim_pipe_kernel<true, 2>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCapBytes),
                           cudaFuncSetAttribute(pipe::solve_elim_pipe_kernel<false, 2>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCapBytes),
                           true);
      (void)once3;
      const int grid = std::min(nrec, nsm);
      constexpr int nthr = 2 * pipe::kGroup + 32;
      if (forward)
        pipe::solve_elim_pipe_kernel<true, 2><<<grid, nthr, psm, s>>>(recs, nrec, idx, fac, fac_len, v, nrhs, contrib,
                                                                      max_nc, max_nq, stages);
      else
        pipe::solve_elim_pipe_kernel<false, 2><<<grid, nthr, psm, s>>>(recs, nrec, idx, fac, fac_len, v, nrhs,
                                                                       contrib, max_nc, max_nq, stages);
      return;
    }
  }
  static bool once = (cudaFuncSetAttribute(solve_elim_fwd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kSmemCapBytes),
                      cudaFuncSetAttribute(solve_elim_bwd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kSmemCapBytes),
                      true);
  (void)once;
  static bool once2 = (cudaFuncSetAttribute(solve_elim_fwd_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)kSmemCapBytes),
                       cudaFuncSetAttribute(solve_elim_bwd_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)kSmemCapBytes),
                       true);
  (void)once2;
  if (nrhs >= kMmaMinRhs) {
    if (forward) solve_elim_fwd_mma_kernel<<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, contrib);
    else solve_elim_bwd_mma_kernel<<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs);
    return;
  }
  if (forward) solve_elim_fwd_small_kernel<<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, contrib);
  else solve_elim_bwd_small_kernel<<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs);
}

size_t solve_skel_small_smem(int max_r, int max_k, int nrhs) {
  const size_t ld = nrhs >= kMmaMinRhs ? (size_t)mma_ld(nrhs) : (size_t)nrhs;
  return sizeof(double) * (2 * (size_t)max_k * max_r + (size_t)max_r * (max_r + 1) / 2 + (size_t)max_k * ld +
                           2 * (size_t)max_r * ld);
}

void launch_solve_skel_small(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac, double* v,
                             int nrhs, size_t smem, int forward, cudaStream_t s) {
  if (nrec <= 0) return;
  static bool once = (cudaFuncSetAttribute(solve_skel_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kSmemCapBytes),
                      true);
  (void)once;
  static bool once2 = (cudaFuncSetAttribute(solve_skel_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)kSmemCapBytes),
                       true);
  (void)once2;
  if (nrhs >= kMmaMinRhs) {
    solve_skel_mma_kernel<<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, forward);
    return;
  }
  solve_skel_small_kernel<<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, forward);
}

void launch_solve_reduce(const int32_t* targets, const int64_t* ptr, const int64_t* ent,
                         int ntargets, const double* contrib, double* v, int nrhs, cudaStream_t s,
                         double sign) {
  if (ntargets <= 0) return;
  const int64_t total = (int64_t)ntargets * nrhs;
  const int blocks = (int)((total + 255) / 256);
  solve_reduce_kernel<<<blocks, 256, 0, s>>>(targets, ptr, ent, ntargets, contrib, v, nrhs, sign);
}

void launch_solve_elim_bwd(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac,
                           double* v, int nrhs, double* scratch, int64_t scratch_per_rec,
                           size_t smem, cudaStream_t s) {
  if (nrec <= 0) return;
  static bool once = (set_smem_attr((const void*)solve_elim_bwd_kernel<false>),
                      set_smem_attr((const void*)solve_elim_bwd_kernel<true>), true);
  (void)once;
  if (nrhs >= kDmmaMinRhs)
    solve_elim_bwd_kernel<true><<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, scratch, scratch_per_rec);
  else
    solve_elim_bwd_kernel<false><<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, scratch, scratch_per_rec);
}

void launch_solve_skel(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac,
                       double* v, int nrhs, int forward, double* scratch,
                       int64_t scratch_per_rec, size_t smem, cudaStream_t s) {
  if (nrec <= 0) return;
  static bool once = (set_smem_attr((const void*)solve_skel_kernel<false>),
                      set_smem_attr((const void*)solve_skel_kernel<true>), true);
  (void)once;
  if (nrhs >= kDmmaMinRhs)
    solve_skel_kernel<true><<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, forward, scratch, scratch_per_rec);
  else
    solve_skel_kernel<false><<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, forward, scratch, scratch_per_rec);
}

void launch_apply_elim(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac, double* v, int nrhs,
                       double* contrib, double* scratch, int64_t scratch_per_rec, size_t smem, int fwdinv,
                       cudaStream_t s) {
  if (nrec <= 0) return;
  static bool once = (set_smem_attr((const void*)apply_elim_kernel), true);
  (void)once;
  apply_elim_kernel<<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, contrib, scratch, scratch_per_rec, fwdinv);
}

void launch_apply_skel(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac, double* v, int nrhs,
                       double* scratch, int64_t scratch_per_rec, size_t smem, int fwdinv, cudaStream_t s) {
  if (nrec <= 0) return;
  static bool once = (set_smem_attr((const void*)apply_skel_kernel), true);
  (void)once;
  apply_skel_kernel<<<nrec, NT, smem, s>>>(recs, idx, fac, v, nrhs, scratch, scratch_per_rec, fwdinv);
}

}  // namespace hifde
