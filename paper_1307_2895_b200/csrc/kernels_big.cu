// Blocked, multi-CTA elimination of large cells (sm_100a).
//
// A cell whose front does not fit one CTA's shared memory is factored in
// place in the factor arena by a short sequence of launches per level:
//
//   big_assemble_kernel   grid (row chunks x cells): rows of the front
//                         [F_cc | F_cq] (in the record's C and W slots) and the
//                         q x q clique part U (block arena), each front row
//                         owned by exactly one CTA -> deterministic.
//   for every 64-column panel p:
//     panel_chol_kernel   1 CTA per cell: Cholesky of the diagonal block.
//     panel_trsm_kernel   rows below the panel  L_rp = F_rp L_pp^-T  and the
//                         panel rows of W       W_p  = L_pp^-1 W_p, in chunks.
//     panel_update_kernel 64 x 64 DMMA tiles: F_rs -= L_rp L_sp^T (lower
//                         trailing part) and W_r -= L_rp W_p (rows below).
//   schur_tile_kernel     U -= W^T W (kernels_factor.cu).
//   big_finish_kernel     singular-pivot check, zero the upper triangle of C.
//
// Same semantics as the single-CTA path (src/dense.py:187-219,
// src/factor_ops.py:138-159): right-looking blocked Cholesky of A_cc with the
// dpotrf indefinite rule and the 1e-14 singular rule.
#include <cfloat>
#include <cstdint>

#include "hifde_internal.h"

namespace hifde {

namespace {

constexpr double kSingularRtol = 1e-14;  // src/dense.py:38
constexpr int PB = kPanelB;               // panel width
constexpr int kInvLocal = kInvLocalCols;     // packed-inverse columns kept in local memory

__device__ __forceinline__ int bsearch_i32(const int32_t* s, int n, int32_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (s[mid] < key) lo = mid + 1; else hi = mid;
  }
  return (lo < n && s[lo] == key) ? lo : -1;
}

__device__ __forceinline__ int front_pos(const int32_t* dofs, int nc, int nq, int32_t g) {
  int p = bsearch_i32(dofs, nc, g);
  if (p >= 0) return p;
  p = bsearch_i32(dofs + nc, nq, g);
  return p >= 0 ? nc + p : -1;
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

}  // namespace

// ---------------------------------------------------------------------------
// Assembly.  Work item: int4 {cell, r0, r1, 0} -> front rows [r0, r1).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) big_assemble_kernel(const ElimTask* __restrict__ tasks,
                                                           const int4* __restrict__ work, Arenas A,
                                                           double* __restrict__ diag_scale) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int nsel;
  const int4 w = work[blockIdx.x];
  const ElimTask t = tasks[w.x];
  const int nc = t.nc, nq = t.nq, nf = nc + nq;
  const int r0 = w.y, r1 = w.z;
  int32_t* sdofs = reinterpret_cast<int32_t*>(smem);
  int32_t* smap = sdofs + nf;
  int32_t* ssel = smap + t.maxnb;
  double* F = A.fac + t.C_off;   // nc x nc
  double* W = A.fac + t.W_off;   // nc x nq
  double* U = A.bvals + t.U_off; // nq x nq
  const int32_t* gd = A.idx + t.dofs_off;
  for (int i = threadIdx.x; i < nf; i += 256) sdofs[i] = gd[i];
  for (int r = r0 + (int)threadIdx.x; r < r1 && r < nc; r += 256) A.active[gd[r]] = 0;
  // zero the owned rows (warp per row)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int r = r0 + wid; r < r1; r += 8) {
    if (r < nc) {
      for (int j = lane; j < nc; j += 32) F[(size_t)r * nc + j] = 0.0;
      for (int j = lane; j < nq; j += 32) W[(size_t)r * nq + j] = 0.0;
    } else {
      for (int j = lane; j < nq; j += 32) U[(size_t)(r - nc) * nq + j] = 0.0;
    }
  }
  __syncthreads();
  for (int p = r0 + (int)threadIdx.x; p < r1 && p < nc; p += 256) {
    const int g = sdofs[p];
    for (int64_t k = A.indptr[g]; k < A.indptr[g + 1]; ++k) {
      const int pj = front_pos(sdofs, nc, nq, A.indices[k]);
      if (pj < 0) continue;
      if (pj < nc) F[(size_t)p * nc + pj] += A.a0[k];
      else W[(size_t)p * nq + pj - nc] += A.a0[k];
    }
  }
  __syncthreads();
  const int32_t* bl = A.lists + t.blk_off;
  for (int b = 0; b < t.nblk; ++b) {
    const int bid = bl[b];
    const int nb = A.blk_n[bid];
    const int32_t* bd = A.idx + A.blk_dof_off[bid];
    const double* bv = A.bvals + A.blk_val_off[bid];
    if (threadIdx.x == 0) nsel = 0;
    __syncthreads();
    for (int k = threadIdx.x; k < nb; k += 256) {
      const int p = front_pos(sdofs, nc, nq, bd[k]);
      smap[k] = p;
      if (p >= r0 && p < r1) ssel[atomicAdd(&nsel, 1)] = k;  // rows this CTA owns
    }
    __syncthreads();
    const int ns = nsel;
    for (int s = wid; s < ns; s += 8) {  // warp per owned block row
      const int k = ssel[s];
      const int pk = smap[k];
      const double* brow = bv + (size_t)k * nb;
      for (int l = lane; l < nb; l += 32) {
        const int pl = smap[l];
        if (pl < 0) continue;
        if (pk < nc) {
          if (pl < nc) F[(size_t)pk * nc + pl] += brow[l];
          else W[(size_t)pk * nq + pl - nc] += brow[l];
        } else if (pl >= nc) {
          U[(size_t)(pk - nc) * nq + pl - nc] += brow[l];
        }
      }
    }
    __syncthreads();
  }
  // max |diag(A_cc)| of the owned rows, for the singular-pivot rule
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int r = r0; r < r1 && r < nc; ++r) m = fmax(m, fabs(F[(size_t)r * nc + r]));
    if (r0 < nc) {
      unsigned long long* p = reinterpret_cast<unsigned long long*>(diag_scale + w.x);
      atomicMax(p, (unsigned long long)__double_as_longlong(m));  // m >= 0: bit order == value order
    }
  }
}

// ---------------------------------------------------------------------------
// Panel Cholesky: one CTA per cell with nc > p0.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) panel_chol_kernel(const ElimTask* __restrict__ tasks,
                                                         const int32_t* __restrict__ cells, int p0,
                                                         Arenas A, double* __restrict__ dmin) {
  __shared__ double D[PB][PB + 1];
  const int cell = cells[blockIdx.x];
  if (A.status[cell] != 0) return;
  const ElimTask t = tasks[cell];
  const int nc = t.nc;
  if (p0 >= nc) return;
  const int pw = min(PB, nc - p0);
  double* F = A.fac + t.C_off;
  for (int e = threadIdx.x; e < pw * pw; e += 256) {
    const int i = e / pw, j = e - i * pw;
    D[i][j] = (j <= i) ? F[(size_t)(p0 + i) * nc + p0 + j] : 0.0;
  }
  double dm = DBL_MAX, prev_piv = 0.0, prev_inv = 0.0;
  for (int k = 0; k < pw; ++k) {
    __syncthreads();
    const double akk = D[k][k];
    if (!(akk > 0.0)) {
      if (threadIdx.x == 0) A.status[cell] = 1;
      return;
    }
    const double rakk = 1.0 / akk;
    dm = fmin(dm, akk);
    if (k > 0) {
      for (int i = k + threadIdx.x; i < pw; i += 256) D[i][k - 1] *= prev_inv;
      if (threadIdx.x == 0) D[k - 1][k - 1] = prev_piv;
    }
    for (int i = k + 1 + (int)(threadIdx.x >> 5); i < pw; i += 8) {  // warp per row
      const double dik = D[i][k];
      for (int j = k + 1 + (int)(threadIdx.x & 31); j <= i; j += 32) D[i][j] -= dik * (D[j][k] * rakk);
    }
    prev_piv = sqrt(akk);
    prev_inv = 1.0 / prev_piv;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    D[pw - 1][pw - 1] = prev_piv;
    dmin[cell] = fmin(dmin[cell], dm);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < pw * pw; e += 256) {
    const int i = e / pw, j = e - i * pw;
    if (j <= i) F[(size_t)(p0 + i) * nc + p0 + j] = D[i][j];
  }
}

// ---------------------------------------------------------------------------
// Panel triangular solves.  Work item int4 {cell, kind, start, 0}:
//   kind 0: rows [start, start+128) below the panel:  X L_pp^T = F_rows
//   kind 1: W columns [start, start+128):              L_pp Y = W_p
// One thread per row / column, L_pp and the chunk in shared memory.
// ---------------------------------------------------------------------------
constexpr int kChunk = 128;

__global__ void __launch_bounds__(kChunk) panel_trsm_kernel(const ElimTask* __restrict__ tasks,
                                                            const int4* __restrict__ work, int p0,
                                                            Arenas A) {
  extern __shared__ __align__(16) double dsm[];
  double (*Lp)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(dsm);
  double (*X)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(dsm + PB * (PB + 1));
  const int4 w = work[blockIdx.x];
  const int cell = w.x;
  if (A.status[cell] != 0) return;
  const ElimTask t = tasks[cell];
  const int nc = t.nc, nq = t.nq;
  if (p0 >= nc || (w.y == 0 ? w.z >= nc : w.z >= nq)) return;
  const int pw = min(PB, nc - p0);
  const double* F = A.fac + t.C_off;
  for (int e = threadIdx.x; e < pw * pw; e += kChunk) {
    const int i = e / pw, j = e - i * pw;
    Lp[i][j] = F[(size_t)(p0 + i) * nc + p0 + j];
  }
  if (w.y == 0) {
    double* Fw = A.fac + t.C_off;
    const int rows = min(kChunk, nc - w.z);
    for (int e = threadIdx.x; e < rows * pw; e += kChunk) {
      const int i = e / pw, j = e - i * pw;
      X[i][j] = Fw[(size_t)(w.z + i) * nc + p0 + j];
    }
    __syncthreads();
    const int i = threadIdx.x;
    if (i < rows) {
      for (int j = 0; j < pw; ++j) {
        double s = X[i][j];
        for (int l = 0; l < j; ++l) s -= X[i][l] * Lp[j][l];
        X[i][j] = s / Lp[j][j];
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * pw; e += kChunk) {
      const int r = e / pw, j = e - r * pw;
      Fw[(size_t)(w.z + r) * nc + p0 + j] = X[r][j];
    }
  } else {
    double* W = A.fac + t.W_off;
    const int cols = min(kChunk, nq - w.z);
    // X[j][i]: column j of the chunk, row i of the panel
    for (int e = threadIdx.x; e < pw * cols; e += kChunk) {
      const int i = e / cols, j = e - i * cols;
      X[j][i] = W[(size_t)(p0 + i) * nq + w.z + j];
    }
    __syncthreads();
    const int j = threadIdx.x;
    if (j < cols) {
      for (int i = 0; i < pw; ++i) {
        double s = X[j][i];
        for (int l = 0; l < i; ++l) s -= Lp[i][l] * X[j][l];
        X[j][i] = s / Lp[i][i];
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < pw * cols; e += kChunk) {
      const int i = e / cols, jj = e - i * cols;
      W[(size_t)(p0 + i) * nq + w.z + jj] = X[jj][i];
    }
  }
}

// ---------------------------------------------------------------------------
// Trailing update tiles.  Work item int4 {cell, kind, a0, b0} (64 x 64 tile):
//   kind 0: F[a0.., b0..] -= L[a0.., p] L[b0.., p]^T   (b0 <= a0; lower part)
//   kind 1: W[a0.., b0..] -= L[a0.., p] W[p, b0..]
// 128 threads = 2 x 2 warps of 32 x 32, FP64 DMMA m8n8k4.
// ---------------------------------------------------------------------------
constexpr int kT = 64, kKs = 16, kLd = 68;

__global__ void __launch_bounds__(128) panel_update_kernel(const ElimTask* __restrict__ tasks,
                                                           const int4* __restrict__ work, int p0,
                                                           Arenas A) {
  __shared__ double As[kKs][kLd];
  __shared__ double Bs[kKs][kLd];
  const int4 w = work[blockIdx.x];
  const int cell = w.x;
  if (A.status[cell] != 0) return;
  const ElimTask t = tasks[cell];
  const int nc = t.nc, nq = t.nq;
  const int a0 = w.z, b0 = w.w;
  if (p0 >= nc || a0 >= nc || (w.y == 1 && b0 >= nq)) return;
  const int pw = min(PB, nc - p0);
  double* F = A.fac + t.C_off;
  double* W = A.fac + t.W_off;
  const bool kindW = w.y == 1;
  const int nrow = nc, ncol = kindW ? nq : nc;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wy = wid >> 1, wx = wid & 1;
  double acc[4][4][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  for (int k0 = 0; k0 < pw; k0 += kKs) {
    __syncthreads();
    for (int e = threadIdx.x; e < kKs * kT; e += 128) {
      const int r = e / kKs, kk = e - r * kKs;   // row-major source: consecutive kk
      const int k = k0 + kk;
      const int ra = a0 + r;
      As[kk][r] = (k < pw && ra < nrow) ? F[(size_t)ra * nc + p0 + k] : 0.0;
      if (!kindW) {
        const int rb = b0 + r;
        Bs[kk][r] = (k < pw && rb < nrow) ? F[(size_t)rb * nc + p0 + k] : 0.0;
      }
    }
    if (kindW) {
      for (int e = threadIdx.x; e < kKs * kT; e += 128) {
        const int kk = e / kT, c = e - kk * kT;
        const int k = k0 + kk;
        Bs[kk][c] = (k < pw && b0 + c < ncol) ? W[(size_t)(p0 + k) * nq + b0 + c] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kKs; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) af[m] = As[kk + (lane & 3)][wy * 32 + m * 8 + (lane >> 2)];
#pragma unroll
      for (int n = 0; n < 4; ++n) bf[n] = Bs[kk + (lane & 3)][wx * 32 + n * 8 + (lane >> 2)];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) dmma_8x8x4(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
    }
  }
  const bool diag = !kindW && a0 == b0;
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = a0 + wy * 32 + m * 8 + (lane >> 2);
        const int b = b0 + wx * 32 + n * 8 + 2 * (lane & 3) + h;
        if (a >= nrow || b >= ncol) continue;
        if (kindW) W[(size_t)a * nq + b] -= acc[m][n][h];
        else if (!diag || b <= a) F[(size_t)a * nc + b] -= acc[m][n][h];
      }
}

// ---------------------------------------------------------------------------
// Finish: singular-pivot rule and the zero upper triangle of C.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) big_finish_kernel(const ElimTask* __restrict__ tasks, Arenas A,
                                                         const double* __restrict__ dmin,
                                                         const double* __restrict__ diag_scale) {
  const int cell = blockIdx.x;
  const ElimTask t = tasks[cell];
  const int nc = t.nc;
  double* F = A.fac + t.C_off;
  for (size_t e = threadIdx.x; e < (size_t)nc * nc; e += 256) {
    const int i = (int)(e / nc), j = (int)(e - (size_t)i * nc);
    if (j > i) F[e] = 0.0;
  }
  if (threadIdx.x == 0 && A.status[cell] == 0) {
    const double scale = diag_scale[cell];
    if (dmin[cell] <= kSingularRtol * fmax(scale, 1e-300)) A.status[cell] = 2;
  }
}

// Packed lower inverse of C for the solve: one thread per column (work item
// int4 {cell, col0}), C row-major in the record, P packed row-major.
__global__ void __launch_bounds__(128) big_inverse_kernel(const ElimTask* __restrict__ tasks,
                                                          const int4* __restrict__ work, Arenas A) {
  const int4 w = work[blockIdx.x];
  if (A.status[w.x] != 0) return;
  const ElimTask t = tasks[w.x];
  const int nc = t.nc;
  const int j = w.y + (int)threadIdx.x;
  if (j >= nc) return;
  const double* C = A.fac + t.C_off;
  double* P = A.fac + t.P_off;
  if (nc <= kInvLocal) {
    // the column lives in (L1-cached, thread-private) local memory
    double x[kInvLocal];
    x[j] = 1.0 / C[(size_t)j * nc + j];
    P[(size_t)j * (j + 1) / 2 + j] = x[j];
    for (int i = j + 1; i < nc; ++i) {
      const double* ci = C + (size_t)i * nc;
      double s0 = 0.0, s1 = 0.0;
      int l = j;
      for (; l + 1 < i; l += 2) {
        s0 += ci[l] * x[l];
        s1 += ci[l + 1] * x[l + 1];
      }
      if (l < i) s0 += ci[l] * x[l];
      x[i] = -(s0 + s1) / ci[i];
      P[(size_t)i * (i + 1) / 2 + j] = x[i];
    }
    return;
  }
  // larger cells take the blocked path (inv_diag_kernel / inv_tile_kernel)
}

// ---------------------------------------------------------------------------
// Blocked packed inverse P = C^-1 for large cells (nc > kInvLocal), right-
// looking over 64-wide panels.  P(i, j) lives at P[i(i+1)/2 + j], j <= i.
//   inv_diag_kernel:  P_pp = C_pp^-1 for every panel at once (1 CTA each);
//   inv_tile_kernel, panel p, work {cell, kind, i0, j0}:
//     kind 0 (j0 < p0):  P_pj := P_pp * S_pj,   S_pj accumulated in place;
//     kind 1 (i0 > p0):  P_ij := [P_ij] - C_ip * P_pj   (assign when j0 == p0).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(64) inv_diag_kernel(const ElimTask* __restrict__ tasks,
                                                      const int4* __restrict__ work, Arenas A) {
  __shared__ double L[PB][PB + 1];
  const int4 w = work[blockIdx.x];
  if (A.status[w.x] != 0) return;
  const ElimTask t = tasks[w.x];
  const int nc = t.nc, p0 = w.y;
  if (p0 >= nc) return;  // planned on an upper bound of nc (large skeleton groups)
  const int pw = min(PB, nc - p0);
  const double* C = A.fac + t.C_off;
  double* P = A.fac + t.P_off;
  for (int e = threadIdx.x; e < pw * pw; e += 64) {
    const int i = e / pw, j = e - i * pw;
    L[i][j] = j <= i ? C[(size_t)(p0 + i) * nc + p0 + j] : 0.0;
  }
  __syncthreads();
  const int j = threadIdx.x;
  if (j >= pw) return;
  double x[PB];  // column j of the inverse (thread-private)
  x[j] = 1.0 / L[j][j];
  P[(size_t)(p0 + j) * (p0 + j + 1) / 2 + p0 + j] = x[j];
  for (int i = j + 1; i < pw; ++i) {
    double s0 = 0.0;
    for (int l = j; l < i; ++l) s0 += L[i][l] * x[l];
    x[i] = -s0 / L[i][i];
    P[(size_t)(p0 + i) * (p0 + i + 1) / 2 + p0 + j] = x[i];
  }
}

__global__ void __launch_bounds__(128) inv_tile_kernel(const ElimTask* __restrict__ tasks,
                                                       const int4* __restrict__ work, int p0, Arenas A) {
  __shared__ double As[kKs][kLd];
  __shared__ double Bs[kKs][kLd];
  const int4 w = work[blockIdx.x];
  if (A.status[w.x] != 0) return;
  const ElimTask t = tasks[w.x];
  const int nc = t.nc;
  const bool upd = w.y == 1;
  const int i0 = w.z, j0 = w.w;
  if (p0 >= nc || (upd && i0 >= nc)) return;
  const int pw = min(PB, nc - p0);
  const double* C = A.fac + t.C_off;
  double* P = A.fac + t.P_off;
  auto pk = [](int i, int j) { return (size_t)i * (i + 1) / 2 + j; };
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wy = wid >> 1, wx = wid & 1;
  double acc[4][4][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  for (int k0 = 0; k0 < pw; k0 += kKs) {
    __syncthreads();
    for (int e = threadIdx.x; e < kKs * kT; e += 128) {
      const int r = e / kKs, kk = e - r * kKs;
      const int k = p0 + k0 + kk, ra = (upd ? i0 : p0) + r;
      double a = 0.0;
      if (k0 + kk < pw && ra < nc) {
        if (upd) a = C[(size_t)ra * nc + k];                 // C_ip
        else if (k <= ra) a = P[pk(ra, k)];                  // P_pp (lower)
      }
      As[kk][r] = a;
    }
    for (int e = threadIdx.x; e < kKs * kT; e += 128) {
      const int kk = e / kT, c = e - kk * kT;
      const int k = p0 + k0 + kk, cb = j0 + c;
      Bs[kk][c] = (k0 + kk < pw && cb <= k) ? P[pk(k, cb)] : 0.0;  // S_pj / P_pj
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kKs; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) af[m] = As[kk + (lane & 3)][wy * 32 + m * 8 + (lane >> 2)];
#pragma unroll
      for (int n = 0; n < 4; ++n) bf[n] = Bs[kk + (lane & 3)][wx * 32 + n * 8 + (lane >> 2)];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) dmma_8x8x4(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
    }
  }
  __syncthreads();  // kind 0 overwrites its own B operand
  const int r0 = upd ? i0 : p0;
  const bool first = j0 == p0;
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = r0 + wy * 32 + m * 8 + (lane >> 2);
        const int b = j0 + wx * 32 + n * 8 + 2 * (lane & 3) + h;
        if (a >= nc || b >= j0 + kT || b > a) continue;
        if (!upd) {
          if (b < p0) P[pk(a, b)] = acc[m][n][h];
        } else {
          const double old = first ? 0.0 : P[pk(a, b)];
          P[pk(a, b)] = old - acc[m][n][h];
        }
      }
}

// ---------------------------------------------------------------------------
void launch_big_inverse(const ElimTask* tasks, const int4* work, int nwork, const Arenas& A, cudaStream_t s) {
  if (nwork > 0) big_inverse_kernel<<<nwork, 128, 0, s>>>(tasks, work, A);
}

void launch_inv_diag(const ElimTask* tasks, const int4* work, int nwork, const Arenas& A, cudaStream_t s) {
  if (nwork > 0) inv_diag_kernel<<<nwork, 64, 0, s>>>(tasks, work, A);
}

void launch_inv_tiles(const ElimTask* tasks, const int4* work, int nwork, int p0, const Arenas& A,
                      cudaStream_t s) {
  if (nwork > 0) inv_tile_kernel<<<nwork, 128, 0, s>>>(tasks, work, p0, A);
}

void launch_big_assemble(const ElimTask* tasks, const int4* work, int nwork, const Arenas& A,
                         double* diag_scale, size_t smem, cudaStream_t s) {
  if (nwork <= 0) return;
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(big_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemCapBytes);
    once = true;
  }
  big_assemble_kernel<<<nwork, 256, smem, s>>>(tasks, work, A, diag_scale);
}

void launch_panel_chol(const ElimTask* tasks, const int32_t* cells, int ncells, int p0, const Arenas& A,
                       double* dmin, cudaStream_t s) {
  if (ncells <= 0) return;
  panel_chol_kernel<<<ncells, 256, 0, s>>>(tasks, cells, p0, A, dmin);
}

void launch_panel_trsm(const ElimTask* tasks, const int4* work, int nwork, int p0, const Arenas& A,
                       cudaStream_t s) {
  if (nwork <= 0) return;
  const size_t smem = sizeof(double) * (size_t)(PB + kChunk) * (PB + 1);
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(panel_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    once = true;
  }
  panel_trsm_kernel<<<nwork, kChunk, smem, s>>>(tasks, work, p0, A);
}

void launch_panel_update(const ElimTask* tasks, const int4* work, int nwork, int p0, const Arenas& A,
                         cudaStream_t s) {
  if (nwork <= 0) return;
  panel_update_kernel<<<nwork, 128, 0, s>>>(tasks, work, p0, A);
}

void launch_big_finish(const ElimTask* tasks, int ncells, const Arenas& A, const double* dmin,
                       const double* diag_scale, cudaStream_t s) {
  if (ncells <= 0) return;
  big_finish_kernel<<<ncells, 256, 0, s>>>(tasks, A, dmin, diag_scale);
}

}  // namespace hifde
