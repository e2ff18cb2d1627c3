// sm_100a kernels of the HIF-DE factorization.
//
// Work decomposition:
//   * elim_small_kernel  -- one CTA per cell whose whole front fits in shared
//                           memory: assembly, Cholesky, TRSM and Schur update.
//   * large cells        -- blocked multi-CTA path in kernels_big.cu; their
//                           Schur update U -= W^T W is done by
//   * schur_tile_kernel  -- many CTAs per cell, 64 x 64 tiles on FP64 DMMA
//                           tensor cores (mma.sync m8n8k4 f64).
//   * skel_kernel        -- one CTA per skeletonization group: ID by
//                           column-pivoted QR (LAPACK dlaqp2 pivoting and norm
//                           downdating, early stop at the rank cut), congruence,
//                           inner elimination of rd against sk, delta block.
//   * skel_ordered_kernel -- the same in the reference's sequential order, one
//                           cooperative launch with per-group done flags.
//   * skel_cluster_kernel -- exact order with a CTA cluster per large group
//                           (column slices, DSMEM pivot exchange).
//
// Reference semantics followed:
//   elimination   src/factor_ops.py:138-159, src/dense.py:187-219
//   skeletonize   src/factor_ops.py:162-214
//   CPQR / ID     src/dense.py:239-264
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda/atomic>

#include "hifde_internal.h"

namespace hifde {

namespace {

constexpr double kSingularRtol = 1e-14;  // src/dense.py:38

__device__ __forceinline__ int bsearch_i32(const int32_t* s, int n, int32_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (s[mid] < key) lo = mid + 1; else hi = mid;
  }
  return (lo < n && s[lo] == key) ? lo : -1;
}

// Position of global DOF g in the front (c ascending, then q ascending).
__device__ __forceinline__ int front_pos(const int32_t* dofs, int nc, int nq, int32_t g) {
  int p = bsearch_i32(dofs, nc, g);
  if (p >= 0) return p;
  p = bsearch_i32(dofs + nc, nq, g);
  return p >= 0 ? nc + p : -1;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum over aligned groups of G lanes (G a power of two <= 32)
__device__ __forceinline__ double group_sum(double v, int G) {
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Thread teams of the one-group device code: a whole CTA (the one-CTA
// kernels) or one warp of a multi-warp CTA that works on its own group
// (skel_warp_kernel); `sync` is the team's barrier.
template <int NT_>
struct CtaTeam {
  static constexpr int NT = NT_;
  __device__ __forceinline__ static int tid() { return (int)threadIdx.x; }
  __device__ __forceinline__ static void sync() { __syncthreads(); }
};
struct WarpTeam {
  static constexpr int NT = 32;
  __device__ __forceinline__ static int tid() { return (int)(threadIdx.x & 31); }
  __device__ __forceinline__ static void sync() { __syncwarp(); }
};

template <class Tm>
__device__ double block_max_t(double v, double* red) {
  constexpr int NT = Tm::NT;
  constexpr int NW = NT / 32;
  const int lane = Tm::tid() & 31, wid = Tm::tid() >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  Tm::sync();
  if (lane == 0) red[wid] = v;
  Tm::sync();
  double s = red[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) s = fmax(s, red[w]);
  return s;
}
template <int NT>
__device__ double block_max(double v, double* red) {
  return block_max_t<CtaTeam<NT>>(v, red);
}

__device__ __forceinline__ size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// In-place Cholesky of the lower triangle of A (n x n, row-major, ld).
// Right-looking with the column scaling deferred by one step, so every step
// needs a single barrier.  Status: 1 indefinite (pivot <= 0 or NaN, dpotrf
// info > 0), 2 singular (min D <= 1e-14 max|diag A|, src/dense.py:102-113).
template <class Tm>
__device__ int chol_1sync_t(double* A, int n, int ld, double* red) {
  constexpr int NT = Tm::NT;
  if (n == 0) return 0;
  double sc = 0.0;
  for (int i = Tm::tid(); i < n; i += NT) sc = fmax(sc, fabs(A[(size_t)i * ld + i]));
  double scale = block_max_t<Tm>(sc, red);
  if (scale == 0.0) {
    double s2 = 0.0;
    for (int e = Tm::tid(); e < n * n; e += NT) {
      const int i = e / n, j = e - i * n;
      if (j <= i) s2 = fmax(s2, fabs(A[(size_t)i * ld + j]));
    }
    scale = block_max_t<Tm>(s2, red);
  }
  double dmin = DBL_MAX, prev_piv = 0.0, prev_inv = 0.0;
  for (int k = 0; k < n; ++k) {
    Tm::sync();
    const double akk = A[(size_t)k * ld + k];
    if (!(akk > 0.0)) return 1;
    const double piv = sqrt(akk);
    const double rakk = 1.0 / akk;
    dmin = fmin(dmin, akk);
    if (k > 0) {  // finish column k-1 (no longer read by anyone)
      for (int i = k + Tm::tid(); i < n; i += NT) A[(size_t)i * ld + k - 1] *= prev_inv;
      if (Tm::tid() == 0) A[(size_t)(k - 1) * ld + k - 1] = prev_piv;
    }
    // trailing update, lower triangle: warp per row, lanes over columns.
    // A lane's column factors A[j][k] / akk are formed once per step (same
    // rounding as forming them per row) and kept in registers.
    const int lane = (int)(Tm::tid() & 31);
    if (n - k - 1 <= 128) {
      double tj[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int j = k + 1 + lane + 32 * m;
        tj[m] = j < n ? A[(size_t)j * ld + k] * rakk : 0.0;
      }
      for (int i = k + 1 + (int)(Tm::tid() >> 5); i < n; i += NT / 32) {
        const double aik = A[(size_t)i * ld + k];
        double* Ai = A + (size_t)i * ld;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int j = k + 1 + lane + 32 * m;
          if (j <= i) Ai[j] -= aik * tj[m];
        }
      }
    } else {
      for (int i = k + 1 + (int)(Tm::tid() >> 5); i < n; i += NT / 32) {
        const double aik = A[(size_t)i * ld + k];
        for (int j = k + 1 + lane; j <= i; j += 32) A[(size_t)i * ld + j] -= aik * (A[(size_t)j * ld + k] * rakk);
      }
    }
    prev_piv = piv;
    prev_inv = 1.0 / piv;
  }
  Tm::sync();
  if (Tm::tid() == 0) A[(size_t)(n - 1) * ld + n - 1] = prev_piv;
  Tm::sync();
  if (dmin <= kSingularRtol * fmax(scale, 1e-300)) return 2;
  return 0;
}
template <int NT>
__device__ int chol_1sync(double* A, int n, int ld, double* red) {
  return chol_1sync_t<CtaTeam<NT>>(A, n, ld, red);
}

// B (n x m, row-major, ldb) <- C^{-1} B, C lower (row-major, ldc); one barrier
// per row (row scaling deferred by one step).
template <class Tm>
__device__ void trsm_1sync_t(const double* C, int n, int ldc, double* B, int m, int ldb) {
  constexpr int NT = Tm::NT;
  double prev = 0.0;
  for (int i = 0; i < n; ++i) {
    Tm::sync();
    const double cinv = 1.0 / C[(size_t)i * ldc + i];
    if (i > 0)
      for (int j = Tm::tid(); j < m; j += NT) B[(size_t)(i - 1) * ldb + j] *= prev;
    for (int l = i + 1 + (int)(Tm::tid() >> 5); l < n; l += NT / 32) {  // warp per row
      const double c = C[(size_t)l * ldc + i];
      for (int j = (int)(Tm::tid() & 31); j < m; j += 32) B[(size_t)l * ldb + j] -= c * (B[(size_t)i * ldb + j] * cinv);
    }
    prev = cinv;
  }
  Tm::sync();
  if (n > 0)
    for (int j = Tm::tid(); j < m; j += NT) B[(size_t)(n - 1) * ldb + j] *= prev;
  Tm::sync();
}
template <int NT>
__device__ void trsm_1sync(const double* C, int n, int ldc, double* B, int m, int ldb) {
  trsm_1sync_t<CtaTeam<NT>>(C, n, ldc, B, m, ldb);
}

// Packed row-major lower inverse of the lower-triangular C (n x n, ld),
// written to P[i(i+1)/2 + j]; one thread per column, no barriers (each
// thread reads back only its own column).
// Packed lower-triangular front storage (row i at i (i + 1) / 2): the
// elimination kernels touch only the lower triangle of the symmetric front,
// so a front takes half the shared memory (twice the cells per SM).
struct PackedLower {
  double* p;
  __device__ __forceinline__ double* row(int i) const { return p + (size_t)i * (i + 1) / 2; }
};

template <int NT>
__device__ void tri_inverse_packed(PackedLower C, int n, double* __restrict__ P) {
  for (int j = threadIdx.x; j < n; j += NT) {
    P[(size_t)j * (j + 1) / 2 + j] = 1.0 / C.row(j)[j];
    for (int i = j + 1; i < n; ++i) {
      double s = 0.0;
      const double* Ci = C.row(i);
      for (int l = j; l < i; ++l) s += Ci[l] * P[(size_t)l * (l + 1) / 2 + j];
      P[(size_t)i * (i + 1) / 2 + j] = -s / Ci[i];
    }
  }
}

template <int NT>
__device__ void trsm_1sync(const double* C, int n, int ldc, double* B, int m, int ldb);

// Packed lower inverse via B = C^-1 I in the workspace X (n x n), then a
// coalesced packed store.  All threads busy, one barrier per row.
template <class Tm>
__device__ void tri_inverse_packed_ws_t(const double* C, int n, int ld, double* X, double* __restrict__ P) {
  constexpr int NT = Tm::NT;
  Tm::sync();
  for (int e = Tm::tid(); e < n * n; e += NT) {
    const int i = e / n, j = e - i * n;
    X[e] = (i == j) ? 1.0 : 0.0;
  }
  trsm_1sync_t<Tm>(C, n, ld, X, n, n);
  for (int e = Tm::tid(); e < n * n; e += NT) {
    const int i = e / n, j = e - i * n;
    if (j <= i) P[(size_t)i * (i + 1) / 2 + j] = X[e];
  }
}
template <int NT>
__device__ void tri_inverse_packed_ws(const double* C, int n, int ld, double* X, double* __restrict__ P) {
  tri_inverse_packed_ws_t<CtaTeam<NT>>(C, n, ld, X, P);
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Lower-triangular tile index tt -> (ti, tj), tj <= ti.
__device__ __forceinline__ void tri_tile(int tt, int& ti, int& tj) {
  int i = (int)((sqrtf(8.0f * (float)tt + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= tt) ++i;
  while (i * (i + 1) / 2 > tt) --i;
  ti = i;
  tj = tt - i * (i + 1) / 2;
}

// 8 x 8 diagonal block at (p0, p0) of F (pw <= 8 rows), factored by one warp
// in registers, lane l holding row l: L_kk = sqrt(a_kk), L_lk = a_lk / L_kk,
// a_lj -= L_lk L_jk (the scaled form: with the deferred-scaling association
// of chol_1sync instead, config 3's exact-tie rank decisions at levels
// 4.5-6.5 drift by -2..-5%).  The factor goes to Lp[l*8 + j] and its inverse
// diagonal to Lp[64 + l].
__device__ __forceinline__ void diag_factor_warp(PackedLower F, int p0, int pw, double* Lp, int& bad, double& dmin) {
  const int l = threadIdx.x & 31;
  double r[8];
  const double* Fl = F.row(p0 + (l < pw ? l : 0)) + p0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = (l < pw && j <= l) ? Fl[j] : 0.0;
  bool ok = true;  // (locals: the reference parameters were kept in local memory across the steps)
  double dm = dmin;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (k < pw) {  // warp-uniform
      const double akk = __shfl_sync(0xffffffffu, r[k], k);
      ok = ok && akk > 0.0;
      dm = fmin(dm, akk);
      const double lkk = sqrt(akk);
      const double inv = __drcp_rn(lkk);
      if (l == k) r[k] = lkk;
      else if (l > k) r[k] *= inv;
#pragma unroll
      for (int j = k + 1; j < 8; ++j) {
        const double ljk = __shfl_sync(0xffffffffu, r[k], j);
        if (j <= l && l < pw) r[j] -= r[k] * ljk;
      }
    }
  }
  if (!ok) bad = 1;
  dmin = dm;
  if (l < 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) Lp[l * 8 + j] = (l < pw && j <= l) ? r[j] : 0.0;
    double rl = r[0];  // r[l] without a dynamic register index (which sends r to local memory)
#pragma unroll
    for (int j = 1; j < 8; ++j)
      if (j == l) rl = r[j];
    Lp[64 + l] = l < pw ? __drcp_rn(rl) : 0.0;
  }
}

// Blocked partial Cholesky of a front F (nf x nf, row-major, ld nf; lower
// triangle used) over its first nc columns, 8-wide panels:
//   * every thread solves one row of the panel below the diagonal block;
//   * the trailing lower triangle takes the rank-8 update as 8 x 8 FP64 DMMA
//     tiles (mma.sync m8n8k4); warp 0 updates the next diagonal tile first
//     and factors it (diag_factor_warp) while the other warps update the rest
//     (look-ahead: the diagonal chain overlaps the trailing update).
// Two barriers per panel.  Afterwards F holds C (rows < nc), L_qc = W^T =
// F_qc C^-T (rows >= nc, columns < nc) and the lower triangle of U = F_qq -
// W^T W.  Status as chol_1sync: 1 indefinite (a pivot <= 0 or NaN), 2
// singular (min D <= 1e-14 max|diag A|, src/dense.py:102-113).
// Lw: 2 x 72 doubles (the factored diagonal block, double-buffered).
template <int NT>
__device__ int front_chol_blocked(PackedLower F, int nc, int nf, double* red, double* Lw) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __shared__ int s_bad;
  if (nc == 0) return 0;
  double sc = 0.0;
  for (int i = threadIdx.x; i < nc; i += NT) sc = fmax(sc, fabs(F.row(i)[i]));
  double scale = block_max<NT>(sc, red);
  if (scale == 0.0) {
    double s2 = 0.0;
    for (int e = threadIdx.x; e < nc * nc; e += NT) {
      const int i = e / nc, j = e - i * nc;
      if (j <= i) s2 = fmax(s2, fabs(F.row(i)[j]));
    }
    scale = block_max<NT>(s2, red);
  }
  double dmin = DBL_MAX;  // warp 0's
  int bad = 0;
  if (wid == 0) {
    diag_factor_warp(F, 0, min(8, nc), Lw, bad, dmin);
    if (lane == 0) s_bad = bad;
  }
  __syncthreads();
  int buf = 0;
  for (int p0 = 0; p0 < nc; p0 += 8) {
    if (s_bad) return 1;
    const int pw = min(8, nc - p0), p1 = p0 + pw;
    const double* Lp = Lw + 72 * buf;
    // panel below the diagonal block: row i <- row i C_pp^-T
    for (int i = p1 + threadIdx.x; i < nf; i += NT) {
      double x[8];
      double* Fi = F.row(i) + p0;
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = k < pw ? Fi[k] : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        double sk = x[k];
#pragma unroll
        for (int m = 0; m < k; ++m) sk -= x[m] * Lp[k * 8 + m];
        x[k] = k < pw ? sk * Lp[64 + k] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < pw) Fi[k] = x[k];
    }
    __syncthreads();
    // trailing lower triangle from p1: F[i][j] -= sum_k L[i][p0+k] L[j][p0+k];
    // tile 0 (the next diagonal block) by warp 0, which then factors it
    const int nt = (nf - p1 + 7) / 8, ntt = nt * (nt + 1) / 2;
    auto tile = [&](int ti, int tj) {
      const int rb = p1 + 8 * ti, cb = p1 + 8 * tj;
      double c0 = 0.0, c1 = 0.0;
      const int ra = rb + (lane >> 2), rc = cb + (lane >> 2);
      const double* Fa = F.row(ra < nf ? ra : p0) + p0;
      const double* Fc = F.row(rc < nf ? rc : p0) + p0;
#pragma unroll
      for (int ks = 0; ks < 8; ks += 4) {
        const int k = ks + (lane & 3);
        const double a = (k < pw && ra < nf) ? Fa[k] : 0.0;
        const double b = (k < pw && rc < nf) ? Fc[k] : 0.0;
        dmma_8x8x4(c0, c1, a, b);
      }
      const int row = rb + (lane >> 2);
      if (row < nf) {
        double* Fr = F.row(row);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = cb + 2 * (lane & 3) + h;
          if (col <= row) Fr[col] -= h ? c1 : c0;
        }
      }
    };
    if (wid == 0) {
      if (lane < pw) {  // this panel's factored diagonal block into place
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j <= lane) F.row(p0 + lane)[p0 + j] = Lp[lane * 8 + j];
      }
      if (ntt > 0) {
        tile(0, 0);
        __syncwarp();
        if (p1 < nc) {
          diag_factor_warp(F, p1, min(8, nc - p1), Lw + 72 * (buf ^ 1), bad, dmin);
          if (lane == 0) s_bad = bad;
        }
      }
      // warp 0's share beyond tile 0; (ti, tj) of tile tt = ti (ti + 1) / 2 + tj
      // advanced incrementally (tri_tile's float sqrt per tile was ~8% of the
      // samples)
      int ti = 0, tj = 0;
      for (int tt = NW; tt < ntt; tt += NW) {
        tj += NW;
        while (tj > ti) { tj -= ti + 1; ++ti; }
        tile(ti, tj);
      }
    } else {
      int ti, tj;
      tri_tile(wid, ti, tj);
      for (int tt = wid; tt < ntt; tt += NW) {
        tile(ti, tj);
        tj += NW;
        while (tj > ti) { tj -= ti + 1; ++ti; }
      }
    }
    buf ^= 1;
    __syncthreads();
  }
  if (threadIdx.x == 0) red[0] = dmin;  // warp 0 factored every diagonal block
  __syncthreads();
  dmin = red[0];
  __syncthreads();
  if (dmin <= kSingularRtol * fmax(scale, 1e-300)) return 2;
  return 0;
}

// In place: the lower C (n x n, row-major ld) becomes X = C^-1, block row by
// block row: X_b,<b = -C_bb^-1 (C_b,<b X_<b) (the product on DMMA tiles into
// Y, 8 x n), X_bb = C_bb^-1, by one thread per column.  The strictly upper
// part is not touched.
template <int NT>
__device__ void tri_inverse_inplace(PackedLower C, int n, double* Y, double* Lp) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int b0 = 0; b0 < n; b0 += 8) {
    const int bw = min(8, n - b0);
    __syncthreads();  // X_<b complete
    const int nct = (b0 + 7) / 8;
    for (int ct = wid; ct < nct; ct += NW) {
      const int j0 = 8 * ct;
      double c0 = 0.0, c1 = 0.0;
      for (int k0 = j0 & ~3; k0 < b0; k0 += 4) {  // X[k][j] = 0 for k < j
        const int k = k0 + (lane & 3);
        const int ra = b0 + (lane >> 2), jb = j0 + (lane >> 2);
        const double a = (ra < n && k < b0) ? C.row(ra)[k] : 0.0;
        const double b = (k < b0 && jb <= k) ? C.row(k)[jb] : 0.0;  // X, lower part only
        dmma_8x8x4(c0, c1, a, b);
      }
      const int row = lane >> 2;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = j0 + 2 * (lane & 3) + h;
        if (col < b0) Y[row * n + col] = h ? c1 : c0;
      }
    }
    if (threadIdx.x < 64) {  // the diagonal block and its inverse diagonal
      const int i = threadIdx.x >> 3, j = threadIdx.x & 7;
      Lp[threadIdx.x] = (i < bw && j <= i) ? C.row(b0 + i)[b0 + j] : 0.0;
      if (j == 0) Lp[64 + i] = i < bw ? 1.0 / C.row(b0 + i)[b0 + i] : 0.0;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < b0 + bw; j += NT) {  // columns of the block row
      double x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double sacc = (j == b0 + i ? 1.0 : 0.0) - (i < bw && j < b0 ? Y[i * n + j] : 0.0);
#pragma unroll
        for (int m = 0; m < i; ++m) sacc -= Lp[i * 8 + m] * x[m];
        x[i] = i < bw ? sacc * Lp[64 + i] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < bw && j <= b0 + i) C.row(b0 + i)[j] = x[i];
    }
  }
  __syncthreads();
}

}  // namespace

// ---------------------------------------------------------------------------
// Small cells: the whole front in shared memory.
// F = A0[c+q, c] parts + sum of consumed clique blocks; C C^T = F_cc;
// W = C^-1 F_cq; U = F_qq - W^T W.  Also the terminal block (nq == 0).
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(NT, 768 / NT) elim_small_kernel(const ElimTask* __restrict__ tasks, Arenas A) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[NT / 32];
  const ElimTask t = tasks[blockIdx.x];
  const int nc = t.nc, nq = t.nq, nf = nc + nq;
  int32_t* sdofs = reinterpret_cast<int32_t*>(smem);
  int32_t* smap = sdofs + nf;
  const size_t ibytes = align_up(sizeof(int32_t) * (size_t)(nf + t.maxnb), 16);
  double* Fp = reinterpret_cast<double*>(smem + ibytes);  // packed lower front, nf (nf + 1) / 2
  const PackedLower F{Fp};
  const int nfp = nf * (nf + 1) / 2;
  const int32_t* gd = A.idx + t.dofs_off;
  for (int i = threadIdx.x; i < nf; i += NT) sdofs[i] = gd[i];
  for (int i = threadIdx.x; i < nc; i += NT) A.active[gd[i]] = 0;  // the cell retires
  for (int e = threadIdx.x; e < nfp; e += NT) Fp[e] = 0.0;
  __syncthreads();
  // A0 rows of c: eight entry slots per row, so the loads of a row's entries
  // are in flight together (each front entry has one CSR entry: no races);
  // the lower triangle only: (p, pj) for pj <= p in c, (pj, p) for pj in q
  for (int e = threadIdx.x; e < 8 * nc; e += NT) {
    const int p = e >> 3, slot = e & 7;
    const int g = sdofs[p];
    const int64_t k0 = A.indptr[g], k1 = A.indptr[g + 1];
    for (int64_t k = k0 + slot; k < k1; k += 8) {
      const int pj = front_pos(sdofs, nc, nq, A.indices[k]);
      if (pj < 0) continue;
      if (pj > p && pj < nc) continue;  // upper part of A_cc (its mirror is in row pj)
      const double v = A.a0[k];
      if (pj >= nc) F.row(pj)[p] += v;
      else F.row(p)[pj] += v;
    }
  }
  __syncthreads();
  const int32_t* bl = A.lists + t.blk_off;
  for (int b = 0; b < t.nblk; ++b) {
    const int bid = bl[b];
    const int nb = A.blk_n[bid];
    const int32_t* bd = A.idx + A.blk_dof_off[bid];
    const double* bv = A.bvals + A.blk_val_off[bid];
    for (int k = threadIdx.x; k < nb; k += NT) smap[k] = front_pos(sdofs, nc, nq, bd[k]);
    __syncthreads();
    // warp per block row, four rows' loads in flight per lane
    for (int k0 = (int)(threadIdx.x >> 5) * 4; k0 < nb; k0 += NT / 8) {
      for (int l = (int)(threadIdx.x & 31); l < nb; l += 32) {
        const int pl = smap[l];
        double val[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) val[u] = (k0 + u < nb && pl >= 0) ? bv[(size_t)(k0 + u) * nb + l] : 0.0;
        if (pl < 0) continue;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (k0 + u >= nb) break;
          const int pk = smap[k0 + u];
          if (pk >= pl) F.row(pk)[pl] += val[u];  // the lower triangle (the block is symmetric)
        }
      }
    }
    __syncthreads();
  }
  __shared__ double Lw[2 * 72];
  const int st = front_chol_blocked<NT>(F, nc, nf, red, Lw);
  if (st != 0) {
    if (threadIdx.x == 0) A.status[blockIdx.x] = st;
    return;
  }
  // outputs: W = (L_qc)^T row-major nc x nq, U = F_qq - W^T W (symmetric from
  // its lower triangle), P = C^-1 packed
  if (nq > 0) {
    double* W = A.fac + t.W_off;
    for (int e = threadIdx.x; e < nc * nq; e += NT) {
      const int i = e / nq, j = e - i * nq;
      W[e] = F.row(nc + j)[i];
    }
    double* U = A.bvals + t.U_off;
    for (int e = threadIdx.x; e < nq * nq; e += NT) {
      const int a = e / nq, b = e - a * nq;
      const int hi = a > b ? a : b, lo = a > b ? b : a;
      U[e] = F.row(nc + hi)[nc + lo];
    }
  }
  // packed C^-1 for the solve: inverted in place (Y: the 8 x nc block-row
  // product, after the front); rows < nc of the packed front are then P
  if (t.scratch_off == -2) {
    tri_inverse_inplace<NT>(F, nc, Fp + nfp, Lw);
    double* P = A.fac + t.P_off;
    for (int e = threadIdx.x; e < nc * (nc + 1) / 2; e += NT) P[e] = Fp[e];
  } else {
    tri_inverse_packed<NT>(F, nc, A.fac + t.P_off);
  }
  if (threadIdx.x == 0) A.status[blockIdx.x] = 0;
}

// ---------------------------------------------------------------------------
// Large cells, Schur update: U[a,b] -= sum_k W[k,a] W[k,b] on 64 x 64 tiles
// (upper-triangular tile pairs, mirrored), FP64 DMMA m8n8k4.
// 128 threads = 2 x 2 warps, each warp a 32 x 32 sub-tile (4 x 4 MMA tiles).
// ---------------------------------------------------------------------------
constexpr int kTile = kSchurTile, kKc = 32, kLdS = 68;

// Rows of W are staged 32 at a time; the next stage is prefetched into
// registers while the DMMA loop runs on the current one.
__global__ void __launch_bounds__(128, 3) schur_tile_kernel(const ElimTask* __restrict__ tasks,
                                                         const int4* __restrict__ tiles, Arenas A) {
  __shared__ double Wa[kKc][kLdS];
  __shared__ double Wb[kKc][kLdS];
  const int4 tl = tiles[blockIdx.x];
  const ElimTask t = tasks[tl.x];
  const int nc = t.nc, nq = t.nq;
  const int a0 = tl.y * kTile, b0 = tl.z * kTile;
  if (a0 >= nq || b0 >= nq) return;
  const double* W = A.fac + t.W_off;
  double* U = A.bvals + t.U_off;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wy = wid >> 1, wx = wid & 1;
  double acc[4][4][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  double pa[16], pb[16];
  auto load = [&](int k0) {  // thread e = tid + 128 u: row e / 64, column e % 64 (coalesced)
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = (int)threadIdx.x + 128 * u;
      const int k = k0 + (e >> 6), aa = e & 63;
      pa[u] = (k < nc && a0 + aa < nq) ? W[(size_t)k * nq + a0 + aa] : 0.0;
      pb[u] = (k < nc && b0 + aa < nq) ? W[(size_t)k * nq + b0 + aa] : 0.0;
    }
  };
  load(0);
  for (int k0 = 0; k0 < nc; k0 += kKc) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = (int)threadIdx.x + 128 * u;
      Wa[e >> 6][e & 63] = pa[u];
      Wb[e >> 6][e & 63] = pb[u];
    }
    __syncthreads();
    if (k0 + kKc < nc) load(k0 + kKc);
#pragma unroll
    for (int kk = 0; kk < kKc; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) af[m] = Wa[kk + (lane & 3)][wy * 32 + m * 8 + (lane >> 2)];
#pragma unroll
      for (int n = 0; n < 4; ++n) bf[n] = Wb[kk + (lane & 3)][wx * 32 + n * 8 + (lane >> 2)];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) dmma_8x8x4(acc[m][n][0], acc[m][n][1], af[m], bf[n]);
    }
  }
  const bool diag = tl.y == tl.z;
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = a0 + wy * 32 + m * 8 + (lane >> 2);
        const int b = b0 + wx * 32 + n * 8 + 2 * (lane & 3) + h;
        if (a >= nq || b >= nq) continue;
        if (diag && b > a) continue;
        const double v = U[(size_t)a * nq + b] - acc[m][n][h];
        U[(size_t)a * nq + b] = v;
        if (a != b) U[(size_t)b * nq + a] = v;
      }
}

// ---------------------------------------------------------------------------
// Skeletonization of one group.
//   M = A[c+q, c]: A_cc (nc x nc) and Mq = A_qc (nq x nc), column-major.
//   CPQR of Mq: columns stay in place; every warp picks the pivot from the
//   double-buffered partial norms (LAPACK position map for ties) and G-lane
//   sub-warps update the trailing columns and downdate their norms -- one
//   barrier per step.  The Householder vectors are never needed again (only
//   R), so they are not even scaled into place.
// ---------------------------------------------------------------------------
struct NoWait {
  __device__ void operator()() const {}
};
// Full-rank certificate on / off (HIFDE_NO_RANK_CERT clears it: the tests'
// A/B against the plain pivoted QR, which must give the same records).
__device__ int d_rank_cert = 1;
static void rank_cert_init() {
  static const bool once = [] {
    if (getenv("HIFDE_NO_RANK_CERT")) {
      const int z = 0;
      cudaMemcpyToSymbol(d_rank_cert, &z, sizeof z);
    }
    return true;
  }();
  (void)once;
}
struct NoPublish {
  __device__ void operator()(int, const int32_t*, const int32_t*, int) const {}
};

// After the pivoted QR of a group: T = R11^-1 R12 from the R rows of Mq
// (columns in place, LAPACK order perm), ascending sk/rd lists, the
// congruence B_sr / B_rr from A_cc, the inner Cholesky, W, the delta block
// and the record (T | packed C^-1 | W).  Z is the post-CPQR workspace
// (3 q4 + 2 nc^2 doubles); red holds NT/32 partials.
template <class Tm>
__device__ void skel_tail_t(const SkelTask& t, const Arenas& A, int nc, int k, double* Mq, int ldm,
                          const int32_t* perm, int32_t* skl, int32_t* rdl, int32_t* sko, int32_t* rdo,
                          const int32_t* sdofs, const double* Acc, double* Z, double* red) {
  constexpr int NT = Tm::NT;
  const int r = nc - k;
  const size_t q4 = (size_t)nc * nc / 4 + nc;
  double* Ts = Z;                                      // k x r
  double* Bsr = Ts + q4;                               // k x r
  double* Wm = Bsr + q4;                               // r x k
  double* Brr = Wm + q4;                               // r x r
  // T = R11^-1 R12 (back substitution, one thread per column of R12)
  for (int j = Tm::tid(); j < r; j += NT) {
    double* col = Mq + (size_t)perm[k + j] * ldm;
    for (int i = k - 1; i >= 0; --i) {
      double s = col[i];
      for (int l = i + 1; l < k; ++l) s -= Mq[i + (size_t)perm[l] * ldm] * col[l];
      col[i] = s / Mq[i + (size_t)perm[i] * ldm];
    }
  }
  // ascending sk / rd with their pivot positions
  for (int a = Tm::tid(); a < nc; a += NT) {
    const int pv = perm[a];
    int rank = 0;
    if (a < k) {
      for (int b = 0; b < k; ++b) rank += perm[b] < pv;
      skl[rank] = pv;
      sko[rank] = a;
    } else {
      for (int b = k; b < nc; ++b) rank += perm[b] < pv;
      rdl[rank] = pv;
      rdo[rank] = a - k;
    }
  }
  Tm::sync();
  int32_t* out = A.idx + t.out_off;
  for (int a = Tm::tid(); a < k; a += NT) out[a] = sdofs[skl[a]];
  for (int a = Tm::tid(); a < r; a += NT) out[k + a] = sdofs[rdl[a]];
  if (Tm::tid() == 0) A.kout[t.group] = k;
  if (r == 0) {
    if (Tm::tid() == 0) A.status[t.group] = 0;
    return;
  }
  for (int e = Tm::tid(); e < k * r; e += NT) {
    const int a = e / r, b = e - a * r;
    Ts[e] = Mq[sko[a] + (size_t)perm[k + rdo[b]] * ldm];
  }
  Tm::sync();
  // B_sr = A_sr - A_ss T
  for (int e = Tm::tid(); e < k * r; e += NT) {
    const int a = e / r, b = e - a * r;
    const double* arow = Acc + skl[a] * nc;
    double s = arow[rdl[b]];
    for (int l = 0; l < k; ++l) s -= arow[skl[l]] * Ts[l * r + b];
    Bsr[e] = s;
  }
  Tm::sync();
  // B_rr = A_rr - A_sr^T T - T^T B_sr  (then symmetrized)
  for (int e = Tm::tid(); e < r * r; e += NT) {
    const int a = e / r, b = e - a * r;
    double s = Acc[rdl[a] * nc + rdl[b]];
    for (int l = 0; l < k; ++l)
      s -= Acc[skl[l] * nc + rdl[a]] * Ts[l * r + b] + Ts[l * r + a] * Bsr[l * r + b];
    Brr[e] = s;
  }
  Tm::sync();
  for (int e = Tm::tid(); e < r * r; e += NT) {
    const int a = e / r, b = e - a * r;
    if (a < b) {
      const double m = 0.5 * (Brr[e] + Brr[b * r + a]);
      Brr[e] = m;
      Brr[b * r + a] = m;
    }
  }
  Tm::sync();
  const int st = chol_1sync_t<Tm>(Brr, r, r, red);
  if (st != 0) {
    if (Tm::tid() == 0) A.status[t.group] = st;
    return;
  }
  for (int e = Tm::tid(); e < r * k; e += NT) {
    const int a = e / k, b = e - a * k;
    Wm[e] = Bsr[b * r + a];
  }
  if (k > 0) trsm_1sync_t<Tm>(Brr, r, r, Wm, k, k);
  Tm::sync();
  double* dl = A.bvals + t.delta_off;
  for (int e = Tm::tid(); e < k * k; e += NT) {
    const int a = e / k, b = e - a * k;
    double s = 0.0;
    for (int l = 0; l < r; ++l) s -= Wm[l * k + a] * Wm[l * k + b];
    dl[e] = s;
  }
  double* rec = A.fac + t.rec_off;
  for (int e = Tm::tid(); e < k * r; e += NT) rec[e] = Ts[e];
  double* C = rec + (size_t)k * r;
  tri_inverse_packed_ws_t<Tm>(Brr, r, r, Brr + (size_t)nc * nc, C);  // packed C^-1 for the solve
  double* Wo = C + (size_t)r * r;
  for (int e = Tm::tid(); e < r * k; e += NT) Wo[e] = Wm[e];
  if (Tm::tid() == 0) A.status[t.group] = 0;
}
template <int NT>
__device__ void skel_tail(const SkelTask& t, const Arenas& A, int nc, int k, double* Mq, int ldm,
                          const int32_t* perm, int32_t* skl, int32_t* rdl, int32_t* sko, int32_t* rdo,
                          const int32_t* sdofs, const double* Acc, double* Z, double* red) {
  skel_tail_t<CtaTeam<NT>>(t, A, nc, k, Mq, ldm, perm, skl, rdl, sko, rdo, sdofs, Acc, Z, red);
}

// One skeletonization group.  The front is assembled assuming every neighbour
// row is alive, then `wait()` runs (exact order: until the earlier
// neighbouring groups are done), then rows of DOFs retired meanwhile are
// zeroed -- so the assembly is off the dependency chain's critical path.
// red: NT / 32 doubles, shk: one int -- the team's shared scalars.
// GNT: the CTA size whose lane split (lanes per column) the CPQR uses, so a
// warp team reproduces the GNT-thread CTA's sums exactly.
template <class Tm, int GNT, class Wait, class Publish = NoPublish>
__device__ void skel_group_t(const SkelTask& t, const Arenas& A, double eps, unsigned char* smem, const Wait& wait,
                             const Publish& publish, double* red, int* shk) {
  constexpr int NT = Tm::NT;
  constexpr int NW = NT / 32;
  int& sh_k = *shk;
  const int nc = t.nc, nq = t.nq, nf = nc + nq;
  const int lane = Tm::tid() & 31, wid = Tm::tid() >> 5;
  auto mark = [&](int which) {  // debug timestamps (HIFDE_SKEL_TLOG)
    if (A.tlog && Tm::tid() == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      A.tlog[(size_t)t.group * 16 + which] = g;
    }
  };

  int32_t* sdofs = reinterpret_cast<int32_t*>(smem);
  int32_t* salive = sdofs + nf;
  int32_t* smap = salive + nf;
  int32_t* perm = smap + t.maxnb;
  int32_t* skl = perm + nc;
  int32_t* rdl = skl + nc;
  int32_t* sko = rdl + nc;
  int32_t* rdo = sko + nc;
  int32_t* dcol = rdo + nc;                            // column pivoted yet
  int32_t* cpos = dcol + nc;                           // LAPACK position -> column, x2
  const size_t ibytes = align_up(sizeof(int32_t) * (size_t)(2 * nf + t.maxnb + 8 * nc), 16);
  // CPQR vectors (double-buffered norms, next-step Householder norms, R_ii)
  double* cq = reinterpret_cast<double*>(smem + ibytes);
  double* rdiag = cq + 4 * nc;                         // vn1 x2 | xn x2 | R_ii
  // workspace placement (host-chosen): 0 all shared; 1 Mq + norms shared,
  // A_cc and the post-CPQR matrices global; 2 all global
  double* wsh = cq + 5 * nc;
  double* wgl = A.scratch + (t.scratch_off > 0 ? t.scratch_off : 0);
  const int ldq = t.mode <= 1 ? skel_ldq(nq) : nq;    // Mq column-major (padded in shared memory)
  double *Acc, *Mq, *vn1, *vn2, *Z;
  if (t.mode == 1) {
    Mq = wsh;
    vn1 = Mq + (size_t)ldq * nc;
    vn2 = vn1 + nc;
    Acc = wgl;
    Z = Acc + (size_t)nc * nc;
  } else if (t.mode == 3) {  // Mq in global, compressed to its R factor in shared memory
    Acc = wgl;
    Mq = Acc + (size_t)nc * nc;
    Z = Mq + (size_t)nq * nc;
    vn1 = wsh + (size_t)(nc + t.chunk) * nc;
    vn2 = vn1 + nc;
  } else {
    double* ws = t.mode == 0 ? wsh : wgl;
    Acc = ws;                                          // nc x nc, row-major (symmetric)
    Mq = Acc + (size_t)nc * nc;                        // nq x nc, ld ldq
    vn1 = Mq + (size_t)ldq * nc;
    vn2 = vn1 + nc;
    Z = vn2 + nc;                                      // post-CPQR workspace
  }

  const int32_t* gd = A.idx + t.dofs_off;
  for (int i = Tm::tid(); i < nf; i += NT) {
    const int g = gd[i];
    sdofs[i] = g;
    salive[i] = 1;
  }
  for (int i = Tm::tid(); i < nc; i += NT) perm[i] = i;
  for (int e = Tm::tid(); e < nc * nc; e += NT) Acc[e] = 0.0;
  for (size_t e = Tm::tid(); e < (size_t)ldq * nc; e += NT) Mq[e] = 0.0;
  Tm::sync();
  for (int p = Tm::tid(); p < nc; p += NT) {
    const int g = sdofs[p];
    for (int64_t k = A.indptr[g]; k < A.indptr[g + 1]; ++k) {
      const int pj = front_pos(sdofs, nc, nq, A.indices[k]);
      if (pj < 0 || !salive[pj]) continue;
      const double v = A.a0[k];
      if (pj < nc) Acc[p * nc + pj] += v;
      else Mq[(pj - nc) + (size_t)p * ldq] += v;
    }
  }
  Tm::sync();
  const int32_t* bl = A.lists + t.blk_off;
  for (int b = 0; b < t.nblk; ++b) {
    const int bid = bl[b];
    const int nb = A.blk_n[bid];
    const int32_t* bd = A.idx + A.blk_dof_off[bid];
    const double* bv = A.bvals + A.blk_val_off[bid];
    if (Tm::tid() == 0) sh_k = 0;
    Tm::sync();
    for (int k = Tm::tid(); k < nb; k += NT) {
      const int p = front_pos(sdofs, nc, nq, bd[k]);
      smap[k] = (p >= 0 && salive[p]) ? p : -1;
      if (p >= 0 && p < nc && salive[p]) skl[atomicAdd(&sh_k, 1)] = k;  // block columns landing in c
    }
    Tm::sync();
    // only the columns of c are assembled (A_cc and Mq = A_qc): warp per
    // block row over the compact column list, four rows' loads in flight per
    // lane (each front entry still takes one add per block)
    const int ncc = sh_k;
    if (ncc <= 16) {
      // few columns land in c (the small groups): a warp per block row would
      // leave most lanes idle, so the (row, column) pairs are dealt to the
      // threads instead, four loads in flight per thread
      const int total = nb * ncc;
      const float rcc = 1.0f / (float)ncc;
      for (int e0 = (int)Tm::tid(); e0 < total; e0 += 4 * NT) {
        double val[4];
        int pk[4], pl[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = e0 + u * NT;
          pk[u] = -1;
          pl[u] = 0;
          val[u] = 0.0;
          if (e < total) {
            int kr = (int)((float)e * rcc);
            if (kr * ncc > e) --kr;
            else if ((kr + 1) * ncc <= e) ++kr;
            const int l = skl[e - kr * ncc];
            pl[u] = smap[l];
            pk[u] = smap[kr];
            if (pk[u] >= 0) val[u] = bv[(size_t)kr * nb + l];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (pk[u] < 0) continue;
          if (pk[u] < nc) Acc[pk[u] * nc + pl[u]] += val[u];
          else Mq[(pk[u] - nc) + (size_t)pl[u] * ldq] += val[u];
        }
      }
    } else
    for (int k0 = (int)(Tm::tid() >> 5) * 4; k0 < nb; k0 += NT / 8) {
      for (int j = (int)(Tm::tid() & 31); j < ncc; j += 32) {
        const int l = skl[j], pl = smap[l];
        double val[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) val[u] = (k0 + u < nb && smap[k0 + u] >= 0) ? bv[(size_t)(k0 + u) * nb + l] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (k0 + u >= nb) break;
          const int pk = smap[k0 + u];
          if (pk < 0) continue;
          if (pk < nc) Acc[pk * nc + pl] += val[u];
          else Mq[(pk - nc) + (size_t)pl * ldq] += val[u];
        }
      }
    }
    Tm::sync();
  }

  wait();
  Tm::sync();
  // rows of DOFs retired by earlier groups (written by other CTAs)
  for (int i = nc + Tm::tid(); i < nf; i += NT) {
    if (!__ldcg(A.active + sdofs[i])) {
      salive[i] = 0;
      for (int j = 0; j < nc; ++j) Mq[(size_t)(i - nc) + (size_t)j * ldq] = 0.0;
    }
  }
  Tm::sync();
  mark(4);

  // ---- mode 3: R factor of Mq by chunked Householder QR in shared memory --
  // [R ; chunk] is reduced column by column.  G lanes per trailing column,
  // all trailing columns at once; the chunk norm of column i + 1 is
  // accumulated while it is updated at step i, so every thread builds the
  // reflector itself and a column step has one barrier.
  int nqm = nq, ldm = ldq;
  if (t.mode == 3) {
    const int h = t.chunk, lds = nc + h;
    double* S = wsh;
    double* cn2 = cq;  // chunk-part squared norms (the CPQR vectors are not live yet)
    int Gq = 32;
    while (Gq > 8 && GNT / Gq < nc) Gq >>= 1;  // the lane split of a GNT-thread CTA (same sums)
    const int nsq = NT / Gq, slq = lane & (Gq - 1), slotq = wid * (32 / Gq) + lane / Gq;
    for (int e = Tm::tid(); e < lds * nc; e += NT) S[e] = 0.0;
    for (int r0 = 0; r0 < nq; r0 += h) {
      const int hh = min(h, nq - r0);
      Tm::sync();
      for (int e = Tm::tid(); e < h * nc; e += NT) {
        const int j = e / h, rr = e - j * h;
        S[nc + rr + (size_t)j * lds] = rr < hh ? Mq[(size_t)(r0 + rr) + (size_t)j * ldq] : 0.0;
      }
      Tm::sync();
      for (int base = 0; base < nc; base += nsq) {
        const int j = base + slotq;
        const double* col = S + (size_t)min(j, nc - 1) * lds;
        double a = 0.0;
        for (int r = nc + slq; r < nc + hh; r += Gq) a += col[r] * col[r];
        a = group_sum(a, Gq);
        if (j < nc && slq == 0) cn2[j] = a;
      }
      Tm::sync();
      for (int i = 0; i < nc; ++i) {
        // x = [S_ii ; chunk rows of column i]; the R rows below i are zero
        const double* v = S + (size_t)i * lds;
        const double xnorm = sqrt(cn2[i]);
        const double alpha = v[i];
        double beta, tau, scal;
        if (xnorm == 0.0) { beta = alpha; tau = 0.0; scal = 0.0; }
        else {
          beta = -copysign(hypot(alpha, xnorm), alpha);
          tau = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
        if (tau != 0.0) {
          for (int base = i + 1; base < nc; base += nsq) {
            const int j = base + slotq;
            const bool act = j < nc;
            double* col = S + (size_t)(act ? j : i) * lds;  // inactive: harmless reads of v
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int r = nc + slq;
            const int rend = act ? nc + hh : 0;  // inactive slots: no loads, shuffles only
            for (; r + 3 * Gq < rend; r += 4 * Gq) {
              s0 += v[r] * col[r];
              s1 += v[r + Gq] * col[r + Gq];
              s2 += v[r + 2 * Gq] * col[r + 2 * Gq];
              s3 += v[r + 3 * Gq] * col[r + 3 * Gq];
            }
            for (; r < rend; r += Gq) s0 += v[r] * col[r];
            const double sd = group_sum((s0 + s1) + (s2 + s3), Gq);
            const double w = tau * (col[i] + scal * sd);
            const double ws2 = w * scal;
            double a0 = 0.0, a1 = 0.0;
            r = nc + slq;
            for (; r + Gq < rend; r += 2 * Gq) {
              const double x0 = col[r] - ws2 * v[r];
              const double x1 = col[r + Gq] - ws2 * v[r + Gq];
              if (act) {
                col[r] = x0;
                col[r + Gq] = x1;
              }
              a0 += x0 * x0;
              a1 += x1 * x1;
            }
            for (; r < rend; r += Gq) {
              const double x = col[r] - ws2 * v[r];
              if (act) col[r] = x;
              a0 += x * x;
            }
            const double an = group_sum(a0 + a1, Gq);
            if (act && slq == 0) {
              col[i] -= w;
              cn2[j] = an;
            }
          }
        }
        Tm::sync();
        if (Tm::tid() == 0) S[i + (size_t)i * lds] = beta;
      }
    }
    Tm::sync();
    Mq = S;      // the CPQR runs on R (nc x nc, column-major, ld lds)
    nqm = nc;
    ldm = lds;
  }

  // ---- CPQR (dgeqp3 pivoting) of the shared-memory matrix Mc ----------
  // Columns are never moved: every warp tracks the LAPACK column order in
  // registers (position -> column, identical copies), picks the pivot itself
  // from the double-buffered partial norms, and the next step's Householder
  // norm of every candidate is accumulated during the update -- one barrier
  // per step.
  double* Mc = t.mode == 0 ? wsh + (size_t)nc * nc : wsh;
  if (t.mode != 3) { nqm = nq; ldm = ldq; }
  // ---- full-rank certificate (small groups, eps well above rounding) ------
  // Every |R_ii| of the pivoted QR is at least sigma_min(Mq), and R_11 is the
  // largest column norm.  If G - tau^2 I (G = Mq^T Mq, tau = kCertSafety eps
  // max_j |Mq e_j|) has an LDL^T with pivots above tau^2, then sigma_min > tau
  // and no pivot can reach the cut eps |R_11| (tau^2 is >= 1e-11 |G|, five
  // orders above the rounding of G and of its factorization): the rank is nc,
  // sk = c, nothing is eliminated -- the same record the QR ends in, without
  // its nc dependent pivot steps.  A group that fails the test takes the QR.
  bool certified = false;
  if (t.mode == 0 && nc <= kCertMaxNc && nqm >= nc && eps >= kCertMinEps && d_rank_cert) {
    double* Gm = Z;  // nc x nc (lower triangle used); Z is idle until the tail
    const int npair = nc * (nc + 1) / 2;
    for (int e = Tm::tid(); e < npair; e += NT) {
      int a = 0;
      while ((a + 1) * (a + 2) / 2 <= e) ++a;
      const int b = e - a * (a + 1) / 2;  // b <= a
      const double* ca = Mc + (size_t)a * ldm;
      const double* cb = Mc + (size_t)b * ldm;
      double s0 = 0.0, s1 = 0.0;
      int r = 0;
      for (; r + 1 < nqm; r += 2) {
        s0 += ca[r] * cb[r];
        s1 += ca[r + 1] * cb[r + 1];
      }
      if (r < nqm) s0 += ca[r] * cb[r];
      Gm[a * nc + b] = s0 + s1;
    }
    Tm::sync();
    double gmax = 0.0;
    for (int j = 0; j < nc; ++j) gmax = fmax(gmax, Gm[j * nc + j]);
    const double tau2 = (kCertSafety * eps) * (kCertSafety * eps) * gmax;
    certified = gmax > 0.0;
    for (int j = 0; j < nc && certified; ++j) {
      const double d = Gm[j * nc + j] - tau2;  // the same value in every thread
      if (!(d > tau2)) { certified = false; break; }
      const double dinv = 1.0 / d;
      const int m = nc - 1 - j, mp = m * (m + 1) / 2;
      for (int e = Tm::tid(); e < mp; e += NT) {
        int a = 0;
        while ((a + 1) * (a + 2) / 2 <= e) ++a;
        const int b = e - a * (a + 1) / 2;
        const int ia = j + 1 + a, ib = j + 1 + b;
        Gm[ia * nc + ib] -= Gm[ia * nc + j] * Gm[ib * nc + j] * dinv;
      }
      Tm::sync();
    }
    if (certified) {
      for (int pos = Tm::tid(); pos < 2 * nc; pos += NT) cpos[pos] = pos < nc ? pos : pos - nc;
      Tm::sync();
    }
  }
  int nq_alive = 0;
  if (Tm::tid() == 0 && !certified) {
    for (int i = nc; i < nf; ++i) nq_alive += salive[i];
    sh_k = nq_alive;
  }
  for (int j = wid; j < nc && !certified; j += NW) {
    const double* col = Mc + (size_t)j * ldm;
    double s1 = 0.0;
    for (int r = 1 + lane; r < nqm; r += 32) s1 += col[r] * col[r];
    s1 = warp_sum(s1);                            // rows >= 1
    const double c0 = nqm > 0 ? col[0] : 0.0;
    if (lane == 0) {
      const double nv = sqrt(c0 * c0 + s1);
      cq[j] = nv;
      vn2[j] = nv;
      cq[2 * nc + j] = sqrt(s1);
      dcol[j] = 0;
      cpos[j] = j;
    }
  }
  Tm::sync();
  mark(5);
  nq_alive = sh_k;
  const int kmax = nqm < nc ? nqm : nc;
  const double tol3z = sqrt(DBL_EPSILON * 0.5);  // sqrt(dlamch('E'))
  int G = 32;  // lanes per trailing column
  while (G > 8 && GNT / G < nc) G >>= 1;  // the lane split of a GNT-thread CTA (same sums)
  const int nslots = NT / G, sl = lane & (G - 1), slot = wid * (32 / G) + lane / G;
  double thr = 0.0;
  int k = kmax;
  for (int i = 0; i < kmax && !certified; ++i) {
    const int cur = (i & 1) * nc, nxt = nc - cur;
    const double* vn1 = cq + cur;
    double* vn1o = cq + nxt;
    const double* xn = cq + 2 * nc + cur;
    double* xno = cq + 2 * nc + nxt;
    const int32_t* cat = cpos + cur;
    int32_t* cato = cpos + nxt;
    // pivot: largest partial norm, lowest position on ties (idamax)
    double bv = -1.0;
    int bp = nc, bc = 0;
    for (int pos = i + lane; pos < nc; pos += 32) {
      const int c = cat[pos];
      const double v = vn1[c];
      if (v > bv) { bv = v; bp = pos; bc = c; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; bc = oc; }
    }
    const int p = bc;
    if (wid == NW - 1) {  // next position map: LAPACK swaps positions i and bp
      const int ci = cat[i];
      for (int pos = lane; pos < nc; pos += 32) cato[pos] = pos == i ? p : (pos == bp ? ci : cat[pos]);
    }
    if (i == 0 && bv == 0.0) { k = 0; break; }  // zero block: everything redundant
    const double* v = Mc + (size_t)p * ldm;     // Householder vector: rows > i
    const double alpha = v[i];
    const double xnorm = xn[p];
    double beta, tau, scal;
    if (xnorm == 0.0) { beta = alpha; tau = 0.0; scal = 0.0; }
    else {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    const double rii = fabs(beta);
    if (i == 0) thr = eps > 0.0 ? eps * rii : (double)(nq_alive > nc ? nq_alive : nc) * DBL_EPSILON * rii;
    if (rii <= thr) { k = i; break; }
    if (Tm::tid() == 0) { rdiag[i] = beta; dcol[p] = 1; }
    // trailing columns: G lanes per column, NT / G columns at once (the
    // step's latency is one column's dependency chain, not NW of them)
    for (int base = 0; base < nc; base += nslots) {
      const int j = base + slot;
      const bool act = j < nc && j != p && !dcol[j];
      double* col = Mc + (size_t)(act ? j : p) * ldm;  // inactive: harmless reads of v
      const int nqa = act ? nqm : 0;                   // inactive slots: no row loads, shuffles only
      double acc = 0.0;                                // sum of squares of rows >= i + 2
      if (tau != 0.0) {
        // 4 rows in flight per lane: the loops are load-latency bound
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int r = i + 1 + sl;
        for (; r + 3 * G < nqa; r += 4 * G) {
          s0 += v[r] * col[r];
          s1 += v[r + G] * col[r + G];
          s2 += v[r + 2 * G] * col[r + 2 * G];
          s3 += v[r + 3 * G] * col[r + 3 * G];
        }
        for (; r < nqa; r += G) s0 += v[r] * col[r];
        const double sd = group_sum((s0 + s1) + (s2 + s3), G);
        const double w = tau * (col[i] + scal * sd);
        __syncwarp();
        if (act && sl == 0) col[i] -= w;
        const double ws2 = w * scal;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        r = i + 1 + sl;
        if (r == i + 1 && r < nqa) {  // row i + 1: updated, not in the next norm
          const double x = col[r] - ws2 * v[r];
          col[r] = x;
          r += G;
        }
        for (; r + 3 * G < nqa; r += 4 * G) {
          const double x0 = col[r] - ws2 * v[r];
          const double x1 = col[r + G] - ws2 * v[r + G];
          const double x2 = col[r + 2 * G] - ws2 * v[r + 2 * G];
          const double x3 = col[r + 3 * G] - ws2 * v[r + 3 * G];
          col[r] = x0;
          col[r + G] = x1;
          col[r + 2 * G] = x2;
          col[r + 3 * G] = x3;
          a0 += x0 * x0;
          a1 += x1 * x1;
          a2 += x2 * x2;
          a3 += x3 * x3;
        }
        for (; r < nqa; r += G) {
          const double x = col[r] - ws2 * v[r];
          col[r] = x;
          a0 += x * x;
        }
        acc = (a0 + a1) + (a2 + a3);
      } else {
        double a0 = 0.0, a1 = 0.0;
        int r = i + 2 + sl;
        for (; r + G < nqa; r += 2 * G) {
          a0 += col[r] * col[r];
          a1 += col[r + G] * col[r + G];
        }
        for (; r < nqa; r += G) a0 += col[r] * col[r];
        acc = a0 + a1;
      }
      acc = group_sum(acc, G);
      __syncwarp();
      if (act) {
        const double cn = i + 1 < nqm ? col[i + 1] : 0.0;
        double nv = vn1[j];
        if (nv != 0.0) {
          double tmp = fabs(col[i]) / nv;
          tmp = 1.0 - tmp * tmp;
          tmp = tmp > 0.0 ? tmp : 0.0;
          const double ratio = nv / vn2[j];
          if (tmp * ratio * ratio <= tol3z) {
            nv = (i + 1 < nqm) ? sqrt(cn * cn + acc) : 0.0;
            if (sl == 0) vn2[j] = nv;
          } else {
            nv *= sqrt(tmp);
          }
        }
        if (sl == 0) { vn1o[j] = nv; xno[j] = sqrt(acc); }
      }
    }
    Tm::sync();
  }
  mark(6);
  // LAPACK order of the columns (the redundant ones as of step k), R_ii into place
  {
    const int32_t* cat = cpos + (k & 1) * nc;
    for (int pos = Tm::tid(); pos < nc; pos += NT) perm[pos] = cat[pos];
  }
  Tm::sync();
  if (!certified)
    for (int i = Tm::tid(); i < k; i += NT) Mc[i + (size_t)perm[i] * ldm] = rdiag[i];
  Mq = Mc;
  Tm::sync();
  // the redundant set is known: later groups may start (exact order) while
  // this one finishes its interpolation and elimination off the chain
  publish(k, perm, sdofs, nc);

  skel_tail_t<Tm>(t, A, nc, k, Mq, ldm, perm, skl, rdl, sko, rdo, sdofs, Acc, Z, red);
}
template <int NT, class Wait, class Publish = NoPublish>
__device__ void skel_group(const SkelTask& t, const Arenas& A, double eps, unsigned char* smem, const Wait& wait,
                           const Publish& publish = Publish{}) {
  __shared__ double red[NT / 32];
  __shared__ int sh_k;
  skel_group_t<CtaTeam<NT>, NT>(t, A, eps, smem, wait, publish, red, &sh_k);
}

template <int NT>
__global__ void __launch_bounds__(NT) skel_kernel(const SkelTask* __restrict__ tasks, Arenas A, double eps) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SkelTask t = tasks[blockIdx.x];
  skel_group<NT>(t, A, eps, smem, NoWait{});
}

// A group per CTA of NTC threads with the lane split of a GNT-thread CTA
// (bit-identical to skel_kernel<GNT>): smaller CTAs, more groups per SM.
template <int NTC, int GNT>
__global__ void __launch_bounds__(NTC) skel_team_kernel(const SkelTask* __restrict__ tasks, Arenas A, double eps) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[NTC / 32];
  __shared__ int shk;
  const SkelTask t = tasks[blockIdx.x];
  skel_group_t<CtaTeam<NTC>, GNT>(t, A, eps, smem, NoWait{}, NoPublish{}, red, &shk);
}

// Snapshot levels of many small groups (those the 128-thread skel_kernel
// takes): one warp per group, W groups per CTA, each warp with its own slice
// of the dynamic shared memory and only warp barriers.  The CPQR keeps the
// 128-thread CTA's lane split (GNT = 128), so every sum -- and every rank
// decision -- is the one-CTA kernel's; the pivot search, reflector scalars
// and bookkeeping a 4-warp CTA ran four times over run once.
template <int W>
__global__ void __launch_bounds__(32 * W) skel_warp_kernel(const SkelTask* __restrict__ tasks, int ntasks, Arenas A,
                                                           double eps, int per_group) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[W];
  __shared__ int shk[W];
  const int w = (int)(threadIdx.x >> 5);
  const int g = (int)blockIdx.x * W + w;
  if (g >= ntasks) return;  // warp-uniform: no CTA-wide barrier follows
  const SkelTask t = tasks[g];
  skel_group_t<WarpTeam, 128>(t, A, eps, smem + (size_t)w * per_group, NoWait{}, NoPublish{}, red + w, shk + w);
}

// Exact (reference) order in one launch: co-resident CTAs walk the groups in
// reference order; a group starts once every earlier neighbouring group has
// finished (its redundant DOFs are then retired in the device active mask),
// exactly the state the reference's sequential loop gives it
// (src/driver.py:190-194, src/factor_ops.py:208).  Deadlock-free: groups are
// claimed in a topological order, so a claimed group's predecessors are all
// claimed by running CTAs.
// Groups are claimed dynamically in `order` (the reference order sorted
// stably by dependency depth, a topological order): a CTA never holds a group
// whose predecessors are still unclaimed, so the chain is not delayed behind
// groups waiting elsewhere (static round-robin assignment was: config 3
// level 3.5 ran its 62-link chain in 7.4 ms with 3.2 ms of work on it).
// done[ntasks] is the claim counter.
template <int NT>
__global__ void __launch_bounds__(NT) skel_ordered_kernel(const SkelTask* __restrict__ tasks, int ntasks,
                                                          const int64_t* __restrict__ pred_ptr,
                                                          const int32_t* __restrict__ pred,
                                                          const int32_t* __restrict__ order,
                                                          int* __restrict__ done, Arenas A, double eps) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_claim;
  auto stamp = [&](int j, int which) {
    if (A.tlog && threadIdx.x == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      A.tlog[(size_t)j * 16 + which] = g;
    }
  };
  for (;;) {
    if (threadIdx.x == 0) s_claim = atomicAdd(done + ntasks, 1);
    __syncthreads();
    const int i = s_claim;
    __syncthreads();
    if (i >= ntasks) break;
    const int j = order[i];
    const SkelTask t = tasks[j];
    stamp(j, 0);
    auto wait = [&]() {
      // one thread per predecessor polls its flag
      // relaxed polling (an acquire load would invalidate the SM's L1 on
      // every probe, stalling the co-resident groups), then one fence
      bool polled = false;
      for (int64_t p = pred_ptr[j] + threadIdx.x; p < pred_ptr[j + 1]; p += NT) {
        cuda::atomic_ref<int, cuda::thread_scope_device> f(done[pred[p]]);
        while (f.load(cuda::memory_order_relaxed) == 0) __nanosleep(32);
        polled = true;
      }
      if (polled) cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
      __syncthreads();
      stamp(j, 1);
    };
    auto publish = [&](int k, const int32_t* perm, const int32_t* sdofs, int nc) {
      for (int a = k + threadIdx.x; a < nc; a += NT) A.active[sdofs[perm[a]]] = 0;
      __syncthreads();
      if (threadIdx.x == 0) {
        cuda::atomic_ref<int, cuda::thread_scope_device> f(done[j]);
        f.store(1, cuda::memory_order_release);
      }
      stamp(j, 2);
    };
    skel_group<NT>(t, A, eps, smem, wait, publish);
    __syncthreads();
    stamp(j, 3);
  }
}

// ---------------------------------------------------------------------------
// Exact order with a CTA cluster per group (the large 2D groups): the
// neighbour block's columns are dealt round-robin to the kClusterSkel CTAs
// (each keeps its slice in its own shared memory, so the per-step update is
// split kClusterSkel ways); per pivot step the CTAs exchange one candidate
// each and copy the pivot column from its owner over DSMEM -- one cluster
// barrier per step.  Rank 0 waits for the predecessors, publishes the
// redundant set, gathers the R rows and runs the tail (skel_tail).
// Shared layout per CTA: ints as skel_group | vn1 x2 | xn x2 | R_ii | vn2 |
// v (nq) | own slice (ldq x ceil(nc / kClusterSkel)).  Global scratch per
// group (t.scratch_off): A_cc (nc^2) | R rows (nc^2) | tail workspace.
// ---------------------------------------------------------------------------
template <int NT, int CS>
__global__ void __launch_bounds__(NT) skel_cluster_kernel(const SkelTask* __restrict__ tasks, int ntasks,
                                                          const int64_t* __restrict__ pred_ptr,
                                                          const int32_t* __restrict__ pred,
                                                          int* __restrict__ done, Arenas A, double eps) {
  namespace cg = cooperative_groups;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[NW];
  __shared__ double cand[2][3];
  __shared__ double sh_x;
  __shared__ int sh_k;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int ncls = gridDim.x / CS, cid = blockIdx.x / CS;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int j = cid; j < ntasks; j += ncls) {
    const SkelTask t = tasks[j];
    const int nc = t.nc, nq = t.nq, nf = nc + nq;
    int32_t* sdofs = reinterpret_cast<int32_t*>(smem);
    int32_t* salive = sdofs + nf;
    int32_t* smap = salive + nf;
    int32_t* perm = smap + t.maxnb;
    int32_t* skl = perm + nc;
    int32_t* rdl = skl + nc;
    int32_t* sko = rdl + nc;
    int32_t* rdo = sko + nc;
    int32_t* dcol = rdo + nc;
    int32_t* cpos = dcol + nc;
    const size_t ibytes = align_up(sizeof(int32_t) * (size_t)(2 * nf + t.maxnb + 8 * nc), 16);
    double* cq = reinterpret_cast<double*>(smem + ibytes);
    double* rdiag = cq + 4 * nc;
    double* vn2 = cq + 5 * nc;
    double* vbuf = vn2 + nc;
    double* Ms = vbuf + nq;                         // own column slice, ld ldq
    const int ldq = skel_ldq(nq);
    const int ncl = (nc - rank + CS - 1) / CS;      // owned columns rank, rank + CS, ...
    double* Acc = A.scratch + t.scratch_off;
    double* Rf = Acc + (size_t)nc * nc;
    double* Z = Rf + (size_t)nc * nc;
    const int32_t* gd = A.idx + t.dofs_off;
    for (int i = threadIdx.x; i < nf; i += NT) {
      sdofs[i] = gd[i];
      salive[i] = 1;
    }
    for (size_t e = threadIdx.x; e < (size_t)ldq * ncl; e += NT) Ms[e] = 0.0;
    if (rank == 0)
      for (int e = threadIdx.x; e < nc * nc; e += NT) Acc[e] = 0.0;
    __syncthreads();
    // assembly of the own slice (and of A_cc by rank 0), same order as skel_group
    for (int p = threadIdx.x; p < nc; p += NT) {
      const bool mine = p % CS == rank;
      if (!mine && rank != 0) continue;
      const int g = sdofs[p];
      for (int64_t kk = A.indptr[g]; kk < A.indptr[g + 1]; ++kk) {
        const int pj = front_pos(sdofs, nc, nq, A.indices[kk]);
        if (pj < 0) continue;
        const double v = A.a0[kk];
        if (pj < nc) {
          if (rank == 0) Acc[p * nc + pj] += v;
        } else if (mine) {
          Ms[(pj - nc) + (size_t)(p / CS) * ldq] += v;
        }
      }
    }
    __syncthreads();
    const int32_t* bl = A.lists + t.blk_off;
    for (int b = 0; b < t.nblk; ++b) {
      const int bid = bl[b];
      const int nb = A.blk_n[bid];
      const int32_t* bd = A.idx + A.blk_dof_off[bid];
      const double* bv = A.bvals + A.blk_val_off[bid];
      for (int kk = threadIdx.x; kk < nb; kk += NT) smap[kk] = front_pos(sdofs, nc, nq, bd[kk]);
      __syncthreads();
      for (int kk = wid; kk < nb; kk += NW) {
        const int pk = smap[kk];
        if (pk < 0) continue;
        for (int l = lane; l < nb; l += 32) {
          const int pl = smap[l];
          if (pl < 0 || pl >= nc) continue;
          if (pk < nc) {
            if (rank == 0) Acc[pk * nc + pl] += bv[(size_t)kk * nb + l];
          } else if (pl % CS == rank) {
            Ms[(pk - nc) + (size_t)(pl / CS) * ldq] += bv[(size_t)kk * nb + l];
          }
        }
      }
      __syncthreads();
    }
    // exact order: rank 0 waits for the earlier neighbouring groups
    if (rank == 0) {
      bool polled = false;
      for (int64_t q = pred_ptr[j] + threadIdx.x; q < pred_ptr[j + 1]; q += NT) {
        cuda::atomic_ref<int, cuda::thread_scope_device> f(done[pred[q]]);
        while (f.load(cuda::memory_order_relaxed) == 0) __nanosleep(32);
        polled = true;
      }
      if (polled) cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
    }
    cl.sync();
    if (threadIdx.x == 0) cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
    __syncthreads();
    for (int i = nc + threadIdx.x; i < nf; i += NT) {
      if (!__ldcg(A.active + sdofs[i])) {
        salive[i] = 0;
        for (int jl = 0; jl < ncl; ++jl) Ms[(size_t)(i - nc) + (size_t)jl * ldq] = 0.0;
      }
    }
    __syncthreads();
    // CPQR over the slices
    if (threadIdx.x == 0) {
      int na = 0;
      for (int i = nc; i < nf; ++i) na += salive[i];
      sh_k = na;
    }
    for (int jl = wid; jl < ncl; jl += NW) {
      const double* col = Ms + (size_t)jl * ldq;
      double s1 = 0.0;
      for (int r = 1 + lane; r < nq; r += 32) s1 += col[r] * col[r];
      s1 = warp_sum(s1);
      const double c0 = nq > 0 ? col[0] : 0.0;
      if (lane == 0) {
        const int jj = rank + CS * jl;
        const double nv = sqrt(c0 * c0 + s1);
        cq[jj] = nv;
        vn2[jj] = nv;
        cq[2 * nc + jj] = sqrt(s1);
      }
    }
    for (int jj = threadIdx.x; jj < nc; jj += NT) {
      dcol[jj] = 0;
      cpos[jj] = jj;
    }
    __syncthreads();
    const int nq_alive = sh_k;
    const int kmax = nq < nc ? nq : nc;
    const double tol3z = sqrt(DBL_EPSILON * 0.5);
    int Gl = 32;
    while (Gl > 8 && NT / Gl < ncl) Gl >>= 1;
    const int nslots = NT / Gl, sl = lane & (Gl - 1), slot = wid * (32 / Gl) + lane / Gl;
    double thr = 0.0;
    int k = kmax;
    for (int i = 0; i < kmax; ++i) {
      const int cur = (i & 1) * nc, nxt = nc - cur;
      const double* vn1 = cq + cur;
      double* vn1o = cq + nxt;
      const double* xn = cq + 2 * nc + cur;
      double* xno = cq + 2 * nc + nxt;
      const int32_t* cat = cpos + cur;
      int32_t* cato = cpos + nxt;
      if (wid == 0) {  // this CTA's best candidate (largest norm, lowest LAPACK position)
        double bv = -1.0;
        int bp = nc, bc = 0;
        for (int pos = i + lane; pos < nc; pos += 32) {
          const int c = cat[pos];
          if (c % CS != rank) continue;
          const double v = vn1[c];
          if (v > bv) { bv = v; bp = pos; bc = c; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int op = __shfl_xor_sync(0xffffffffu, bp, o);
          const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
          if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; bc = oc; }
        }
        if (lane == 0) {
          cand[i & 1][0] = bv;
          cand[i & 1][1] = bp;
          cand[i & 1][2] = bc;
        }
      }
      cl.sync();  // every candidate (and every owner's updated slice) visible
      double gbv = -1.0;
      int gbp = nc, p = 0;
      for (int q = 0; q < CS; ++q) {
        const double* cr = cl.map_shared_rank(&cand[i & 1][0], q);
        const double v = cr[0];
        const int pp = (int)cr[1];
        if (v > gbv || (v == gbv && pp < gbp)) { gbv = v; gbp = pp; p = (int)cr[2]; }
      }
      if (wid == NW - 1) {
        const int ci = cat[i];
        for (int pos = lane; pos < nc; pos += 32) cato[pos] = pos == i ? p : (pos == gbp ? ci : cat[pos]);
      }
      if (i == 0 && gbv == 0.0) { k = 0; break; }
      // the pivot column (rows >= i) and its Householder norm, from the owner
      const int owner = p % CS;
      const double* Mo = cl.map_shared_rank(Ms, owner) + (size_t)(p / CS) * ldq;
      for (int r = i + threadIdx.x; r < nq; r += NT) vbuf[r] = Mo[r];
      if (threadIdx.x == 0) sh_x = cl.map_shared_rank(cq + 2 * nc + cur, owner)[p];
      __syncthreads();
      const double alpha = vbuf[i], xnorm = sh_x;
      double beta, tau, scal;
      if (xnorm == 0.0) { beta = alpha; tau = 0.0; scal = 0.0; }
      else {
        beta = -copysign(hypot(alpha, xnorm), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      const double rii = fabs(beta);
      if (i == 0) thr = eps > 0.0 ? eps * rii : (double)(nq_alive > nc ? nq_alive : nc) * DBL_EPSILON * rii;
      if (rii <= thr) { k = i; break; }
      if (threadIdx.x == 0) { rdiag[i] = beta; dcol[p] = 1; }
      const double* v = vbuf;
      for (int base = 0; base < ncl; base += nslots) {
        const int jl = base + slot;
        const int jj = rank + CS * jl;
        const bool act = jl < ncl && jj != p && !dcol[jj];
        double* col = Ms + (size_t)(act ? jl : 0) * ldq;
        double acc = 0.0;
        if (tau != 0.0) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
          int r = i + 1 + sl;
          for (; r + 3 * Gl < nq; r += 4 * Gl) {
            s0 += v[r] * col[r];
            s1 += v[r + Gl] * col[r + Gl];
            s2 += v[r + 2 * Gl] * col[r + 2 * Gl];
            s3 += v[r + 3 * Gl] * col[r + 3 * Gl];
          }
          for (; r < nq; r += Gl) s0 += v[r] * col[r];
          const double sd = group_sum((s0 + s1) + (s2 + s3), Gl);
          const double w = tau * (col[i] + scal * sd);
          __syncwarp();
          if (act && sl == 0) col[i] -= w;
          const double ws2 = w * scal;
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          r = i + 1 + sl;
          if (r == i + 1 && r < nq) {
            const double x = col[r] - ws2 * v[r];
            if (act) col[r] = x;
            r += Gl;
          }
          for (; r + 3 * Gl < nq; r += 4 * Gl) {
            const double x0 = col[r] - ws2 * v[r];
            const double x1 = col[r + Gl] - ws2 * v[r + Gl];
            const double x2 = col[r + 2 * Gl] - ws2 * v[r + 2 * Gl];
            const double x3 = col[r + 3 * Gl] - ws2 * v[r + 3 * Gl];
            if (act) {
              col[r] = x0;
              col[r + Gl] = x1;
              col[r + 2 * Gl] = x2;
              col[r + 3 * Gl] = x3;
            }
            a0 += x0 * x0;
            a1 += x1 * x1;
            a2 += x2 * x2;
            a3 += x3 * x3;
          }
          for (; r < nq; r += Gl) {
            const double x = col[r] - ws2 * v[r];
            if (act) col[r] = x;
            a0 += x * x;
          }
          acc = (a0 + a1) + (a2 + a3);
        } else {
          double a0 = 0.0, a1 = 0.0;
          int r = i + 2 + sl;
          for (; r + Gl < nq; r += 2 * Gl) {
            a0 += col[r] * col[r];
            a1 += col[r + Gl] * col[r + Gl];
          }
          for (; r < nq; r += Gl) a0 += col[r] * col[r];
          acc = a0 + a1;
        }
        acc = group_sum(acc, Gl);
        __syncwarp();
        if (act) {
          const double cn = i + 1 < nq ? col[i + 1] : 0.0;
          double nv = vn1[jj];
          if (nv != 0.0) {
            double tmp = fabs(col[i]) / nv;
            tmp = 1.0 - tmp * tmp;
            tmp = tmp > 0.0 ? tmp : 0.0;
            const double ratio = nv / vn2[jj];
            if (tmp * ratio * ratio <= tol3z) {
              nv = (i + 1 < nq) ? sqrt(cn * cn + acc) : 0.0;
              if (sl == 0) vn2[jj] = nv;
            } else {
              nv *= sqrt(tmp);
            }
          }
          if (sl == 0) { vn1o[jj] = nv; xno[jj] = sqrt(acc); }
        }
      }
      __syncthreads();
    }
    {
      const int32_t* cat = cpos + (k & 1) * nc;
      for (int pos = threadIdx.x; pos < nc; pos += NT) perm[pos] = cat[pos];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += NT) {
      const int pc = perm[i];
      if (pc % CS == rank) Ms[i + (size_t)(pc / CS) * ldq] = rdiag[i];
    }
    if (rank == 0) {  // publish: later groups may start
      for (int a = k + threadIdx.x; a < nc; a += NT) A.active[sdofs[perm[a]]] = 0;
      __syncthreads();
      if (threadIdx.x == 0) {
        cuda::atomic_ref<int, cuda::thread_scope_device> f(done[j]);
        f.store(1, cuda::memory_order_release);
      }
    }
    cl.sync();  // R rows complete in every slice
    if (rank == 0)
      for (int e = threadIdx.x; e < k * nc; e += NT) {
        const int jc = e / k, i = e - jc * k;
        Rf[i + (size_t)jc * nc] = cl.map_shared_rank(Ms, jc % CS)[i + (size_t)(jc / CS) * ldq];
      }
    cl.sync();  // the slices may be reused
    if (rank == 0) skel_tail<NT>(t, A, nc, k, Rf, nc, perm, skl, rdl, sko, rdo, sdofs, Acc, Z, red);
    __syncthreads();
  }
}

// Retire the redundant DOFs of a finished batch (device active mask).
__global__ void apply_rd_kernel(const SkelTask* __restrict__ tasks, Arenas A) {
  const SkelTask t = tasks[blockIdx.x];
  const int k = A.kout[t.group];
  const int32_t* out = A.idx + t.out_off;
  for (int a = k + threadIdx.x; a < t.nc; a += blockDim.x) A.active[out[a]] = 0;
}

// ---------------------------------------------------------------------------
template <class K>
static void allow_smem(K kern) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCapBytes);
}

// Four warps per cell: with the packed front (level-0 cell of config 3:
// 24 KB) six cells share an SM (register-bound); eight-warp CTAs were three
// (config 3 level 0: 6.2 ms at 8 warps / full-square front, 5.1 ms here).
void launch_elim_small(const ElimTask* d_tasks, int ntasks, const Arenas& A, size_t smem, int nt,
                       cudaStream_t s) {
  if (ntasks <= 0) return;
  (void)nt;
  static bool once = false;
  if (!once) {
    allow_smem(elim_small_kernel<128>);
    once = true;
  }
  elim_small_kernel<128><<<ntasks, 128, smem, s>>>(d_tasks, A);
}

void launch_schur_tiles(const ElimTask* d_tasks, const int4* d_tiles, int ntiles, const Arenas& A,
                        cudaStream_t s) {
  if (ntiles <= 0) return;
  schur_tile_kernel<<<ntiles, 128, 0, s>>>(d_tasks, d_tiles, A);
}

void launch_skel(const SkelTask* d_tasks, int ntasks, const Arenas& A, double eps, size_t smem, int nt, int max_nc,
                 int max_nq, cudaStream_t s) {
  if (ntasks <= 0) return;
  rank_cert_init();
  static bool once = false;
  if (!once) {
    allow_smem(skel_kernel<128>);
    allow_smem(skel_kernel<512>);
    once = true;
  }
  // (HIFDE_NO_SKEL_WARP: the one-CTA kernels of the level's lane split
  // instead -- the tests' A/B, which must agree bit for bit)
  static const bool no_warp = getenv("HIFDE_NO_SKEL_WARP") != nullptr;
  // many tiny groups (config 3 level 0.5: 7 x 44, 4.4 -> 2.6 ms; config 5
  // level 1/3: 9 x 92, 5.7 -> 4.1 ms; the 15-column groups of config 3 level
  // 1.5 are slower by warp, 2.7 -> 3.9 ms): a warp each (bit-identical)
  if (!no_warp && nt <= 128 && max_nc <= 12 && ntasks >= 4096) {
    static bool once_w = (allow_smem(skel_warp_kernel<8>), true);
    (void)once_w;
    const size_t per = (smem + 15) / 16 * 16;
    const int W = (int)std::min<size_t>(8, std::max<size_t>(1, (kSmemCapBytes - 2048) / std::max<size_t>(per, 16)));
    if (W == 8) {
      skel_warp_kernel<8><<<(ntasks + 7) / 8, 256, per * 8, s>>>(d_tasks, ntasks, A, eps, (int)per);
      return;
    }
  }
  // half-size CTAs with the full-size CTA's lane split (bit-identical),
  // more groups per SM: 15-column groups (config 3 level 1.5: 2.71 -> 2.40
  // ms on 64 threads) and 512-thread groups with short neighbour blocks
  // (config 3 level 2.5: 3.16 -> 2.56 ms on 256 threads; the tall ones of
  // config 5 level 1 2/3 are slower: 30 -> 36 ms)
  if (!no_warp) {
    static bool once_t = (allow_smem(skel_team_kernel<64, 128>), allow_smem(skel_team_kernel<256, 512>), true);
    (void)once_t;
    if (nt <= 128) {
      skel_team_kernel<64, 128><<<ntasks, 64, smem, s>>>(d_tasks, A, eps);
      return;
    }
    if (max_nq <= 256) {
      skel_team_kernel<256, 512><<<ntasks, 256, smem, s>>>(d_tasks, A, eps);
      return;
    }
  }
  if (nt <= 128) skel_kernel<128><<<ntasks, 128, smem, s>>>(d_tasks, A, eps);
  else skel_kernel<512><<<ntasks, 512, smem, s>>>(d_tasks, A, eps);
}

int skel_ordered_capacity(size_t smem, int nt) {
  int per_sm = 0, dev = 0, nsm = 0;
  if (nt <= 128) {
    allow_smem(skel_ordered_kernel<128>);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, skel_ordered_kernel<128>, 128, smem);
  } else {
    allow_smem(skel_ordered_kernel<512>);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, skel_ordered_kernel<512>, 512, smem);
  }
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * nsm;
}

cudaError_t launch_skel_ordered(const SkelTask* d_tasks, int ntasks, const int64_t* pred_ptr, const int32_t* pred,
                                const int32_t* order, int* done, const Arenas& A, double eps, size_t smem, int nt,
                                int grid, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  rank_cert_init();
  Arenas Ac = A;
  void* args[] = {(void*)&d_tasks, (void*)&ntasks, (void*)&pred_ptr, (void*)&pred, (void*)&order, (void*)&done,
                  (void*)&Ac, (void*)&eps};
  if (nt <= 128)
    return cudaLaunchCooperativeKernel((const void*)skel_ordered_kernel<128>, dim3((unsigned)grid), dim3(128), args,
                                       smem, s);
  return cudaLaunchCooperativeKernel((const void*)skel_ordered_kernel<512>, dim3((unsigned)grid), dim3(512), args,
                                     smem, s);
}

template <int CS>
static int cluster_capacity(size_t smem) {
  auto kern = skel_cluster_kernel<kClusterThreads, CS>;
  allow_smem(kern);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(CS * 148);
  cfg.blockDim = dim3(kClusterThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int skel_cluster_capacity(size_t smem, int cs) {
  return cs == 4 ? cluster_capacity<4>(smem) : cluster_capacity<2>(smem);
}

template <int CS>
static cudaError_t cluster_launch(const SkelTask* d_tasks, int ntasks, const int64_t* pred_ptr, const int32_t* pred,
                                  int* done, const Arenas& A, double eps, size_t smem, int nclusters,
                                  cudaStream_t s) {
  auto kern = skel_cluster_kernel<kClusterThreads, CS>;
  allow_smem(kern);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  // the waits spin, so every cluster must be resident: the grid never exceeds
  // cudaOccupancyMaxActiveClusters (skel_cluster_capacity) for this launch
  cfg.gridDim = dim3((unsigned)(CS * nclusters));
  cfg.blockDim = dim3(kClusterThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, d_tasks, ntasks, pred_ptr, pred, done, A, eps);
}

cudaError_t launch_skel_cluster(const SkelTask* d_tasks, int ntasks, const int64_t* pred_ptr, const int32_t* pred,
                                int* done, const Arenas& A, double eps, size_t smem, int nclusters, int cs,
                                cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  return cs == 4 ? cluster_launch<4>(d_tasks, ntasks, pred_ptr, pred, done, A, eps, smem, nclusters, s)
                 : cluster_launch<2>(d_tasks, ntasks, pred_ptr, pred, done, A, eps, smem, nclusters, s);
}

void launch_apply_rd(const SkelTask* d_tasks, int ntasks, const Arenas& A, cudaStream_t s) {
  if (ntasks <= 0) return;
  apply_rd_kernel<<<ntasks, 64, 0, s>>>(d_tasks, A);
}

}  // namespace hifde
