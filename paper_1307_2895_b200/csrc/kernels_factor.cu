// sm_100a kernels of the HIF-DE factorization.
//
// One CTA owns one cell (elimination) or one group (skeletonization).  The
// front is assembled from the original stencil matrix A0 and the live clique
// blocks, then factored in shared memory when
// it fits, otherwise in an L2-resident global scratch slab.
//
// Reference semantics followed:
//   elimination   src/factor_ops.py:138-159, src/dense.py:187-219
//   skeletonize   src/factor_ops.py:162-214
//   CPQR / ID     src/dense.py:239-264 (LAPACK dgeqp3 / dlaqp2 pivoting and
//                 column-norm downdating, rank = first |R_jj| <= eps |R_11|)
#include <cfloat>
#include <cstdint>

#include "hifde_internal.h"

namespace hifde {

namespace {

constexpr int NT = kThreads;
constexpr int NWARP = NT / 32;
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

// Block-wide sum; every thread gets the result.  red must hold NWARP doubles.
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NWARP; ++w) s += red[w];
  return s;
}

__device__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = red[0];
#pragma unroll
  for (int w = 1; w < NWARP; ++w) s = fmax(s, red[w]);
  return s;
}

// Block-wide argmax (largest value, lowest index on ties -- idamax).
__device__ int block_argmax(double v, int idx, double* redv, int* redi) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
  __syncthreads();
  if (lane == 0) { redv[wid] = v; redi[wid] = idx; }
  __syncthreads();
  double bv = redv[0];
  int bi = redi[0];
#pragma unroll
  for (int w = 1; w < NWARP; ++w) {
    if (redv[w] > bv || (redv[w] == bv && redi[w] < bi)) { bv = redv[w]; bi = redi[w]; }
  }
  return bi;
}

// In-place right-looking Cholesky of the n x n lower triangle of A (row-major,
// leading dimension ld).  Returns HIFDE status: 1 indefinite (a pivot <= 0 or
// NaN, dpotrf info > 0), 2 singular (min D <= 1e-14 max|diag|), 0 ok.
__device__ int chol_inplace(double* A, int n, int ld, double* red) {
  if (n == 0) return 0;
  double sc = 0.0;
  for (int i = threadIdx.x; i < n; i += NT) sc = fmax(sc, fabs(A[(size_t)i * ld + i]));
  double scale = block_max(sc, red);
  if (scale == 0.0) {
    double s2 = 0.0;
    for (int e = threadIdx.x; e < n * n; e += NT) {
      int i = e / n, j = e - i * n;
      if (j <= i) s2 = fmax(s2, fabs(A[(size_t)i * ld + j]));
    }
    scale = block_max(s2, red);
  }
  double dmin = DBL_MAX;
  for (int k = 0; k < n; ++k) {
    __syncthreads();
    const double akk = A[(size_t)k * ld + k];
    __syncthreads();
    if (!(akk > 0.0)) return 1;
    const double piv = sqrt(akk);
    const double inv = 1.0 / piv;
    dmin = fmin(dmin, piv * piv);
    if (threadIdx.x == 0) A[(size_t)k * ld + k] = piv;
    for (int i = k + 1 + threadIdx.x; i < n; i += NT) A[(size_t)i * ld + k] *= inv;
    __syncthreads();
    const int m = n - k - 1;
    for (int e = threadIdx.x; e < m * m; e += NT) {
      const int ii = e / m, jj = e - ii * m;
      if (jj <= ii) {
        const int i = k + 1 + ii, j = k + 1 + jj;
        A[(size_t)i * ld + j] -= A[(size_t)i * ld + k] * A[(size_t)j * ld + k];
      }
    }
  }
  __syncthreads();
  if (dmin <= kSingularRtol * fmax(scale, 1e-300)) return 2;
  return 0;
}

// B (n x m, row-major, ld ldb) <- C^{-1} B with C lower (row-major, ld ldc).
__device__ void trsm_lower(const double* C, int n, int ldc, double* B, int m, int ldb) {
  for (int i = 0; i < n; ++i) {
    __syncthreads();
    const double cii = C[(size_t)i * ldc + i];
    for (int j = threadIdx.x; j < m; j += NT) B[(size_t)i * ldb + j] /= cii;
    __syncthreads();
    const int rows = n - i - 1;
    for (int e = threadIdx.x; e < rows * m; e += NT) {
      const int l = i + 1 + e / m, j = e % m;
      B[(size_t)l * ldb + j] -= C[(size_t)l * ldc + i] * B[(size_t)i * ldb + j];
    }
  }
  __syncthreads();
}

__device__ __forceinline__ size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

// ---------------------------------------------------------------------------
// Elimination: F = A0[c+q, c+q] (minus the q x q part of A0) + sum of consumed
// clique blocks; C C^T = F_cc; W = C^-1 F_cq; U = F_qq - W^T W.
// Also used for the terminal block (nq == 0).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) elim_kernel(const ElimTask* __restrict__ tasks, Arenas A) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[NWARP];
  const ElimTask t = tasks[blockIdx.x];
  const int nc = t.nc, nq = t.nq, nf = nc + nq;
  int32_t* sdofs = reinterpret_cast<int32_t*>(smem);
  int32_t* smap = sdofs + nf;
  const size_t ibytes = align_up(sizeof(int32_t) * (size_t)(nf + t.maxnb), 16);
  double* F = t.scratch_off < 0 ? reinterpret_cast<double*>(smem + ibytes) : A.scratch + t.scratch_off;
  const int32_t* gd = A.idx + t.dofs_off;
  for (int i = threadIdx.x; i < nf; i += NT) sdofs[i] = gd[i];
  for (int i = threadIdx.x; i < nc; i += NT) A.active[gd[i]] = 0;  // the cell retires
  for (int e = threadIdx.x; e < nf * nf; e += NT) F[e] = 0.0;
  __syncthreads();

  // original stencil couplings of the c rows (A0[c,c], A0[c,q] and mirror)
  for (int p = threadIdx.x; p < nc; p += NT) {
    const int g = sdofs[p];
    for (int64_t k = A.indptr[g]; k < A.indptr[g + 1]; ++k) {
      const int pj = front_pos(sdofs, nc, nq, A.indices[k]);
      if (pj < 0) continue;
      const double v = A.a0[k];
      F[(size_t)p * nf + pj] += v;
      if (pj >= nc) F[(size_t)pj * nf + p] += v;
    }
  }
  __syncthreads();
  // consumed clique blocks, in ascending block id (deterministic extend-add)
  const int32_t* bl = A.lists + t.blk_off;
  for (int b = 0; b < t.nblk; ++b) {
    const int bid = bl[b];
    const int nb = A.blk_n[bid];
    const int32_t* bd = A.idx + A.blk_dof_off[bid];
    const double* bv = A.bvals + A.blk_val_off[bid];
    for (int k = threadIdx.x; k < nb; k += NT) smap[k] = front_pos(sdofs, nc, nq, bd[k]);
    __syncthreads();
    for (int e = threadIdx.x; e < nb * nb; e += NT) {
      const int k = e / nb, l = e - k * nb;
      const int pk = smap[k], pl = smap[l];
      if (pk >= 0 && pl >= 0) F[(size_t)pk * nf + pl] += bv[e];
    }
    __syncthreads();
  }

  int st = chol_inplace(F, nc, nf, red);
  if (st != 0) {
    if (threadIdx.x == 0) A.status[blockIdx.x] = st;
    return;
  }
  if (nq > 0) {
    trsm_lower(F, nc, nf, F + nc, nq, nf);
    double* U = A.bvals + t.U_off;
    for (int e = threadIdx.x; e < nq * nq; e += NT) {
      const int a = e / nq, b = e - a * nq;
      double s = F[(size_t)(nc + a) * nf + nc + b];
      for (int k = 0; k < nc; ++k) s -= F[(size_t)k * nf + nc + a] * F[(size_t)k * nf + nc + b];
      U[e] = s;
    }
    double* W = A.fac + t.W_off;
    for (int e = threadIdx.x; e < nc * nq; e += NT) {
      const int i = e / nq, j = e - i * nq;
      W[e] = F[(size_t)i * nf + nc + j];
    }
  }
  double* C = A.fac + t.C_off;
  for (int e = threadIdx.x; e < nc * nc; e += NT) {
    const int i = e / nc, j = e - i * nc;
    C[e] = (j <= i) ? F[(size_t)i * nf + j] : 0.0;
  }
  if (threadIdx.x == 0) A.status[blockIdx.x] = 0;
}

// ---------------------------------------------------------------------------
// Skeletonization of one group: M = A[c+q, c] (column-major), CPQR of the q
// rows with early stop at the rank cut, T = R11^-1 R12, congruence, inner
// elimination of rd against sk, delta clique block -W^T W over sk.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) skel_kernel(const SkelTask* __restrict__ tasks, Arenas A,
                                                  double eps) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[NWARP];
  __shared__ int redi[NWARP];
  const SkelTask t = tasks[blockIdx.x];
  const int nc = t.nc, nq = t.nq, nf = nc + nq;
  const int ld = nf;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  // integer workspace (always shared)
  int32_t* sdofs = reinterpret_cast<int32_t*>(smem);
  int32_t* salive = sdofs + nf;
  int32_t* smap = salive + nf;
  int32_t* perm = smap + t.maxnb;
  int32_t* skl = perm + nc;
  int32_t* rdl = skl + nc;
  int32_t* sko = rdl + nc;
  int32_t* rdo = sko + nc;
  const size_t ibytes = align_up(sizeof(int32_t) * (size_t)(2 * nf + t.maxnb + 5 * nc), 16);
  double* ws = t.scratch_off < 0 ? reinterpret_cast<double*>(smem + ibytes) : A.scratch + t.scratch_off;
  const size_t q4 = (size_t)nc * nc / 4 + nc;
  double* M = ws;                                  // nf x nc, column-major
  double* vn1 = M + (size_t)nf * nc;
  double* vn2 = vn1 + nc;
  double* Tp = vn2 + nc;                           // k x r, pivot order
  double* Ts = Tp + q4;                            // k x r, sorted
  double* Bsr = Ts + q4;                           // k x r
  double* Wm = Bsr + q4;                           // r x k
  double* Brr = Wm + q4;                           // r x r

  const int32_t* gd = A.idx + t.dofs_off;
  for (int i = threadIdx.x; i < nf; i += NT) {
    const int g = gd[i];
    sdofs[i] = g;
    salive[i] = (i < nc) ? 1 : (int)A.active[g];
  }
  for (int i = threadIdx.x; i < nc; i += NT) perm[i] = i;
  for (size_t e = threadIdx.x; e < (size_t)nf * nc; e += NT) M[e] = 0.0;
  __syncthreads();

  for (int p = threadIdx.x; p < nc; p += NT) {
    const int g = sdofs[p];
    for (int64_t k = A.indptr[g]; k < A.indptr[g + 1]; ++k) {
      const int pj = front_pos(sdofs, nc, nq, A.indices[k]);
      if (pj < 0 || !salive[pj]) continue;
      const double v = A.a0[k];
      if (pj < nc) M[p + (size_t)pj * ld] += v;
      else M[pj + (size_t)p * ld] += v;
    }
  }
  __syncthreads();
  const int32_t* bl = A.lists + t.blk_off;
  for (int b = 0; b < t.nblk; ++b) {
    const int bid = bl[b];
    const int nb = A.blk_n[bid];
    const int32_t* bd = A.idx + A.blk_dof_off[bid];
    const double* bv = A.bvals + A.blk_val_off[bid];
    for (int k = threadIdx.x; k < nb; k += NT) {
      const int p = front_pos(sdofs, nc, nq, bd[k]);
      smap[k] = (p >= 0 && salive[p]) ? p : -1;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nb * nb; e += NT) {
      const int k = e / nb, l = e - k * nb;
      const int pk = smap[k], pl = smap[l];
      if (pk >= 0 && pl >= 0 && pl < nc) M[pk + (size_t)pl * ld] += bv[e];
    }
    __syncthreads();
  }

  // ---- column-pivoted QR of Mq = M[nc:, :] (dlaqp2 semantics) ----------
  double* Mq = M + nc;
  int nq_alive = 0;
  for (int i = nc + threadIdx.x; i < nf; i += NT) nq_alive += salive[i];
  nq_alive = (int)block_sum((double)nq_alive, red);
  for (int j = wid; j < nc; j += NWARP) {
    double s = 0.0;
    for (int r = lane; r < nq; r += 32) { const double x = Mq[r + (size_t)j * ld]; s += x * x; }
    s = warp_sum(s);
    if (lane == 0) { vn1[j] = sqrt(s); vn2[j] = vn1[j]; }
  }
  __syncthreads();
  const int kmax = nq < nc ? nq : nc;
  const double tol3z = sqrt(DBL_EPSILON * 0.5);  // sqrt(dlamch('E'))
  int k = kmax;
  double thr = 0.0;
  for (int i = 0; i < kmax; ++i) {
    double bv = -1.0;
    int bi = nc;
    for (int j = i + threadIdx.x; j < nc; j += NT) {
      const double v = vn1[j];
      if (v > bv || (v == bv && j < bi)) { bv = v; bi = j; }
    }
    const int pvt = block_argmax(bv, bi, red, redi);
    if (i == 0 && vn1[pvt] == 0.0) { k = 0; break; }   // zero block: all redundant
    __syncthreads();
    if (pvt != i) {
      for (int r = threadIdx.x; r < nq; r += NT) {
        const double a = Mq[r + (size_t)i * ld];
        Mq[r + (size_t)i * ld] = Mq[r + (size_t)pvt * ld];
        Mq[r + (size_t)pvt * ld] = a;
      }
      if (threadIdx.x == 0) {
        const int pi = perm[i]; perm[i] = perm[pvt]; perm[pvt] = pi;
        vn1[pvt] = vn1[i];
        vn2[pvt] = vn2[i];
      }
    }
    __syncthreads();
    // Householder reflector of Mq[i:, i] (dlarfg)
    double xs = 0.0;
    for (int r = i + 1 + threadIdx.x; r < nq; r += NT) { const double x = Mq[r + (size_t)i * ld]; xs += x * x; }
    const double xnorm = sqrt(block_sum(xs, red));
    const double alpha = Mq[i + (size_t)i * ld];
    double beta, tau;
    if (xnorm == 0.0) { beta = alpha; tau = 0.0; }
    else { beta = -copysign(hypot(alpha, xnorm), alpha); tau = (beta - alpha) / beta; }
    const double rii = fabs(beta);
    if (i == 0) {
      thr = eps > 0.0 ? eps * rii : (double)(nq_alive > nc ? nq_alive : nc) * DBL_EPSILON * rii;
    }
    if (rii <= thr) { k = i; break; }
    __syncthreads();
    if (xnorm != 0.0) {
      const double scal = 1.0 / (alpha - beta);
      for (int r = i + 1 + threadIdx.x; r < nq; r += NT) Mq[r + (size_t)i * ld] *= scal;
    }
    if (threadIdx.x == 0) Mq[i + (size_t)i * ld] = beta;
    __syncthreads();
    // apply H_i to the trailing columns and downdate their norms (warp/column)
    for (int j = i + 1 + wid; j < nc; j += NWARP) {
      double* col = Mq + (size_t)j * ld;
      const double* v = Mq + (size_t)i * ld;
      if (tau != 0.0) {
        double s = (lane == 0) ? col[i] : 0.0;
        for (int r = i + 1 + lane; r < nq; r += 32) s += v[r] * col[r];
        s = warp_sum(s) * tau;
        if (lane == 0) col[i] -= s;
        for (int r = i + 1 + lane; r < nq; r += 32) col[r] -= s * v[r];
      }
      __syncwarp();
      double nv = vn1[j];
      int recompute = 0;
      if (nv != 0.0) {
        double tmp = fabs(col[i]) / nv;
        tmp = 1.0 - tmp * tmp;
        tmp = tmp > 0.0 ? tmp : 0.0;
        const double ratio = nv / vn2[j];
        const double tmp2 = tmp * ratio * ratio;
        if (tmp2 <= tol3z) recompute = 1;
        else nv = nv * sqrt(tmp);
      }
      if (recompute) {
        double s = 0.0;
        for (int r = i + 1 + lane; r < nq; r += 32) s += col[r] * col[r];
        s = warp_sum(s);
        nv = (i + 1 < nq) ? sqrt(s) : 0.0;
        if (lane == 0) { vn1[j] = nv; vn2[j] = nv; }
      } else if (lane == 0) {
        vn1[j] = nv;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  const int r = nc - k;

  // T = R11^-1 R12 (back substitution, in place on Mq rows 0..k-1)
  for (int i = k - 1; i >= 0; --i) {
    __syncthreads();
    const double d = Mq[i + (size_t)i * ld];
    for (int j = threadIdx.x; j < r; j += NT) Mq[i + (size_t)(k + j) * ld] /= d;
    __syncthreads();
    for (int e = threadIdx.x; e < i * r; e += NT) {
      const int l = e % i, j = e / i;
      Mq[l + (size_t)(k + j) * ld] -= Mq[l + (size_t)i * ld] * Mq[i + (size_t)(k + j) * ld];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * r; e += NT) {
    const int a = e / r, b = e - a * r;
    Tp[e] = Mq[a + (size_t)(k + b) * ld];
  }
  // ascending sk / rd with their pivot positions
  for (int a = threadIdx.x; a < nc; a += NT) {
    const int v = perm[a];
    int rank = 0;
    if (a < k) {
      for (int b = 0; b < k; ++b) rank += perm[b] < v;
      skl[rank] = v;
      sko[rank] = a;
    } else {
      for (int b = k; b < nc; ++b) rank += perm[b] < v;
      rdl[rank] = v;
      rdo[rank] = a - k;
    }
  }
  __syncthreads();
  int32_t* out = A.idx + t.out_off;
  for (int a = threadIdx.x; a < k; a += NT) out[a] = sdofs[skl[a]];
  for (int a = threadIdx.x; a < r; a += NT) out[k + a] = sdofs[rdl[a]];
  if (threadIdx.x == 0) A.kout[t.group] = k;
  if (r == 0) {
    if (threadIdx.x == 0) A.status[t.group] = 0;
    return;
  }
  for (int e = threadIdx.x; e < k * r; e += NT) {
    const int a = e / r, b = e - a * r;
    Ts[e] = Tp[(size_t)sko[a] * r + rdo[b]];
  }
  __syncthreads();
  // B_sr = A_sr - A_ss T
#define ACC(x, y) M[(size_t)(x) + (size_t)(y) * ld]
  for (int e = threadIdx.x; e < k * r; e += NT) {
    const int a = e / r, b = e - a * r;
    const int sa = skl[a];
    double s = ACC(sa, rdl[b]);
    for (int l = 0; l < k; ++l) s -= ACC(sa, skl[l]) * Ts[(size_t)l * r + b];
    Bsr[e] = s;
  }
  __syncthreads();
  // B_rr = A_rr - A_sr^T T - T^T B_sr
  for (int e = threadIdx.x; e < r * r; e += NT) {
    const int a = e / r, b = e - a * r;
    double s = ACC(rdl[a], rdl[b]);
    for (int l = 0; l < k; ++l)
      s -= ACC(skl[l], rdl[a]) * Ts[(size_t)l * r + b] + Ts[(size_t)l * r + a] * Bsr[(size_t)l * r + b];
    Brr[e] = s;
  }
#undef ACC
  __syncthreads();
  for (int e = threadIdx.x; e < r * r; e += NT) {
    const int a = e / r, b = e - a * r;
    if (a < b) {
      const double m = 0.5 * (Brr[e] + Brr[(size_t)b * r + a]);
      Brr[e] = m;
      Brr[(size_t)b * r + a] = m;
    }
  }
  __syncthreads();
  const int st = chol_inplace(Brr, r, r, red);
  if (st != 0) {
    if (threadIdx.x == 0) A.status[t.group] = st;
    return;
  }
  // W = C^-1 B_sr^T (r x k)
  for (int e = threadIdx.x; e < r * k; e += NT) {
    const int a = e / k, b = e - a * k;
    Wm[e] = Bsr[(size_t)b * r + a];
  }
  __syncthreads();
  if (k > 0) trsm_lower(Brr, r, r, Wm, k, k);
  double* dl = A.bvals + t.delta_off;
  for (int e = threadIdx.x; e < k * k; e += NT) {
    const int a = e / k, b = e - a * k;
    double s = 0.0;
    for (int l = 0; l < r; ++l) s -= Wm[(size_t)l * k + a] * Wm[(size_t)l * k + b];
    dl[e] = s;
  }
  double* rec = A.fac + t.rec_off;
  for (int e = threadIdx.x; e < k * r; e += NT) rec[e] = Ts[e];
  double* C = rec + (size_t)k * r;
  for (int e = threadIdx.x; e < r * r; e += NT) {
    const int a = e / r, b = e - a * r;
    C[e] = (b <= a) ? Brr[e] : 0.0;
  }
  double* W = C + (size_t)r * r;
  for (int e = threadIdx.x; e < r * k; e += NT) W[e] = Wm[e];
  if (threadIdx.x == 0) A.status[t.group] = 0;
}

// Retire the redundant DOFs of a finished batch (device active mask).
__global__ void apply_rd_kernel(const SkelTask* __restrict__ tasks, Arenas A) {
  const SkelTask t = tasks[blockIdx.x];
  const int k = A.kout[t.group];
  const int32_t* out = A.idx + t.out_off;
  for (int a = k + threadIdx.x; a < t.nc; a += blockDim.x) A.active[out[a]] = 0;
}

void launch_elim(const ElimTask* d_tasks, int ntasks, const Arenas& A, size_t smem,
                 int /*smem_cap_doubles*/, cudaStream_t s) {
  if (ntasks <= 0) return;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(elim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  elim_kernel<<<ntasks, NT, smem, s>>>(d_tasks, A);
}

void launch_skel(const SkelTask* d_tasks, int ntasks, const Arenas& A, double eps, size_t smem,
                 int /*smem_cap_doubles*/, cudaStream_t s) {
  if (ntasks <= 0) return;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(skel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  skel_kernel<<<ntasks, NT, smem, s>>>(d_tasks, A, eps);
}

void launch_apply_rd(const SkelTask* d_tasks, int ntasks, const Arenas& A, cudaStream_t s) {
  if (ntasks <= 0) return;
  apply_rd_kernel<<<ntasks, 64, 0, s>>>(d_tasks, A);
}

}  // namespace hifde
