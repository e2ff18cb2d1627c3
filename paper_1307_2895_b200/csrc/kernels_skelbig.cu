// Skeletonization of groups too large for one CTA (sm_100a).
//
// Pipeline per batch of large groups (src/factor_ops.py:162-214,
// src/dense.py:239-264):
//   skelbig_posmap_kernel    front position of every consumed block entry.
//   skelbig_assemble_kernel  rows of A_cc (row-major) and Mq = A_qc
//                            (column-major) into scratch; one CTA per row chunk.
//   cpqr_coop_kernel         column-pivoted QR of Mq with the rank cut, by
//                            G co-resident CTAs per group (cooperative launch,
//                            the batch's groups share all SMs).  Columns are
//                            owned round-robin and never moved (pivoting = a
//                            pivot list); each step every CTA rebuilds the
//                            reflector from the pivot column, updates and
//                            downdates its own columns, and posts its best
//                            remaining norm; one group barrier per step.
//                            dlaqp2 semantics.
//   skelbig_gram_kernel +    (loose tolerances, eps >= kGramMinEps, instead of
//   pchol_mc_kernel          the CPQR) G = Mq^T Mq on DMMA tiles, then a
//                            cooperative pivoted Cholesky of G writing the
//                            CPQR's outputs (same pivots and rank cut in
//                            exact arithmetic).
//   skelbig_sort_kernel      sk / rd ascending, output index lists, inner task.
//   skelbig_t*_kernel        T = R11^-1 R12, blocked back substitution (64-row
//                            diagonal solves + DMMA updates), then written
//                            row-permuted to ascending sk order in the record.
//   skelbig_bsr_kernel       B_sr = A_sr - A_ss T   (DMMA), stored as W^T input.
//   skelbig_brr_kernel       B_rr = A_rr - A_sr^T T - T^T B_sr (DMMA).
//   skelbig_symm_kernel      B_rr <- (B_rr + B_rr^T)/2, max |diag|.
// The inner elimination of rd against sk (Cholesky of B_rr, W, delta block
// -W^T W) reuses the blocked large-cell kernels of kernels_big.cu.
#include <cfloat>
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda/atomic>
#include <utility>
#include <vector>

#include "hifde_internal.h"

namespace hifde {

namespace {

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

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Warp-strided dot product / axpy over rows [r0, n) with 8 independent loads
// in flight per lane (the columns live in L2/HBM).
__device__ __forceinline__ double wdot(const double* __restrict__ a, const double* __restrict__ b, int r0, int n,
                                       int lane) {
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int r = r0 + lane;
  for (; r + 7 * 32 < n; r += 8 * 32) {
#pragma unroll
    for (int u = 0; u < 8; ++u) s[u] += a[r + 32 * u] * b[r + 32 * u];
  }
  for (; r < n; r += 32) s[0] += a[r] * b[r];
  return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}
__device__ __forceinline__ void waxpy(double* __restrict__ y, const double* __restrict__ x, double alpha, int r0,
                                      int n, int lane) {
  int r = r0 + lane;
  for (; r + 7 * 32 < n; r += 8 * 32) {
    double yv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) yv[u] = y[r + 32 * u];
#pragma unroll
    for (int u = 0; u < 8; ++u) y[r + 32 * u] = yv[u] - alpha * x[r + 32 * u];
  }
  for (; r < n; r += 32) y[r] -= alpha * x[r];
}

// Barrier among the G co-resident CTAs of one group (cooperative launch):
// a monotonic arrival counter, each CTA waits for G * round arrivals.
__device__ __forceinline__ void group_barrier(unsigned int* ctr, unsigned int G, unsigned int& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += G;
    cuda::atomic_ref<unsigned int, cuda::thread_scope_device> a(*ctr);
    a.fetch_add(1u, cuda::memory_order_release);
    while (a.load(cuda::memory_order_acquire) < target) __nanosleep(32);
  }
  __syncthreads();
}

// scratch layout of one large group (doubles)
struct BigWs {
  double *Acc, *Mq, *Tp, *vn1, *vn2, *rdiag, *cand, *G;
  int32_t *piv, *skl, *sko, *rdl;
};
__device__ __forceinline__ BigWs big_ws(const SkelBigTask& t, const Arenas& A) {
  BigWs w;
  const size_t nc = t.nc, nq = t.nq;
  w.Acc = A.scratch + t.ws_off;
  w.Mq = w.Acc + nc * nc;
  w.Tp = w.Mq + nq * nc;
  w.vn1 = w.Tp + (nc * nc / 4 + nc);
  w.vn2 = w.vn1 + nc;
  w.rdiag = w.vn2 + nc;
  w.cand = w.rdiag + nc;  // 2 x kMaxG x (value, index)
  w.G = w.cand + 4 * kMaxG + 8;  // Gram matrix Mq^T Mq (nc x nc), the Gram path only
  w.piv = A.iscratch + t.iws_off;
  w.skl = w.piv + nc;
  w.sko = w.skl + nc;
  w.rdl = w.sko + nc;
  return w;
}

}  // namespace

// ---------------------------------------------------------------------------
// Per (group, block): the block's entries that land in the front, as two
// arrays sorted by front position -- first the entries in c (positions < nc),
// then those in q -- so an assembly CTA finds its rows by binary search and
// takes the c columns as a prefix, instead of scanning every entry.  Work
// item int4 {task, block, offset}; region = [cnt_c, cnt_q, pos[nb], ent[nb]].
// The block's DOFs ascend, so its c entries and its q entries each ascend in
// position: a stable partition (ballots + warp offsets) sorts them.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) skelbig_posmap_kernel(const SkelBigTask* __restrict__ tasks,
                                                             const int4* __restrict__ work, Arenas A) {
  __shared__ int wsum[2][8];
  __shared__ int base[2];
  __shared__ int ctot;
  const int4 wk = work[blockIdx.x];
  const SkelBigTask t = tasks[wk.x];
  const int nc = t.nc, nq = t.nq;
  const int32_t* gd = A.idx + t.dofs_off;
  const int bid = A.lists[t.blk_off + wk.y];
  const int nb = A.blk_n[bid];
  const int32_t* bd = A.idx + A.blk_dof_off[bid];
  int32_t* reg = A.iscratch + t.map_off + wk.z;
  int32_t* pos = reg + 2;
  int32_t* ent = pos + nb;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto position = [&](int k) {
    int p = front_pos(gd, nc, nq, bd[k]);
    if (p >= nc && !A.active[gd[p]]) p = -1;
    return p;
  };
  int c = 0;  // pass 1: the number of c entries
  for (int k = threadIdx.x; k < nb; k += 256) {
    const int p = position(k);
    c += (p >= 0 && p < nc) ? 1 : 0;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if (lane == 0) wsum[0][wid] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < 8; ++w) tot += wsum[0][w];
    ctot = tot;
    base[0] = 0;
    base[1] = tot;
  }
  __syncthreads();
  for (int k0 = 0; k0 < nb; k0 += 256) {  // pass 2: stable partition, 256 entries at a time
    const int k = k0 + (int)threadIdx.x;
    const int p = k < nb ? position(k) : -1;
    const bool isc = p >= 0 && p < nc, isq = p >= nc;
    const unsigned mc = __ballot_sync(0xffffffffu, isc), mq = __ballot_sync(0xffffffffu, isq);
    if (lane == 0) {
      wsum[0][wid] = __popc(mc);
      wsum[1][wid] = __popc(mq);
    }
    __syncthreads();
    int oc = base[0], oq = base[1];
    for (int w = 0; w < wid; ++w) {
      oc += wsum[0][w];
      oq += wsum[1][w];
    }
    const unsigned lt = (1u << lane) - 1u;
    if (isc) {
      const int o = oc + __popc(mc & lt);
      pos[o] = p;
      ent[o] = k;
    }
    if (isq) {
      const int o = oq + __popc(mq & lt);
      pos[o] = p;
      ent[o] = k;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 0; w < 8; ++w) {
        base[0] += wsum[0][w];
        base[1] += wsum[1][w];
      }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    reg[0] = ctot;
    reg[1] = base[1] - ctot;
  }
}

// ---------------------------------------------------------------------------
// Assembly of [A_cc ; Mq].  Work item int4 {task, r0, r1, 0}: front rows.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) skelbig_assemble_kernel(const SkelBigTask* __restrict__ tasks,
                                                               const int4* __restrict__ work, Arenas A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int4 wk = work[blockIdx.x];
  const SkelBigTask t = tasks[wk.x];
  const int nc = t.nc, nq = t.nq, nf = nc + nq;
  const int r0 = wk.y, r1 = wk.z;
  int32_t* sdofs = reinterpret_cast<int32_t*>(smem);
  int32_t* salive = sdofs + nf;
  const BigWs w = big_ws(t, A);
  const int32_t* gd = A.idx + t.dofs_off;
  for (int i = threadIdx.x; i < nf; i += 256) {
    sdofs[i] = gd[i];
    salive[i] = i < nc ? 1 : (int)A.active[gd[i]];
  }
  for (int r = r0; r < r1; ++r) {
    if (r < nc) for (int j = threadIdx.x; j < nc; j += 256) w.Acc[(size_t)r * nc + j] = 0.0;
    else for (int j = threadIdx.x; j < nc; j += 256) w.Mq[(size_t)(r - nc) + (size_t)j * nq] = 0.0;
  }
  __syncthreads();
  // original couplings: c rows give A_cc, alive q rows give their c columns
  for (int r = r0 + (int)threadIdx.x; r < r1; r += 256) {
    if (!salive[r]) continue;
    const int g = sdofs[r];
    for (int64_t k = A.indptr[g]; k < A.indptr[g + 1]; ++k) {
      const int pj = bsearch_i32(sdofs, nc, A.indices[k]);
      if (pj < 0) continue;
      if (r < nc) w.Acc[(size_t)r * nc + pj] += A.a0[k];
      else w.Mq[(size_t)(r - nc) + (size_t)pj * nq] += A.a0[k];
    }
  }
  __syncthreads();
  const int32_t* bl = A.lists + t.blk_off;
  const int32_t* reg = A.iscratch + t.map_off;  // per block: [cnt_c, cnt_q, pos[nb], ent[nb]] by position
  for (int b = 0; b < t.nblk; ++b) {
    const int bid = bl[b];
    const int nb = A.blk_n[bid];
    const double* bv = A.bvals + A.blk_val_off[bid];
    const int ncn = reg[0], ntot = reg[0] + reg[1];
    const int32_t* pos = reg + 2;
    const int32_t* ent = pos + nb;
    // this CTA's rows: positions in [r0, r1), a contiguous range of the list
    int lo = 0, hi = ntot;
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if (pos[m] < r0) lo = m + 1; else hi = m;
    }
    const int s0 = lo;
    hi = ntot;
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if (pos[m] < r1) lo = m + 1; else hi = m;
    }
    const int ns = lo - s0;
    // every (row, c column) pair: one source per destination entry in a block
    for (int e = threadIdx.x; e < ns * ncn; e += 256) {
      const int sr = e / ncn, cc = e - sr * ncn;
      const int k = ent[s0 + sr], l = ent[cc];
      const int pk = pos[s0 + sr], pl = pos[cc];
      const double val = bv[(size_t)k * nb + l];
      if (pk < nc) w.Acc[(size_t)pk * nc + pl] += val;
      else w.Mq[(size_t)(pk - nc) + (size_t)pl * nq] += val;
    }
    reg += 2 + 2 * nb;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Multi-CTA CPQR.  Cooperative launch; CTAs [gstart[t], gstart[t+1]) serve
// task t and synchronize through a per-task software barrier.
// ---------------------------------------------------------------------------
// kCluster: thread-block clusters of kCL CTAs (hardware cluster barrier),
// otherwise a cooperative launch with a software barrier per group.
template <bool kCluster>
__global__ void __launch_bounds__(256) cpqr_mc_kernel(const SkelBigTask* __restrict__ tasks, int ntasks,
                                                      const int* __restrict__ gstart,
                                                      unsigned int* __restrict__ bar, Arenas A, double eps) {
  extern __shared__ __align__(16) double vsm[];  // reflector column (nq doubles)
  __shared__ double red[8];
  __shared__ double spart[16];  // split-column partial dots
  __shared__ double sh_best;
  __shared__ int sh_pvt;
  __shared__ unsigned char done[kMaxBigNc];
  int tix = 0, rb = 0, CL = 1;
  if (kCluster) {
    cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    rb = (int)cl.block_rank();
    CL = (int)cl.num_blocks();
    tix = (int)blockIdx.x / CL;
  } else {
    while (tix + 1 < ntasks && (int)blockIdx.x >= gstart[tix + 1]) ++tix;
    rb = (int)blockIdx.x - gstart[tix];
    CL = gstart[tix + 1] - gstart[tix];
  }
  unsigned int* ctr = bar + tix;
  unsigned int target = 0;
  auto gsync = [&]() {
    if (kCluster) cooperative_groups::this_cluster().sync();
    else group_barrier(ctr, (unsigned)CL, target);
  };
  const SkelBigTask t = tasks[tix];
  const int nc = t.nc, nq = t.nq;
  const BigWs w = big_ws(t, A);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ldq = nq;
  for (int j = threadIdx.x; j < nc; j += 256) done[j] = 0;
  int nq_alive = 0;  // rows of inactive DOFs are exact zeros; count the live ones
  {
    const int32_t* gd = A.idx + t.dofs_off;
    int c = 0;
    for (int i = threadIdx.x; i < nq; i += 256) c += A.active[gd[nc + i]] ? 1 : 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) red[wid] = c;
    __syncthreads();
    for (int i = 0; i < 8; ++i) nq_alive += (int)red[i];
    __syncthreads();
  }
  // initial norms of the owned columns and the first candidate
  double best = -1.0;
  int bidx = nc;
  for (int j = rb + CL * wid; j < nc; j += CL * 8) {
    const double* col = w.Mq + (size_t)j * ldq;
    double s = wdot(col, col, 0, nq, lane);
    s = sqrt(warp_sum(s));
    if (lane == 0) { w.vn1[j] = s; w.vn2[j] = s; }
    if (s > best || (s == best && j < bidx)) { best = s; bidx = j; }
  }
  // block argmax of (best, bidx) -> this CTA's candidate slot
  __shared__ double wbest[8];
  __shared__ int widx[8];
  auto block_best = [&](double v, int ix, int slot) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, ix, o);
      if (ov > v || (ov == v && oi < ix)) { v = ov; ix = oi; }
    }
    if (lane == 0) { wbest[wid] = v; widx[wid] = ix; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bv = wbest[0];
      int bi = widx[0];
      for (int q = 1; q < 8; ++q)
        if (wbest[q] > bv || (wbest[q] == bv && widx[q] < bi)) { bv = wbest[q]; bi = widx[q]; }
      w.cand[(size_t)(slot * CL + rb) * 2] = bv;
      w.cand[(size_t)(slot * CL + rb) * 2 + 1] = (double)bi;
    }
  };
  block_best(best, bidx, 0);
  gsync();

  const int kmax = nq < nc ? nq : nc;
  const double tol3z = sqrt(DBL_EPSILON * 0.5);
  double thr = 0.0;
  int k = kmax;
  for (int i = 0; i < kmax; ++i) {
    const int slot = i & 1;
    {
      // all candidates read in parallel, block argmax (lowest index on ties)
      double bv = -1.0;
      int bi = nc;
      for (int q = threadIdx.x; q < CL; q += 256) {
        const double v = __ldcg(&w.cand[(size_t)(slot * CL + q) * 2]);
        const int ix = (int)__ldcg(&w.cand[(size_t)(slot * CL + q) * 2 + 1]);
        if (v > bv || (v == bv && ix < bi)) { bv = v; bi = ix; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { wbest[wid] = bv; widx[wid] = bi; }
      __syncthreads();
      if (threadIdx.x == 0) {
        double b2 = wbest[0];
        int i2 = widx[0];
        for (int q = 1; q < 8; ++q)
          if (wbest[q] > b2 || (wbest[q] == b2 && widx[q] < i2)) { b2 = wbest[q]; i2 = widx[q]; }
        sh_best = b2;
        sh_pvt = i2;
      }
    }
    __syncthreads();
    const int P = sh_pvt;
    if (i == 0 && sh_best == 0.0) { k = 0; break; }  // zero block: all redundant

    // reflector from column P rows i.. (every CTA, identical arithmetic)
    const double* colP = w.Mq + (size_t)P * ldq;
    double xs = 0.0;
    for (int r = i + 1 + (int)threadIdx.x; r < nq; r += 256) {
      const double x = __ldcg(colP + r);
      vsm[r] = x;
      xs += x * x;
    }
    xs = warp_sum(xs);
    if (lane == 0) red[wid] = xs;
    __syncthreads();
    double xn2 = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) xn2 += red[q];
    const double xnorm = sqrt(xn2);
    const double alpha = __ldcg(colP + i);
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
    if (rb == 0 && threadIdx.x == 0) {
      w.rdiag[i] = beta;
      w.piv[i] = P;
    }
    best = -1.0;
    bidx = nc;
    // owned, not yet pivoted columns of this CTA
    int nown = 0;
    for (int j = rb; j < nc; j += CL) nown += (done[j] || j == P) ? 0 : 1;
    if (nown > 0 && nown <= 4) {
      // few columns per CTA (many CTAs per group): the rows of each column
      // are split over S warps, partial dots combined in a fixed order
      const int S = 8 / nown;
      const int c = wid / S, sl = wid - c * S;
      int j = -1;
      if (c < nown) {
        int q = 0;
        for (int jj = rb; jj < nc; jj += CL) {
          if (done[jj] || jj == P) continue;
          if (q++ == c) { j = jj; break; }
        }
      }
      const int m1 = nq - (i + 1);
      const int chunk = ((m1 + S - 1) / S + 31) & ~31;
      const int ra = i + 1 + sl * chunk, rz = min(nq, ra + chunk);
      double* col = j >= 0 ? w.Mq + (size_t)j * ldq : nullptr;
      double ci = 0.0;
      if (j >= 0 && tau != 0.0) {
        ci = col[i];
        const double s = warp_sum(wdot(vsm, col, ra, rz, lane));
        if (lane == 0) spart[wid] = s;
      }
      __syncthreads();
      double nv = 0.0;
      bool recompute = false;
      if (j >= 0) {
        double civ = ci;
        if (tau != 0.0) {
          double s = 0.0;
          for (int q = 0; q < S; ++q) s += spart[c * S + q];
          const double wv = tau * (ci + scal * s);
          civ = ci - wv;
          waxpy(col, vsm, wv * scal, ra, rz, lane);
          if (sl == 0 && lane == 0) col[i] = civ;
        } else {
          civ = col[i];
        }
        nv = w.vn1[j];
        if (nv != 0.0) {
          double tmp = fabs(civ) / nv;
          tmp = 1.0 - tmp * tmp;
          tmp = tmp > 0.0 ? tmp : 0.0;
          const double ratio = nv / w.vn2[j];
          if (tmp * ratio * ratio <= tol3z) recompute = true;
          else nv *= sqrt(tmp);
        }
      }
      if (__syncthreads_or(recompute ? 1 : 0)) {  // rare: norms recomputed from the rows
        if (recompute) {
          const double s = warp_sum(wdot(col, col, ra, rz, lane));
          if (lane == 0) spart[8 + wid] = s;
        }
        __syncthreads();
        if (recompute) {
          double s = 0.0;
          for (int q = 0; q < S; ++q) s += spart[8 + c * S + q];
          nv = (i + 1 < nq) ? sqrt(s) : 0.0;
          if (sl == 0 && lane == 0) w.vn2[j] = nv;
        }
      }
      if (j >= 0 && sl == 0) {
        if (lane == 0) w.vn1[j] = nv;
        if (nv > best || (nv == best && j < bidx)) { best = nv; bidx = j; }
      }
    } else
    // update the owned, not yet pivoted columns (warp per column)
    for (int j = rb + CL * wid; j < nc; j += CL * 8) {
      if (done[j] || j == P) continue;
      double* col = w.Mq + (size_t)j * ldq;
      double civ;  // R(i, j) after this step, kept in a register
      if (tau != 0.0) {
        const double ci = col[i];
        double s = wdot(vsm, col, i + 1, nq, lane);
        s = warp_sum(s);
        const double wv = tau * (ci + scal * s);
        civ = ci - wv;
        __syncwarp();
        if (lane == 0) col[i] = civ;
        waxpy(col, vsm, wv * scal, i + 1, nq, lane);
        __syncwarp();
      } else {
        civ = col[i];
      }
      double nv = w.vn1[j];
      bool recompute = false;
      if (nv != 0.0) {
        double tmp = fabs(civ) / nv;
        tmp = 1.0 - tmp * tmp;
        tmp = tmp > 0.0 ? tmp : 0.0;
        const double ratio = nv / w.vn2[j];
        if (tmp * ratio * ratio <= tol3z) recompute = true;
        else nv *= sqrt(tmp);
      }
      if (recompute) {
        double s = wdot(col, col, i + 1, nq, lane);
        s = warp_sum(s);
        nv = (i + 1 < nq) ? sqrt(s) : 0.0;
        if (lane == 0) w.vn2[j] = nv;
      }
      if (lane == 0) w.vn1[j] = nv;
      if (nv > best || (nv == best && j < bidx)) { best = nv; bidx = j; }
    }
    __syncthreads();
    if (P % CL == rb && threadIdx.x == 0) done[P] = 1;
    block_best(best, bidx, slot ^ 1);
    gsync();
  }
  if (rb == 0 && threadIdx.x == 0) A.kout[t.group] = k;
}

constexpr int kTT = 64, kTK = 16, kTL = 68;  // DMMA tile kernels: 64 x 64 tiles, K chunks of 16

// ---------------------------------------------------------------------------
// Gram path of the large-group ID (tolerances eps >= kGramMinEps, tall groups):
//   skelbig_gram_kernel   G = Mq^T Mq on 64 x 64 DMMA tiles, one pass over Mq
//   pchol_mc_kernel       pivoted Cholesky of G with the CPQR's rank cut
// Pivoted Cholesky of G picks, step by step, the column of Mq whose component
// orthogonal to the columns already chosen is largest: the pivots, the
// rank cut |R_ii| <= eps |R_00| and R itself (up to row signs, which T =
// R11^-1 R12 does not see) are those of the column-pivoted QR of Mq, in exact
// arithmetic.  The Schur diagonal carries an absolute error ~k u |G| against
// the cut at eps^2 |G|; T = G11^-1 G12 is off by ~u cond(G11) ~ u / eps^2, but
// only along the small singular directions of M_sk, so the ID residual
// |M_rd - M_sk T| moves by ~u / eps.  The path is taken only for eps >=
// kGramMinEps = 1e-4, where even the worst-case T error u / eps^2 <= 1e-8 is
// far below eps (config 5, eps = 1e-3: ranks identical to the CPQR path;
// config 4, eps = 1e-6, takes the CPQR).  Traffic: one read of Mq plus O(nc k) per step against O(nq nc) per step
// for the CPQR on Mq itself.
// ---------------------------------------------------------------------------
// Work item int4 {task, a0, b0, split}: rows [split * kGramRows, +kGramRows)
// of the 64 x 64 tile (a0, b0), a0 <= b0.  One split: G directly; several:
// the tile's partial goes to part[item] and skelbig_gram_reduce_kernel sums
// the splits in order (deterministic).  Rows are staged 32 at a time with the
// next stage prefetched into registers during the DMMA loop.
constexpr int kGK = 32;
__global__ void __launch_bounds__(128) skelbig_gram_kernel(const SkelBigTask* __restrict__ tasks,
                                                           const int4* __restrict__ work, Arenas A,
                                                           double* __restrict__ part) {
  __shared__ double As[kGK][kTL];
  __shared__ double Bs[kGK][kTL];
  const int4 wk = work[blockIdx.x];
  const SkelBigTask t = tasks[wk.x];
  const BigWs w = big_ws(t, A);
  const int nc = t.nc, nq = t.nq;
  const int a0 = wk.y, b0 = wk.z;
  const int r_lo = wk.w * kGramRows, r_hi = min(nq, r_lo + kGramRows);
  const bool split = nq > kGramRows;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wy = wid >> 1, wx = wid & 1;
  double acc[4][4][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  double pa[16], pb[16];
  // thread e = tid + 128 u stages row (e & 31) of column (e >> 5): a warp reads
  // 32 consecutive rows of one column (256 contiguous bytes)
  auto load = [&](int r0) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = (int)threadIdx.x + 128 * u;
      const int r = r0 + (e & 31), x = e >> 5;
      pa[u] = (r < r_hi && a0 + x < nc) ? __ldcg(w.Mq + (size_t)r + (size_t)(a0 + x) * nq) : 0.0;
      pb[u] = (r < r_hi && b0 + x < nc) ? __ldcg(w.Mq + (size_t)r + (size_t)(b0 + x) * nq) : 0.0;
    }
  };
  load(r_lo);
  for (int r0 = r_lo; r0 < r_hi; r0 += kGK) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = (int)threadIdx.x + 128 * u;
      As[e & 31][e >> 5] = pa[u];
      Bs[e & 31][e >> 5] = pb[u];
    }
    __syncthreads();
    if (r0 + kGK < r_hi) load(r0 + kGK);
#pragma unroll
    for (int kk = 0; kk < kGK; kk += 4) {
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
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ta = wy * 32 + m * 8 + (lane >> 2);
        const int tb = wx * 32 + n * 8 + 2 * (lane & 3) + h;
        if (split) {
          part[(size_t)blockIdx.x * 4096 + ta * 64 + tb] = acc[m][n][h];
          continue;
        }
        const int a = a0 + ta, b = b0 + tb;
        // G is symmetric: each (a, b), a <= b, written once and mirrored
        if (a < nc && b < nc && (a0 != b0 || a <= b)) {
          w.G[(size_t)a + (size_t)b * nc] = acc[m][n][h];
          w.G[(size_t)b + (size_t)a * nc] = acc[m][n][h];
        }
      }
}

// Sum of a tile's row splits in split order.  Work int4 {task, a0, b0, first
// item}; the splits of a tile are consecutive work items.
__global__ void __launch_bounds__(256) skelbig_gram_reduce_kernel(const SkelBigTask* __restrict__ tasks,
                                                                  const int4* __restrict__ work, Arenas A,
                                                                  const double* __restrict__ part) {
  const int4 wk = work[blockIdx.x];
  const SkelBigTask t = tasks[wk.x];
  const BigWs w = big_ws(t, A);
  const int nc = t.nc, nq = t.nq;
  const int ns = (nq + kGramRows - 1) / kGramRows;
  const int a0 = wk.y, b0 = wk.z;
  for (int e = threadIdx.x; e < 4096; e += 256) {
    const int a = a0 + (e >> 6), b = b0 + (e & 63);
    if (a >= nc || b >= nc || (a0 == b0 && a > b)) continue;
    double v = 0.0;
    for (int q = 0; q < ns; ++q) v += part[(size_t)(wk.w + q) * 4096 + e];
    w.G[(size_t)a + (size_t)b * nc] = v;
    w.G[(size_t)b + (size_t)a * nc] = v;
  }
}

// Cooperative launch; CTAs [gstart[t], gstart[t+1]) serve task t.  CTA rb of
// CL owns columns rb, rb + CL, ... and keeps their R rows in shared memory;
// R(i, j) also goes to Mq[i + j nq], the CPQR's output layout (rdiag, piv,
// kout likewise), so the T / congruence kernels run unchanged.
__global__ void __launch_bounds__(256) pchol_mc_kernel(const SkelBigTask* __restrict__ tasks, int ntasks,
                                                       const int* __restrict__ gstart,
                                                       unsigned int* __restrict__ bar, Arenas A, double eps) {
  extern __shared__ __align__(16) double psm[];
  __shared__ double wbest[8];
  __shared__ int widx[8];
  __shared__ double sh_best;
  __shared__ int sh_pvt;
  int tix = 0;
  while (tix + 1 < ntasks && (int)blockIdx.x >= gstart[tix + 1]) ++tix;
  const int rb = (int)blockIdx.x - gstart[tix];
  const int CL = gstart[tix + 1] - gstart[tix];
  unsigned int* ctr = bar + tix;
  unsigned int target = 0;
  const SkelBigTask t = tasks[tix];
  const int nc = t.nc, nq = t.nq;
  const BigWs w = big_ws(t, A);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nown = rb < nc ? (nc - rb + CL - 1) / CL : 0;
  double* Rs = psm;                       // [nc][nown]: R(l, rb + c CL) at l * nown + c
  double* rp = Rs + (size_t)nc * nown;    // R(0..i-1, P)
  double* dd = rp + nc;                   // Schur diagonal of the owned columns (< 0: pivoted)
  double* gcol = dd + nown;               // G(j, P) of the owned columns, this step
  for (int c = threadIdx.x; c < nown; c += 256) {
    const int j = rb + c * CL;
    dd[c] = w.G[(size_t)j + (size_t)j * nc];
  }
  __syncthreads();
  auto post = [&](int slot) {  // this CTA's best remaining column -> candidate slot
    double bv = -1.0;
    int bi = nc;
    for (int c = threadIdx.x; c < nown; c += 256)
      if (dd[c] > bv) { bv = dd[c]; bi = rb + c * CL; }  // ascending j: first max wins
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { wbest[wid] = bv; widx[wid] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b2 = wbest[0];
      int i2 = widx[0];
      for (int q = 1; q < 8; ++q)
        if (wbest[q] > b2 || (wbest[q] == b2 && widx[q] < i2)) { b2 = wbest[q]; i2 = widx[q]; }
      w.cand[(size_t)(slot * CL + rb) * 2] = b2;
      w.cand[(size_t)(slot * CL + rb) * 2 + 1] = (double)i2;
    }
  };
  post(0);
  group_barrier(ctr, (unsigned)CL, target);
  double thr = 0.0;
  int k = nc;
  for (int i = 0; i < nc; ++i) {
    const int slot = i & 1;
    {
      double bv = -1.0;
      int bi = nc;
      for (int q = threadIdx.x; q < CL; q += 256) {
        const double v = __ldcg(&w.cand[(size_t)(slot * CL + q) * 2]);
        const int ix = (int)__ldcg(&w.cand[(size_t)(slot * CL + q) * 2 + 1]);
        if (v > bv || (v == bv && ix < bi)) { bv = v; bi = ix; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { wbest[wid] = bv; widx[wid] = bi; }
      __syncthreads();
      if (threadIdx.x == 0) {
        double b2 = wbest[0];
        int i2 = widx[0];
        for (int q = 1; q < 8; ++q)
          if (wbest[q] > b2 || (wbest[q] == b2 && widx[q] < i2)) { b2 = wbest[q]; i2 = widx[q]; }
        sh_best = b2;
        sh_pvt = i2;
      }
      __syncthreads();
    }
    const int P = sh_pvt;
    const double dP = sh_best;
    if (i == 0 && !(dP > 0.0)) { k = 0; break; }  // zero block: all redundant
    const double rii = sqrt(dP > 0.0 ? dP : 0.0);
    if (i == 0) thr = eps * rii;
    if (rii <= thr || P >= nc) { k = i; break; }
    if (rb == 0 && threadIdx.x == 0) {
      w.rdiag[i] = rii;
      w.piv[i] = P;
    }
    // every load of the step issued together (one L2 latency, not one per column)
    for (int l = threadIdx.x; l < i; l += 256) rp[l] = __ldcg(w.Mq + (size_t)l + (size_t)P * nq);
    for (int c = threadIdx.x; c < nown; c += 256) gcol[c] = __ldcg(w.G + (size_t)(rb + c * CL) + (size_t)P * nc);
    __syncthreads();
    const double inv = 1.0 / rii;
    for (int c = wid; c < nown; c += 8) {
      const int j = rb + c * CL;
      if (dd[c] < 0.0) continue;  // pivoted earlier
      if (j == P) {
        __syncwarp();
        if (lane == 0) dd[c] = -1.0;
        continue;
      }
      double sacc = 0.0;
      for (int l = lane; l < i; l += 32) sacc += rp[l] * Rs[(size_t)l * nown + c];
      sacc = warp_sum(sacc);
      const double rij = (gcol[c] - sacc) * inv;
      __syncwarp();
      if (lane == 0) {
        Rs[(size_t)i * nown + c] = rij;
        w.Mq[(size_t)i + (size_t)j * nq] = rij;
        const double nd = dd[c] - rij * rij;
        dd[c] = nd > 0.0 ? nd : 0.0;
      }
    }
    __syncthreads();
    post(slot ^ 1);
    group_barrier(ctr, (unsigned)CL, target);
  }
  if (rb == 0 && threadIdx.x == 0) A.kout[t.group] = k;
}


// ---------------------------------------------------------------------------
// sk / rd ascending, output lists, inner elimination task (one CTA per group)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) skelbig_sort_kernel(const SkelBigTask* __restrict__ tasks, Arenas A,
                                                           ElimTask* __restrict__ inner, double* __restrict__ dmin,
                                                           double* __restrict__ dscale) {
  __shared__ unsigned char piv_flag[kMaxBigNc];
  const SkelBigTask t = tasks[blockIdx.x];
  const int nc = t.nc;
  const BigWs w = big_ws(t, A);
  const int k = A.kout[t.group], r = nc - k;
  for (int j = threadIdx.x; j < nc; j += 256) piv_flag[j] = 0;
  __syncthreads();
  for (int a = threadIdx.x; a < k; a += 256) piv_flag[w.piv[a]] = 1;
  __syncthreads();
  for (int a = threadIdx.x; a < k; a += 256) {
    const int v = w.piv[a];
    int rank = 0;
    for (int b = 0; b < k; ++b) rank += w.piv[b] < v;
    w.skl[rank] = v;
    w.sko[rank] = a;
  }
  // rd: the non-pivoted columns in ascending order
  for (int j = threadIdx.x; j < nc; j += 256) {
    if (piv_flag[j]) continue;
    int rank = 0;
    for (int l = 0; l < j; ++l) rank += piv_flag[l] ? 0 : 1;
    w.rdl[rank] = j;
  }
  __syncthreads();
  const int32_t* gd = A.idx + t.dofs_off;
  int32_t* out = A.idx + t.out_off;
  for (int a = threadIdx.x; a < k; a += 256) out[a] = gd[w.skl[a]];
  for (int b = threadIdx.x; b < r; b += 256) out[k + b] = gd[w.rdl[b]];
  if (threadIdx.x == 0) {
    ElimTask e;
    e.nc = r;
    e.nq = k;
    e.nblk = 0;
    e.maxnb = 0;
    e.dofs_off = 0;
    e.blk_off = 0;
    e.scratch_off = -1;
    e.C_off = t.rec_off + (int64_t)k * r;
    e.W_off = e.C_off + (int64_t)r * r;
    e.U_off = t.delta_off;
    // packed inverse after the largest T | C | W footprint of the record
    e.P_off = t.rec_off + (int64_t)nc * nc + 2 * ((int64_t)nc * nc / 4 + nc);
    inner[blockIdx.x] = e;
    dmin[blockIdx.x] = DBL_MAX;
    dscale[blockIdx.x] = 0.0;
    A.status[blockIdx.x] = 0;
  }
}

// ---------------------------------------------------------------------------
// T = R11^-1 R12 by blocked back substitution over 64-row blocks (bottom-up):
//   skelbig_tinit_kernel    Tp = R12                (work {task, row0})
//   skelbig_tsolve_kernel   diagonal block solve    (work {task, col0}, block b0)
//   skelbig_tupdate_kernel  rows above -= R11 Tp    (work {task, a0, c0}, block b0)
//   skelbig_tperm_kernel    record T = Tp rows in ascending sk order
// R11[a][l] = Mq[a + piv[l] nq], R12[a][c] = Mq[a + rd_c nq] (pivot order).
// Block loops run on the size bound; the kernels skip rows >= k.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) skelbig_tinit_kernel(const SkelBigTask* __restrict__ tasks,
                                                            const int4* __restrict__ work, Arenas A) {
  const int4 wk = work[blockIdx.x];
  const SkelBigTask t = tasks[wk.x];
  const BigWs w = big_ws(t, A);
  const int k = A.kout[t.group], r = t.nc - k;
  for (int a = wk.y; a < min(wk.y + 64, k); ++a)
    for (int c = threadIdx.x; c < r; c += 256) w.Tp[(size_t)a * r + c] = w.Mq[a + (size_t)w.rdl[c] * t.nq];
}

__global__ void __launch_bounds__(128) skelbig_tsolve_kernel(const SkelBigTask* __restrict__ tasks,
                                                             const int4* __restrict__ work, int b0, Arenas A) {
  __shared__ double R[64][65];
  const int4 wk = work[blockIdx.x];
  const SkelBigTask t = tasks[wk.x];
  const BigWs w = big_ws(t, A);
  const int k = A.kout[t.group], r = t.nc - k;
  if (b0 >= k || wk.y >= r) return;
  const int b1 = min(b0 + 64, k), bw = b1 - b0;
  for (int e = threadIdx.x; e < bw * bw; e += 128) {
    const int i = e / bw, j = e - i * bw;
    R[i][j] = (j > i) ? w.Mq[(size_t)(b0 + i) + (size_t)w.piv[b0 + j] * t.nq] : 0.0;
  }
  __syncthreads();
  const int c = wk.y + (int)threadIdx.x;
  if (c >= r) return;
  double x[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) x[i] = 0.0;
  for (int i = bw - 1; i >= 0; --i) {
    double v = w.Tp[(size_t)(b0 + i) * r + c];
#pragma unroll 8
    for (int j = i + 1; j < 64; ++j)
      if (j < bw) v -= R[i][j] * x[j];
    // x[i] with a dynamic index would spill; select by unrolled compare
    const double xi = v / w.rdiag[b0 + i];
#pragma unroll
    for (int q = 0; q < 64; ++q)
      if (q == i) x[q] = xi;
  }
#pragma unroll
  for (int i = 0; i < 64; ++i)
    if (i < bw) w.Tp[(size_t)(b0 + i) * r + c] = x[i];
}

__global__ void __launch_bounds__(128) skelbig_tupdate_kernel(const SkelBigTask* __restrict__ tasks,
                                                              const int4* __restrict__ work, int b0, Arenas A) {
  __shared__ double As[kTK][kTL];
  __shared__ double Bs[kTK][kTL];
  const int4 wk = work[blockIdx.x];
  const SkelBigTask t = tasks[wk.x];
  const BigWs w = big_ws(t, A);
  const int k = A.kout[t.group], r = t.nc - k;
  const int a0 = wk.y, c0 = wk.z;
  if (b0 >= k || a0 >= b0 || c0 >= r) return;
  const int b1 = min(b0 + 64, k), bw = b1 - b0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wy = wid >> 1, wx = wid & 1;
  double acc[4][4][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  for (int l0 = 0; l0 < bw; l0 += kTK) {
    __syncthreads();
    for (int e = threadIdx.x; e < kTK * kTT; e += 128) {
      const int ll = e / kTT, x = e - ll * kTT;
      const int l = b0 + l0 + ll;
      As[ll][x] = (l < b1 && a0 + x < b0) ? w.Mq[(size_t)(a0 + x) + (size_t)w.piv[l] * t.nq] : 0.0;
      Bs[ll][x] = (l < b1 && c0 + x < r) ? w.Tp[(size_t)l * r + c0 + x] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; kk += 4) {
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
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = a0 + wy * 32 + m * 8 + (lane >> 2);
        const int c = c0 + wx * 32 + n * 8 + 2 * (lane & 3) + h;
        if (a < b0 && c < r) w.Tp[(size_t)a * r + c] -= acc[m][n][h];
      }
}

__global__ void __launch_bounds__(256) skelbig_tperm_kernel(const SkelBigTask* __restrict__ tasks,
                                                            const int4* __restrict__ work, Arenas A) {
  const int4 wk = work[blockIdx.x];
  const SkelBigTask t = tasks[wk.x];
  const BigWs w = big_ws(t, A);
  const int k = A.kout[t.group], r = t.nc - k;
  double* T = A.fac + t.rec_off;
  for (int a = wk.y; a < min(wk.y + 64, k); ++a)
    for (int c = threadIdx.x; c < r; c += 256) T[(size_t)a * r + c] = w.Tp[(size_t)w.sko[a] * r + c];
}

// ---------------------------------------------------------------------------
// Congruence products on 64 x 64 tiles (DMMA m8n8k4, 2 x 2 warps of 32 x 32)
//   kind 0 (tile a over sk, b over rd): B_sr[a,b] = A_cc[sk_a, rd_b]
//            - sum_l A_cc[sk_a, sk_l] T[l,b];  stored transposed into W (r x k)
//   kind 1 (a, b over rd):  B_rr[a,b] = A_cc[rd_a, rd_b]
//            - sum_l A_cc[rd_a, sk_l] T[l,b] - sum_l T[l,a] B_sr[l,b]; into C
// work item int4 {task, kind, a0, b0}
// ---------------------------------------------------------------------------
constexpr int kT = 64, kKs = 16, kLd = 68;

__global__ void __launch_bounds__(128) skelbig_congruence_kernel(const SkelBigTask* __restrict__ tasks,
                                                                 const int4* __restrict__ work, Arenas A) {
  __shared__ double As[kGK][kTL];
  __shared__ double Bs[kGK][kTL];
  const int4 wk = work[blockIdx.x];
  const SkelBigTask t = tasks[wk.x];
  const int nc = t.nc;
  const BigWs w = big_ws(t, A);
  const int k = A.kout[t.group], r = nc - k;
  const int kind = wk.y, a0 = wk.z, b0 = wk.w;
  const int na = kind == 0 ? k : r;
  if (r == 0 || a0 >= na || b0 >= r) return;
  const double* T = A.fac + t.rec_off;            // k x r, ascending sk rows
  double* C = A.fac + t.rec_off + (size_t)k * r;   // r x r
  double* W = C + (size_t)r * r;                   // r x k  (= B_sr^T)
  const int32_t* ra = kind == 0 ? w.skl : w.rdl;   // row index set of the tile
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wy = wid >> 1, wx = wid & 1;
  double acc[4][4][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  // 32-deep stages, the next one prefetched into registers during the DMMA loop
  double pa[16], pb[16];
  auto load = [&](int pass, int l0) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = (int)threadIdx.x + 128 * u;
      const int l = l0 + (e >> 6), x = e & 63;
      double av = 0.0, bv = 0.0;
      if (l < k) {
        if (a0 + x < na) {
          if (pass == 0) av = w.Acc[(size_t)ra[a0 + x] * nc + w.skl[l]];   // A[row][sk_l]
          else av = T[(size_t)l * r + a0 + x];                             // T[l][a]
        }
        if (b0 + x < r) {
          if (pass == 0) bv = T[(size_t)l * r + b0 + x];                   // T[l][b]
          else bv = W[(size_t)(b0 + x) * k + l];                           // B_sr[l][b]
        }
      }
      pa[u] = av;
      pb[u] = bv;
    }
  };
  const int npass = kind == 0 ? 1 : 2;
  const int nst = (k + kGK - 1) / kGK;
  if (nst > 0) load(0, 0);
  for (int it = 0; it < npass * nst; ++it) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = (int)threadIdx.x + 128 * u;
      As[e >> 6][e & 63] = pa[u];
      Bs[e >> 6][e & 63] = pb[u];
    }
    __syncthreads();
    if (it + 1 < npass * nst) load((it + 1) / nst, ((it + 1) % nst) * kGK);
#pragma unroll
    for (int kk = 0; kk < kGK; kk += 4) {
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
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = a0 + wy * 32 + m * 8 + (lane >> 2);
        const int b = b0 + wx * 32 + n * 8 + 2 * (lane & 3) + h;
        if (a >= na || b >= r) continue;
        const double v = w.Acc[(size_t)ra[a] * nc + w.rdl[b]] - acc[m][n][h];
        if (kind == 0) W[(size_t)b * k + a] = v;
        else C[(size_t)a * r + b] = v;
      }
}

// B_rr <- (B_rr + B_rr^T) / 2 and max |diag|; work item int4 {task, row0, 0, 0}
__global__ void __launch_bounds__(256) skelbig_symm_kernel(const SkelBigTask* __restrict__ tasks,
                                                           const int4* __restrict__ work, Arenas A,
                                                           const int32_t* __restrict__ task_of, double* dscale) {
  const int4 wk = work[blockIdx.x];
  const SkelBigTask t = tasks[wk.x];
  const int k = A.kout[t.group], r = t.nc - k;
  double* C = A.fac + t.rec_off + (size_t)k * r;
  double m = 0.0;
  for (int a = wk.y; a < min(wk.y + 64, r); ++a) {
    for (int b = threadIdx.x; b < a; b += 256) {
      const double v = 0.5 * (C[(size_t)a * r + b] + C[(size_t)b * r + a]);
      C[(size_t)a * r + b] = v;
      C[(size_t)b * r + a] = v;
    }
    if (threadIdx.x == 0) m = fmax(m, fabs(C[(size_t)a * r + a]));
  }
  (void)task_of;
  if (threadIdx.x == 0 && wk.y < r) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(dscale + wk.x);
    atomicMax(p, (unsigned long long)__double_as_longlong(m));
  }
}

// ---------------------------------------------------------------------------
void launch_skelbig_posmap(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A, cudaStream_t s) {
  if (nwork > 0) skelbig_posmap_kernel<<<nwork, 256, 0, s>>>(tasks, work, A);
}

void launch_skelbig_assemble(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A,
                             size_t smem, cudaStream_t s) {
  if (nwork <= 0) return;
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(skelbig_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemCapBytes);
    once = true;
  }
  skelbig_assemble_kernel<<<nwork, 256, smem, s>>>(tasks, work, A);
}

int cpqr_coop_capacity(size_t smem) {
  // cached per shared-memory size (the occupancy query is slow enough to
  // starve the GPU between batches)
  static std::vector<std::pair<size_t, int>> cache;
  for (const auto& c : cache)
    if (c.first == smem) return c.second;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(cpqr_mc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCapBytes);
    attr = true;
  }
  int per_sm = 0, dev = 0, nsm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cpqr_mc_kernel<false>, 256, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int cap = per_sm * nsm;  // the cooperative co-residency limit
  cache.emplace_back(smem, cap);
  return cap;
}

cudaError_t launch_cpqr_coop(const SkelBigTask* tasks, int ntasks, const int* d_gstart, int nblocks,
                             unsigned int* d_bar, int max_nq, const Arenas& A, double eps, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  size_t smem = sizeof(double) * (size_t)max_nq;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(cpqr_mc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCapBytes);
    attr = true;
  }
  Arenas Ac = A;
  void* args[] = {(void*)&tasks, (void*)&ntasks, (void*)&d_gstart, (void*)&d_bar, (void*)&Ac, (void*)&eps};
  return cudaLaunchCooperativeKernel((const void*)cpqr_mc_kernel<false>, dim3((unsigned)nblocks), dim3(256), args,
                                     smem, s);
}

void launch_skelbig_gram(const SkelBigTask* tasks, const int4* work, int nwork, const int4* tiles, int ntiles,
                         double* part, const Arenas& A, cudaStream_t s) {
  if (nwork <= 0) return;
  skelbig_gram_kernel<<<nwork, 128, 0, s>>>(tasks, work, A, part);
  if (ntiles > 0) skelbig_gram_reduce_kernel<<<ntiles, 256, 0, s>>>(tasks, tiles, A, part);
}

size_t pchol_smem(int nc, int G) {
  const size_t nown = (size_t)((nc + G - 1) / G);
  return sizeof(double) * ((size_t)nc * nown + (size_t)nc + 2 * nown);
}

int pchol_min_ctas(int nc) {
  for (int G = 1; G <= kMaxG; ++G)
    if (pchol_smem(nc, G) <= kSmemCapBytes) return G;
  return -1;
}

int pchol_coop_capacity(size_t smem) {
  static std::vector<std::pair<size_t, int>> cache;
  for (const auto& c : cache)
    if (c.first == smem) return c.second;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pchol_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCapBytes);
    attr = true;
  }
  int per_sm = 0, dev = 0, nsm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pchol_mc_kernel, 256, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int cap = per_sm * nsm;
  cache.emplace_back(smem, cap);
  return cap;
}

cudaError_t launch_pchol_coop(const SkelBigTask* tasks, int ntasks, const int* d_gstart, int nblocks,
                              unsigned int* d_bar, size_t smem, const Arenas& A, double eps, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pchol_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCapBytes);
    attr = true;
  }
  Arenas Ac = A;
  void* args[] = {(void*)&tasks, (void*)&ntasks, (void*)&d_gstart, (void*)&d_bar, (void*)&Ac, (void*)&eps};
  return cudaLaunchCooperativeKernel((const void*)pchol_mc_kernel, dim3((unsigned)nblocks), dim3(256), args, smem,
                                     s);
}


void launch_skelbig_sort(const SkelBigTask* tasks, int ntasks, const Arenas& A, ElimTask* inner, double* dmin,
                         double* dscale, cudaStream_t s) {
  if (ntasks <= 0) return;
  skelbig_sort_kernel<<<ntasks, 256, 0, s>>>(tasks, A, inner, dmin, dscale);
}

void launch_skelbig_tinit(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A, cudaStream_t s) {
  if (nwork > 0) skelbig_tinit_kernel<<<nwork, 256, 0, s>>>(tasks, work, A);
}
void launch_skelbig_tsolve(const SkelBigTask* tasks, const int4* work, int nwork, int b0, const Arenas& A,
                           cudaStream_t s) {
  if (nwork > 0) skelbig_tsolve_kernel<<<nwork, 128, 0, s>>>(tasks, work, b0, A);
}
void launch_skelbig_tupdate(const SkelBigTask* tasks, const int4* work, int nwork, int b0, const Arenas& A,
                            cudaStream_t s) {
  if (nwork > 0) skelbig_tupdate_kernel<<<nwork, 128, 0, s>>>(tasks, work, b0, A);
}
void launch_skelbig_tperm(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A, cudaStream_t s) {
  if (nwork > 0) skelbig_tperm_kernel<<<nwork, 256, 0, s>>>(tasks, work, A);
}

void launch_skelbig_congruence(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A,
                               cudaStream_t s) {
  if (nwork <= 0) return;
  skelbig_congruence_kernel<<<nwork, 128, 0, s>>>(tasks, work, A);
}

void launch_skelbig_symm(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A, double* dscale,
                         cudaStream_t s) {
  if (nwork <= 0) return;
  skelbig_symm_kernel<<<nwork, 256, 0, s>>>(tasks, work, A, nullptr, dscale);
}

}  // namespace hifde
