// Device symbolic pass of the level sweep.
//
// On the fine levels the host used to spend most of the factorization on
// integer bookkeeping: the level partition, every cell's neighbour set
// (src/sparse.py:164-173 on the clique-block store), block membership, task
// tables and arena offsets.  Here the same steps run on the GPU, on the
// device-resident structure (active mask, block table, index arena), with
// results identical to the host path:
//   * partition: the reference's keys (keys.h), a stable radix sort of the
//     active DOFs by key (members ascending within a group, groups in key
//     order, src/partition.py:40-92,108-181);
//   * membership: per level a DOF -> live-block CSR over the active DOFs;
//   * fronts: per group the live blocks touching it and its neighbour set q
//     = active DOFs coupled through a block or A0, not in the group; hashed in
//     shared memory, then sorted (count pass, then fill pass);
//   * sizes and offsets: the host's sizing rules (hifde_internal.h) and
//     prefix sums in the host's task order, so arena offsets, block ids and
//     therefore every summation order match the host path bit for bit;
//   * exact-order dependency chains: predecessor CSR and the longest chain by
//     relaxation (the exact / snapshot choice of the host path).
#include <cfloat>
#include <climits>
#include <cstdint>

#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "hifde_internal.h"
#include "keys.h"

namespace hifde {

namespace {

constexpr int kSymNT = 128;
constexpr int32_t kEmpty = INT32_MAX;

__device__ __forceinline__ void dof_coords(int64_t d, int dim, int side, int* x) {
  for (int ax = 0; ax < dim; ++ax) {
    x[ax] = (int)(d % side) + 1;
    d /= side;
  }
}

__device__ __forceinline__ uint32_t hash_slot(int32_t key, int logh) {
  return ((uint32_t)key * 2654435761u) >> (32 - logh);
}

// Insert key into an open-addressing set of 2^logh slots; returns false when
// the set overflows (more than half full or no free slot within the probes).
__device__ __forceinline__ bool set_insert(int32_t* t, int logh, int32_t key, int* count, int* ovf) {
  const uint32_t mask = (1u << logh) - 1;
  uint32_t h = hash_slot(key, logh);
  for (int p = 0; p <= (int)mask; ++p) {
    const int32_t old = atomicCAS(&t[h], kEmpty, key);
    if (old == kEmpty) {
      if (atomicAdd(count, 1) >= (int)(mask + 1) / 2) *ovf = 1;
      return true;
    }
    if (old == key) return true;
    h = (h + 1) & mask;
  }
  *ovf = 1;
  return false;
}

__device__ __forceinline__ int bsearch_sorted(const int32_t* s, int n, int32_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (s[mid] < key) lo = mid + 1; else hi = mid;
  }
  return (lo < n && s[lo] == key) ? lo : -1;
}

// Compact the non-empty slots of t[0, H) into out[0, n) (slot order), n
// returned to every thread.  One barrier-separated block scan.
template <int NT>
__device__ int compact_set(const int32_t* t, int H, int32_t* out) {
  typedef cub::BlockScan<int, NT> Scan;
  __shared__ typename Scan::TempStorage ts;
  __shared__ int total;
  const int per = (H + NT - 1) / NT;
  const int lo = threadIdx.x * per, hi = min(lo + per, H);
  int c = 0;
  for (int i = lo; i < hi; ++i) c += t[i] != kEmpty;
  int off = 0, tot = 0;
  Scan(ts).ExclusiveSum(c, off, tot);
  for (int i = lo; i < hi; ++i)
    if (t[i] != kEmpty) out[off++] = t[i];
  if (threadIdx.x == 0) total = tot;
  __syncthreads();
  return total;
}

// Ascending bitonic sort of s[0, n) in place (s has room for the next power of two).
template <int NT>
__device__ void sort_small(int32_t* s, int n) {
  int p = 1;
  while (p < n) p <<= 1;
  for (int i = n + threadIdx.x; i < p; i += NT) s[i] = kEmpty;
  __syncthreads();
  for (int k = 2; k <= p; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < p; i += NT) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int32_t a = s[i], b = s[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            s[i] = b;
            s[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// Partition
// ---------------------------------------------------------------------------
__global__ void sym_keys_kernel(const int32_t* __restrict__ act, const int64_t* __restrict__ nact, int64_t nact_ub,
                                int dim, int side, int w, int k, int kind, int32_t nkeys, int32_t* __restrict__ keys) {
  const int64_t na = *nact;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nact_ub; i += (int64_t)gridDim.x * blockDim.x) {
    int key = -1;
    if (i < na) {
      int x[3] = {0, 0, 0};
      dof_coords(act[i], dim, side, x);
      key = kind == 3 ? 0 : kind == 0 ? interior_key(x, dim, w, k) : interface_key(x, dim, w, k, kind == 2);
    }
    keys[i] = key < 0 ? nkeys : key;  // nkeys: no group (sorts last)
  }
}

// Group offsets of the sorted members: goff[g] = first member of group g,
// goff[ng] = members; group_of[d] = g (skeleton levels; -1 elsewhere).
__global__ void sym_groups_kernel(const int32_t* __restrict__ skeys, const int32_t* __restrict__ gid,
                                  const int32_t* __restrict__ gmem, const int64_t* __restrict__ nact, int32_t nkeys,
                                  int64_t* __restrict__ goff, int32_t* __restrict__ ng, int32_t* group_of) {
  const int64_t na = *nact;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t key = skeys[i];
    if (key == nkeys) continue;
    const int g = gid[i] - 1;  // inclusive scan of the head flags
    if (i == 0 || skeys[i - 1] != key) goff[g] = i;
    if (i + 1 == na || skeys[i + 1] == nkeys) {
      goff[g + 1] = i + 1;
      *ng = g + 1;
    }
    if (group_of) group_of[gmem[i]] = g;
  }
}

__global__ void sym_heads_kernel(const int32_t* __restrict__ skeys, int64_t n, int32_t nkeys,
                                 int32_t* __restrict__ head) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t key = skeys[i];
    head[i] = key != nkeys && (i == 0 || skeys[i - 1] != key);
  }
}

__global__ void sym_reset_group_of(const int32_t* __restrict__ gmem, const int64_t* __restrict__ goff,
                                   const int32_t* __restrict__ ng, int32_t* __restrict__ group_of) {
  const int64_t n = goff[*ng];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    group_of[gmem[i]] = -1;
}

// ---------------------------------------------------------------------------
// Membership: DOF -> live blocks, over the active DOFs
// ---------------------------------------------------------------------------
__global__ void sym_member_count(const int32_t* __restrict__ alive_list, const int64_t* __restrict__ nalive,
                                 const int32_t* __restrict__ blk_n, const int64_t* __restrict__ blk_dof_off,
                                 const int32_t* __restrict__ idx, const uint8_t* __restrict__ active,
                                 int32_t* __restrict__ cnt) {
  const int64_t nb = *nalive;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = w0; j < nb; j += nw) {
    const int32_t b = alive_list[j];
    const int32_t* d = idx + blk_dof_off[b];
    for (int i = lane; i < blk_n[b]; i += 32)
      if (active[d[i]]) atomicAdd(&cnt[d[i]], 1);
  }
}

__global__ void sym_member_fill(const int32_t* __restrict__ alive_list, const int64_t* __restrict__ nalive,
                                const int32_t* __restrict__ blk_n, const int64_t* __restrict__ blk_dof_off,
                                const int32_t* __restrict__ idx, const uint8_t* __restrict__ active,
                                int32_t* __restrict__ pos, int32_t* __restrict__ mblk) {
  const int64_t nb = *nalive;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = w0; j < nb; j += nw) {
    const int32_t b = alive_list[j];
    const int32_t* d = idx + blk_dof_off[b];
    for (int i = lane; i < blk_n[b]; i += 32)
      if (active[d[i]]) mblk[atomicAdd(&pos[d[i]], 1)] = b;
  }
}

// ---------------------------------------------------------------------------
// Fronts: live blocks touching the group, neighbour set q, predecessors
// ---------------------------------------------------------------------------
// Warp tier (kWarpTierW below): one warp per group of at most 64 DOFs with
// per-warp sets of 32 blocks / 128 neighbours / 64 predecessors; config 3's
// 130,560 edge groups of level 0.5 (7 DOFs, ~50 neighbours) took one
// 128-thread CTA each, whose barriers and dependent loads (a chain of ~10
// global reads per phase) left the pass latency-bound at 16 groups per SM.
// The sets and the sorted outputs are those of the CTA tiers (they do not
// depend on insertion order); a group whose sets outgrow the warp's goes to
// the CTA tier's list (flag 1).
__device__ __forceinline__ int warp_compact(const int32_t* t, int H, int32_t* out, int lane) {
  int base = 0;
  for (int i0 = 0; i0 < H; i0 += 32) {
    const int32_t v = t[i0 + lane];
    const unsigned m = __ballot_sync(0xffffffffu, v != kEmpty);
    if (v != kEmpty) out[base + __popc(m & ((1u << lane) - 1u))] = v;
    base += __popc(m);
  }
  __syncwarp();
  return base;
}
// dst[rank(v)] = v for the n distinct values of src (rank = number smaller)
__device__ __forceinline__ void warp_rank_sort(const int32_t* src, int n, int32_t* dst, int lane) {
  for (int i = lane; i < n; i += 32) {
    const int32_t v = src[i];
    int r = 0;
    for (int k = 0; k < n; ++k) r += src[k] < v;
    dst[r] = v;
  }
}

constexpr int kWLQ = 7, kWLB = 5, kWLP = 6, kWNC = 64, kWarpTierW = 8;

template <bool FILL>
__global__ void __launch_bounds__(32 * kWarpTierW) sym_front_warp_kernel(SymFront P) {
  constexpr int HQ = 1 << kWLQ, HB = 1 << kWLB, HP = 1 << kWLP;
  constexpr int kPer = kWNC + HB + HQ + HP + HQ;
  __shared__ __align__(16) int32_t sh[kWarpTierW][kPer];
  __shared__ int cnt[kWarpTierW][4];  // blocks, neighbours, predecessors, overflow
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t* c = sh[w];
  int32_t* hb = c + kWNC;
  int32_t* hq = hb + HB;
  int32_t* hp = hq + HQ;
  int32_t* buf = hp + HP;
  int* ct = cnt[w];
  const int ngr = *P.ng;
  for (int g = blockIdx.x * kWarpTierW + w; g < ngr; g += gridDim.x * kWarpTierW) {
    if (FILL && P.flag[g] != 0) continue;
    const int64_t c0 = P.goff[g];
    const int nc = (int)(P.goff[g + 1] - c0);
    if (nc > kWNC) {  // count pass only (the fill sees flag 1)
      if (lane == 0) {
        P.flag[g] = 1;
        P.retry2[atomicAdd(P.nretry2, 1)] = g;
      }
      continue;
    }
    for (int i = lane; i < HB; i += 32) hb[i] = kEmpty;
    for (int i = lane; i < HQ; i += 32) hq[i] = kEmpty;
    for (int i = lane; i < HP; i += 32) hp[i] = kEmpty;
    if (lane < 4) ct[lane] = 0;
    for (int i = lane; i < nc; i += 32) c[i] = P.gmem[c0 + i];
    __syncwarp();
    for (int i = lane; i < nc; i += 32) {  // live blocks touching the group
      const int32_t d = c[i];
      for (int32_t t = P.mptr[d]; t < P.mptr[d + 1]; ++t) set_insert(hb, kWLB, P.mblk[t], &ct[0], &ct[3]);
    }
    __syncwarp();
    int nb = 0, maxnb = 0;
    if (!ct[3]) {
      nb = warp_compact(hb, HB, buf, lane);
      for (int j = 0; j < nb; ++j) {  // q candidates: the blocks' DOFs, then A0 rows of c
        const int32_t b = buf[j];
        const int n = P.blk_n[b];
        maxnb = max(maxnb, n);
        const int32_t* d = P.idx + P.blk_dof_off[b];
        for (int i = lane; i < n; i += 32) {
          const int32_t e = d[i];
          if (P.active[e] && bsearch_sorted(c, nc, e) < 0) set_insert(hq, kWLQ, e, &ct[1], &ct[3]);
        }
      }
      for (int i = lane; i < nc; i += 32) {
        const int32_t d = c[i];
        for (int64_t t = P.indptr[d]; t < P.indptr[d + 1]; ++t) {
          const int32_t e = P.indices[t];
          if (P.active[e] && bsearch_sorted(c, nc, e) < 0) set_insert(hq, kWLQ, e, &ct[1], &ct[3]);
        }
      }
    }
    __syncwarp();
    if (!ct[3] && P.group_of) {  // predecessors: earlier groups owning a DOF of q
      for (int i = lane; i < HQ; i += 32) {
        const int32_t e = hq[i];
        if (e == kEmpty) continue;
        const int32_t go = P.group_of[e];
        if (go >= 0 && go < g) set_insert(hp, kWLP, go, &ct[2], &ct[3]);
      }
    }
    __syncwarp();
    if (ct[3]) {
      if (lane == 0) {
        if (!FILL) {
          P.flag[g] = 1;
          P.retry2[atomicAdd(P.nretry2, 1)] = g;
        } else {
          atomicExch(P.fatal, 1);  // the count pass fitted these sets
        }
      }
      __syncwarp();
      continue;
    }
    const int nqk = ct[1], npk = ct[2];
    if (!FILL) {
      if (P.group_of && P.pred_tmp) {  // unsorted predecessor lists for the chain
        int64_t pstart = 0;
        if (lane == 0) {
          pstart = (int64_t)atomicAdd((unsigned long long*)P.pred_alloc, (unsigned long long)npk);
          if (pstart + npk > P.pred_cap) atomicExch(P.pred_ovf, 1);
          P.pred_start[g] = pstart;
        }
        pstart = __shfl_sync(0xffffffffu, pstart, 0);
        if (pstart + npk <= P.pred_cap) warp_compact(hp, HP, P.pred_tmp + pstart, lane);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxnb = max(maxnb, __shfl_xor_sync(0xffffffffu, maxnb, o));
      if (lane == 0) {
        P.nq[g] = nqk;
        P.nb[g] = nb;
        P.maxnb[g] = maxnb;
        P.npred[g] = npk;
        P.flag[g] = 0;
      }
      __syncwarp();
      continue;
    }
    // fill: c, sorted blocks, sorted q, sorted predecessors
    const int64_t* ex = P.exc + (size_t)g * P.exc_stride;
    int32_t* out = P.idx_out + P.idx_base + ex[P.o_nf];
    for (int i = lane; i < nc; i += 32) out[i] = c[i];
    warp_rank_sort(buf, nb, P.lists + ex[P.o_nb], lane);
    __syncwarp();
    const int nq = warp_compact(hq, HQ, buf, lane);
    warp_rank_sort(buf, nq, out + nc, lane);
    __syncwarp();
    if (P.group_of) {
      const int np = warp_compact(hp, HP, buf, lane);
      warp_rank_sort(buf, np, P.preds + ex[P.o_pred], lane);
    }
    __syncwarp();
  }
}

template <int LQ, int LB, int LP, int NCMAX, bool FILL>
__global__ void __launch_bounds__(kSymNT) sym_front_kernel(SymFront P) {
  constexpr int HQ = 1 << LQ, HB = 1 << LB, HP = 1 << LP;
  extern __shared__ __align__(16) int32_t sm[];
  int32_t* c = sm;                 // NCMAX
  int32_t* hb = c + NCMAX;         // HB
  int32_t* hq = hb + HB;           // HQ
  int32_t* hp = hq + HQ;           // HP
  int32_t* buf = hp + HP;          // HQ (sort buffer)
  __shared__ int nbk, nqk, npk, ovf, maxnb;
  const bool big_tier = LQ > 10;
  const int nwork = big_tier ? *P.nretry : *P.nretry2;  // groups the tier before could not take
  for (int wi = blockIdx.x; wi < nwork; wi += gridDim.x) {
    const int g = big_tier ? P.retry[wi] : P.retry2[wi];
    if (!big_tier && P.flag[g] != 1 && FILL) continue;  // the big tier fills it
    const int64_t c0 = P.goff[g];
    const int nc = (int)(P.goff[g + 1] - c0);
    if (threadIdx.x == 0) { nbk = nqk = npk = ovf = maxnb = 0; }
    for (int i = threadIdx.x; i < HB; i += kSymNT) hb[i] = kEmpty;
    for (int i = threadIdx.x; i < HQ; i += kSymNT) hq[i] = kEmpty;
    for (int i = threadIdx.x; i < HP; i += kSymNT) hp[i] = kEmpty;
    __syncthreads();
    if (nc > NCMAX) {
      if (threadIdx.x == 0) ovf = 1;
    } else {
      for (int i = threadIdx.x; i < nc; i += kSymNT) c[i] = P.gmem[c0 + i];
    }
    __syncthreads();
    if (!ovf) {
      // live blocks touching the group
      for (int i = threadIdx.x; i < nc; i += kSymNT) {
        const int32_t d = c[i];
        for (int32_t t = P.mptr[d]; t < P.mptr[d + 1]; ++t) set_insert(hb, LB, P.mblk[t], &nbk, &ovf);
      }
    }
    __syncthreads();
    int nb = 0;
    if (!ovf) nb = compact_set<kSymNT>(hb, HB, buf);  // unique blocks (slot order)
    __syncthreads();
    if (!ovf) {
      // q candidates: the blocks' DOFs (warp per block), then A0 rows of c
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
      for (int j = wid; j < nb; j += kSymNT / 32) {
        const int32_t b = buf[j];
        const int n = P.blk_n[b];
        if (lane == 0) atomicMax(&maxnb, n);
        const int32_t* d = P.idx + P.blk_dof_off[b];
        for (int i = lane; i < n; i += 32) {
          const int32_t e = d[i];
          if (P.active[e] && bsearch_sorted(c, nc, e) < 0) set_insert(hq, LQ, e, &nqk, &ovf);
        }
      }
      for (int i = threadIdx.x; i < nc; i += kSymNT) {
        const int32_t d = c[i];
        for (int64_t t = P.indptr[d]; t < P.indptr[d + 1]; ++t) {
          const int32_t e = P.indices[t];
          if (P.active[e] && bsearch_sorted(c, nc, e) < 0) set_insert(hq, LQ, e, &nqk, &ovf);
        }
      }
    }
    __syncthreads();
    if (!ovf && P.group_of) {  // predecessors: earlier groups owning a DOF of q
      for (int i = threadIdx.x; i < HQ; i += kSymNT) {
        const int32_t e = hq[i];
        if (e == kEmpty) continue;
        const int32_t go = P.group_of[e];
        if (go >= 0 && go < g) set_insert(hp, LP, go, &npk, &ovf);
      }
    }
    __syncthreads();
    if (ovf) {
      if (!FILL && threadIdx.x == 0) {
        if (!big_tier) {
          P.flag[g] = 2;
          P.retry[atomicAdd(P.nretry, 1)] = g;
        } else {
          atomicExch(P.fatal, 1);
        }
      }
      __syncthreads();
      continue;
    }
    if (!FILL) {
      // predecessor lists for the dependency-chain relaxation, right away
      // (unsorted, at an atomically allocated place: the chain does not need
      // the arenas, so the level's exact / snapshot choice travels with the
      // count totals in one readback)
      __shared__ int64_t pstart;
      if (P.group_of && P.pred_tmp) {
        if (threadIdx.x == 0) {
          pstart = atomicAdd((unsigned long long*)P.pred_alloc, (unsigned long long)npk);
          if (pstart + npk > P.pred_cap) atomicExch(P.pred_ovf, 1);
          P.pred_start[g] = pstart;
        }
        __syncthreads();
        if (pstart + npk <= P.pred_cap) {
          const int np = compact_set<kSymNT>(hp, HP, buf);
          for (int i = threadIdx.x; i < np; i += kSymNT) P.pred_tmp[pstart + i] = buf[i];
        }
      }
      if (threadIdx.x == 0) {
        P.nq[g] = nqk;
        P.nb[g] = nb;
        P.maxnb[g] = maxnb;
        P.npred[g] = npk;
      }
      __syncthreads();
      continue;
    }
    // fill: c, sorted q, sorted blocks, sorted predecessors
    const int64_t* ex = P.exc + (size_t)g * P.exc_stride;
    const int64_t doff = P.idx_base + ex[P.o_nf];
    int32_t* out = P.idx_out + doff;
    for (int i = threadIdx.x; i < nc; i += kSymNT) out[i] = c[i];
    sort_small<kSymNT>(buf, nb);
    int32_t* lo = P.lists + ex[P.o_nb];
    for (int i = threadIdx.x; i < nb; i += kSymNT) lo[i] = buf[i];
    __syncthreads();
    const int nq = compact_set<kSymNT>(hq, HQ, buf);
    sort_small<kSymNT>(buf, nq);
    for (int i = threadIdx.x; i < nq; i += kSymNT) out[nc + i] = buf[i];
    __syncthreads();
    if (P.group_of) {
      const int np = compact_set<kSymNT>(hp, HP, buf);
      sort_small<kSymNT>(buf, np);
      int32_t* po = P.preds + ex[P.o_pred];
      for (int i = threadIdx.x; i < np; i += kSymNT) po[i] = buf[i];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Elimination level: sizes, prefix sums, task tables, block table updates
// ---------------------------------------------------------------------------
struct ElimIncOp {
  __device__ __forceinline__ ElimInc operator()(const ElimInc& a, const ElimInc& b) const {
    ElimInc r;
#pragma unroll
    for (int i = 0; i < kElimIncN; ++i) r.v[i] = a.v[i] + b.v[i];
    return r;
  }
};
struct SkelIncOp {
  __device__ __forceinline__ SkelInc operator()(const SkelInc& a, const SkelInc& b) const {
    SkelInc r;
#pragma unroll
    for (int i = 0; i < kSkelIncN; ++i) r.v[i] = a.v[i] + b.v[i];
    return r;
  }
};

__device__ __forceinline__ void amax64(int64_t* p, int64_t v) {
  atomicMax((unsigned long long*)p, (unsigned long long)v);
}


// Maxima of a grid-stride loop: per thread over its items, then per block
// (warp shuffles, shared memory), then one atomic per block and field -- the
// per-item atomics on the few LevelTotals words serialized at L2 (config 3
// level 0.5: 130,560 groups x 8 fields, 0.47 ms).  Values are >= 0.
template <int NF>
struct BlockMax {
  int64_t v[NF];
  __device__ BlockMax() {
#pragma unroll
    for (int i = 0; i < NF; ++i) v[i] = 0;
  }
  __device__ void put(int i, int64_t x) { v[i] = x > v[i] ? x : v[i]; }
  // every thread of the block calls it (blockDim.x <= 1024, a multiple of 32)
  __device__ void commit(int64_t* const (&dst)[NF]) {
    __shared__ int64_t sh[32][NF];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < NF; ++i) {
      int64_t x = v[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t y = __shfl_xor_sync(0xffffffffu, x, o);
        x = y > x ? y : x;
      }
      if (lane == 0) sh[w][i] = x;
    }
    __syncthreads();
    if (threadIdx.x < NF) {
      int64_t x = 0;
      for (int k = 0; k < nw; ++k) x = sh[k][threadIdx.x] > x ? sh[k][threadIdx.x] : x;
      if (x > 0) amax64(dst[threadIdx.x], x);
    }
  }
};

__global__ void elim_size_kernel(const SymFront P, int is_top, ElimInc* __restrict__ inc, LevelTotals* tot) {
  const int ng = *P.ng;
  BlockMax<7> m;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
    const int nc = (int)(P.goff[g + 1] - P.goff[g]), nq = P.nq[g], nb = P.nb[g], mb = P.maxnb[g];
    const ElimSizes z = elim_sizes(nc, nq, mb, is_top != 0);
    ElimInc I;
    I.v[0] = nc + nq;                                                  // idx
    I.v[1] = nb;                                                       // lists
    I.v[2] = (int64_t)nc * nc + (z.big ? (int64_t)nc * (nc + 1) / 2 : 0) + (int64_t)nc * nq;  // fac
    I.v[3] = (int64_t)nq * nq;                                         // block arena
    I.v[4] = nq;                                                       // contribution rows
    I.v[5] = nq > 0;                                                   // new blocks
    I.v[6] = !z.big;                                                   // small cells
    I.v[7] = z.big;                                                    // big cells
    inc[g] = I;
    if (z.big) {
      m.put(0, (int64_t)elim_big_smem(nc + nq, mb));
      m.put(1, nc);
    } else {
      m.put(2, (int64_t)z.smem);
      m.put(3, nc + nq);
    }
    m.put(4, nc + nq);
    m.put(5, nc);
    m.put(6, nq);
  }
  int64_t* const dst[7] = {&tot->smem_big, &tot->max_big_nc, &tot->smem, &tot->max_small_nf, &tot->max_front,
                           &tot->max_nc, &tot->max_nq};
  m.commit(dst);
}

__global__ void elim_total_kernel(const int32_t* __restrict__ ng, const ElimInc* __restrict__ inc,
                                  const ElimInc* __restrict__ exc, LevelTotals* tot) {
  const int n = *ng;
  tot->ng = n;
  for (int i = 0; i < kElimIncN; ++i) tot->sum[i] = n ? exc[n - 1].v[i] + inc[n - 1].v[i] : 0;
}

__global__ void elim_fill_kernel(const SymFront P, ElimFillArgs A) {
  const int ng = *P.ng;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
    const int nc = (int)(P.goff[g + 1] - P.goff[g]), nq = P.nq[g], nb = P.nb[g], mb = P.maxnb[g];
    const ElimSizes z = elim_sizes(nc, nq, mb, A.is_top != 0);
    const ElimInc& o = A.exc[g];
    ElimTask T;
    T.nc = nc;
    T.nq = nq;
    T.nblk = nb;
    T.maxnb = mb;
    T.dofs_off = A.idx_base + o.v[0];
    T.blk_off = o.v[1];
    T.scratch_off = z.scratch_off;
    T.C_off = A.fac_base + o.v[2];
    T.P_off = z.big ? T.C_off + (int64_t)nc * nc : T.C_off;
    T.W_off = T.C_off + (int64_t)nc * nc + (z.big ? (int64_t)nc * (nc + 1) / 2 : 0);
    T.U_off = nq > 0 ? A.bv_base + o.v[3] : 0;
    if (z.big) A.big[o.v[7]] = T;
    else A.small[o.v[6]] = T;
    SolveRec R;
    R.nc = nc;
    R.nq = nq;
    R.idx_off = T.dofs_off;
    R.C_off = T.P_off;  // the solve applies the packed inverse
    R.W_off = T.W_off;
    R.T_off = 0;
    R.contrib_off = o.v[4];
    R.inv = 1;
    R.pad = 0;
    A.recs[g] = R;
    hifde_record_t X;
    X.kind = A.is_top ? 2 : 0;
    X.nc = nc;
    X.nq = nq;
    X.nr = 0;
    X.cell_off = T.dofs_off;
    X.idx_off = T.dofs_off;
    X.P_off = T.P_off;
    X.W_off = T.W_off;
    X.T_off = 0;
    A.xrec[g] = X;
    const int64_t nblk0 = *A.nblk;
    if (nq > 0) {
      const int64_t id = nblk0 + o.v[5];
      A.blk_dof_off[id] = T.dofs_off + nc;
      A.blk_n[id] = nq;
      A.blk_val_off[id] = T.U_off;
      A.blk_alive[id] = 1;
    }
    const int32_t* bl = A.lists + T.blk_off;
    for (int j = 0; j < nb; ++j) A.blk_alive[bl[j]] = 0;  // consumed (a block touches one cell of a level)
    // solve-side reduction pairs: (neighbour DOF, contribution row)
    const int32_t* q = A.idx + T.dofs_off + nc;
    for (int i = 0; i < nq; ++i) {
      A.red_key[o.v[4] + i] = q[i];
      A.red_val[o.v[4] + i] = o.v[4] + i;
    }
    // level statistics (SURVEY 8(d) work per cell, the reference's m_f accounting)
    const double dc = nc, dq = nq;
    const double gf = (dc * dc * dc / 3 + dc * dc * dq + dc * dq + dc * dq * dq) * 1e-9;
    const double gb = 8.0 * ((dc + dq) * (dc + dq) + dc * dc + dc + dc * dq + 2 * dq * dq) * 1e-9;
    A.cellstat[g] = make_double4(gf, gb, 8.0 * (dc * dc + dc + dc * dq), dc * (dc + 1) / 2 + dc * dq);
    A.cellcls[g] = (uint8_t)z.big;
  }
}

// ---- level statistics: two-stage reduction in a fixed order (deterministic)
struct StatAcc {
  double d[8];
  int64_t sum[4], mx[4];
};
constexpr int kStatGrid = 148;

__device__ void stat_block_reduce(StatAcc& a, StatAcc* out) {
  __shared__ double rd[256];
  __shared__ int64_t ri[256];
  for (int i = 0; i < 8; ++i) {
    rd[threadIdx.x] = a.d[i];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (threadIdx.x < s) rd[threadIdx.x] += rd[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) out->d[i] = rd[0];
    __syncthreads();
  }
  for (int i = 0; i < 8; ++i) {
    ri[threadIdx.x] = i < 4 ? a.sum[i] : a.mx[i - 4];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (threadIdx.x < s) ri[threadIdx.x] = i < 4 ? ri[threadIdx.x] + ri[threadIdx.x + s] : max(ri[threadIdx.x], ri[threadIdx.x + s]);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      if (i < 4) out->sum[i] = ri[0];
      else out->mx[i - 4] = ri[0];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) elim_stats_part(const int32_t* __restrict__ ng, const double4* __restrict__ cs,
                                                       const uint8_t* __restrict__ cls, const SymFront P,
                                                       StatAcc* __restrict__ part) {
  const int n = *ng;
  const int lo = (int)((int64_t)n * blockIdx.x / gridDim.x), hi = (int)((int64_t)n * (blockIdx.x + 1) / gridDim.x);
  StatAcc a;
  for (int i = 0; i < 8; ++i) a.d[i] = 0.0;
  for (int i = 0; i < 4; ++i) a.sum[i] = a.mx[i] = 0;
  for (int g = lo + threadIdx.x; g < hi; g += 256) {
    const double4 v = cs[g];
    const int c = cls[g];
    a.d[0] += v.x;
    a.d[1] += v.y;
    a.d[2 + 2 * c] += v.x;
    a.d[3 + 2 * c] += v.y;
    a.d[6] += v.w;
    const int nc = (int)(P.goff[g + 1] - P.goff[g]), nq = P.nq[g];
    a.sum[0] += (int64_t)v.z;
    a.sum[1] += nc + nq;
    a.mx[0] = max(a.mx[0], (int64_t)nc);
    a.mx[1] = max(a.mx[1], (int64_t)nq);
    a.mx[2] = max(a.mx[2], (int64_t)(nc + nq));
  }
  stat_block_reduce(a, part + blockIdx.x);
}

// Second stage of the fixed-order level statistics: the kStatGrid partials
// reduced by one 256-thread block as a tree (a single thread summing them
// in a row took ~40 us per level on the factor's critical path).
__device__ StatAcc stat_partials(const StatAcc* __restrict__ part, int np) {
  StatAcc a;
  for (int i = 0; i < 8; ++i) a.d[i] = 0.0;
  for (int i = 0; i < 4; ++i) a.sum[i] = a.mx[i] = 0;
  if ((int)threadIdx.x < np) a = part[threadIdx.x];
  __shared__ StatAcc r;
  stat_block_reduce(a, &r);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) elim_stats_final(const int32_t* __restrict__ ng,
                                                        const StatAcc* __restrict__ part, int np, LevelStat* st,
                                                        const int64_t* __restrict__ nblk_inc, int64_t* nblk) {
  const StatAcc a = stat_partials(part, np);
  if (threadIdx.x != 0) return;
  const int n = *ng;
  st->ngroups = n;
  st->gflop = a.d[0];
  st->gbytes = a.d[1];
  st->gf_cls[0] = a.d[2];
  st->gb_cls[0] = a.d[3];
  st->gf_cls[1] = a.d[4];
  st->gb_cls[1] = a.d[5];
  st->solve_fac = a.d[6];
  st->solve_rows = (double)a.sum[1];
  st->mf_bytes = a.sum[0];
  st->nrecs = n;
  st->max_nc = a.mx[0];
  st->max_nq = a.mx[1];
  st->max_front = a.mx[2];
  *nblk += *nblk_inc;
}

// ---------------------------------------------------------------------------
// Skeletonization level
// ---------------------------------------------------------------------------
__global__ void skel_size_kernel(const SymFront P, double promote_work, int gram_eps_ok, SkelInc* __restrict__ inc,
                                 LevelTotals* tot) {
  const int ng = *P.ng;
  BlockMax<8> m;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
    const int nc = (int)(P.goff[g + 1] - P.goff[g]), nq = P.nq[g], nb = P.nb[g], mb = P.maxnb[g];
    const SkelSizes z = skel_sizes(nc, nq, mb);
    const bool promote = (z.mode == 1 || z.mode == 3) && (double)nq * nc * nc >= promote_work && gram_eps_ok &&
                         nq >= 2 * nc && nc <= 1024;
    SkelInc I;
    I.v[0] = nc + nq;                                                  // idx (fronts)
    I.v[1] = nb;                                                       // lists
    I.v[2] = (int64_t)z.scr;                                           // scratch
    I.v[3] = (int64_t)(z.fac + ((z.mode == 2 || promote) ? z.fac_big : 0));  // fac
    I.v[4] = (int64_t)nc * nc;                                         // delta blocks
    I.v[5] = P.npred[g];                                               // predecessors
    I.v[6] = nc;                                                       // sk/rd output lists
    I.v[7] = (int64_t)skel_cluster_scratch(nc);                        // cluster workspace
    inc[g] = I;
    m.put(0, (int64_t)z.smem);
    m.put(1, nc);
    m.put(2, nq);
    m.put(3, nc + nq);
    m.put(4, (int64_t)skel_cluster_need(nc, nq, mb, 4));
    m.put(5, (int64_t)skel_cluster_need(nc, nq, mb, 2));
    if (z.mode == 2) m.put(6, 1);
    if (promote && (double)nq * nc * nc >= 4e6) m.put(7, 1);
  }
  int64_t* const dst[8] = {&tot->smem, &tot->max_nc, &tot->max_nq, &tot->max_front, &tot->cl_need4, &tot->cl_need2,
                           &tot->any_mode2, &tot->any_promote};
  m.commit(dst);
}

__global__ void skel_total_kernel(const int32_t* __restrict__ ng, const SkelInc* __restrict__ inc,
                                  const SkelInc* __restrict__ exc, LevelTotals* tot) {
  const int n = *ng;
  tot->ng = n;
  for (int i = 0; i < kSkelIncN; ++i) tot->sum[i] = n ? exc[n - 1].v[i] + inc[n - 1].v[i] : 0;
}

__global__ void skel_fill_kernel(const SymFront P, SkelFillArgs A) {
  const int ng = *P.ng;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
    const int nc = (int)(P.goff[g + 1] - P.goff[g]), nq = P.nq[g], nb = P.nb[g], mb = P.maxnb[g];
    const SkelSizes z = skel_sizes(nc, nq, mb);
    const SkelInc& o = A.exc[g];
    SkelTask T;
    T.nc = nc;
    T.nq = nq;
    T.nblk = nb;
    T.maxnb = mb;
    T.dofs_off = A.idx_base + o.v[0];
    T.blk_off = o.v[1];
    T.scratch_off = z.scr ? A.scr_base + o.v[2] : -1;
    T.rec_off = A.fac_base + o.v[3];
    T.delta_off = A.bv_base + o.v[4];
    T.out_off = A.idx_base + A.tot_nf + o.v[6];
    T.group = g;
    T.mode = z.mode;
    T.chunk = z.chunk;
    T.pad2 = 0;
    A.tasks[g] = T;
    A.pred_ptr[g] = o.v[5];
    if (g == ng - 1) A.pred_ptr[ng] = o.v[5] + P.npred[g];
    A.cl_rel[g] = o.v[7];
    int32_t* out = A.idx + T.out_off;
    for (int i = 0; i < nc; ++i) out[i] = 0;
  }
}

// cluster path: per-group global workspace in scratch_off
__global__ void skel_cluster_tasks(SkelTask* __restrict__ tasks, const int64_t* __restrict__ cl_rel, int64_t base,
                                   const int32_t* __restrict__ ng) {
  const int n = *ng;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x)
    tasks[g].scratch_off = base + cl_rel[g];
}

// Longest dependency chain: b[t] = 1 + max b[p] over predecessors p (Jacobi
// sweeps from 0; after i sweeps b = min(chain, i)); iteration it stops early
// once the previous sweep changed nothing.
__global__ void skel_relax_kernel(const int64_t* __restrict__ pred_start, const int32_t* __restrict__ npred,
                                  const int32_t* __restrict__ preds, const int32_t* __restrict__ ng,
                                  const int32_t* __restrict__ bin, int32_t* __restrict__ bout, int32_t* changed,
                                  int it) {
  if (it > 0 && changed[it - 1] == 0) return;
  const int n = *ng;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    int b = 0;
    const int64_t p0 = pred_start[t];
    for (int64_t p = p0; p < p0 + npred[t]; ++p) b = max(b, bin[preds[p]] + 1);
    bout[t] = b;
    if (b != bin[t]) changed[it] = 1;
  }
}

// The same sweeps in one cooperative launch (grid-wide barrier between
// sweeps), stopping once a sweep changed nothing: a 2D fine level's 65 sweeps
// cost one launch instead of 65.
__global__ void __launch_bounds__(256) skel_relax_coop(const int64_t* __restrict__ pred_start,
                                                       const int32_t* __restrict__ npred,
                                                       const int32_t* __restrict__ preds,
                                                       const int32_t* __restrict__ ng, int32_t* b0, int32_t* b1,
                                                       int32_t* changed, int iters, int cap, LevelTotals* tot) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int n = *ng;
  int m = 0;  // max depth this thread wrote in the last sweep that ran
  if (cap > 0) {
    // AUTO order only asks whether the chain exceeds `cap`: relax in place
    // (every value stays a lower bound of its depth and only grows, so the
    // fixed point is the Jacobi sweeps' and is reached no later) and stop as
    // soon as any depth passes the cap -- a fine level's chain of thousands
    // shows after a few sweeps instead of cap + 1.  The level then runs in
    // snapshot order and its depths are not used; a chain within the cap
    // converges to the exact depths as before.
    for (int it = 0; it < iters; ++it) {
      int ch = 0;
      for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        int b = 0;
        const int64_t p0 = pred_start[t];
        for (int64_t p = p0; p < p0 + npred[t]; ++p) b = max(b, __ldcg(b0 + preds[p]) + 1);
        if (b > __ldcg(b0 + t)) {
          __stcg(b0 + t, b);
          ch = 1;
        }
        m = max(m, b);
      }
      const int any = __syncthreads_or(ch | (m > cap ? 2 : 0));
      if (threadIdx.x == 0) {
        if (any & 1) atomicExch(changed + it, 1);
        if (any & 2) atomicExch(changed + iters, 1);  // past the cap
      }
      grid.sync();
      if (__ldcg(changed + it) == 0 || __ldcg(changed + iters) != 0) break;  // uniform: read after the barrier
    }
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) b1[t] = __ldcg(b0 + t);
    typedef cub::BlockReduce<int, 256> R0;
    __shared__ typename R0::TempStorage rt0;
    m = R0(rt0).Reduce(m, cub::Max());
    if (threadIdx.x == 0 && m > 0) amax64(&tot->max_chain, m);
    return;
  }
  for (int it = 0; it < iters; ++it) {
    if (it > 0 && __ldcg(changed + it - 1) == 0) break;  // uniform: read after the barrier
    const int32_t* bin = (it % 2 == 0) ? b0 : b1;
    int32_t* bout = (it % 2 == 0) ? b1 : b0;
    int ch = 0;
    m = 0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
      int b = 0;
      const int64_t p0 = pred_start[t];
      for (int64_t p = p0; p < p0 + npred[t]; ++p) b = max(b, __ldcg(bin + preds[p]) + 1);
      __stcg(bout + t, b);
      ch |= b != __ldcg(bin + t);
      m = max(m, b);
    }
    if (__syncthreads_or(ch) && threadIdx.x == 0) atomicExch(changed + it, 1);
    grid.sync();
  }
  // the longest chain (was a one-block reduction over every group's depth
  // after the sweeps: 0.23 ms at config 3 level 0.5)
  typedef cub::BlockReduce<int, 256> R;
  __shared__ typename R::TempStorage rt;
  m = R(rt).Reduce(m, cub::Max());
  if (threadIdx.x == 0 && m > 0) amax64(&tot->max_chain, m);
}

// the relaxation's final depths (the buffer the last sweep that ran wrote)
__global__ void skel_depth_kernel(const int32_t* __restrict__ b0, const int32_t* __restrict__ b1,
                                  const int32_t* __restrict__ changed, int iters, const int32_t* __restrict__ ng,
                                  int32_t* __restrict__ depth, int32_t* __restrict__ iota) {
  int last = iters - 1;
  for (int i = 1; i < iters; ++i)
    if (changed[i - 1] == 0) { last = i - 1; break; }
  const int32_t* b = (last % 2 == 0) ? b1 : b0;
  const int n = *ng;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    depth[t] = b[t];
    iota[t] = t;
  }
}

// after the level's kernels: ranks known -> delta blocks, solve records, stats
__global__ void skel_finish_inc(const SkelTask* __restrict__ tasks, const int32_t* __restrict__ kout,
                                const int32_t* __restrict__ ng, int2* __restrict__ inc) {
  const int n = *ng;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
    const int k = kout[g], r = tasks[g].nc - k;
    inc[g] = make_int2(r > 0 && k > 0, r > 0);
  }
}

struct Int2Sum {
  __device__ __forceinline__ int2 operator()(const int2& a, const int2& b) const {
    return make_int2(a.x + b.x, a.y + b.y);
  }
};

__global__ void skel_finish_fill(const SkelTask* __restrict__ tasks, const int32_t* __restrict__ kout,
                                 const int32_t* __restrict__ ng, const int2* __restrict__ exc, SkelFinishArgs A) {
  const int n = *ng;
  const int64_t nblk0 = *A.nblk;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
    const SkelTask& T = tasks[g];
    const int k = kout[g], r = T.nc - k;
    if (r > 0 && k > 0) {
      const int64_t id = nblk0 + exc[g].x;
      A.blk_dof_off[id] = T.out_off;
      A.blk_n[id] = k;
      A.blk_val_off[id] = T.delta_off;
      A.blk_alive[id] = 1;
    }
    hifde_record_t X;
    X.kind = 1;
    X.nc = T.nc;
    X.nq = k;
    X.nr = r;
    X.cell_off = T.dofs_off;
    X.idx_off = T.out_off;
    X.T_off = T.rec_off;
    X.P_off = T.rec_off + (int64_t)k * r;
    X.W_off = T.rec_off + (int64_t)k * r + (int64_t)r * r;
    A.xrec[g] = X;
    if (r > 0) {
      SolveRec R;
      R.nc = r;
      R.nq = k;
      R.idx_off = T.out_off;
      R.T_off = T.rec_off;
      R.C_off = T.rec_off + (int64_t)k * r;
      R.W_off = R.C_off + (int64_t)r * r;
      R.contrib_off = 0;
      R.inv = 1;
      R.pad = 0;
      A.recs[exc[g].y] = R;
    }
  }
}

__global__ void __launch_bounds__(256) skel_stats_part(const SkelTask* __restrict__ tasks,
                                                       const int32_t* __restrict__ kout, const int32_t* __restrict__ ng,
                                                       StatAcc* __restrict__ part) {
  const int n = *ng;
  const int lo = (int)((int64_t)n * blockIdx.x / gridDim.x), hi = (int)((int64_t)n * (blockIdx.x + 1) / gridDim.x);
  StatAcc a;
  for (int i = 0; i < 8; ++i) a.d[i] = 0.0;
  for (int i = 0; i < 4; ++i) a.sum[i] = a.mx[i] = 0;
  for (int g = lo + threadIdx.x; g < hi; g += 256) {
    const SkelTask& T = tasks[g];
    const int kk = kout[g], r = T.nc - kk;
    a.sum[0] += kk;
    a.sum[1] += r;
    a.mx[2] = max(a.mx[2], (int64_t)(T.nc + T.nq));
    const double dc = T.nc, dq = T.nq, dk = kk, dr = r;
    double f = 4 * dq * dc * dk - 2 * dk * dk * (dq + dc) + 4 * dk * dk * dk / 3 + 2 * dq * dc + dk * dk * dr +
               2 * dk * dk * dr + 4 * dk * dr * dr;
    if (r > 0) f += dr * dr * dr / 3 + dr * dr * dk + dk * dk * dr;
    a.d[0] += f * 1e-9;
    a.d[1] += 8.0 * (dq * dc + dc * dc + dk * dr + dr * dr + dr + dr * dk + 2 * dk * dk) * 1e-9;
    if (r > 0) {
      a.sum[2] += 8 * ((int64_t)kk * r + (int64_t)r * r + r + (int64_t)r * kk);
      a.d[2] += dr * (dr + 1) / 2 + 2 * dr * dk;
      a.d[3] += dr + dk;
      a.mx[0] = max(a.mx[0], (int64_t)r);
      a.mx[1] = max(a.mx[1], (int64_t)kk);
    }
  }
  stat_block_reduce(a, part + blockIdx.x);
}

__global__ void __launch_bounds__(256) skel_stats_final(const int32_t* __restrict__ ng,
                                                        const StatAcc* __restrict__ part, int np,
                                                        const int2* __restrict__ exc, const int2* __restrict__ inc,
                                                        LevelStat* st, int64_t* nblk) {
  const StatAcc a = stat_partials(part, np);
  if (threadIdx.x != 0) return;
  const int n = *ng;
  st->ngroups = n;
  st->nskel = a.sum[0];
  st->nred = a.sum[1];
  st->gflop = a.d[0];
  st->gbytes = a.d[1];
  st->gf_cls[0] = a.d[0];
  st->gb_cls[0] = a.d[1];
  st->solve_fac = a.d[2];
  st->solve_rows = a.d[3];
  st->mf_bytes = a.sum[2];
  st->max_nc = a.mx[0];
  st->max_nq = a.mx[1];
  st->max_front = a.mx[2];
  const int2 last = n ? make_int2(exc[n - 1].x + inc[n - 1].x, exc[n - 1].y + inc[n - 1].y) : make_int2(0, 0);
  st->nrecs = last.y;
  *nblk += last.x;
}

// active DOFs -> ascending list (and the count into the previous level's stats)
__global__ void count_to(const int64_t* __restrict__ n, int64_t* dst) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *dst = *n;
}

// ---------------------------------------------------------------------------
// Host-side launchers
// ---------------------------------------------------------------------------
namespace {
int sym_grid(int per_sm) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return nsm * per_sm;
}
}  // namespace

// per-CTA partials of the level statistics (persistent, SymWork-owned)
static StatAcc* stat_parts(SymWork& W, cudaStream_t s) {
  if (!W.stat_part) cudaMallocAsync(&W.stat_part, sizeof(StatAcc) * kStatGrid, s);
  return reinterpret_cast<StatAcc*>(W.stat_part);
}

// temp storage for CUB calls lives at the front of W.cub_tmp; the launcher
// grows it (stream-ordered) when a call needs more
static void ensure_tmp(SymWork& W, size_t bytes, cudaStream_t s) {
  if (bytes <= W.cub_bytes) return;
  if (W.cub_tmp) cudaFreeAsync(W.cub_tmp, s);
  W.cub_bytes = bytes + bytes / 2 + (1 << 20);
  cudaMallocAsync((void**)&W.cub_tmp, W.cub_bytes, s);
}

cudaError_t sym_active_list(const uint8_t* active, int64_t N, int32_t* act, int64_t* nact, SymWork& W,
                            cudaStream_t s) {
  size_t tb = 0;
  cub::CountingInputIterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, tb, it, active, act, nact, (int)N, s);
  ensure_tmp(W, tb, s);
  return cub::DeviceSelect::Flagged(W.cub_tmp, tb, it, active, act, nact, (int)N, s);
}

cudaError_t sym_partition(const SymPartArgs& A, SymWork& W, cudaStream_t s) {
  if (A.nact_ub <= 0) {
    cudaMemsetAsync(A.ng, 0, sizeof(int32_t), s);
    cudaMemsetAsync(A.goff, 0, sizeof(int64_t), s);
    return cudaGetLastError();
  }
  const int grid = sym_grid(8);
  sym_keys_kernel<<<grid, 256, 0, s>>>(A.act, A.nact, A.nact_ub, A.dim, A.side, A.w, A.k, A.kind, A.nkeys, A.keys);
  int bits = 1;
  while ((1ll << bits) <= (int64_t)A.nkeys) ++bits;  // keys in [0, nkeys]
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, A.keys, A.skeys, A.act, A.gmem, (int)A.nact_ub, 0, bits, s);
  ensure_tmp(W, tb, s);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(W.cub_tmp, tb, A.keys, A.skeys, A.act, A.gmem, (int)A.nact_ub,
                                                  0, bits, s);
  if (e != cudaSuccess) return e;
  sym_heads_kernel<<<grid, 256, 0, s>>>(A.skeys, A.nact_ub, A.nkeys, A.head);
  tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, A.head, A.head, (int)A.nact_ub, s);
  ensure_tmp(W, tb, s);
  e = cub::DeviceScan::InclusiveSum(W.cub_tmp, tb, A.head, A.head, (int)A.nact_ub, s);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(A.ng, 0, sizeof(int32_t), s);
  cudaMemsetAsync(A.goff, 0, sizeof(int64_t), s);
  sym_groups_kernel<<<grid, 256, 0, s>>>(A.skeys, A.head, A.gmem, A.nact, A.nkeys, A.goff, A.ng, A.group_of);
  return cudaGetLastError();
}

cudaError_t sym_membership(const SymMemberArgs& A, SymWork& W, cudaStream_t s) {
  // live blocks
  size_t tb = 0;
  cub::CountingInputIterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, tb, it, A.blk_alive, A.alive_list, A.nalive, (int)A.nblk_ub, s);
  ensure_tmp(W, tb, s);
  cudaError_t e = cub::DeviceSelect::Flagged(W.cub_tmp, tb, it, A.blk_alive, A.alive_list, A.nalive,
                                             (int)A.nblk_ub, s);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(A.cnt, 0, sizeof(int32_t) * (size_t)(A.N + 1), s);
  const int grid = sym_grid(8);
  sym_member_count<<<grid, 256, 0, s>>>(A.alive_list, A.nalive, A.blk_n, A.blk_dof_off, A.idx, A.active, A.cnt);
  tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, A.cnt, A.mptr, (int)(A.N + 1), s);
  ensure_tmp(W, tb, s);
  e = cub::DeviceScan::ExclusiveSum(W.cub_tmp, tb, A.cnt, A.mptr, (int)(A.N + 1), s);
  if (e != cudaSuccess) return e;
  cudaMemcpyAsync(A.cnt, A.mptr, sizeof(int32_t) * (size_t)(A.N + 1), cudaMemcpyDeviceToDevice, s);
  sym_member_fill<<<grid, 256, 0, s>>>(A.alive_list, A.nalive, A.blk_n, A.blk_dof_off, A.idx, A.active, A.cnt,
                                       A.mblk);
  return cudaGetLastError();
}

namespace {
constexpr int kSLQ = 10, kSLB = 8, kSLP = 8, kSNC = 512;     // small tier: 1024 / 256 / 256 slots, 512 DOFs
constexpr int kBLQ = 14, kBLB = 11, kBLP = 11, kBNC = 4096;  // big tier
constexpr size_t smem_of(int lq, int lb, int lp, int nc) {
  return sizeof(int32_t) * ((size_t)nc + (1u << lb) + 2 * (1u << lq) + (1u << lp));
}
template <bool FILL>
cudaError_t fronts_pass(const SymFront& P, cudaStream_t s) {
  int wper = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wper, sym_front_warp_kernel<FILL>, 32 * kWarpTierW, 0);
  sym_front_warp_kernel<FILL><<<sym_grid(std::max(wper, 1)), 32 * kWarpTierW, 0, s>>>(P);
  auto ks = sym_front_kernel<kSLQ, kSLB, kSLP, kSNC, FILL>;
  auto kb = sym_front_kernel<kBLQ, kBLB, kBLP, kBNC, FILL>;
  static bool once = false;
  const size_t ss = smem_of(kSLQ, kSLB, kSLP, kSNC), sb = smem_of(kBLQ, kBLB, kBLP, kBNC);
  if (!once) {
    cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ss);
    cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    once = true;
  }
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ks, kSymNT, ss);
  ks<<<sym_grid(std::max(per, 1)), kSymNT, ss, s>>>(P);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kb, kSymNT, sb);
  kb<<<sym_grid(std::max(per, 1)), kSymNT, sb, s>>>(P);
  return cudaGetLastError();
}
}  // namespace

cudaError_t sym_fronts_count(const SymFront& P, cudaStream_t s) {
  cudaMemsetAsync(P.nretry, 0, sizeof(int32_t), s);
  cudaMemsetAsync(P.nretry2, 0, sizeof(int32_t), s);
  return fronts_pass<false>(P, s);
}
cudaError_t sym_fronts_fill(const SymFront& P, cudaStream_t s) { return fronts_pass<true>(P, s); }

cudaError_t sym_elim_sizes(const SymFront& P, int is_top, int ng_ub, ElimInc* inc, ElimInc* exc, LevelTotals* tot,
                           SymWork& W, cudaStream_t s) {
  cudaMemsetAsync(tot, 0, sizeof(LevelTotals), s);
  cudaMemsetAsync(inc, 0, sizeof(ElimInc) * (size_t)ng_ub, s);
  elim_size_kernel<<<sym_grid(4), 256, 0, s>>>(P, is_top, inc, tot);
  size_t tb = 0;
  ElimInc zero;
  for (int i = 0; i < kElimIncN; ++i) zero.v[i] = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, tb, inc, exc, ElimIncOp(), zero, ng_ub, s);
  ensure_tmp(W, tb, s);
  cudaError_t e = cub::DeviceScan::ExclusiveScan(W.cub_tmp, tb, inc, exc, ElimIncOp(), zero, ng_ub, s);
  if (e != cudaSuccess) return e;
  elim_total_kernel<<<1, 1, 0, s>>>(P.ng, inc, exc, tot);
  return cudaGetLastError();
}

cudaError_t sym_elim_fill(const SymFront& P, const ElimFillArgs& A, int64_t nred_ub, SymWork& W, cudaStream_t s) {
  elim_fill_kernel<<<sym_grid(4), 256, 0, s>>>(P, A);
  StatAcc* part = stat_parts(W, s);
  elim_stats_part<<<kStatGrid, 256, 0, s>>>(P.ng, A.cellstat, A.cellcls, P, part);
  elim_stats_final<<<1, 256, 0, s>>>(P.ng, part, kStatGrid, A.stat, A.newblk_total, A.nblk);
  // reduction of the forward sweep: contribution rows grouped by neighbour
  // DOF in record order (stable radix sort), targets = the distinct DOFs
  if (nred_ub > 0) {
    size_t tb = 0;
    int bits = 1;
    while ((1ll << bits) < A.N) ++bits;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, A.red_key, A.red_key2, A.red_val, A.red_ent, (int)nred_ub, 0, bits,
                                    s);
    ensure_tmp(W, tb, s);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(W.cub_tmp, tb, A.red_key, A.red_key2, A.red_val, A.red_ent,
                                                    (int)nred_ub, 0, bits, s);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(A.red_cnt, 0, sizeof(int64_t) * (size_t)(nred_ub + 1), s);
    tb = 0;
    cub::DeviceRunLengthEncode::Encode(nullptr, tb, A.red_key2, A.red_targets, A.red_cnt, A.red_nt, (int)nred_ub, s);
    ensure_tmp(W, tb, s);
    e = cub::DeviceRunLengthEncode::Encode(W.cub_tmp, tb, A.red_key2, A.red_targets, A.red_cnt, A.red_nt,
                                           (int)nred_ub, s);
    if (e != cudaSuccess) return e;
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, A.red_cnt, A.red_ptr, (int)(nred_ub + 1), s);
    ensure_tmp(W, tb, s);
    e = cub::DeviceScan::ExclusiveSum(W.cub_tmp, tb, A.red_cnt, A.red_ptr, (int)(nred_ub + 1), s);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t sym_skel_sizes(const SymFront& P, double promote_work, int gram_eps_ok, int ng_ub, SkelInc* inc,
                           SkelInc* exc, LevelTotals* tot, SymWork& W, cudaStream_t s) {
  cudaMemsetAsync(tot, 0, sizeof(LevelTotals), s);
  cudaMemsetAsync(inc, 0, sizeof(SkelInc) * (size_t)ng_ub, s);
  skel_size_kernel<<<sym_grid(4), 256, 0, s>>>(P, promote_work, gram_eps_ok, inc, tot);
  size_t tb = 0;
  SkelInc zero;
  for (int i = 0; i < kSkelIncN; ++i) zero.v[i] = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, tb, inc, exc, SkelIncOp(), zero, ng_ub, s);
  ensure_tmp(W, tb, s);
  cudaError_t e = cub::DeviceScan::ExclusiveScan(W.cub_tmp, tb, inc, exc, SkelIncOp(), zero, ng_ub, s);
  if (e != cudaSuccess) return e;
  skel_total_kernel<<<1, 1, 0, s>>>(P.ng, inc, exc, tot);
  return cudaGetLastError();
}

cudaError_t sym_skel_fill(const SymFront& P, const SkelFillArgs& A, cudaStream_t s) {
  skel_fill_kernel<<<sym_grid(4), 256, 0, s>>>(P, A);
  return cudaGetLastError();
}

cudaError_t sym_skel_chain(const int64_t* pred_start, const int32_t* npred, const int32_t* preds, const int32_t* ng,
                           int ng_ub, int iters, int cap, int32_t* b0, int32_t* b1, int32_t* changed,
                           LevelTotals* tot, cudaStream_t s) {
  cudaMemsetAsync(b0, 0, sizeof(int32_t) * (size_t)ng_ub, s);
  cudaMemsetAsync(changed, 0, sizeof(int32_t) * ((size_t)iters + 1), s);
  cudaMemsetAsync(&tot->max_chain, 0, sizeof(int64_t), s);
  static int per_sm = 0;
  if (!per_sm) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, skel_relax_coop, 256, 0);
  const int grid = std::max(1, std::min(sym_grid(std::max(per_sm, 1)), (ng_ub + 255) / 256));
  void* args[] = {(void*)&pred_start, (void*)&npred, (void*)&preds, (void*)&ng, (void*)&b0, (void*)&b1,
                  (void*)&changed, (void*)&iters, (void*)&cap, (void*)&tot};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)skel_relax_coop, dim3((unsigned)grid), dim3(256), args, 0, s);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t sym_skel_order(const int32_t* b0, const int32_t* b1, const int32_t* changed, int iters,
                           const int32_t* ng, int ng_ub, int32_t* depth, int32_t* depth_sorted, int32_t* iota,
                           int32_t* order, SymWork& W, cudaStream_t s) {
  skel_depth_kernel<<<std::max(1, (ng_ub + 255) / 256), 256, 0, s>>>(b0, b1, changed, iters, ng, depth, iota);
  int bits = 1;
  while ((1 << bits) <= iters) ++bits;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, depth, depth_sorted, iota, order, ng_ub, 0, bits, s);
  ensure_tmp(W, tb, s);
  return cub::DeviceRadixSort::SortPairs(W.cub_tmp, tb, depth, depth_sorted, iota, order, ng_ub, 0, bits, s);
}

cudaError_t sym_skel_cluster_tasks(SkelTask* tasks, const int64_t* cl_rel, int64_t base, const int32_t* ng,
                                   int ng_ub, cudaStream_t s) {
  skel_cluster_tasks<<<std::max(1, (ng_ub + 255) / 256), 256, 0, s>>>(tasks, cl_rel, base, ng);
  return cudaGetLastError();
}

cudaError_t sym_skel_finish(const SkelTask* tasks, const int32_t* kout, const int32_t* ng, int ng_ub,
                            const SkelFinishArgs& A, SymWork& W, cudaStream_t s) {
  const int grid = std::max(1, std::min(sym_grid(4), (ng_ub + 255) / 256));
  int2* inc = A.inc;
  int2* exc = A.exc;
  cudaMemsetAsync(inc, 0, sizeof(int2) * (size_t)ng_ub, s);
  skel_finish_inc<<<grid, 256, 0, s>>>(tasks, kout, ng, inc);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, tb, inc, exc, Int2Sum(), make_int2(0, 0), ng_ub, s);
  ensure_tmp(W, tb, s);
  cudaError_t e = cub::DeviceScan::ExclusiveScan(W.cub_tmp, tb, inc, exc, Int2Sum(), make_int2(0, 0), ng_ub, s);
  if (e != cudaSuccess) return e;
  skel_finish_fill<<<grid, 256, 0, s>>>(tasks, kout, ng, exc, A);
  StatAcc* part = stat_parts(W, s);
  skel_stats_part<<<kStatGrid, 256, 0, s>>>(tasks, kout, ng, part);
  skel_stats_final<<<1, 256, 0, s>>>(ng, part, kStatGrid, exc, inc, A.stat, A.nblk);
  return cudaGetLastError();
}

cudaError_t sym_reset_groups(const int32_t* gmem, const int64_t* goff, const int32_t* ng, int32_t* group_of,
                             cudaStream_t s) {
  sym_reset_group_of<<<sym_grid(4), 256, 0, s>>>(gmem, goff, ng, group_of);
  return cudaGetLastError();
}

// Elimination levels: every member of every cell retires (the structural
// part of the elimination, so the next level's analysis need not wait for
// the numeric kernels, which clear the same bytes again).
__global__ void sym_retire_members(const int32_t* __restrict__ gmem, const int64_t* __restrict__ goff,
                                   const int32_t* __restrict__ ng, uint8_t* __restrict__ active) {
  const int64_t n = goff[*ng];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    active[gmem[i]] = 0;
}
cudaError_t sym_retire_cells(const int32_t* gmem, const int64_t* goff, const int32_t* ng, uint8_t* active,
                             cudaStream_t s) {
  sym_retire_members<<<sym_grid(4), 256, 0, s>>>(gmem, goff, ng, active);
  return cudaGetLastError();
}

cudaError_t sym_copy_count(const int64_t* n, int64_t* dst, cudaStream_t s) {
  count_to<<<1, 32, 0, s>>>(n, dst);
  return cudaGetLastError();
}

}  // namespace hifde
