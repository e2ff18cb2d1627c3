// Internal structures shared by the host runtime and the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hifde_gpu.h"

namespace hifde {

// Per-cell work item of an elimination level (src/factor_ops.py:138-159).
// Front DOFs are c (ascending) followed by q (ascending) in the idx arena.
struct ElimTask {
  int32_t nc, nq;
  int32_t nblk, maxnb;      // consumed clique blocks, largest block order
  int64_t dofs_off;         // idx arena: c[nc] then q[nq]
  int64_t blk_off;          // list arena: consumed block ids (ascending)
  int64_t scratch_off;      // scratch arena (doubles) for a global front, -1: smem
  int64_t C_off;            // factor arena: Cholesky factor, nc x nc row-major
  int64_t W_off;            // factor arena: W = C^-1 A_cq, nc x nq row-major
  int64_t U_off;            // block arena: new clique block, nq x nq row-major
  int64_t P_off;            // factor arena: packed lower C^-1 (what the solve applies)
};

// Per-group work item of a skeletonization level (src/factor_ops.py:162-214).
struct SkelTask {
  int32_t nc, nq;
  int32_t nblk, maxnb;      // clique blocks touching c (read only)
  int64_t dofs_off;         // idx arena: c[nc] then q[nq]
  int64_t blk_off;          // list arena
  int64_t scratch_off;      // scratch arena workspace, -1: smem
  int64_t rec_off;          // factor arena: T (k x r), C (r x r), W (r x k)
  int64_t delta_off;        // block arena: delta block (k x k)
  int64_t out_off;          // idx arena: sk (ascending) then rd (ascending), global ids
  int32_t group;            // index of the group within its level
  int32_t mode;             // workspace: 0 shared, 1 Mq shared, 3 Mq global + TSQR, 2 large path
  int32_t chunk;            // mode 3: Mq rows per TSQR chunk
  int32_t pad2;
};

// Skeletonization of a group too large for one CTA (kernels_skelbig.cu).
struct SkelBigTask {
  int32_t nc, nq;
  int32_t nblk, maxnb;
  int64_t dofs_off, blk_off;
  int64_t ws_off;           // scratch arena: A_cc, Mq, Tp, norms, candidates
  int64_t iws_off;          // int scratch: pivots, sk / rd orders
  int64_t rec_off, delta_off, out_off;
  int32_t group, pad;
  int64_t map_off;          // int scratch: front position of every block entry (-1: none)
};
constexpr int kMaxG = 1024;                    // most CTAs serving one large-group CPQR
constexpr int kCL = 16;                        // CTAs per cluster (many-group batches)
constexpr int kMaxBigNc = 4096;                // largest group handled by that path

// One tiled product of the solve for large records (kernels_solve.cu):
//   dst(i, :) = src(i, :) + alpha * sum_k A(i, k) X(k, :),  i < M, k < K
// A: amode 0 packed lower P, 1 its transpose, 2 dense row-major (lda), 3 dense
// transposed.  X / src / dst rows: mode 0 = rows of v gathered through the
// index list at *_off, 1 = solve scratch rows from *_off, 2 = contribution rows
// from *_off; smode -1 = no src.
struct TileOp {
  int32_t M, K;
  int32_t amode, xmode, smode, dmode;
  int64_t A_off, lda;
  int64_t x_off, s_off, d_off;
  double alpha;
};

// Solve-sweep record (one per elimination cell / skeleton group with rd != {}).
struct SolveRec {
  int32_t nc;               // |cell| (elimination) or |rd| (skeleton)
  int32_t nq;               // |nbrs| (elimination) or |sk| (skeleton)
  int64_t idx_off;          // idx arena: cell then nbrs / rd then sk
  int64_t C_off, W_off, T_off;  // factor arena
  int64_t contrib_off;      // elimination: row offset in the contribution buffer
  int32_t inv;              // 1: C slot holds the packed lower inverse C^-1; 0: C itself
  int32_t pad;
};

// Device views of the persistent arenas.
struct Arenas {
  const int64_t* indptr;    // A0 (original matrix) CSR
  const int32_t* indices;
  const double* a0;
  int32_t* idx;             // index arena (cells, neighbour lists, sk/rd)
  const int32_t* lists;     // per-level block lists
  const int64_t* blk_dof_off;  // block table: dof list offset in idx
  const int32_t* blk_n;        //              order
  const int64_t* blk_val_off;  //              value offset in the block arena
  double* bvals;            // block arena
  double* fac;              // factor arena
  double* scratch;          // per-level scratch arena
  uint8_t* active;          // device active mask (exact-order batches)
  int* status;              // per-task status words
  int32_t* kout;            // per-group skeleton rank
  int32_t* iscratch;        // per-level integer scratch
  unsigned long long* tlog; // optional per-group timestamps (HIFDE_SKEL_TLOG), else null
};

constexpr size_t kSmemCapBytes = 220 * 1024;  // dynamic shared memory per CTA we use
constexpr int kSchurTile = 64;                 // schur_tile_kernel tile edge
constexpr int kPanelB = 64;                    // blocked Cholesky panel width
constexpr int kMaxSkelNc = 192;
// Column stride of a shared-memory neighbour block: = 8 (mod 16) doubles, so
// the G-lane column slices of one warp's 4 columns fall on disjoint banks
// (2 wavefronts per 64-bit warp access instead of 3-4).
__host__ __device__ inline int skel_ldq(int nq) { return nq < 32 ? nq : nq + ((24 - nq % 16) % 16); }
// cells this wide (or with fronts this large) take the multi-CTA blocked path
// even when the front fits one CTA's shared memory: one CTA per wide cell is
// latency-bound (measured: 0.5 ms for a 93-wide terminal block)
constexpr int kBigCellNc = 64, kBigCellNf = 128;
constexpr size_t kSolveDynSmem = 190 * 1024;   // solve record kernels: dynamic smem beside the 25 KB staging tile                // largest group skeletonized by one CTA (skel_group)

// ---------------------------------------------------------------------------
// Workspace sizing of one cell / group, shared by the host task builder and
// the device symbolic pass (symbolic.cu) so both place work identically.
// ---------------------------------------------------------------------------
__host__ __device__ inline size_t hd_align16(size_t x) { return (x + 15) / 16 * 16; }

struct ElimSizes {
  size_t smem;          // dynamic shared memory of elim_small_kernel (small cells)
  int32_t big;          // 1: the blocked multi-CTA path
  int32_t scratch_off;  // ElimTask.scratch_off: -2 room for the inverse workspace, -1 not
};
__host__ __device__ inline ElimSizes elim_sizes(int nc, int nq, int maxnb, bool is_top) {
  const int nf = nc + nq;
  const size_t ib = hd_align16(sizeof(int32_t) * (size_t)(nf + maxnb));
  // the path choices (one CTA or blocked, in-place or per-column inverse)
  // keep the full-square rule they were tuned with; elim_small_kernel holds
  // the front as a packed lower triangle
  const size_t need = ib + sizeof(double) * (size_t)nf * nf;
  const size_t need_inv = need + sizeof(double) * 8 * (size_t)nc;  // in-place inverse: one 8-row product block
  const size_t packed = ib + sizeof(double) * ((size_t)nf * (nf + 1) / 2);
  ElimSizes z;
  if (need <= kSmemCapBytes && (is_top || (nc < kBigCellNc && nf < kBigCellNf))) {
    z.big = 0;
    z.scratch_off = need_inv <= kSmemCapBytes ? -2 : -1;
    z.smem = z.scratch_off == -2 ? packed + sizeof(double) * 8 * (size_t)nc : packed;
  } else {
    z.big = 1;
    z.scratch_off = -1;
    z.smem = 0;
  }
  return z;
}
// shared memory of big_assemble for a large cell
__host__ __device__ inline size_t elim_big_smem(int nf, int maxnb) {
  return hd_align16(sizeof(int32_t) * (size_t)(nf + 2 * maxnb));
}

struct SkelSizes {
  int32_t mode;   // SkelTask.mode: 0 / 1 / 3 one CTA, 2 the large-group pipeline
  int32_t chunk;  // mode 3: rows per TSQR chunk
  size_t smem;    // dynamic shared memory of the one-CTA kernels
  size_t scr;     // doubles of global scratch
  size_t fac;     // factor-arena doubles without the large-group extra
  size_t fac_big; // extra doubles when the group takes the large-group pipeline
};
// (kernels_factor.cu skel_group: index arrays, then the CPQR vectors)
__host__ __device__ inline SkelSizes skel_sizes(int nc, int nq, int maxnb) {
  const int nf = nc + nq;
  const size_t ib = hd_align16(sizeof(int32_t) * (size_t)(2 * nf + maxnb + 8 * nc)) + sizeof(double) * 5 * (size_t)nc;
  const size_t q4 = (size_t)nc * nc / 4 + nc;
  const size_t lq = (size_t)skel_ldq(nq);  // padded column stride in shared memory
  const size_t wsd = (size_t)(nc + lq) * nc + 2 * (size_t)nc + 3 * q4 + 2 * (size_t)nc * nc;
  const size_t mq = lq * nc + 2 * (size_t)nc;
  SkelSizes z;
  z.chunk = 0;
  z.smem = 0;
  z.scr = 0;
  if (nc > kMaxSkelNc) {
    z.mode = 2;  // beyond the one-CTA CPQR
  } else if (ib + sizeof(double) * wsd <= kSmemCapBytes) {
    z.mode = 0;
    z.smem = ib + sizeof(double) * wsd;
  } else if (ib + sizeof(double) * mq <= kSmemCapBytes) {
    z.mode = 1;
    z.scr = 3 * (size_t)nc * nc + 3 * q4 + 8;
    z.smem = ib + sizeof(double) * mq;
  } else if (nq > nc && nc <= 160 && ib + sizeof(double) * ((size_t)(2 * nc) * nc + 2 * (size_t)nc) <= kSmemCapBytes) {
    // Mq in global scratch, compressed to R (nc x nc) in shared memory by
    // chunked Householder QR: column norms and pivots are unchanged
    z.mode = 3;
    const size_t avail = (kSmemCapBytes - ib) / sizeof(double) - 2 * (size_t)nc;
    const size_t ch = avail / nc - nc;
    z.chunk = (int32_t)(ch < (size_t)nq ? ch : (size_t)nq);
    z.scr = wsd + 8;
    z.smem = ib + sizeof(double) * ((size_t)(nc + z.chunk) * nc + 2 * (size_t)nc);
  } else {
    z.mode = 2;  // too large for one CTA: cluster pipeline (kernels_skelbig.cu)
  }
  z.fac = (size_t)nc * nc + 2 * q4;
  z.fac_big = (size_t)nc * (nc + 1) / 2 + nc;
  return z;
}
// shared memory of skel_cluster_kernel with cs CTAs per group
__host__ __device__ inline size_t skel_cluster_need(int nc, int nq, int maxnb, int cs) {
  const int nf = nc + nq;
  return hd_align16(sizeof(int32_t) * (size_t)(2 * nf + maxnb + 8 * nc)) +
         sizeof(double) * (6 * (size_t)nc + (size_t)nq + (size_t)skel_ldq(nq) * ((nc + cs - 1) / cs));
}
// global workspace (doubles) of a group in skel_cluster_kernel
__host__ __device__ inline size_t skel_cluster_scratch(int nc) {
  const size_t q4 = (size_t)nc * nc / 4 + nc;
  return 4 * (size_t)nc * nc + 3 * q4 + 8;
}

// Kernel launchers (kernels_factor.cu / kernels_solve.cu).
void launch_elim_small(const ElimTask* d_tasks, int ntasks, const Arenas& A, size_t smem, int nt,
                       cudaStream_t s);
void launch_big_assemble(const ElimTask* tasks, const int4* work, int nwork, const Arenas& A,
                         double* diag_scale, size_t smem, cudaStream_t s);
void launch_panel_chol(const ElimTask* tasks, const int32_t* cells, int ncells, int p0, const Arenas& A,
                       double* dmin, cudaStream_t s);
void launch_panel_trsm(const ElimTask* tasks, const int4* work, int nwork, int p0, const Arenas& A,
                       cudaStream_t s);
void launch_panel_update(const ElimTask* tasks, const int4* work, int nwork, int p0, const Arenas& A,
                         cudaStream_t s);
void launch_big_finish(const ElimTask* tasks, int ncells, const Arenas& A, const double* dmin,
                       const double* diag_scale, cudaStream_t s);
void launch_big_inverse(const ElimTask* tasks, const int4* work, int nwork, const Arenas& A, cudaStream_t s);
constexpr int kInvLocalCols = 64;   // cells up to this nc: thread-per-column packed inverse
void launch_inv_diag(const ElimTask* tasks, const int4* work, int nwork, const Arenas& A, cudaStream_t s);
void launch_inv_tiles(const ElimTask* tasks, const int4* work, int nwork, int p0, const Arenas& A,
                      cudaStream_t s);
void launch_schur_tiles(const ElimTask* d_tasks, const int4* d_tiles, int ntiles, const Arenas& A,
                        cudaStream_t s);
void launch_skel(const SkelTask* d_tasks, int ntasks, const Arenas& A, double eps, size_t smem, int nt, int max_nc,
                 int max_nq, cudaStream_t s);
void launch_apply_rd(const SkelTask* d_tasks, int ntasks, const Arenas& A, cudaStream_t s);
int skel_ordered_capacity(size_t smem, int nt);
constexpr int kClusterThreads = 256;           // threads per CTA of the cluster skeleton kernel
constexpr int kClusterMinNc = 24;              // levels whose widest group reaches this may use it
int skel_cluster_capacity(size_t smem, int cs);  // resident clusters of cs CTAs
cudaError_t launch_skel_cluster(const SkelTask* d_tasks, int ntasks, const int64_t* pred_ptr, const int32_t* pred,
                                int* done, const Arenas& A, double eps, size_t smem, int nclusters, int cs,
                                cudaStream_t s);
// order: claim order of the groups (topological: by dependency depth, then
// reference order); done: ntasks + 1 ints, zeroed (the last is the claim counter)
cudaError_t launch_skel_ordered(const SkelTask* d_tasks, int ntasks, const int64_t* pred_ptr, const int32_t* pred,
                                const int32_t* order, int* done, const Arenas& A, double eps, size_t smem, int nt,
                                int grid, cudaStream_t s);

// work int4 {task, block index, map offset of the block, 0}
void launch_skelbig_posmap(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A, cudaStream_t s);
void launch_skelbig_assemble(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A,
                             size_t smem, cudaStream_t s);
int cpqr_coop_capacity(size_t smem);
// Gram path of the large-group ID (kernels_skelbig.cu): G = Mq^T Mq tiles,
// then a cooperative pivoted Cholesky of G with the CPQR's outputs
// Used only when u cond(G11) ~ u / eps^2 <= 1e-8 << eps (T = R11^-1 R12 from
// the Cholesky factor of G loses u cond(G11)); the rank cut eps^2 |G| >> u |G|
constexpr double kGramMinEps = 1e-4;
// Full-rank certificate of a small skeletonization group (skel_group_t): groups
// of at most kCertMaxNc DOFs, tolerances from kCertMinEps up (so that
// (kCertSafety eps)^2 >= 1e-11 stays far above the rounding of the Gram matrix).
constexpr int kCertMaxNc = 12;
constexpr double kCertMinEps = 2e-7;
constexpr double kCertSafety = 16.0;
constexpr double kPromoteWork = 2.5e5;  // nq nc^2 above which a one-CTA group joins the pipeline
constexpr int kGramRows = 1024;  // rows per split of a Gram tile
void launch_skelbig_gram(const SkelBigTask* tasks, const int4* work, int nwork, const int4* tiles, int ntiles,
                         double* part, const Arenas& A, cudaStream_t s);
size_t pchol_smem(int nc, int G);
int pchol_min_ctas(int nc);
int pchol_coop_capacity(size_t smem);
cudaError_t launch_pchol_coop(const SkelBigTask* tasks, int ntasks, const int* d_gstart, int nblocks,
                              unsigned int* d_bar, size_t smem, const Arenas& A, double eps, cudaStream_t s);
cudaError_t launch_cpqr_coop(const SkelBigTask* tasks, int ntasks, const int* d_gstart, int nblocks,
                             unsigned int* d_bar, int max_nq, const Arenas& A, double eps, cudaStream_t s);
void launch_skelbig_sort(const SkelBigTask* tasks, int ntasks, const Arenas& A, ElimTask* inner, double* dmin,
                         double* dscale, cudaStream_t s);
void launch_skelbig_tinit(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A, cudaStream_t s);
void launch_skelbig_tsolve(const SkelBigTask* tasks, const int4* work, int nwork, int b0, const Arenas& A,
                           cudaStream_t s);
void launch_skelbig_tupdate(const SkelBigTask* tasks, const int4* work, int nwork, int b0, const Arenas& A,
                            cudaStream_t s);
void launch_skelbig_tperm(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A, cudaStream_t s);
void launch_skelbig_congruence(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A,
                               cudaStream_t s);
void launch_skelbig_symm(const SkelBigTask* tasks, const int4* work, int nwork, const Arenas& A, double* dscale,
                         cudaStream_t s);

// solve
// small elimination records (nc, nq <= 64, 2..16 RHS): one shared-memory load phase
size_t solve_small_smem(int max_nc, int max_nq, int nrhs);
void launch_solve_rec_rows(const SolveRec* recs, int nrec, const int32_t* idx, int32_t* cmin, int32_t* cmax,
                           cudaStream_t s);
void launch_solve_elim_small(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac, int64_t fac_len,
                             double* v, int nrhs, double* contrib, int max_nc, int max_nq, size_t smem, int forward,
                             cudaStream_t s);
size_t solve_skel_small_smem(int max_r, int max_k, int nrhs);
void launch_solve_skel_small(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac, double* v,
                             int nrhs, size_t smem, int forward, cudaStream_t s);
void launch_solve_elim_fwd(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac,
                           double* v, int nrhs, double* contrib, double* scratch,
                           int64_t scratch_per_rec, size_t smem, cudaStream_t s);
void launch_solve_reduce(const int32_t* targets, const int64_t* ptr, const int64_t* ent,
                         int ntargets, const double* contrib, double* v, int nrhs,
                         cudaStream_t s, double sign = -1.0);
// kernels_krylov.cu (device-resident PCG)
void launch_spmv(const int64_t* ip, const int32_t* ix, const double* va, const double* x, double* y, int64_t n,
                 cudaStream_t s);
void launch_dot(const double* a, const double* c, int64_t n, double* partial, double* out, cudaStream_t s);
int dot_partials();
void launch_cg_xr(double* x, double* r, const double* p, const double* ap, const double* sc, int64_t n,
                  cudaStream_t s);
void launch_cg_p(double* p, const double* z, double* sc, int64_t n, cudaStream_t s);
void launch_sub(double* z, const double* x, const double* y, int64_t n, cudaStream_t s);
void launch_scale(double* x, const double* y, const double* nn, int64_t n, cudaStream_t s);
void launch_apply_elim(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac, double* v, int nrhs,
                       double* contrib, double* scratch, int64_t scratch_per_rec, size_t smem, int fwdinv,
                       cudaStream_t s);
void launch_apply_skel(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac, double* v, int nrhs,
                       double* scratch, int64_t scratch_per_rec, size_t smem, int fwdinv, cudaStream_t s);
void launch_solve_elim_bwd(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac,
                           double* v, int nrhs, double* scratch, int64_t scratch_per_rec,
                           size_t smem, cudaStream_t s);
void launch_solve_skel(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac,
                       double* v, int nrhs, int forward, double* scratch,
                       int64_t scratch_per_rec, size_t smem, cudaStream_t s);
void launch_solve_tiles(const TileOp* ops, const int2* work, int nwork, const int32_t* idx, const double* fac,
                        double* v, int nrhs, double* tscratch, double* contrib, cudaStream_t s);

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// Device symbolic pass (symbolic.cu): partition, membership, fronts, task
// tables and block-table updates of a level on the GPU, identical to the host
// analysis (runtime.cu Factorizer::front_sym / elimination_level /
// skeleton_level / finish_skeleton_level).
// ---------------------------------------------------------------------------
struct SymWork {           // CUB temporary storage (grown on demand, stream-ordered)
  char* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  void* stat_part = nullptr;  // per-CTA partials of the level statistics
};
struct SymPartArgs {
  const int32_t* act;      // active DOFs, ascending (act[0, *nact))
  const int64_t* nact;
  int64_t nact_ub;         // host bound on *nact (sort length)
  int dim, side, w, k, kind;  // kind 0 interior cells, 1 edges, 2 faces
  int32_t nkeys;           // keys are < nkeys; nkeys marks "no group"
  int32_t* keys;
  int32_t* skeys;
  int32_t* gmem;           // members sorted by group (ascending inside a group)
  int32_t* head;           // scratch: group number of each sorted member
  int64_t* goff;           // group offsets (ng + 1)
  int32_t* ng;             // number of groups (device scalar)
  int32_t* group_of;       // skeleton levels: group of each member DOF, else null
};
struct SymMemberArgs {
  const uint8_t* blk_alive;
  int64_t nblk_ub;
  int32_t* alive_list;
  int64_t* nalive;
  const int32_t* blk_n;
  const int64_t* blk_dof_off;
  const int32_t* idx;
  const uint8_t* active;
  int64_t N;
  int32_t* cnt;            // N + 1
  int32_t* mptr;           // N + 1: membership CSR (active DOF -> live blocks)
  int32_t* mblk;
};
struct SymFront {
  const int64_t* goff;
  const int32_t* gmem;
  const int32_t* ng;
  const int32_t* mptr;
  const int32_t* mblk;
  const int32_t* blk_n;
  const int64_t* blk_dof_off;
  const int32_t* idx;
  const int64_t* indptr;
  const int32_t* indices;
  const uint8_t* active;
  const int32_t* group_of;  // predecessors (skeleton levels) when non-null
  // count pass outputs (per group)
  int32_t* nq;
  int32_t* nb;
  int32_t* maxnb;
  int32_t* npred;
  int32_t* flag;            // tier of the group: 0 warp, 1 shared-memory CTA, 2 large CTA
  int32_t* retry;           // groups for the large tier
  int32_t* nretry;
  int32_t* retry2;          // groups for the shared-memory CTA tier (too large for a warp)
  int32_t* nretry2;
  int32_t* fatal;           // even the large tier overflowed (host fallback)
  // count pass, skeleton levels: unsorted predecessor lists for the chain
  int32_t* pred_tmp;        // null: not wanted
  int64_t* pred_start;
  int64_t* pred_alloc;      // allocation cursor (device scalar, zeroed)
  int64_t pred_cap;
  int32_t* pred_ovf;        // the capacity was exceeded
  // fill pass: offsets from the level's prefix sums (int64 words of the
  // per-group increment struct), destinations
  const int64_t* exc;
  int32_t exc_stride, o_nf, o_nb, o_pred;
  int64_t idx_base;
  int32_t* idx_out;
  int32_t* lists;
  int32_t* preds;
};
constexpr int kElimIncN = 8;  // idx, lists, fac, block arena, contributions, new blocks, small, big
struct ElimInc { int64_t v[kElimIncN]; };
constexpr int kSkelIncN = 8;  // idx, lists, scratch, fac, delta blocks, preds, out lists, cluster scratch
struct SkelInc { int64_t v[kSkelIncN]; };
struct LevelTotals {          // read back by the host once per level
  int64_t ng;
  int64_t sum[8];
  int64_t smem, max_small_nf, smem_big, max_big_nc, max_front, max_nc, max_nq;
  int64_t cl_need4, cl_need2, any_mode2, any_promote, max_chain;
  int64_t pad[2];
};
struct LevelStat {            // per device level, read back at the end of the factorization
  int64_t ngroups, nskel, nred, max_front, mf_bytes, nrecs, max_nc, max_nq;
  int64_t ntargets, active_after;
  double gflop, gbytes, solve_fac, solve_rows;
  double gf_cls[2], gb_cls[2];
};
struct ElimFillArgs {
  int is_top;
  int64_t idx_base, fac_base, bv_base;
  const ElimInc* exc;
  ElimTask* small;
  ElimTask* big;
  SolveRec* recs;
  hifde_record_t* xrec;
  int64_t* blk_dof_off;
  int32_t* blk_n;
  int64_t* blk_val_off;
  uint8_t* blk_alive;
  int64_t* nblk;            // device block count (advanced by the stats kernel)
  const int64_t* newblk_total;
  const int32_t* lists;
  const int32_t* idx;
  int32_t* red_key;         // reduction pairs (neighbour DOF, contribution row)
  int64_t* red_val;
  int32_t* red_key2;        // sorted
  int64_t* red_ent;
  int32_t* red_targets;
  int64_t* red_cnt;
  int64_t* red_ptr;
  int64_t* red_nt;          // distinct targets (device scalar)
  int64_t N;
  double4* cellstat;
  uint8_t* cellcls;
  LevelStat* stat;
};
struct SkelFillArgs {
  int64_t idx_base, scr_base, fac_base, bv_base, tot_nf;
  const SkelInc* exc;
  SkelTask* tasks;
  int64_t* pred_ptr;
  int64_t* cl_rel;          // cluster workspace offset of each group (relative)
  int32_t* idx;
};
struct SkelFinishArgs {
  int2* inc;
  int2* exc;
  SolveRec* recs;
  hifde_record_t* xrec;
  int64_t* blk_dof_off;
  int32_t* blk_n;
  int64_t* blk_val_off;
  uint8_t* blk_alive;
  int64_t* nblk;
  LevelStat* stat;
};
cudaError_t sym_active_list(const uint8_t* active, int64_t N, int32_t* act, int64_t* nact, SymWork& W, cudaStream_t s);
cudaError_t sym_partition(const SymPartArgs& A, SymWork& W, cudaStream_t s);
cudaError_t sym_membership(const SymMemberArgs& A, SymWork& W, cudaStream_t s);
cudaError_t sym_fronts_count(const SymFront& P, cudaStream_t s);
cudaError_t sym_fronts_fill(const SymFront& P, cudaStream_t s);
cudaError_t sym_elim_sizes(const SymFront& P, int is_top, int ng_ub, ElimInc* inc, ElimInc* exc, LevelTotals* tot,
                           SymWork& W, cudaStream_t s);
cudaError_t sym_elim_fill(const SymFront& P, const ElimFillArgs& A, int64_t nred_ub, SymWork& W, cudaStream_t s);
cudaError_t sym_skel_sizes(const SymFront& P, double promote_work, int gram_eps_ok, int ng_ub, SkelInc* inc,
                           SkelInc* exc, LevelTotals* tot, SymWork& W, cudaStream_t s);
cudaError_t sym_skel_fill(const SymFront& P, const SkelFillArgs& A, cudaStream_t s);
cudaError_t sym_skel_chain(const int64_t* pred_start, const int32_t* npred, const int32_t* preds, const int32_t* ng,
                           int ng_ub, int iters, int cap, int32_t* b0, int32_t* b1, int32_t* changed,
                           LevelTotals* tot, cudaStream_t s);
// claim order of an exact level: groups sorted stably by dependency depth
// (the final relaxation buffer of sym_skel_chain)
cudaError_t sym_skel_order(const int32_t* b0, const int32_t* b1, const int32_t* changed, int iters,
                           const int32_t* ng, int ng_ub, int32_t* depth, int32_t* depth_sorted, int32_t* iota,
                           int32_t* order, SymWork& W, cudaStream_t s);
cudaError_t sym_skel_cluster_tasks(SkelTask* tasks, const int64_t* cl_rel, int64_t base, const int32_t* ng,
                                   int ng_ub, cudaStream_t s);
cudaError_t sym_skel_finish(const SkelTask* tasks, const int32_t* kout, const int32_t* ng, int ng_ub,
                            const SkelFinishArgs& A, SymWork& W, cudaStream_t s);
cudaError_t sym_retire_cells(const int32_t* gmem, const int64_t* goff, const int32_t* ng, uint8_t* active,
                             cudaStream_t s);
cudaError_t sym_reset_groups(const int32_t* gmem, const int64_t* goff, const int32_t* ng, int32_t* group_of,
                             cudaStream_t s);
cudaError_t sym_copy_count(const int64_t* n, int64_t* dst, cudaStream_t s);

}  // namespace hifde
