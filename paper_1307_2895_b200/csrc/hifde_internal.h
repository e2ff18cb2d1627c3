// Internal structures shared by the host runtime and the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

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
void launch_skel(const SkelTask* d_tasks, int ntasks, const Arenas& A, double eps, size_t smem, int nt,
                 cudaStream_t s);
void launch_apply_rd(const SkelTask* d_tasks, int ntasks, const Arenas& A, cudaStream_t s);
int skel_ordered_capacity(size_t smem, int nt);
constexpr int kClusterThreads = 256;           // threads per CTA of the cluster skeleton kernel
constexpr int kClusterMinNc = 24;              // levels whose widest group reaches this may use it
int skel_cluster_capacity(size_t smem, int cs);  // resident clusters of cs CTAs
cudaError_t launch_skel_cluster(const SkelTask* d_tasks, int ntasks, const int64_t* pred_ptr, const int32_t* pred,
                                int* done, const Arenas& A, double eps, size_t smem, int nclusters, int cs,
                                cudaStream_t s);
cudaError_t launch_skel_ordered(const SkelTask* d_tasks, int ntasks, const int64_t* pred_ptr, const int32_t* pred,
                                int* done, const Arenas& A, double eps, size_t smem, int nt, int grid,
                                cudaStream_t s);

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
constexpr double kPromoteWork = 2.5e5;  // nq nc^2 above which a one-CTA group joins the pipeline
constexpr int kGramRows = 1024;  // rows per split of a Gram tile
void launch_skelbig_gram(const SkelBigTask* tasks, const int4* work, int nwork, const int4* tiles, int ntiles,
                         double* part, const Arenas& A, cudaStream_t s);
size_t pchol_smem(int nc, int G);
int pchol_min_ctas(int nc);
int pchol_coop_capacity(size_t smem);
// one CTA per group, R in shared memory: groups with pchol_1cta_smem(nc) <= kSmemCapBytes
size_t pchol_1cta_smem(int nc);
void launch_pchol_1cta(const SkelBigTask* tasks, int ntasks, size_t smem, const Arenas& A, double eps,
                       cudaStream_t s);
// one cl-CTA cluster per group (cl in 2, 4, 8, 16), smem = pchol_smem(max nc, cl)
cudaError_t launch_pchol_cluster(const SkelBigTask* tasks, int ntasks, int cl, size_t smem, const Arenas& A,
                                 double eps, cudaStream_t s);
cudaError_t launch_pchol_coop(const SkelBigTask* tasks, int ntasks, const int* d_gstart, int nblocks,
                              unsigned int* d_bar, size_t smem, const Arenas& A, double eps, cudaStream_t s);
cudaError_t launch_cpqr_cluster(const SkelBigTask* tasks, int ntasks, int max_nq, const Arenas& A, double eps,
                                cudaStream_t s);
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
void launch_solve_elim_small(const SolveRec* recs, int nrec, const int32_t* idx, const double* fac, double* v,
                             int nrhs, double* contrib, size_t smem, int forward, cudaStream_t s);
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

}  // namespace hifde
