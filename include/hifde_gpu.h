/*
 * hifde_gpu.h -- C ABI of the B200-native HIF-DE factor/solve hot path.
 *
 * The reference (hifde 0.1.0, /root/reference/pkg/src/hifde) is a pure-Python
 * package with no FFI.  These entry points replace, one for one, the Python
 * functions on its hot path; the Python shim in paper_1307_2895_b200/driver.py
 * binds them with ctypes and keeps the reference's names and signatures:
 *
 *   hifde_factor   <- factor_hifde   (src/driver.py:212-225)
 *                     factor_hifde3x (src/driver.py:228-251)
 *                     factor_mf      (src/driver.py:201-209)
 *   hifde_solve    <- GeneralizedLDL.apply_inverse (src/driver.py:113-129)
 *   hifde_apply    <- GeneralizedLDL.apply (src/driver.py:95-111)
 *   hifde_pcg      <- pcg(A, b, F.apply_inverse) (src/krylov.py:48-77)
 *   hifde_power_norm <- _power_norm / estimate_*_error (src/krylov.py:153-201)
 *                     and module-level apply_inverse (src/driver.py:258-259)
 *   hifde_get_info / hifde_get_level
 *                  <- GeneralizedLDL.metrics (src/driver.py:165-171)
 *   hifde_free     <- (Python GC of the factor object)
 *   hifde_last_error
 *                  <- the exception message (FactorizationError family,
 *                     src/dense.py:41-50; cell context as in
 *                     src/factor_ops.py:193-200)
 *
 * Status codes map onto the reference's exception classes:
 *   HIFDE_OK 0, HIFDE_INDEFINITE 1 (IndefiniteBlockError),
 *   HIFDE_SINGULAR 2 (SingularBlockError), HIFDE_BADARG 3 (ValueError),
 *   HIFDE_CUDA 4 (RuntimeError), HIFDE_INTERNAL 5 (AssertionError).
 *
 * Plain C types only: no torch or CUDA types cross this boundary (the stream
 * is an opaque pointer to a cudaStream_t, NULL for the library's own).
 */
#ifndef HIFDE_GPU_H
#define HIFDE_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HIFDE_OK 0
#define HIFDE_INDEFINITE 1
#define HIFDE_SINGULAR 2
#define HIFDE_BADARG 3
#define HIFDE_CUDA 4
#define HIFDE_INTERNAL 5

/* factorization variants (the reference's "skeletonize-fronts" switch) */
#define HIFDE_VARIANT_MF 0      /* factor_mf: elimination only, exact      */
#define HIFDE_VARIANT_HIFDE 1   /* factor_hifde: edges (2D) / faces (3D)   */
#define HIFDE_VARIANT_HIFDE3X 2 /* factor_hifde3x: faces + edges (3D)      */

/* ordering of the groups of one skeletonization level */
#define HIFDE_ORDER_AUTO 0      /* exact order unless the chain is too long */
#define HIFDE_ORDER_SNAPSHOT 1  /* all IDs of a level from one snapshot    */
#define HIFDE_ORDER_EXACT 2     /* reference's sequential semantics        */
/* where the per-level symbolic analysis (partition, neighbour sets, task
 * tables) runs; both give identical factors */
#define HIFDE_SYMBOLIC_AUTO 0   /* on the GPU while levels allow, then host */
#define HIFDE_SYMBOLIC_HOST 1   /* host analysis for every level           */

/*
 * Rank communicator of the sharded factorization: the fine
 * levels are partitioned spatially over the ranks, each group factored by its
 * owner, and only the blocks a rank consumes from another rank's groups are
 * exchanged (NCCL over NVLink); coarse exact-order levels run on rank 0.
 * Every rank passes the same matrix and ends with the whole factor.  The
 * reference has no multi-process path (src/driver.py:183 runs one thread).
 */
typedef struct hifde_comm hifde_comm_t;
#define HIFDE_COMM_ID_BYTES 128

typedef struct hifde_options {
  int variant;          /* HIFDE_VARIANT_*                                  */
  int skip_levels;      /* skeletonization skipped below this level         */
  int spd;              /* 1: Cholesky mode (the only mode implemented)     */
  int order_mode;       /* HIFDE_ORDER_*                                    */
  int exact_max_batches;/* AUTO: exact order when its dependency chain <= this */
  int device;           /* CUDA device ordinal                              */
  int input_on_device;  /* CSR arrays are device pointers                   */
  int verify;           /* 1: check cells of each level are non-interacting */
  double eps;           /* ID relative tolerance (0 -> exact rank)          */
  void* stream;         /* cudaStream_t or NULL                             */
  hifde_comm_t* comm;   /* NULL: one GPU; else shard over comm's ranks      */
  int kernel_log;       /* 1: time the main launches (hifde_kernel_stats)   */
  int symbolic;         /* HIFDE_SYMBOLIC_*: where the level analysis runs  */
  int indptr_int32;     /* 1: indptr points to n + 1 int32 offsets (scipy's
                           default index type), host arrays only; widened
                           by the library instead of by the caller          */
  int async_factor;     /* 1: hifde_factor returns the handle at once and the
                           factorization runs on a library thread (one GPU
                           only; the input arrays must stay valid until
                           hifde_wait or the first call that uses the handle,
                           which wait for it and report its status).  A
                           hifde_solve of page-locked host right-hand sides
                           uploads them while the factorization still runs. */
} hifde_options_t;

typedef struct hifde_factor hifde_factor_t;

typedef struct hifde_info {
  int64_t n;            /* matrix order N                                   */
  int32_t dim;
  int32_t nlevels;      /* number of level records (integer + fractional)   */
  int64_t s_top;        /* size of the terminal dense block                 */
  int64_t m_f_bytes;    /* 8 * nfloats, the reference's accounting          */
  int64_t device_bytes; /* bytes actually held on the device by the factor  */
  double t_f_seconds;   /* host wall time of hifde_factor                   */
  double eps;
  int32_t spd;
  int32_t variant;
  int64_t fac_len;      /* doubles in the factor arena (hifde_copy_arenas)  */
  int64_t idx_len;      /* int32 entries in the index arena                 */
  int32_t nranks;       /* ranks the factorization was sharded over (1)     */
  int32_t factor_whole; /* 1: the factor arena holds every record; 0: real
                           ranks before the first operation that sums them
                           (apply, export, power): each rank holds its own */
  int64_t xfer_bytes;   /* block bytes this rank exchanged with its peers   */
  int64_t solve_xfer_bytes; /* vector bytes the partitioned solves of this
                           rank exchanged; 0 unsharded         */
} hifde_info_t;

/*
 * One record of a level, for export (hifde_level_records): offsets into the
 * factor arena (doubles) and the index arena (int32) copied by
 * hifde_copy_arenas.  Cholesky form: C C^T = the eliminated block, stored as
 * its packed lower inverse P = C^-1 (row i at P_off + i(i+1)/2); the
 * reference's L = C diag(C)^-1, D = diag(C)^2, coupling X = diag(C)^-1 W.
 */
typedef struct hifde_record {
  int32_t kind;         /* 0 elimination cell, 1 skeleton group, 2 terminal */
  int32_t nc;           /* |cell| (0/2) or |group| (1)                      */
  int32_t nq;           /* |nbrs| (0) or k = |sk| (1); 0 for the terminal   */
  int32_t nr;           /* |rd| (1), else 0; 0 = no-op skeleton record      */
  int64_t cell_off;     /* cell / group DOFs, ascending                     */
  int64_t idx_off;      /* 0/2: cell then nbrs; 1: sk[k] then rd[r]         */
  int64_t P_off;        /* packed C^-1 (nc x nc, or r x r)                  */
  int64_t W_off;        /* 0: W (nc x nq) row-major; 1: W (r x k)           */
  int64_t T_off;        /* 1: interpolation T (k x r) row-major             */
} hifde_record_t;

typedef struct hifde_level_info {
  double tag;           /* level tag: l, l+1/2, l+1/3, l+2/3                */
  int32_t kind;         /* 0 elimination, 1 skeletonization                 */
  int32_t nbatches;     /* launches used (exact-order batches)              */
  int64_t ngroups;      /* cells / groups                                   */
  int64_t nskel;        /* sum |sk| (skeleton levels)                       */
  int64_t nredundant;   /* sum |rd| (skeleton levels)                       */
  int64_t active_after; /* active DOFs after the level (active_trace)       */
  int64_t max_front;    /* largest |c|+|q|                                  */
  double seconds;       /* host wall time of the level                      */
  double gflop;         /* algorithmic FLOPs of the level     */
  double gbytes;        /* algorithmic bytes of the level     */
  double gpu_seconds;   /* CUDA-event time of the level's kernels           */
} hifde_level_info_t;

/* Library version string. */
const char* hifde_version(void);

/* Number of visible CUDA devices (0 if no driver / no GPU). */
int hifde_device_count(void);

/* Fill *opt with the reference defaults for `variant`
 * (skip_levels 0 for MF/HIFDE, 1 for HIFDE3X; spd 1; AUTO ordering). */
void hifde_default_options(hifde_options_t* opt, int variant);

/*
 * Factor the symmetric matrix A given as full symmetric CSR
 * (indptr[n+1] int64, indices[nnz] int32, vals[nnz] float64; what
 * SparseSymMatrix.to_scipy() returns, src/sparse.py:105-111) on the
 * uniform grid (dim, n_grid, m_leaf, nlevels) of GridConfig
 * (src/discretize.py:43-74).  A is not modified.
 */
int hifde_factor(const int64_t* indptr, const int32_t* indices, const double* vals,
                 int64_t n, int dim, int n_grid, int m_leaf, int nlevels,
                 const hifde_options_t* opt, hifde_factor_t** out);

/*
 * x = F^{-1} b for an n x nrhs block stored row-major (C order, ld = nrhs),
 * b and x on the host (device_ptrs = 0) or the device (device_ptrs = 1).
 * Reentrant for a finished factor; b and x may alias.
 */
int hifde_solve(const hifde_factor_t* f, const double* b, double* x, int64_t n,
                int nrhs, int device_ptrs, void* stream);

/*
 * Page-locked host blocks from the library's caching pool, for solve/apply
 * outputs (and inputs): hifde_solve DMAs a result straight into such a block,
 * and a freed block is reused by the next request of about its size, so
 * repeated solves pay neither the pinning nor the page faults of a fresh
 * multi-GB host array.  No reference counterpart (the reference returns a
 * fresh numpy array from apply_inverse, src/driver.py:113-129; the Python
 * shim wraps these blocks in numpy arrays with the same semantics).
 */
int hifde_host_alloc(size_t bytes, void** out);
int hifde_host_free(void* p);

/*
 * y = F x (the factored operator, ~ A x), same layout and pointer rules as
 * hifde_solve; apply(apply_inverse(b)) == b up to rounding.
 */
int hifde_apply(const hifde_factor_t* f, const double* x, double* y, int64_t n,
                int nrhs, int device_ptrs, void* stream);

/*
 * Preconditioned CG on A x = b (A in CSR, the matrix the factor approximates)
 * with F^{-1} as preconditioner, run on the device: converged when
 * ||b - A x|| / ||b|| <= tol.  One right-hand side; host (device_ptrs = 0) or
 * device pointers for A, b and x alike.
 */
int hifde_pcg(const hifde_factor_t* f, const int64_t* indptr, const int32_t* indices,
              const double* vals, const double* b, double* x, int64_t n, double tol,
              int max_iter, int device_ptrs, void* stream, int* iters, double* residual,
              int* converged);

/*
 * Power iteration for sqrt(lambda_max(G^T G)) on the device, the reference's
 * _power_norm: kind 0 G = A - F, 1 G = A, 2 G = I - A F^-1 (G^T = I - F^-1 A).
 * x0 (host, length n) is the normalized start vector; stops when two
 * successive estimates agree to rtol, or after max_iter iterations.
 */
int hifde_power_norm(const hifde_factor_t* f, const int64_t* indptr, const int32_t* indices,
                     const double* vals, int64_t n, int kind, const double* x0, double rtol,
                     int max_iter, double* value, int* converged, int* iters);

int hifde_get_info(const hifde_factor_t* f, hifde_info_t* info);

/*
 * Export (hifde_export of SURVEY 8(b)): the records of level `level` in the
 * reference's record order -- every cell of an elimination level, every
 * group of a skeletonization level (no-op groups included), the terminal
 * block as the last level -- into out[0..cap); *count = number of records.
 * With out == NULL only *count is set.
 */
int hifde_level_records(const hifde_factor_t* f, int level, hifde_record_t* out, int64_t cap,
                        int64_t* count);

/*
 * Import (load_factor, src/driver.py:318-376): build a device factor from
 * records in the export layout.  Level li holds recs[rec_ptr[li] ..
 * rec_ptr[li+1]) with tag tags[li] and kind kinds[li] (0 elimination, 1
 * skeletonization, 2 terminal block -- the last level, one record); offsets
 * index the host arenas fac (doubles) and idx (int32), which are copied.
 */
int hifde_import(int64_t n, int dim, double eps, int nlevels, const double* tags, const int32_t* kinds,
                 const int64_t* rec_ptr, const hifde_record_t* recs, const double* fac, int64_t fac_len,
                 const int32_t* idx, int64_t idx_len, int device, hifde_factor_t** out);

/* Copy the factor arena (fac_len doubles) and the index arena (idx_len
 * int32) to host buffers; either pointer may be NULL. */
int hifde_copy_arenas(const hifde_factor_t* f, double* fac, int64_t fac_len, int32_t* idx,
                      int64_t idx_len);
int hifde_get_level(const hifde_factor_t* f, int level, hifde_level_info_t* info);

/* Number of kernel launches issued by the last hifde_factor / hifde_solve
 * on this thread (the bench's gpu_launches count). */
int64_t hifde_last_launch_count(void);

/*
 * Kernel log of a factor created with options.kernel_log = 1: per (kernel,
 * level) the launches, their summed CUDA-event time and the algorithmic bytes
 * and FLOPs of the work they cover.  phase 0: the factorization;
 * phase 1: the last hifde_solve of this factor (per level and direction).
 * With out == NULL only *count is set.  No reference counterpart (the
 * reference times levels with perf_counter, src/driver.py:170).
 */
typedef struct hifde_kernel_stat {
  char name[40];
  double tag;           /* level tag                                        */
  int32_t phase;        /* 0 factor, 1 solve                                */
  int32_t launches;     /* launches (or pipelines) aggregated               */
  double seconds;       /* summed CUDA-event time                           */
  double gbytes;        /* algorithmic GB of the covered work               */
  double gflop;         /* algorithmic GFLOP of the covered work            */
} hifde_kernel_stat_t;
int hifde_kernel_stats(const hifde_factor_t* f, int phase, hifde_kernel_stat_t* out, int64_t cap,
                       int64_t* count);
void hifde_free(hifde_factor_t* f);
/* Waits for an options.async_factor factorization; returns its status (0 at
 * once for a handle that is complete).  Reference: none (factor_hifde,
 * src/driver.py:212-225, returns when the factor is complete). */
int hifde_wait(const hifde_factor_t* f);

/* Thread-local message describing the last non-zero status. */
const char* hifde_last_error(void);

/*
 * Host-only partition hook (no GPU needed): groups of `level_kind`
 * (0 interior, 1 interface-edge, 2 interface-face) at level `ell` over the
 * DOFs with active[i] != 0, in the reference's order
 * (src/partition.py:68-181).  Writes the member DOFs group after group into
 * members[] and the group offsets into offsets[ngroups+1]; returns the number
 * of groups, or -1 if the capacities are too small.
 */
int64_t hifde_partition(int dim, int n_grid, int m_leaf, int ell, int level_kind,
                        const uint8_t* active, int32_t* members, int64_t members_cap,
                        int64_t* offsets, int64_t offsets_cap);

/*
 * Communicators.  Rank 0 creates a unique id (HIFDE_COMM_ID_BYTES bytes) and
 * the caller distributes it; every rank then calls hifde_comm_init with its
 * rank and CUDA device (ncclCommInitRank; libnccl.so.2 is loaded at run time,
 * preferring the copy torch already loaded).  hifde_comm_emulated builds P
 * virtual ranks inside one process on one device (tests: each virtual rank
 * keeps a private block arena, so a missing transfer corrupts the factor).
 */
int hifde_comm_unique_id(uint8_t* id);
int hifde_comm_init(const uint8_t* id, int nranks, int rank, int device, hifde_comm_t** out);
int hifde_comm_emulated(int nranks, int device, hifde_comm_t** out);
/*
 * Host-staged communicator (testing the real-rank path without NCCL, e.g.
 * two processes on one GPU over gloo): the library copies each collective's
 * device data to host buffers and calls
 *   allreduce(ctx, buf, count, dtype (0 int32, 1 uint8, 2 float64), op (0 sum, 1 max, 2 min))
 *   sendrecv(ctx, nsend, send_peer[], send_buf[], send_bytes[], nrecv, recv_peer[], recv_buf[], recv_bytes[])
 * in place; callbacks return 0 on success.
 */
typedef int (*hifde_allreduce_fn)(void* ctx, void* buf, size_t count, int dtype, int op);
typedef int (*hifde_sendrecv_fn)(void* ctx, int nsend, const int* send_peer, void* const* send_buf,
                                 const size_t* send_bytes, int nrecv, const int* recv_peer, void* const* recv_buf,
                                 const size_t* recv_bytes);
int hifde_comm_host(int nranks, int rank, int device, hifde_allreduce_fn allreduce, hifde_sendrecv_fn sendrecv,
                    void* ctx, hifde_comm_t** out);
int hifde_comm_info(const hifde_comm_t* c, int* nranks, int* rank, int* emulated);
void hifde_comm_free(hifde_comm_t* c);
const char* hifde_comm_last_error(void);

/*
 * Host-only sharding hooks (no GPU needed; the CPU multi-process tests):
 * hifde_shard_owner: subdomain rank of each DOF for nranks ranks (boxes split
 * round-robin over the axes by twos).  hifde_shard_plan: the block transfers
 * that make every block listed by a task (task t lists
 * lists[list_ptr[t] .. list_ptr[t+1])) resident on the task's owner, given
 * each block's producer and holders (have[], a bit per rank, updated);
 * out[3i..3i+2] = (src, dst, block) sorted by (src, dst, block).  Returns the
 * number of transfers (out == NULL: count only), -2-count if cap is too small,
 * -1 on bad input.
 */
int hifde_shard_owner(int nranks, int dim, int n_grid, const int32_t* dofs, int64_t count, int32_t* owner);
int64_t hifde_shard_plan(int nranks, int64_t nblocks, const int32_t* producer, uint32_t* have, int64_t ntasks,
                         const int32_t* owner, const int64_t* list_ptr, const int32_t* lists, int32_t* out,
                         int64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* HIFDE_GPU_H */
