// Host runtime of the B200 HIF-DE path: level schedule, symbolic analysis,
// device arenas, kernel orchestration and the C ABI (include/hifde_gpu.h).
//
// Data model: the working matrix A_l is the original stencil
// matrix A0 restricted to the active DOFs plus a set of live dense "clique
// blocks".  An elimination consumes every block touching its cell and emits
// one block over its neighbour set (the Schur update); a skeletonization with
// redundant DOFs emits a delta block over its skeletons.  This reproduces the
// reference's sparsity pattern exactly (src/sparse.py), so neighbour sets,
// partitions and order-dependent steps match the reference.  The host keeps
// only integer structure (DOF lists, block membership); every floating-point
// operation runs in the sm_100a kernels.
//
// Sharding (options.comm, shard.h / comm.h): every rank runs this host
// analysis; a group's kernels run on its owner, consumed blocks are exchanged
// before each level and the state every rank reads is merged after each
// launch; the solve runs each rank's own records, exchanging vector rows.  Exact-order 3D batches queue each large-group tail on a second
// stream so it overlaps the next batch's assembly and ID.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <deque>
#include <exception>
#include <functional>
#include <unordered_map>
#include <thread>
#include <future>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hifde_gpu.h"
#include "hifde_internal.h"
#include "hostprof.h"
#include "partition.h"
#include "comm.h"
#include "shard.h"

#include <omp.h>

namespace hifde {

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;

struct Fail {
  int code;
  std::string msg;
};

#define HCK(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      throw Fail{HIFDE_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)};          \
  } while (0)

constexpr size_t kSmemCap = kSmemCapBytes;

bool trace_on() {
  static const bool on = getenv("HIFDE_TRACE") != nullptr;
  return on;
}
#define HTRACE(...)                                \
  do {                                             \
    if (trace_on()) {                              \
      fprintf(stderr, "[hifde-trace] " __VA_ARGS__); \
      fprintf(stderr, "\n");                       \
      fflush(stderr);                              \
    }                                              \
  } while (0)

double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

size_t align16(size_t x) { return (x + 15) / 16 * 16; }

// Pinned host staging arena for H2D uploads: host data is memcpy'd into it
// and copied with a truly asynchronous cudaMemcpyAsync, so the host never
// waits for the GPU to drain when it uploads the next level's work.  The arena
// is bump-allocated per factorization; if it fills up the stream is drained
// and it is reused.  Kept across factorizations (grown to the peak).
struct PinnedStage {
  char* p = nullptr;
  size_t cap = 0, n = 0, peak = 0;
  size_t failed = SIZE_MAX;  // smallest size a pinned allocation failed at
  cudaStream_t s = nullptr;
  static constexpr size_t kMaxCap = (size_t)256 << 20;  // larger factorizations wrap (drain) instead
  void begin(cudaStream_t st) {
    s = st;
    n = 0;
    // grow only when the last factorization needed more, and then in one
    // step (a pinned allocation runs at ~2.3 GB/s on this host: 256 MB is
    // ~110 ms, so a geometric series of growths costs the repeated calls of
    // a fixed problem twice); a failed size is never retried
    if (peak > cap && cap < kMaxCap) {
      const size_t want = peak > ((size_t)16 << 20) ? kMaxCap : std::min(std::max(4 * peak, 2 * cap), kMaxCap);
      if (want < failed) {
        char* q = nullptr;
        if (cudaHostAlloc((void**)&q, want, cudaHostAllocDefault) == cudaSuccess) {
          if (p) cudaFreeHost(p);
          p = q;
          cap = want;
        } else {
          cudaGetLastError();
          failed = want;
        }
      }
    }
  }
  // returns false when the caller should fall back to a pageable copy
  bool copy(void* dst, const void* src, size_t bytes) {
    const size_t need = (bytes + 255) & ~(size_t)255;
    peak = std::max(peak, n + need);
    if (!p || need > cap) return false;
    if (n + need > cap) {  // full: drain the stream, then reuse from the start
      HCK(cudaStreamSynchronize(s));
      n = 0;
    }
    if (bytes >= (1u << 20)) {  // large uploads: several threads fill the pinned slice
      const int nth = 8;
#pragma omp parallel for num_threads(nth) schedule(static)
      for (int t = 0; t < nth; ++t) {
        const size_t lo = bytes * t / nth, hi = bytes * (t + 1) / nth;
        std::memcpy(p + n + lo, (const char*)src + lo, hi - lo);
      }
    } else {
      std::memcpy(p + n, src, bytes);
    }
    HCK(cudaMemcpyAsync(dst, p + n, bytes, cudaMemcpyHostToDevice, s));
    n += need;
    return true;
  }
};
thread_local PinnedStage* g_stage = nullptr;
PinnedStage& pinned_stage() {
  static PinnedStage ps;
  return ps;
}

// Growable device array with stream-ordered (pooled) allocation.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0, cap = 0;
  void reserve(size_t c, cudaStream_t s) {
    if (c <= cap) return;
    size_t nc = std::max(c, cap + cap / 2 + 4096);
    T* q = nullptr;
    HCK(cudaMallocAsync((void**)&q, nc * sizeof(T), s));
    if (n) HCK(cudaMemcpyAsync(q, p, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (p) HCK(cudaFreeAsync(p, s));
    p = q;
    cap = nc;
  }
  size_t bump(size_t k, cudaStream_t s) {
    reserve(n + k, s);
    size_t off = n;
    n += k;
    return off;
  }
  void upload(const T* h, size_t off, size_t cnt, cudaStream_t s) {
    if (!cnt) return;
    if (g_stage && g_stage->copy(p + off, h, cnt * sizeof(T))) return;
    HCK(cudaMemcpyAsync(p + off, h, cnt * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void release(cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = cap = 0;
  }
};

// Packed-inverse work of a batch of cells (kernels_big.cu): thread-per-column
// for nc <= kInvLocalCols, blocked diagonal-inverse + DMMA tiles above.
struct InvPlan {
  std::vector<int4> loc, diag, tiles;
  std::vector<int64_t> off;  // tiles of panel p: kind 0 [off[2p], off[2p+1]), kind 1 up to off[2p+2]
  DBuf<int4> d_loc, d_diag, d_tiles;
  void build(const std::vector<int>& ncs) {
    int maxnc = 0;
    for (int i = 0; i < (int)ncs.size(); ++i) {
      const int nc = ncs[(size_t)i];
      if (nc <= kInvLocalCols) {
        for (int c0 = 0; c0 < nc; c0 += 128) loc.push_back(make_int4(i, c0, 0, 0));
      } else {
        maxnc = std::max(maxnc, nc);
        for (int p0 = 0; p0 < nc; p0 += kPanelB) diag.push_back(make_int4(i, p0, 0, 0));
      }
    }
    const int np = (maxnc + kPanelB - 1) / kPanelB;
    off.assign((size_t)2 * np + 1, 0);
    for (int p = 0; p < np; ++p) {
      const int p0 = p * kPanelB;
      for (int kind = 0; kind < 2; ++kind) {
        for (int i = 0; i < (int)ncs.size(); ++i) {
          const int nc = ncs[(size_t)i];
          if (nc <= kInvLocalCols || p0 >= nc) continue;
          if (kind == 0) {
            for (int j0 = 0; j0 < p0; j0 += kPanelB) tiles.push_back(make_int4(i, 0, p0, j0));
          } else {
            for (int i0 = p0 + kPanelB; i0 < nc; i0 += kPanelB)
              for (int j0 = 0; j0 <= p0; j0 += kPanelB) tiles.push_back(make_int4(i, 1, i0, j0));
          }
        }
        off[(size_t)2 * p + kind + 1] = (int64_t)tiles.size();
      }
    }
  }
  void upload(cudaStream_t s) {
    for (auto pr : {std::make_pair(&d_loc, &loc), std::make_pair(&d_diag, &diag), std::make_pair(&d_tiles, &tiles)}) {
      pr.first->reserve(pr.second->size(), s);
      pr.first->upload(pr.second->data(), 0, pr.second->size(), s);
    }
  }
  int launch(const ElimTask* tasks, const Arenas& A, cudaStream_t s) {
    int nl = 0;
    if (!loc.empty()) { launch_big_inverse(tasks, d_loc.p, (int)loc.size(), A, s); ++nl; }
    if (!diag.empty()) { launch_inv_diag(tasks, d_diag.p, (int)diag.size(), A, s); ++nl; }
    for (size_t q = 0; q + 1 < off.size(); ++q) {
      const int cnt = (int)(off[q + 1] - off[q]);
      if (cnt == 0) continue;
      launch_inv_tiles(tasks, d_tiles.p + off[q], cnt, (int)(q / 2) * kPanelB, A, s);
      ++nl;
    }
    return nl;
  }
  void release(cudaStream_t s) {
    d_loc.release(s);
    d_diag.release(s);
    d_tiles.release(s);
  }
};

struct LevelRec {
  double tag = 0;
  int kind = 0;  // 0 elimination, 1 skeleton
  int nbatches = 1;
  int64_t ngroups = 0, nskel = 0, nred = 0, active_after = 0, max_front = 0;
  double seconds = 0, gflop = 0, gbytes = 0;
  double gpu_seconds = 0;                 // CUDA-event time of the level's kernels
  double t_part = 0, t_sym = 0, t_upd = 0, t_launch = 0, t_sync = 0;  // host phases
  std::vector<std::pair<const char*, double>> sub;                     // finer host phases (profile)
  double t_lap = 0;
  void lap(const char* what) {
    const double t = now_s();
    if (t_lap > 0) sub.emplace_back(what, t - t_lap);
    t_lap = t;
  }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // solve metadata: records handled one CTA each (recs / d_recs after the
  // split) and the tiled phases of the large records
  std::vector<SolveRec> recs;
  SolveRec* d_recs = nullptr;
  int nsmall = 0;
  SolveRec* d_all = nullptr;  // every record of the level (apply)
  std::vector<hifde_record_t> xrec;  // export view of every record (hifde_level_records)
  hifde_record_t* d_xrec = nullptr;  // device-symbolic levels: the export view on the device (copied on demand)
  int64_t nxrec = 0;
  int dev_stat = -1;                 // device-symbolic levels: index of the level's LevelStat
  int nall = 0, all_max_nc = 0, all_max_nq = 0;
  int max_nc = 0, max_nq = 0;
  struct Phase {
    TileOp* d_ops = nullptr;
    int2* d_work = nullptr;
    int nwork = 0;
  };
  std::vector<Phase> fwd_ph, bwd_ph;
  // elimination forward reduction (targets / CSR of contribution rows)
  int64_t ncontrib = 0;
  int32_t* d_targets = nullptr;
  int64_t* d_ptr = nullptr;
  int64_t* d_ent = nullptr;
  int ntargets = 0;
  // skeleton levels: algorithmic GB / GFLOP of the one-CTA groups [0] and of
  // the large-group pipeline [1] (kernel log)
  double gb_cls[2] = {0, 0}, gf_cls[2] = {0, 0};
  // solve sweep: factor doubles and touched vector rows of the level's records
  double solve_fac = 0, solve_rows = 0;
  // sharded factorization: owner rank of each record of `recs`
  std::vector<uint8_t> rec_own;
  // partitioned solve: the level's records and reduction
  // targets of each rank (real ranks: only this process's entry is filled),
  // and the row exchanges before the forward records [0], before the forward
  // reduction (contribution rows) [1] and before the backward records [2]
  std::vector<LevelRec> rank_view;
  struct XPair {
    int src, dst;
    int64_t off, cnt;  // rows [off, off + cnt) of the step's row list
  };
  struct XStep {
    std::vector<XPair> pairs;
    int32_t* d_rows = nullptr;
  };
  XStep xs[3];
};

// Kernel log (options.kernel_log): CUDA events around the main launches of
// a factorization and of the solves of its factor, with the algorithmic
// bytes / FLOPs of the work each launch covers.  bench.py's
// roofline divides them by the event times (hifde_kernel_stats).
struct KLog {
  struct Entry {
    std::string name;
    double tag;
    int phase;  // 0 factor, 1 solve
    cudaEvent_t e0, e1;
    double gbytes, gflop;
  };
  bool on = false;
  std::vector<Entry> v;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  // returns the entry index, or -1 when the log is off
  int begin(const char* name, double tag, int phase, double gb, double gf, cudaStream_t s) {
    if (!on) return -1;
    Entry E{name, tag, phase, ev(), ev(), gb, gf};
    cudaEventRecord(E.e0, s);
    v.push_back(E);
    return (int)v.size() - 1;
  }
  void end(int i, cudaStream_t s) {
    if (i >= 0) cudaEventRecord(v[(size_t)i].e1, s);
  }
  void clear(int phase) {
    std::vector<Entry> keep;
    for (auto& E : v) {
      if (E.phase == phase) {
        pool.push_back(E.e0);
        pool.push_back(E.e1);
      } else {
        keep.push_back(E);
      }
    }
    v.swap(keep);
  }
  ~KLog() {
    for (auto& E : v) {
      cudaEventDestroy(E.e0);
      cudaEventDestroy(E.e1);
    }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

}  // namespace
}  // namespace hifde

struct hifde_factor {
  int64_t n = 0;
  int dim = 0, variant = 0, spd = 1, device = 0;
  double eps = 0;
  int64_t s_top = 0, m_f_bytes = 0;
  int nranks = 1;           // ranks the factorization was sharded over
  int64_t xfer_bytes = 0;   // block bytes moved between ranks
  double t_f = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  hifde::DBuf<double> fac;
  hifde::DBuf<int32_t> idx;
  std::vector<hifde::LevelRec> levels;  // last entry = terminal block (kind 2)
  int64_t max_contrib = 0;
  int64_t tile_rows = 0;  // solve scratch rows of the tiled phases
  char* meta = nullptr;  // every level's solve metadata (one allocation)
  mutable hifde::KLog klog;  // options.kernel_log (the solve appends its launches)
  // banded host solve (solve_pipelined): per level-0 record, the prefix max
  // of its largest cell DOF and the suffix min of its smallest, built once
  mutable std::mutex band_m;
  mutable bool band_done = false;
  mutable std::vector<int32_t> band_pmax, band_smin;
  std::vector<void*> dev_allocs;  // device-symbolic levels' solve / export tables
  mutable std::mutex klog_m;
  // Partitioned solve of a sharded factorization: every rank
  // runs only its own records; vector rows and contribution rows cross ranks
  // as the per-level plans say (LevelRec::xs).  Real ranks hold only their
  // records' factor values until an operation that needs the whole factor
  // (apply, export, power iteration) sums the arenas once (ensure_whole).
  const hifde_comm* comm = nullptr;  // the factorization's communicator (must outlive the solves)
  bool part = false;                 // partitioned solve plans built
  bool emu = false;                  // virtual ranks in this process
  int me = 0;
  uint8_t* d_holder = nullptr;       // rank holding each solved row after the backward sweep
  hifde::LevelRec::XStep gather;     // emulated: rows of ranks 1.. into rank 0's vector
  mutable bool whole = true;         // factor arena holds every record
  mutable std::mutex whole_m;
  mutable std::atomic<int64_t> solve_xfer_bytes{0};  // vector bytes this rank exchanged in solves
  // options.async_factor: the factorization runs on `worker`; every entry
  // point that reads the factor joins it first (async_done)
  mutable std::thread worker;
  mutable std::mutex async_m;
  int async_status = 0;
  std::string async_err;
  std::atomic<int> inputs_issued{1};  // 0 until the worker has queued its own uploads
  mutable std::atomic<int> async_pending{0};  // 1 from the worker's start to its join
  std::mutex ev_m;
  cudaEvent_t ev_inputs = nullptr;  // the matrix values' upload (while the factorization owns it)
  ~hifde_factor() {
    if (worker.joinable()) worker.join();
    // stream-ordered frees: no device-wide synchronization on release
    cudaSetDevice(device);
    if (meta) cudaFreeAsync(meta, stream);
    for (void* q : dev_allocs) cudaFreeAsync(q, stream);
    if (fac.p) cudaFreeAsync(fac.p, stream);
    if (idx.p) cudaFreeAsync(idx.p, stream);
    if (own_stream && stream) {
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
};

namespace hifde {
namespace {


// Growable array of trivially copyable T whose resize does not initialize
// (the index arena's host mirror is always written before it is read).
template <class T>
struct PodVec {
  std::unique_ptr<T[]> p;
  size_t n = 0, cap = 0;
  T* data() { return p.get(); }
  const T* data() const { return p.get(); }
  size_t size() const { return n; }
  T& operator[](size_t i) { return p[i]; }
  const T& operator[](size_t i) const { return p[i]; }
  void reserve(size_t c) {
    if (c <= cap) return;
    std::unique_ptr<T[]> q(new T[c]);
    if (n) std::memcpy(q.get(), p.get(), n * sizeof(T));
    p.swap(q);
    cap = c;
  }
  void resize(size_t m) {
    if (m > cap) reserve(std::max(m, cap + cap / 2));
    n = m;
  }
  void assign(const T* b, const T* e) {
    resize((size_t)(e - b));
    if (n) std::memcpy(p.get(), b, n * sizeof(T));
  }
  void swap(PodVec& o) {
    p.swap(o.p);
    std::swap(n, o.n);
    std::swap(cap, o.cap);
  }
};

// Solve metadata of a whole factorization packed into one device allocation
// and one asynchronous upload (instead of an allocation + blocking copy each).
struct MetaPack {
  PodVec<char> h;
  std::vector<std::pair<void**, size_t>> slots;
  template <class T>
  void add(T** slot, const std::vector<T>& v) {
    *slot = nullptr;
    if (v.empty()) return;
    const size_t off = (h.size() + 255) & ~(size_t)255;
    h.resize(off + v.size() * sizeof(T));  // PodVec: grows x1.5, no zero fill
    std::memcpy(h.data() + off, v.data(), v.size() * sizeof(T));
    slots.emplace_back((void**)slot, off);
  }
  // returns the device block (owned by the caller)
  char* commit(cudaStream_t s, const std::function<void(void*, const void*, size_t)>& up) {
    if (h.size() == 0) return nullptr;
    char* d = nullptr;
    HCK(cudaMallocAsync((void**)&d, h.size(), s));
    up(d, h.data(), h.size());
    for (auto& sl : slots) *sl.first = d + sl.second;
    return d;
  }
};

// Live clique blocks containing each DOF: up to kInline ids stored inline per
// DOF, the rare overflow in a side table.
struct Membership {
  static constexpr int kInline = 8;
  std::unique_ptr<int32_t[]> ids;
  std::vector<uint8_t> cnt;
  std::vector<std::vector<int32_t>> over;  // overflow lists, pre-sized; slots taken atomically
  std::atomic<int32_t> nover{0};
  std::vector<int32_t> over_slot;          // per DOF, -1 if none
  void init(int64_t n) {
    ids.reset(new int32_t[(size_t)n * kInline]);
    cnt.assign((size_t)n, 0);
    over_slot.assign((size_t)n, -1);
    over.clear();
    over.resize(1024);
    nover = 0;
  }
  // empty every list (storage kept)
  void reset() {
    const int64_t n = (int64_t)cnt.size();
#pragma omp parallel for schedule(static) if (n > (1 << 16))
    for (int64_t i = 0; i < n; ++i) {
      cnt[(size_t)i] = 0;
      over_slot[(size_t)i] = -1;
    }
    const int32_t used = std::min<int32_t>(nover.load(), (int32_t)over.size());
    for (int32_t i = 0; i < used; ++i) over[(size_t)i].clear();
    nover = 0;
  }
  // serial phases only: keep room for the overflow slots a parallel phase may take
  void ensure_room(size_t extra) {
    const size_t need = (size_t)nover.load() + extra;
    if (need > over.size()) over.resize(std::max(need, over.size() * 2));
  }
  // add / remove: safe concurrently for distinct DOFs (after ensure_room)
  void add(int32_t d, int32_t b) {
    uint8_t& c = cnt[(size_t)d];
    if (c < kInline) { ids[(size_t)d * kInline + c] = b; ++c; return; }
    int32_t& sl = over_slot[(size_t)d];
    if (sl < 0) sl = nover.fetch_add(1);
    over[(size_t)sl].push_back(b);
  }
  void remove(int32_t d, int32_t b) {
    int32_t* v = &ids[(size_t)d * kInline];
    uint8_t& c = cnt[(size_t)d];
    for (int i = 0; i < c; ++i)
      if (v[i] == b) {
        const int32_t sl = over_slot[(size_t)d];
        if (sl >= 0 && !over[(size_t)sl].empty()) {  // refill from the overflow
          v[i] = over[(size_t)sl].back();
          over[(size_t)sl].pop_back();
        } else {
          v[i] = v[c - 1];
          --c;
        }
        return;
      }
    const int32_t sl = over_slot[(size_t)d];
    if (sl >= 0) {
      auto& o = over[(size_t)sl];
      auto it = std::find(o.begin(), o.end(), b);
      if (it != o.end()) { *it = o.back(); o.pop_back(); }
    }
  }
  template <class Fn>
  void for_each(int32_t d, Fn&& fn) const {
    const int32_t* v = &ids[(size_t)d * kInline];
    for (int i = 0; i < cnt[(size_t)d]; ++i) fn(v[i]);
    const int32_t sl = over_slot[(size_t)d];
    if (sl >= 0)
      for (int32_t b : over[(size_t)sl]) fn(b);
  }
};

// Host scratch kept across factorizations of the same grid (coordinates,
// per-thread stamp arrays, block membership storage): avoids re-touching
// O(N) memory on every call.  hifde_factor holds g_host_mutex while it runs.
struct HostCache;
HostCache& host_cache();

// Per-thread scratch of the symbolic analysis.
struct SymCtx {
  std::vector<int32_t> dstamp, bstamp;
  int32_t stamp = 0;
  std::vector<int32_t> qbuf, bbuf;  // concatenated outputs of this thread
};

struct HostCache {
  GridDesc g;
  bool valid = false;
  Coords X;
  std::vector<SymCtx> ctx;
  Membership member;
  // arena sizes reached by the last factorization of this grid / variant:
  // reserved up front next time so the arenas do not grow (and copy) mid-run
  int variant = -1;
  size_t hint_fac = 0, hint_bv = 0, hint_idx = 0, hint_scr = 0, hint_meta = 0;
  // pinned host copies of a device-resident CSR pattern (input_on_device):
  // DMA lands in them directly, pages stay resident across factorizations
  struct Pinned {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
      if (bytes <= cap) return p;
      if (p) cudaFreeHost(p);
      cap = bytes + bytes / 8;
      if (cudaHostAlloc(&p, cap, cudaHostAllocDefault) != cudaSuccess) {
        p = nullptr;
        cap = 0;
      }
      return p;
    }
  } pat_ip, pat_ix, wide_ip;  // wide_ip: int64 copy of an int32 indptr (options.indptr_int32)
  // host mirror of the index arena and the solve-metadata staging buffer,
  // lent to each factorization: their pages stay mapped (a fresh multi-100 MB
  // buffer per factorization costs its page faults on first touch)
  PodVec<int32_t> idx_buf;
  PodVec<char> meta_buf;
};
HostCache& host_cache() {
  static HostCache hc;
  return hc;
}
std::mutex g_host_mutex;

struct FrontSym {  // result of the symbolic analysis of one cell / group
  int tid;
  int64_t q_off, b_off;
  int nq, nb, maxnb;
};

// ---------------------------------------------------------------------------
// Factorization state
// ---------------------------------------------------------------------------
// Host <-> device copies of the user's pageable right-hand sides/solutions
// through a persistent pinned double buffer: chunks are copied by several
// host threads into pinned memory while the previous chunk's DMA runs (a
// pageable cudaMemcpy stages through the driver at one thread's memcpy speed).
struct PinnedXfer {
  static constexpr size_t kChunk = 32u << 20;
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int dev = -1;
  std::mutex m;
  bool ready(int device) {
    if (buf[0] && dev == device) return true;
    if (buf[0]) return false;  // bound to another device: fall back to plain copies
    for (int i = 0; i < 2; ++i) {
      if (cudaHostAlloc((void**)&buf[i], kChunk, cudaHostAllocDefault) != cudaSuccess) return false;
      if (cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess) return false;
    }
    dev = device;
    return true;
  }
  // host memory the driver already has page-locked (cudaHostAlloc'ed or
  // registered, e.g. a pinned torch tensor): DMA straight from / into it
  static bool page_locked(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  }
  static int copy_threads() {
    static const int n = std::max(1, std::min(16, omp_get_num_procs()));
    return n;
  }
  static void pmemcpy(char* d, const char* s, size_t n) {
    const int nth = n >= (1u << 20) ? copy_threads() : 1;
#pragma omp parallel for num_threads(nth) schedule(static)
    for (int t = 0; t < nth; ++t) {
      const size_t lo = n * t / nth, hi = n * (t + 1) / nth;
      std::memcpy(d + lo, s + lo, hi - lo);
    }
  }
  void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    int device = 0;
    HCK(cudaGetDevice(&device));
    std::lock_guard<std::mutex> lk(m);
    if (bytes < (1u << 20) || page_locked(src) || !ready(device)) {
      HCK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
      return;
    }
    for (size_t off = 0, c = 0; off < bytes; off += kChunk, ++c) {
      const int b = (int)(c & 1);
      const size_t n = std::min(kChunk, bytes - off);
      HCK(cudaEventSynchronize(ev[b]));  // the slot's previous DMA is done
      pmemcpy(buf[b], (const char*)src + off, n);
      HCK(cudaMemcpyAsync((char*)dst + off, buf[b], n, cudaMemcpyHostToDevice, s));
      HCK(cudaEventRecord(ev[b], s));
    }
    HCK(cudaEventSynchronize(ev[0]));  // the slots may be reused by the next call at once
    HCK(cudaEventSynchronize(ev[1]));
  }
  // Fault in the pages of a fresh pageable destination on all copy threads,
  // one write per 4 KiB page (the caller overwrites the buffer anyway): run
  // while the GPU still computes, the staged copy-out then meets no faults.
  static void prefault(void* dst, size_t bytes) {
    if (bytes < (8u << 20) || page_locked(dst)) return;
    char* d = (char*)dst;
    const int64_t npg = (int64_t)((bytes + 4095) / 4096);
#pragma omp parallel for num_threads(copy_threads()) schedule(static)
    for (int64_t i = 0; i < npg; ++i) d[(size_t)i * 4096] = 0;
  }
  // The column chunks c (device blocks vb[c], N x (c0[c+1] - c0[c]) row-major,
  // complete after their events es[c]) back into the host block x (N x nrhs):
  // row pieces gathered from every chunk by strided DMAs into a pinned slot
  // (whole rows, nrhs wide), copied out contiguously by the host threads
  // while the other slot's DMAs run.
  void d2h_columns(double* x, int nrhs, const std::vector<double*>& vb, const std::vector<int>& c0, int64_t N,
                   const std::vector<cudaEvent_t>& es, cudaStream_t s) {
    if (page_locked(x)) {  // page-locked output: each chunk's columns DMA'd straight into x
      for (size_t c = 0; c + 1 < c0.size(); ++c) {
        const int w = c0[c + 1] - c0[c];
        HCK(cudaStreamWaitEvent(s, es[c], 0));
        HCK(cudaMemcpy2DAsync(x + c0[c], (size_t)nrhs * sizeof(double), vb[c], (size_t)w * sizeof(double),
                              (size_t)w * sizeof(double), (size_t)N, cudaMemcpyDeviceToHost, s));
      }
      return;
    }
    int device = 0;
    HCK(cudaGetDevice(&device));
    std::lock_guard<std::mutex> lk(m);
    if (!ready(device)) throw Fail{HIFDE_CUDA, "pinned staging buffers unavailable"};
    for (const cudaEvent_t e : es) HCK(cudaStreamWaitEvent(s, e, 0));
    const int64_t rows = std::max<int64_t>(1, (int64_t)(kChunk / ((size_t)nrhs * sizeof(double))));
    const int64_t npc = (N + rows - 1) / rows;
    auto issue = [&](int64_t k) {
      const int64_t r0 = k * rows, r1 = std::min(N, r0 + rows);
      for (size_t c = 0; c + 1 < c0.size(); ++c) {
        const int w = c0[c + 1] - c0[c];
        HCK(cudaMemcpy2DAsync((double*)buf[k & 1] + c0[c], (size_t)nrhs * sizeof(double), vb[c] + r0 * w,
                              (size_t)w * sizeof(double), (size_t)w * sizeof(double), (size_t)(r1 - r0),
                              cudaMemcpyDeviceToHost, s));
      }
      HCK(cudaEventRecord(ev[k & 1], s));
    };
    issue(0);
    for (int64_t k = 0; k < npc; ++k) {
      HCK(cudaEventSynchronize(ev[k & 1]));
      if (k + 1 < npc) issue(k + 1);
      const int64_t r0 = k * rows, r1 = std::min(N, r0 + rows);
      pmemcpy((char*)(x + (size_t)r0 * nrhs), buf[k & 1], (size_t)(r1 - r0) * nrhs * sizeof(double));
    }
  }
  void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    int device = 0;
    HCK(cudaGetDevice(&device));
    std::lock_guard<std::mutex> lk(m);
    if (bytes < (1u << 20) || page_locked(dst) || !ready(device)) {
      HCK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
      HCK(cudaStreamSynchronize(s));
      return;
    }
    const size_t nch = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t c) {
      const int b = (int)(c & 1);
      const size_t off = c * kChunk, n = std::min(kChunk, bytes - off);
      HCK(cudaMemcpyAsync(buf[b], (const char*)src + off, n, cudaMemcpyDeviceToHost, s));
      HCK(cudaEventRecord(ev[b], s));
    };
    issue(0);
    for (size_t c = 0; c < nch; ++c) {
      const int b = (int)(c & 1);
      HCK(cudaEventSynchronize(ev[b]));
      if (c + 1 < nch) issue(c + 1);  // the other slot's DMA overlaps this copy-out
      const size_t off = c * kChunk, n = std::min(kChunk, bytes - off);
      pmemcpy((char*)dst + off, buf[b], n);
    }
  }
};
PinnedXfer& pinned_xfer() {
  static PinnedXfer x;
  return x;
}

// Caching allocator of page-locked host blocks for solve/apply outputs
// (hifde_host_alloc / hifde_host_free): the result of a solve is DMA'd
// straight into its pages, and a freed block serves the next request of about
// its size, so neither the pinning nor the first-touch faults of a fresh
// multi-GB host array recur per call.  Free blocks beyond kCacheCap are
// returned to the driver.
struct HostPool {
  static constexpr size_t kGran = (size_t)2 << 20;
  static constexpr size_t kCacheCap = (size_t)16 << 30;
  std::mutex m;
  std::vector<std::pair<size_t, void*>> free_;  // cached blocks, most recently freed last
  std::unordered_map<void*, size_t> live;       // block -> size
  size_t cached = 0;
  void* alloc(size_t bytes) {
    const size_t want = (std::max<size_t>(bytes, 1) + kGran - 1) / kGran * kGran;
    {
      std::lock_guard<std::mutex> lk(m);
      // the most recently freed block that fits without wasting over a quarter
      for (size_t i = free_.size(); i-- > 0;) {
        if (free_[i].first < want || free_[i].first > want + want / 4) continue;
        void* p = free_[i].second;
        live[p] = free_[i].first;
        cached -= free_[i].first;
        free_.erase(free_.begin() + (std::ptrdiff_t)i);
        return p;
      }
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, want, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      trim(0);  // give the cached blocks back and retry once
      if (cudaHostAlloc(&p, want, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
    }
    std::lock_guard<std::mutex> lk(m);
    live[p] = want;
    return p;
  }
  bool release(void* p) {
    std::lock_guard<std::mutex> lk(m);
    auto it = live.find(p);
    if (it == live.end()) return false;
    free_.emplace_back(it->second, p);
    cached += it->second;
    live.erase(it);
    trim_locked(kCacheCap);
    return true;
  }
  void trim_locked(size_t keep) {  // least recently freed blocks go first
    size_t i = 0;
    while (cached > keep && i < free_.size()) {
      cudaFreeHost(free_[i].second);
      cached -= free_[i].first;
      ++i;
    }
    free_.erase(free_.begin(), free_.begin() + (std::ptrdiff_t)i);
  }
  void trim(size_t keep) {
    std::lock_guard<std::mutex> lk(m);
    trim_locked(keep);
  }
};
HostPool& host_pool() {
  static HostPool p;
  return p;
}

// One background host thread per factorization for work that only the solve
// needs (reductions, solve plans): jobs run in order, off the level loop.
struct Helper {
  // Persistent worker (one per process, g_host_mutex serializes factorizations):
  // jobs run in order; wait(seq) blocks until job `seq` has finished.
  std::thread th;
  std::mutex m;
  std::condition_variable cv, cv_done;
  std::deque<std::function<void()>> q;
  uint64_t posted = 0, finished = 0;
  bool started = false, inline_mode = false;
  std::exception_ptr err;
  void ensure_started() {
    if (started) return;
    started = true;
    th = std::thread([this]() {
      for (;;) {
        std::function<void()> job;
        {
          std::unique_lock<std::mutex> lk(m);
          cv.wait(lk, [&]() { return !q.empty(); });
          job = std::move(q.front());
          q.pop_front();
        }
        if (!job) return;  // shutdown
        try {
          job();
        } catch (...) {
          std::lock_guard<std::mutex> lk(m);
          if (!err) err = std::current_exception();
        }
        {
          std::lock_guard<std::mutex> lk(m);
          ++finished;
        }
        cv_done.notify_all();
      }
    });
  }
  uint64_t post(std::function<void()> job) {
    if (inline_mode) { job(); return 0; }
    ensure_started();
    uint64_t id;
    {
      std::lock_guard<std::mutex> lk(m);
      q.push_back(std::move(job));
      id = ++posted;
    }
    cv.notify_one();
    return id;
  }
  void wait(uint64_t id) {
    if (inline_mode || id == 0) return;
    std::unique_lock<std::mutex> lk(m);
    cv_done.wait(lk, [&]() { return finished >= id; });
  }
  void drain() {  // every posted job finished; rethrow (and clear) the first failure
    uint64_t id;
    {
      std::lock_guard<std::mutex> lk(m);
      id = posted;
    }
    wait(id);
    std::exception_ptr e;
    {
      std::lock_guard<std::mutex> lk(m);
      e = err;
      err = nullptr;
    }
    if (e) std::rethrow_exception(e);
  }
  ~Helper() {
    if (!started) return;
    {
      std::lock_guard<std::mutex> lk(m);
      q.push_back(nullptr);
    }
    cv.notify_one();
    th.join();
  }
};
Helper& helper_thread() {
  static Helper h;
  return h;
}

struct Factorizer {
  // host CSR upload in flight on the helper thread: the pattern (which the
  // symbolic analysis needs) first, then the values on their own copy
  // stream (needed by the numeric kernels only), overlapping the level-0
  // analysis
  uint64_t a0_job = 0, a0_pat_job = 0;
  cudaError_t a0_err = cudaSuccess;
  cudaStream_t a0_s = nullptr;
  cudaEvent_t ev_a0 = nullptr;  // the values' copy is done (device-side wait)
  void a0_pattern_ready() {
    if (a0_pat_job) {
      helper.wait(a0_pat_job);
      a0_pat_job = 0;
    }
  }
  void a0_ready() {
    a0_pattern_ready();
    if (a0_job) {  // the copy is issued (and, from pageable memory, done): the stream waits for it
      helper.wait(a0_job);
      a0_job = 0;
      if (a0_err == cudaSuccess && ev_a0) HCK(cudaStreamWaitEvent(s, ev_a0, 0));
    }
    if (a0_err != cudaSuccess) {
      const cudaError_t e = a0_err;
      a0_err = cudaSuccess;
      throw Fail{HIFDE_CUDA, std::string("A0 upload: ") + cudaGetErrorString(e)};
    }
  }
  ~Factorizer() {
    // jobs capture this factorizer: none may outlive it (also on error paths)
    try {
      helper.drain();
    } catch (...) {
    }
    // a failed factorization (IndefiniteBlockError, CUDA error, ...) leaves
    // its working buffers here: free them so a caller that retries does not
    // run out of HBM
    release_all();
    if (tail_s) {
      cudaStreamSynchronize(tail_s);
      cudaStreamDestroy(tail_s);
      cudaEventDestroy(ev_id);
      cudaEventDestroy(ev_tail);
      cudaEventDestroy(ev_inv);
    }
    if (a0_s) {
      cudaStreamSynchronize(a0_s);
      cudaStreamDestroy(a0_s);
      if (F) {
        std::lock_guard<std::mutex> lk(F->ev_m);
        F->ev_inputs = nullptr;
      }
      if (ev_a0) cudaEventDestroy(ev_a0);
    }
    if (pat_s) {
      cudaStreamSynchronize(pat_s);
      cudaStreamDestroy(pat_s);
      cudaEventDestroy(ev_pat);
    }
    if (sym_s) {
      cudaStreamSynchronize(sym_s);
      cudaStreamDestroy(sym_s);
      cudaStreamSynchronize(sym_hi);
      cudaStreamDestroy(sym_hi);
      cudaEventDestroy(ev_symdone);
      cudaEventDestroy(ev_symjoin);
    }
  }
  // Frees every working buffer of the factorization (stream-ordered) and
  // hands the borrowed host buffers back to the cache; idempotent.
  bool released = false;
  void release_all() {
    if (released) return;
    released = true;
    if (pat_pending) {  // (not pat_wait: release_all also runs on error paths and must not throw)
      pat_pending = false;
      cudaEventSynchronize(ev_pat);
    }
    if (tail_s) join_inv();  // the deferred inverses read buffers freed here
    if (borrowed) {
      HostCache& hc = host_cache();
      hc.idx_buf.swap(h_idx);
      hc.meta_buf.swap(meta.h);
      borrowed = false;
    }
    bvals.release(s);
    for (auto& l : lanes) l.release(s);
    for (auto* d : {&xsend, &xrecv}) d->release(s);
    xseg.release(s);
    xiseg.release(s);
    xret.release(s);
    xi32.release(s);
    agree.release(s);
    gpart.release(s);
    scratch.release(s);
    lists.release(s);
    lists_alt.release(s);
    status.release(s);
    kout.release(s);
    iscratch.release(s);
    d_blk_dof_off.release(s);
    d_blk_n.release(s);
    d_blk_val_off.release(s);
    if (own_a0) {
      if (d_indptr) cudaFreeAsync(d_indptr, s);
      if (d_indices) cudaFreeAsync(d_indices, s);
      if (d_a0) cudaFreeAsync(d_a0, s);
      d_indptr = nullptr;
      d_indices = nullptr;
      d_a0 = nullptr;
      own_a0 = false;
    }
    if (d_active) cudaFreeAsync(d_active, s);
    d_active = nullptr;
    dev_release();
    for (auto& L : F ? F->levels : no_levels) {  // a failed run leaves level events behind
      if (L.ev0) cudaEventDestroy(L.ev0);
      if (L.ev1) cudaEventDestroy(L.ev1);
      L.ev0 = L.ev1 = nullptr;
    }
  }
  bool borrowed = false;
  std::vector<LevelRec> no_levels;
  LevelRec prof;  // setup / finish phase timings
  MetaPack meta;  // solve metadata, uploaded once at the end
  size_t meta_bytes = 0;
  GridDesc g;
  hifde_options_t opt;
  hifde_factor_t* F = nullptr;
  hifde_factor_t* F_ = nullptr;  // alias used by the solve planner
  cudaStream_t s = nullptr;
  int64_t N;
  // A0 (host + device); the host pattern aliases the caller's arrays when
  // they are host arrays
  std::vector<int64_t> indptr_own;
  std::vector<int32_t> indices_own;
  const int64_t* indptr = nullptr;
  const int32_t* indices = nullptr;
  Coords& X = host_cache().X;
  std::vector<int32_t> act;  // ascending active DOFs
  std::vector<SymCtx>& ctx = host_cache().ctx;
  int nthreads = 1;
  int64_t* d_indptr = nullptr;
  int32_t* d_indices = nullptr;
  double* d_a0 = nullptr;
  bool own_a0 = false;
  // activity
  std::vector<uint8_t> active;
  uint8_t* d_active = nullptr;
  // idx arena host mirror
  PodVec<int32_t> h_idx;  // host mirror of the index arena (grows without zero-filling)
  // block table
  std::vector<int64_t> blk_dof_off;
  std::vector<int32_t> blk_n;
  std::vector<int64_t> blk_val_off;
  std::vector<uint8_t> blk_alive;
  DBuf<int64_t> d_blk_dof_off;
  DBuf<int32_t> d_blk_n;
  DBuf<int64_t> d_blk_val_off;
  size_t blk_uploaded = 0;
  Membership& member = host_cache().member;
  DBuf<double> bvals;
  DBuf<double> scratch;
  DBuf<int32_t> lists;
  DBuf<int> status;
  DBuf<int32_t> kout;
  DBuf<int32_t> iscratch;
  // stamps (serial paths)
  int64_t stamp = 0;
  // block-foreign cache for adaptive partitioning
  std::vector<int64_t> bf_key;
  std::vector<uint8_t> bf_val;
  int64_t bf_epoch = 0;
  size_t idx_uploaded = 0;

  // --- sharding over ranks (opt.comm, shard.h) -------------------------------
  // Every rank runs this host analysis identically; a group's kernels run on
  // its owner only.  Real ranks (NCCL): the blocks a rank's groups consume
  // from other ranks arrive before the launch; after each launch the ranks
  // and sk/rd lists are merged by all-reduces over the level's slices (max
  // over slices the non-owners left at 0) and every rank retires the other
  // ranks' DOFs in its own active mask.  Each rank keeps only its records'
  // factor values: the solve is partitioned the same way (build_shard_solve).
  // Emulated ranks: one process launches every virtual rank's groups with
  // that rank's private block arena.
  const hifde_comm* comm = nullptr;
  int P = 1, me = 0;
  bool emu = false, real = false;
  ShardGeom geom;
  BlockLedger ledger;
  std::vector<DBuf<double>> lanes;  // emulated: block arenas of virtual ranks 1..P-1 (rank 0: bvals)
  DBuf<double> xsend, xrecv;        // packed block transfers
  DBuf<int64_t> xseg;               // segment tables of the packs
  DBuf<int> agree;                  // status agreement scalar
  DBuf<double> gpart;               // split-tile partials of the Gram matrices
  std::vector<uint8_t> own_;        // owner rank per group of the current level
  // Large-group pipelines: the tail of a batch (T, congruence, inner
  // elimination, inverse) runs on a second stream while the next batch's
  // assembly and ID proceed on the main one -- the next batch depends only on
  // the ranks and the retired rows, not on the tail.
  cudaStream_t tail_s = nullptr;
  cudaEvent_t ev_id = nullptr, ev_tail = nullptr;
  // Device symbolic of a skeleton level overlapped with the numeric kernels
  // of the elimination level before it (structure only: partition, fronts,
  // tables -- nothing of the factor's values): run on sym_s after
  // ev_symdone (the elimination's symbolic fill and cell retirement), joined
  // back into the main stream before the level's numeric launches.
  cudaStream_t sym_s = nullptr;
  cudaEvent_t ev_symdone = nullptr, ev_symjoin = nullptr;
  bool symdone_ok = false;
  DBuf<int32_t> lists_alt;  // the skeleton symbolic's block lists while the elimination reads `lists`
  // The overlapped analysis runs on a high-priority stream (sym_hi swapped
  // in at the first overlap): it is a chain of ~40 small launches with a
  // readback in the middle, and at normal priority its CTAs queue behind the
  // elimination's (config 3: the level-0.5 analysis then ran in the tail of
  // the level-0 elimination, 1.1 ms of mostly idle SMs; at high priority it
  // ends 3 ms before the elimination does and the pair takes 0.3 ms less).
  cudaStream_t sym_hi = nullptr;
  int sym_overlaps = 0;
  // Device-resident input: the host copy of the CSR pattern is only read by
  // the host analysis.  While the device symbolic pass runs the levels the
  // copy (117 MB on config 3: 2.1 ms of a 41 ms factorization when waited for
  // up front) goes over a copy engine on its own stream; the hand-over to the
  // host analysis and the end of the run wait for it.
  cudaStream_t pat_s = nullptr;
  cudaEvent_t ev_pat = nullptr;
  bool pat_pending = false;
  void pat_wait() {
    if (!pat_pending) return;
    pat_pending = false;
    HCK(cudaEventSynchronize(ev_pat));
  }
  cudaStream_t sym_stream() {
    if (!sym_s) {
      int lo = 0, hi = 0;
      HCK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      HCK(cudaStreamCreateWithFlags(&sym_s, cudaStreamNonBlocking));
      HCK(cudaStreamCreateWithPriority(&sym_hi, cudaStreamNonBlocking, hi));
      HCK(cudaEventCreateWithFlags(&ev_symdone, cudaEventDisableTiming));
      HCK(cudaEventCreateWithFlags(&ev_symjoin, cudaEventDisableTiming));
    }
    return sym_s;
  }
  bool tail_pending = false;
  cudaStream_t tail_stream() {
    if (!tail_s) {
      HCK(cudaStreamCreateWithFlags(&tail_s, cudaStreamNonBlocking));
      HCK(cudaEventCreateWithFlags(&ev_id, cudaEventDisableTiming));
      HCK(cudaEventCreateWithFlags(&ev_tail, cudaEventDisableTiming));
      HCK(cudaEventCreateWithFlags(&ev_inv, cudaEventDisableTiming));
    }
    return tail_s;
  }
  // Packed inverses of a device elimination level's blocked cells run on the
  // tail stream (only the solve reads them), under the next skeleton level;
  // joined before anything they read or write can move: the next
  // elimination's analysis (it rewrites the big-cell task table), a growth of
  // the factor or status arenas, the hand-over to the host, the end.
  cudaEvent_t ev_inv = nullptr;
  bool inv_pending = false;
  void join_inv() {
    if (!inv_pending) return;
    HCK(cudaEventRecord(ev_inv, tail_s));
    HCK(cudaStreamWaitEvent(s, ev_inv, 0));
    inv_pending = false;
  }
  // main stream waits for every tail issued so far
  void join_tails() {
    if (!tail_pending || !tail_s) return;
    HCK(cudaEventRecord(ev_tail, tail_s));
    HCK(cudaStreamWaitEvent(s, ev_tail, 0));
    tail_pending = false;
  }
  int64_t xfer_blocks = 0, xfer_bytes = 0;  // totals (metrics)

  bool sharded() const { return comm != nullptr && P > 1; }
  // ranks whose groups this process launches: all (unsharded / emulated) or its own
  int rank_lo() const { return sharded() && !emu ? me : 0; }
  int rank_hi() const { return sharded() && !emu ? me + 1 : (sharded() ? P : 1); }
  DBuf<double>& bv_of(int r) { return (emu && r > 0) ? lanes[(size_t)r - 1] : bvals; }
  Arenas arenas_for(int r) {
    Arenas A = arenas();
    A.bvals = bv_of(r).p;
    return A;
  }
  // owner of a group: the subdomain box of its first DOF
  uint8_t owner_of(const int32_t* c) const { return sharded() ? (uint8_t)shard_owner(geom, X, c[0]) : 0; }
  // after a bump of the block arena: the emulated lanes follow its size, and
  // the new region of every virtual rank is NaN until its producer writes it
  void bvals_grown(size_t old_n) {
    if (!emu || bvals.n == old_n) return;
    const size_t add = bvals.n - old_n;
    for (auto& l : lanes) {
      l.reserve(bvals.n, s);
      l.n = bvals.n;
      HCK(cudaMemsetAsync(l.p + old_n, 0xFF, add * sizeof(double), s));
    }
    HCK(cudaMemsetAsync(bvals.p + old_n, 0xFF, add * sizeof(double), s));
  }
  // real ranks: non-owners must contribute zeros to the final factor sum
  void fac_grown(size_t off, size_t cnt) {
    if (real && cnt) HCK(cudaMemsetAsync(F->fac.p + off, 0, cnt * sizeof(double), s));
  }
  // Real ranks: merge the ranks kout[0, nk) and the index-arena regions
  // [off[i], off[i] + len[i]) (sk/rd lists, zero on non-owners: packed,
  // max-reduced, scattered back), then retire every region's DOFs past its
  // rank kout[kid[i]] (kid == nullptr: cells, all of them) in the local active
  // mask -- the owners' kernels retired theirs already; no rank exchanges the
  // N-byte mask.
  DBuf<int32_t> xi32;
  DBuf<int64_t> xiseg, xret;
  void union_state(const int64_t* off, const int* len, const int32_t* kid, int nreg, int64_t nk) {
    if (!real) return;
    try {
      if (nk > 0) comm_allreduce(comm, kout.p, (size_t)nk, kI32, kMax, s);
      if (nreg > 0 && kid) {
        std::vector<int64_t> seg((size_t)3 * nreg);
        int64_t tot = 0;
        for (int i = 0; i < nreg; ++i) {
          seg[(size_t)i] = off[i];
          seg[(size_t)nreg + i] = tot;
          seg[(size_t)2 * nreg + i] = len[i];
          tot += len[i];
        }
        if (tot > 0) {
          xiseg.reserve(seg.size(), s);
          xiseg.upload(seg.data(), 0, seg.size(), s);
          xi32.reserve((size_t)tot, s);
          launch_seg_copy_i32(F->idx.p, xi32.p, xiseg.p, xiseg.p + nreg, xiseg.p + 2 * nreg, nreg, s);
          comm_allreduce(comm, xi32.p, (size_t)tot, kI32, kMax, s);
          launch_seg_copy_i32(xi32.p, F->idx.p, xiseg.p + nreg, xiseg.p, xiseg.p + 2 * nreg, nreg, s);
          g_launches += 2;
        }
      }
      if (nreg > 0) {
        std::vector<int64_t> ret((size_t)3 * nreg);
        for (int i = 0; i < nreg; ++i) {
          ret[(size_t)i] = off[i];
          ret[(size_t)nreg + i] = len[i];
          ret[(size_t)2 * nreg + i] = kid ? kid[i] : -1;
        }
        xret.reserve(ret.size(), s);
        xret.upload(ret.data(), 0, ret.size(), s);
        launch_retire_regions(F->idx.p, xret.p, xret.p + nreg, xret.p + 2 * nreg, kout.p, nreg, d_active, s);
        ++g_launches;
      }
    } catch (const std::exception& e) {
      throw Fail{HIFDE_CUDA, e.what()};
    }
  }
  void union_level(const std::vector<SkelTask>& tasks, int64_t nt) {
    if (!real) return;
    std::vector<int64_t> off((size_t)nt);
    std::vector<int> len((size_t)nt);
    std::vector<int32_t> kid((size_t)nt);
    for (int64_t t = 0; t < nt; ++t) {
      off[(size_t)t] = tasks[(size_t)t].out_off;
      len[(size_t)t] = tasks[(size_t)t].nc;
      kid[(size_t)t] = (int32_t)t;
    }
    union_state(off.data(), len.data(), kid.data(), (int)nt, nt);
  }
  // Make every block listed by the tasks resident on the task's owner.
  void exchange_blocks(int64_t nt, const uint8_t* owner, const int64_t* ptr, const int32_t* cnt,
                       const int32_t* lists) {
    if (!sharded()) return;
    std::vector<Xfer> xf;
    ledger.plan(nt, owner, ptr, cnt, lists, xf);
    if (xf.empty()) return;
    // pairs in plan order; blocks packed contiguously per pair in block order
    struct Pair {
      int src, dst;
      size_t lo, hi;  // xf range
      int64_t doubles;
    };
    std::vector<Pair> pairs;
    for (size_t i = 0; i < xf.size(); ++i) {
      const int64_t nb = blk_n[(size_t)xf[i].blk];
      if (pairs.empty() || pairs.back().src != xf[i].src || pairs.back().dst != xf[i].dst)
        pairs.push_back(Pair{xf[i].src, xf[i].dst, i, i, 0});
      pairs.back().hi = i + 1;
      pairs.back().doubles += nb * nb;
    }
    for (const Xfer& x : xf) {
      const int64_t nb = blk_n[(size_t)x.blk];
      ++xfer_blocks;
      xfer_bytes += 8 * nb * nb;
    }
    // segment table: (src_off, dst_off, len) triples, one table per launch
    std::vector<int64_t> seg;
    auto pack_table = [&](const Pair& p, bool pack, int64_t base) {
      const size_t n0 = seg.size();
      const size_t cnt_seg = p.hi - p.lo;
      seg.resize(n0 + 3 * cnt_seg);
      int64_t o = base;
      for (size_t i = p.lo; i < p.hi; ++i) {
        const int32_t b = xf[i].blk;
        const int64_t len = (int64_t)blk_n[(size_t)b] * blk_n[(size_t)b];
        const size_t j = i - p.lo;
        seg[n0 + j] = pack ? blk_val_off[(size_t)b] : o;
        seg[n0 + cnt_seg + j] = pack ? o : blk_val_off[(size_t)b];
        seg[n0 + 2 * cnt_seg + j] = len;
        o += len;
      }
      return n0;
    };
    if (emu) {
      for (const Pair& p : pairs) {
        seg.clear();
        xsend.reserve((size_t)p.doubles, s);
        const size_t a = pack_table(p, true, 0);
        const size_t b = pack_table(p, false, 0);
        xseg.reserve(seg.size(), s);
        xseg.upload(seg.data(), 0, seg.size(), s);
        const int ns = (int)(p.hi - p.lo);
        launch_seg_copy(bv_of(p.src).p, xsend.p, xseg.p + a, xseg.p + a + ns, xseg.p + a + 2 * ns, ns, s);
        launch_seg_copy(xsend.p, bv_of(p.dst).p, xseg.p + b, xseg.p + b + ns, xseg.p + b + 2 * ns, ns, s);
        g_launches += 2;
        // the staging buffer is reused by the next pair: keep the stream order
      }
      return;
    }
    int64_t nsend = 0, nrecv = 0;
    for (const Pair& p : pairs) {
      if (p.src == me) nsend += p.doubles;
      if (p.dst == me) nrecv += p.doubles;
    }
    xsend.reserve((size_t)std::max<int64_t>(nsend, 1), s);
    xrecv.reserve((size_t)std::max<int64_t>(nrecv, 1), s);
    std::vector<P2P> sends, recvs;
    std::vector<std::pair<size_t, int>> packs, unpacks;  // (table offset, segments)
    int64_t so = 0, ro = 0;
    for (const Pair& p : pairs) {
      const int ns = (int)(p.hi - p.lo);
      if (p.src == me) {
        packs.emplace_back(pack_table(p, true, so), ns);
        sends.push_back(P2P{p.dst, xsend.p + so, (size_t)p.doubles * sizeof(double)});
        so += p.doubles;
      }
      if (p.dst == me) {
        unpacks.emplace_back(pack_table(p, false, ro), ns);
        recvs.push_back(P2P{p.src, xrecv.p + ro, (size_t)p.doubles * sizeof(double)});
        ro += p.doubles;
      }
    }
    if (seg.empty()) return;
    xseg.reserve(seg.size(), s);
    xseg.upload(seg.data(), 0, seg.size(), s);
    for (auto& pk : packs) {
      const int64_t* t = xseg.p + pk.first;
      launch_seg_copy(bvals.p, xsend.p, t, t + pk.second, t + 2 * pk.second, pk.second, s);
      ++g_launches;
    }
    try {
      comm_sendrecv(comm, sends.data(), (int)sends.size(), recvs.data(), (int)recvs.size(), s);
    } catch (const std::exception& e) {
      throw Fail{HIFDE_CUDA, e.what()};
    }
    for (auto& up : unpacks) {
      const int64_t* t = xseg.p + up.first;
      launch_seg_copy(xrecv.p, bvals.p, t, t + up.second, t + 2 * up.second, up.second, s);
      ++g_launches;
    }
  }

  void upload_idx() {
    F->idx.reserve(h_idx.size(), s);
    F->idx.n = h_idx.size();
    F->idx.upload(h_idx.data() + idx_uploaded, idx_uploaded, h_idx.size() - idx_uploaded, s);
    idx_uploaded = h_idx.size();
  }
  void upload_blocks() {
    size_t nb = blk_n.size();
    if (nb == blk_uploaded) return;
    d_blk_dof_off.reserve(nb, s);
    d_blk_n.reserve(nb, s);
    d_blk_val_off.reserve(nb, s);
    d_blk_dof_off.upload(blk_dof_off.data() + blk_uploaded, blk_uploaded, nb - blk_uploaded, s);
    d_blk_n.upload(blk_n.data() + blk_uploaded, blk_uploaded, nb - blk_uploaded, s);
    d_blk_val_off.upload(blk_val_off.data() + blk_uploaded, blk_uploaded, nb - blk_uploaded, s);
    d_blk_dof_off.n = d_blk_n.n = d_blk_val_off.n = nb;
    blk_uploaded = nb;
  }
  Arenas arenas() {
    a0_ready();  // every launch site takes its arenas here
    Arenas A;
    A.indptr = d_indptr;
    A.indices = d_indices;
    A.a0 = d_a0;
    A.idx = F->idx.p;
    A.lists = lists.p;
    A.blk_dof_off = d_blk_dof_off.p;
    A.blk_n = d_blk_n.p;
    A.blk_val_off = d_blk_val_off.p;
    A.bvals = bvals.p;
    A.fac = F->fac.p;
    A.scratch = scratch.p;
    A.active = d_active;
    A.status = status.p;
    A.kout = kout.p;
    A.iscratch = iscratch.p;
    A.tlog = nullptr;
    return A;
  }

  // block table entry only (membership updated by the caller)
  int32_t new_block(int64_t dof_off, int32_t nb, int64_t val_off, int producer) {
    int32_t id = (int32_t)blk_n.size();
    if (sharded()) ledger.add(id, producer);
    blk_dof_off.push_back(dof_off);
    blk_n.push_back(nb);
    blk_val_off.push_back(val_off);
    blk_alive.push_back(1);
    bf_key.push_back(-2);
    bf_val.push_back(0);
    return id;
  }
  void kill_block(int32_t b) {
    blk_alive[(size_t)b] = 0;
    const int32_t* d = h_idx.data() + blk_dof_off[(size_t)b];
    for (int32_t i = 0; i < blk_n[(size_t)b]; ++i) member.remove(d[i], b);
  }

  // Neighbour set q of the group c and the live blocks touching c
  // (src/sparse.py:164-173 on the clique representation), appended to the
  // thread's buffers.
  FrontSym front_sym(SymCtx& x, int tid, const int32_t* c, int nc) {
    if (x.stamp > INT32_MAX - 4) {
      std::fill(x.dstamp.begin(), x.dstamp.end(), 0);
      std::fill(x.bstamp.begin(), x.bstamp.end(), 0);
      x.stamp = 0;
    }
    const int32_t tc = ++x.stamp;
    const int32_t tq = ++x.stamp;
    FrontSym r;
    r.tid = tid;
    r.q_off = (int64_t)x.qbuf.size();
    r.b_off = (int64_t)x.bbuf.size();
    for (int i = 0; i < nc; ++i) x.dstamp[(size_t)c[i]] = tc;
    for (int i = 0; i < nc; ++i)
      member.for_each(c[i], [&](int32_t b) {
        if (x.bstamp[(size_t)b] != tq) {
          x.bstamp[(size_t)b] = tq;
          x.bbuf.push_back(b);
        }
      });
    std::sort(x.bbuf.begin() + r.b_off, x.bbuf.end());
    int maxnb = 0;
    auto consider = [&](int32_t d) {
      int32_t& st = x.dstamp[(size_t)d];
      if (st != tc && st != tq && active[(size_t)d]) {
        st = tq;
        x.qbuf.push_back(d);
      }
    };
    for (int64_t j = r.b_off; j < (int64_t)x.bbuf.size(); ++j) {
      const int32_t b = x.bbuf[(size_t)j];
      const int32_t* d = h_idx.data() + blk_dof_off[(size_t)b];
      maxnb = std::max(maxnb, blk_n[(size_t)b]);
      for (int32_t i = 0; i < blk_n[(size_t)b]; ++i) consider(d[i]);
    }
    for (int i = 0; i < nc; ++i)
      for (int64_t k = indptr[c[i]]; k < indptr[c[i] + 1]; ++k) consider(indices[k]);
    std::sort(x.qbuf.begin() + r.q_off, x.qbuf.end());
    r.nq = (int)((int64_t)x.qbuf.size() - r.q_off);
    r.nb = (int)((int64_t)x.bbuf.size() - r.b_off);
    r.maxnb = maxnb;
    return r;
  }

  // Symbolic analysis of every group of a level, in parallel over groups.
  std::vector<FrontSym> fronts(const Groups& gr) {
    const int64_t nt = gr.size();
    std::vector<FrontSym> out((size_t)nt);
    for (auto& x : ctx) {
      x.qbuf.clear();
      x.bbuf.clear();
      if (x.bstamp.size() < blk_n.size()) x.bstamp.resize(blk_n.size() + blk_n.size() / 2 + 1024, 0);
    }
    // few large groups (coarse levels) are worth threads too: weight by size
    int64_t work = 0;
    for (int64_t t = 0; t < nt; ++t) work += gr.count(t);
    const int nthr = (nt >= 8 && work >= 4096) ? (int)std::min<int64_t>(nthreads, nt) : 1;
    const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(32, nt / (4 * std::max(nthr, 1))));
#pragma omp parallel for num_threads(nthr) schedule(dynamic, chunk)
    for (int64_t t = 0; t < nt; ++t) {
      const int tid = omp_get_thread_num();
      out[(size_t)t] = front_sym(ctx[(size_t)tid], tid, gr.begin(t), gr.count(t));
    }
    return out;
  }
  const int32_t* sym_q(const FrontSym& f) const { return ctx[(size_t)f.tid].qbuf.data() + f.q_off; }
  const int32_t* sym_b(const FrontSym& f) const { return ctx[(size_t)f.tid].bbuf.data() + f.b_off; }

  // cells of an elimination level must not interact (assert_noninteracting,
  // src/partition.py:230-241)
  void check_noninteracting(const Groups& gr, double tag) {
    std::vector<int64_t> cell_of((size_t)N, -1);
    for (int64_t gi = 0; gi < gr.size(); ++gi)
      for (int i = 0; i < gr.count(gi); ++i) cell_of[(size_t)gr.begin(gi)[i]] = gi;
    std::vector<FrontSym> fs = fronts(gr);
    for (int64_t gi = 0; gi < gr.size(); ++gi) {
      const int32_t* q = sym_q(fs[(size_t)gi]);
      for (int i = 0; i < fs[(size_t)gi].nq; ++i)
        if (cell_of[(size_t)q[i]] >= 0 && cell_of[(size_t)q[i]] != gi) {
          char buf[128];
          snprintf(buf, sizeof buf, "cells interact at level %g", tag);
          throw Fail{HIFDE_INTERNAL, buf};
        }
    }
  }

  struct Pending {
    int64_t off, cnt;
    double tag;
    const char* what;
  };
  std::vector<Pending> pending;
  size_t status_checked = 0;
  // Per-task status words of every launch since the last check: one D2H copy
  // at the next synchronization point (no extra stream syncs per level).
  void check_status() {
    int code = 0;
    std::string msg;
    if (status.n != status_checked) {
      const size_t cnt = status.n - status_checked;
      std::vector<int> st(cnt);
      HCK(cudaMemcpyAsync(st.data(), status.p + status_checked, cnt * sizeof(int), cudaMemcpyDeviceToHost, s));
      HCK(cudaStreamSynchronize(s));
      for (const Pending& P : pending) {
        for (int64_t i = 0; i < P.cnt && !code; ++i) {
          const int v = st[(size_t)(P.off - (int64_t)status_checked + i)];
          if (v != 0) {
            char buf[256];
            const char* kind = v == 1 ? "matrix is not positive definite" : "singular pivot";
            snprintf(buf, sizeof buf, "%s (%s %lld of level %g)", kind, P.what, (long long)i, P.tag);
            code = v == 1 ? HIFDE_INDEFINITE : HIFDE_SINGULAR;
            msg = buf;
          }
        }
        if (code) break;
      }
    }
    status_checked = status.n;
    pending.clear();
    if (real) {  // every rank reaches this point: agree on the outcome
      agree.reserve(1, s);
      HCK(cudaMemcpyAsync(agree.p, &code, sizeof(int), cudaMemcpyHostToDevice, s));
      try {
        comm_allreduce(comm, agree.p, 1, kI32, kMax, s);
      } catch (const std::exception& e) {
        throw Fail{HIFDE_CUDA, e.what()};
      }
      int all = 0;
      HCK(cudaMemcpyAsync(&all, agree.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      HCK(cudaStreamSynchronize(s));
      if (all && !code) {
        code = all;
        msg = "factorization failed on another rank";
      }
    }
    if (code) throw Fail{code, msg};
  }

  // -------------------------------------------------------------------------
  void elimination_level(const Groups& gr, double tag, LevelRec& L, bool is_top) {
    HTRACE("elim level %g: %lld cells", tag, (long long)gr.size());
    const double t_begin = now_s();
    const int64_t nt = gr.size();
    L.kind = is_top ? 2 : 0;
    L.ngroups = nt;
    std::vector<ElimTask> tasks((size_t)nt);
    std::vector<uint8_t> is_big((size_t)nt, 0);
    std::vector<int32_t> hl;  // block lists of this level
    size_t smem_small = 0, smem_big = 0;
    int max_small_nf = 0;
    scratch.n = 0;
    L.lap(nullptr);
    const std::vector<FrontSym> fs = fronts(gr);
    L.lap("fronts");
    // sizes and placement per cell (parallel), offsets (prefix), fill (parallel)
    std::vector<size_t> smem_need((size_t)nt, 0);
    const int nthr = nt >= 256 ? nthreads : 1;
#pragma omp parallel for num_threads(nthr) schedule(static)
    for (int64_t t = 0; t < nt; ++t) {
      const int nc = gr.count(t);
      const FrontSym& f = fs[(size_t)t];
      const int nq = f.nq, nf = nc + nq;
      ElimTask& T = tasks[(size_t)t];
      T.nc = nc;
      T.nq = nq;
      T.nblk = f.nb;
      T.maxnb = f.maxnb;
      (void)nf;
      const ElimSizes z = elim_sizes(nc, nq, T.maxnb, is_top);  // -2: room for the inverse workspace too
      T.scratch_off = z.scratch_off;
      is_big[(size_t)t] = (uint8_t)z.big;
      smem_need[(size_t)t] = z.smem;
    }
    int64_t idx_tot = 0, hl_tot = 0;
    size_t fac_tot = 0, bv_tot = 0;
    L.recs.resize((size_t)nt);
    for (int64_t t = 0; t < nt; ++t) {
      ElimTask& T = tasks[(size_t)t];
      const int nc = T.nc, nq = T.nq, nf = nc + nq;
      T.dofs_off = idx_tot;
      idx_tot += nf;
      T.blk_off = hl_tot;
      hl_tot += T.nblk;
      if (!is_big[(size_t)t]) {
        smem_small = std::max(smem_small, smem_need[(size_t)t]);
        max_small_nf = std::max(max_small_nf, nf);
      } else {
        smem_big = std::max(smem_big, elim_big_smem(nf, T.maxnb));
      }
      T.C_off = (int64_t)fac_tot;
      fac_tot += (size_t)nc * nc;
      if (is_big[(size_t)t]) {
        T.P_off = (int64_t)fac_tot;
        fac_tot += (size_t)nc * (nc + 1) / 2;
      } else {
        T.P_off = T.C_off;
      }
      T.W_off = (int64_t)fac_tot;
      fac_tot += (size_t)nc * nq;
      T.U_off = (int64_t)bv_tot;
      bv_tot += (size_t)nq * nq;
      L.max_front = std::max<int64_t>(L.max_front, nf);
      SolveRec& R = L.recs[(size_t)t];
      R.nc = nc;
      R.nq = nq;
      R.contrib_off = L.ncontrib;
      R.T_off = 0;
      R.inv = 1;
      R.pad = 0;
      L.ncontrib += nq;
      L.max_nc = std::max(L.max_nc, nc);
      L.max_nq = std::max(L.max_nq, nq);
      F->m_f_bytes += 8 * ((int64_t)nc * nc + nc + (int64_t)nc * nq);
      const double dc = nc, dq = nq;
      const double gf = (dc * dc * dc / 3 + dc * dc * dq + dc * dq + dc * dq * dq) * 1e-9;
      const double gb = 8.0 * ((dc + dq) * (dc + dq) + dc * dc + dc + dc * dq + 2 * dq * dq) * 1e-9;
      L.gflop += gf;
      L.gbytes += gb;
      L.gf_cls[is_big[(size_t)t]] += gf;
      L.gb_cls[is_big[(size_t)t]] += gb;
    }
    const int64_t idx_base = (int64_t)h_idx.size();
    h_idx.resize((size_t)(idx_base + idx_tot));
    hl.resize((size_t)hl_tot);
    const int64_t fac_base = (int64_t)F->fac.bump(fac_tot, s);
    fac_grown((size_t)fac_base, fac_tot);
    const size_t bv_old = bvals.n;
    const int64_t bv_base = bv_tot ? (int64_t)bvals.bump(bv_tot, s) : 0;
    bvals_grown(bv_old);
    own_.assign((size_t)nt, 0);
    if (sharded())
      for (int64_t t = 0; t < nt; ++t) own_[(size_t)t] = owner_of(gr.begin(t));
    if (sharded()) L.rec_own = own_;
#pragma omp parallel for num_threads(nthr) schedule(dynamic, 64)
    for (int64_t t = 0; t < nt; ++t) {
      ElimTask& T = tasks[(size_t)t];
      const FrontSym& f = fs[(size_t)t];
      T.dofs_off += idx_base;
      T.C_off += fac_base;
      T.P_off += fac_base;
      T.W_off += fac_base;
      T.U_off = T.nq > 0 ? T.U_off + bv_base : 0;
      int32_t* d = h_idx.data() + T.dofs_off;
      std::copy(gr.begin(t), gr.begin(t) + T.nc, d);
      std::copy(sym_q(f), sym_q(f) + T.nq, d + T.nc);
      std::copy(sym_b(f), sym_b(f) + f.nb, hl.data() + T.blk_off);
      SolveRec& R = L.recs[(size_t)t];
      R.idx_off = T.dofs_off;
      R.C_off = T.P_off;  // the solve applies the packed inverse
      R.W_off = T.W_off;
    }
    L.xrec.resize((size_t)nt);
    for (int64_t t = 0; t < nt; ++t) {
      const ElimTask& T = tasks[(size_t)t];
      hifde_record_t& X = L.xrec[(size_t)t];
      X.kind = is_top ? 2 : 0;
      X.nc = T.nc;
      X.nq = T.nq;
      X.nr = 0;
      X.cell_off = T.dofs_off;
      X.idx_off = T.dofs_off;
      X.P_off = T.P_off;
      X.W_off = T.W_off;
      X.T_off = 0;
    }
    double tp = now_s();
    L.t_sym = tp - t_begin;
    L.lap("tasks");
    HTRACE("  symbolic done");
    // host structure updates: consumed blocks die, new neighbour blocks live
    {
      std::vector<int32_t> newid((size_t)nt, -1);
      size_t nadd = 0;
      for (int64_t t = 0; t < nt; ++t) {
        const ElimTask& T = tasks[(size_t)t];
        for (int j = 0; j < T.nblk; ++j) blk_alive[(size_t)hl[(size_t)(T.blk_off + j)]] = 0;
        if (T.nq > 0) newid[(size_t)t] = new_block(T.dofs_off + T.nc, T.nq, T.U_off, own_[(size_t)t]);
        nadd += (size_t)T.nq;
      }
      member.ensure_room(nadd);
      // every thread applies the membership edits of its own DOF range
      const int nthu = nt >= 64 ? nthreads : 1;
#pragma omp parallel num_threads(nthu)
      {
        const int tid = omp_get_thread_num(), nth = omp_get_num_threads();
        const int64_t lo = N * tid / nth, hi = N * (tid + 1) / nth;
        for (int64_t t = 0; t < nt; ++t) {
          const ElimTask& T = tasks[(size_t)t];
          for (int j = 0; j < T.nblk; ++j) {
            const int32_t b = hl[(size_t)(T.blk_off + j)];
            const int32_t* d = h_idx.data() + blk_dof_off[(size_t)b];
            for (int32_t i = 0; i < blk_n[(size_t)b]; ++i)
              if (d[i] >= lo && d[i] < hi) member.remove(d[i], b);
          }
        }
        for (int64_t t = 0; t < nt; ++t) {
          const ElimTask& T = tasks[(size_t)t];
          if (T.nq <= 0) continue;
          const int32_t* d = h_idx.data() + T.dofs_off + T.nc;
          for (int i = 0; i < T.nq; ++i)
            if (d[i] >= lo && d[i] < hi) member.add(d[i], newid[(size_t)t]);
        }
#pragma omp for schedule(static)
        for (int64_t t = 0; t < nt; ++t) {
          const int32_t* c = gr.begin(t);
          for (int i = 0; i < gr.count(t); ++i) active[(size_t)c[i]] = 0;
        }
      }
    }
    L.t_upd = now_s() - tp;
    L.lap("blocks");
    tp = now_s();
    // blocks this process's groups consume from other ranks
    if (sharded()) {
      std::vector<int64_t> bptr((size_t)nt);
      std::vector<int32_t> bcnt((size_t)nt);
      for (int64_t t = 0; t < nt; ++t) {
        bptr[(size_t)t] = tasks[(size_t)t].blk_off;
        bcnt[(size_t)t] = tasks[(size_t)t].nblk;
      }
      exchange_blocks(nt, own_.data(), bptr.data(), bcnt.data(), hl.data());
    }
    upload_idx();
    upload_blocks();
    lists.reserve(std::max<size_t>(hl.size(), 1), s);
    lists.n = hl.size();
    lists.upload(hl.data(), 0, hl.size(), s);
    HCK(cudaEventCreate(&L.ev0));
    HCK(cudaEventCreate(&L.ev1));
    HCK(cudaEventRecord(L.ev0, s));
    // the groups of rank r (all of them unsharded): shared-memory path and
    // blocked large-front path
    auto launch_rank = [&](int r) {
    std::vector<ElimTask> small, big;
    for (int64_t t = 0; t < nt; ++t) {
      if (sharded() && own_[(size_t)t] != r) continue;
      const ElimTask& T = tasks[(size_t)t];
      (is_big[(size_t)t] ? big : small).push_back(T);
    }
    HTRACE("  host updates done (%zu small / %zu big)", small.size(), big.size());
    L.lap("e-lists");
    DBuf<ElimTask> d_small, d_big;
    d_small.reserve(small.size(), s);
    d_small.upload(small.data(), 0, small.size(), s);
    d_big.reserve(big.size(), s);
    d_big.upload(big.data(), 0, big.size(), s);
    const int64_t st_small = (int64_t)status.bump(small.size(), s);
    const char* what = is_top ? "top block" : "cell";
    pending.push_back({st_small, (int64_t)small.size(), tag, what});
    L.lap("e-uploads");
    Arenas A = arenas_for(r);
    if (!small.empty()) {
      A.status = status.p + st_small;
      const int kl = F->klog.begin(is_top ? "elim_small_kernel(top)" : "elim_small_kernel", tag, 0, L.gb_cls[0],
                                   L.gf_cls[0], s);
      launch_elim_small(d_small.p, (int)small.size(), A, smem_small, max_small_nf <= 64 ? 128 : 256, s);
      F->klog.end(kl, s);
      ++g_launches;
    }
    launch_big_cells(big, d_big.p, smem_big, A, tag, is_top, L.gb_cls[1], L.gf_cls[1]);
    L.lap("e-launches");
    d_small.release(s);
    d_big.release(s);
    };
    for (int r = rank_lo(); r < rank_hi(); ++r) launch_rank(r);
    HCK(cudaEventRecord(L.ev1, s));
    HCK(cudaGetLastError());
    HTRACE("  launched");
    if (trace_on()) { HCK(cudaStreamSynchronize(s)); HTRACE("  kernels done"); }
    // (the kernels retire the cells in the device active mask themselves;
    // real ranks retire the other ranks' cells locally)
    if (real) {
      std::vector<int64_t> off((size_t)nt);
      std::vector<int> len((size_t)nt);
      for (int64_t t = 0; t < nt; ++t) {
        off[(size_t)t] = tasks[(size_t)t].dofs_off;
        len[(size_t)t] = tasks[(size_t)t].nc;
      }
      union_state(off.data(), len.data(), nullptr, (int)nt, 0);
    }
    L.t_launch = now_s() - tp;
    L.lap("launch");
    tp = now_s();
    if (is_top) check_status();
    // solve-side reduction structure for the shared neighbour DOFs
    if (!is_top) build_reduction((size_t)(&L - F->levels.data()), L);
    L.t_sync = now_s() - tp;
  }

  // Blocked multi-CTA path of the large cells of an elimination level
  // (kernels_big.cu): per-cell work lists on the host from (nc, nq), the
  // cells' ElimTasks already on the device at d_big.
  void launch_big_cells(const std::vector<ElimTask>& big, const ElimTask* d_big, size_t smem_big, Arenas A,
                        double tag, bool is_top, double gb, double gf, bool defer_inverse = false) {
    if (big.empty()) return;
    std::vector<int4> tiles, asm_work;
    int max_big_nc = 0;
    for (int bi = 0; bi < (int)big.size(); ++bi) {
      const ElimTask& T = big[(size_t)bi];
      max_big_nc = std::max(max_big_nc, T.nc);
      const int nf = T.nc + T.nq;
      for (int r0 = 0; r0 < nf; r0 += 64) asm_work.push_back(make_int4(bi, r0, std::min(r0 + 64, nf), 0));
      const int ntl = (T.nq + kSchurTile - 1) / kSchurTile;
      for (int a = 0; a < ntl; ++a)
        for (int b = a; b < ntl; ++b) tiles.push_back(make_int4(bi, a, b, 0));
    }
    InvPlan inv;  // packed inverses of the big cells
    {
      std::vector<int> ncs;
      for (const ElimTask& T : big) ncs.push_back(T.nc);
      inv.build(ncs);
    }
    // per-panel work lists of the blocked Cholesky / TRSM
    const int npanel = (max_big_nc + kPanelB - 1) / kPanelB;
    std::vector<int32_t> pcells;
    std::vector<int4> ptrsm, pupd;
    std::vector<int64_t> pc_off(npanel + 1, 0), pt_off(npanel + 1, 0), pu_off(npanel + 1, 0);
    for (int p = 0; p < npanel; ++p) {
      const int p0 = p * kPanelB;
      for (int bi = 0; bi < (int)big.size(); ++bi) {
        const ElimTask& T = big[(size_t)bi];
        if (T.nc <= p0) continue;
        const int p1 = std::min(p0 + kPanelB, T.nc);
        pcells.push_back(bi);
        for (int r0 = p1; r0 < T.nc; r0 += 128) ptrsm.push_back(make_int4(bi, 0, r0, 0));
        for (int c0 = 0; c0 < T.nq; c0 += 128) ptrsm.push_back(make_int4(bi, 1, c0, 0));
        for (int a0 = p1; a0 < T.nc; a0 += 64) {
          for (int b0 = p1; b0 <= a0; b0 += 64) pupd.push_back(make_int4(bi, 0, a0, b0));
          for (int b0 = 0; b0 < T.nq; b0 += 64) pupd.push_back(make_int4(bi, 1, a0, b0));
        }
      }
      pc_off[(size_t)p + 1] = (int64_t)pcells.size();
      pt_off[(size_t)p + 1] = (int64_t)ptrsm.size();
      pu_off[(size_t)p + 1] = (int64_t)pupd.size();
    }
    DBuf<int4> d_tiles, d_asm, d_ptrsm, d_pupd;
    DBuf<int32_t> d_pcells;
    DBuf<double> d_dmin, d_scale;
    auto up4 = [&](DBuf<int4>& d, const std::vector<int4>& h) { d.reserve(h.size(), s); d.upload(h.data(), 0, h.size(), s); };
    up4(d_tiles, tiles);
    up4(d_asm, asm_work);
    up4(d_ptrsm, ptrsm);
    up4(d_pupd, pupd);
    inv.upload(s);
    d_pcells.reserve(pcells.size(), s);
    d_pcells.upload(pcells.data(), 0, pcells.size(), s);
    std::vector<double> dm(big.size(), DBL_MAX);
    d_dmin.reserve(big.size(), s);
    d_dmin.upload(dm.data(), 0, dm.size(), s);
    d_scale.reserve(big.size(), s);
    HCK(cudaMemsetAsync(d_scale.p, 0, big.size() * sizeof(double), s));
    const int64_t st_big = (int64_t)status.bump(big.size(), s);
    HCK(cudaMemsetAsync(status.p + st_big, 0, big.size() * sizeof(int), s));
    pending.push_back({st_big, (int64_t)big.size(), tag, is_top ? "top block" : "cell"});
    A.status = status.p + st_big;
    const int kl = F->klog.begin(is_top ? "elim_blocked_pipeline(top)" : "elim_blocked_pipeline", tag, 0, gb, gf, s);
    launch_big_assemble(d_big, d_asm.p, (int)asm_work.size(), A, d_scale.p, smem_big, s);
    ++g_launches;
    for (int p = 0; p < npanel; ++p) {
      const int p0 = p * kPanelB;
      launch_panel_chol(d_big, d_pcells.p + pc_off[(size_t)p], (int)(pc_off[(size_t)p + 1] - pc_off[(size_t)p]), p0,
                        A, d_dmin.p, s);
      launch_panel_trsm(d_big, d_ptrsm.p + pt_off[(size_t)p], (int)(pt_off[(size_t)p + 1] - pt_off[(size_t)p]), p0, A,
                        s);
      launch_panel_update(d_big, d_pupd.p + pu_off[(size_t)p], (int)(pu_off[(size_t)p + 1] - pu_off[(size_t)p]), p0,
                          A, s);
      g_launches += 3;
    }
    if (!tiles.empty()) {
      launch_schur_tiles(d_big, d_tiles.p, (int)tiles.size(), A, s);
      ++g_launches;
    }
    launch_big_finish(d_big, (int)big.size(), A, d_dmin.p, d_scale.p, s);
    if (defer_inverse) {
      const cudaStream_t ts = tail_stream();
      HCK(cudaEventRecord(ev_id, s));
      HCK(cudaStreamWaitEvent(ts, ev_id, 0));
      g_launches += 1 + inv.launch(d_big, A, ts);
      inv.release(ts);
      inv_pending = true;
    } else {
      g_launches += 1 + inv.launch(d_big, A, s);
      inv.release(s);
    }
    F->klog.end(kl, s);
    d_tiles.release(s);
    d_asm.release(s);
    d_ptrsm.release(s);
    d_pupd.release(s);
    d_pcells.release(s);
    d_dmin.release(s);
    d_scale.release(s);
  }

  // Solve-side reduction of one elimination level: for every neighbour DOF the
  // contribution rows (record order) summed by solve_reduce_kernel.  Linear
  // counting sort by DOF (targets in first-touch order); uploaded at the end.
  struct Reduction {
    std::vector<int32_t> targets;
    std::vector<int64_t> ptr, ent;
  };
  std::vector<std::pair<size_t, Reduction>> reductions;
  std::vector<int32_t> red_slot;  // per DOF: target index during a build, else -1

  Helper& helper = helper_thread();

  // Copies the level's neighbour lists now (h_idx keeps growing) and builds
  // the reduction on the helper thread.
  void build_reduction(size_t level_index, const LevelRec& L) {
    std::vector<int32_t> qflat;
    std::vector<int64_t> qptr{0}, coff;
    qflat.reserve((size_t)L.ncontrib);
    for (const SolveRec& R : L.recs) {
      const int32_t* q = h_idx.data() + R.idx_off + R.nc;
      qflat.insert(qflat.end(), q, q + R.nq);
      qptr.push_back((int64_t)qflat.size());
      coff.push_back(R.contrib_off);
    }
    F->max_contrib = std::max(F->max_contrib, L.ncontrib);
    helper.post([this, level_index, qflat = std::move(qflat), qptr = std::move(qptr), coff = std::move(coff)]() {
      if ((int64_t)red_slot.size() != N) red_slot.assign((size_t)N, -1);
      Reduction r;
      std::vector<int64_t> cnt;
      for (int32_t d : qflat) {
        int32_t& sl = red_slot[(size_t)d];
        if (sl < 0) {
          sl = (int32_t)r.targets.size();
          r.targets.push_back(d);
          cnt.push_back(0);
        }
        ++cnt[(size_t)sl];
      }
      r.ptr.assign(r.targets.size() + 1, 0);
      for (size_t i = 0; i < cnt.size(); ++i) r.ptr[i + 1] = r.ptr[i] + cnt[i];
      r.ent.resize((size_t)r.ptr.back());
      std::vector<int64_t> pos(r.ptr.begin(), r.ptr.end() - 1);
      for (size_t rec = 0; rec + 1 < qptr.size(); ++rec)
        for (int64_t a = qptr[rec]; a < qptr[rec + 1]; ++a)
          r.ent[(size_t)pos[(size_t)red_slot[(size_t)qflat[(size_t)a]]]++] = coff[rec] + (a - qptr[rec]);
      for (int32_t d : r.targets) red_slot[(size_t)d] = -1;
      reductions.emplace_back(level_index, std::move(r));
    });
  }

  void finish_reductions() {
    for (auto& pr : reductions) {
      const Reduction& r = pr.second;
      LevelRec& L = F->levels[pr.first];
      L.ntargets = (int)r.targets.size();
      meta.add(&L.d_targets, r.targets);
      meta.add(&L.d_ptr, r.ptr);
      meta.add(&L.d_ent, r.ent);
    }
    reductions.clear();
  }

  // -------------------------------------------------------------------------
  void skeleton_level(const Groups& gr, double tag, LevelRec& L) {
    HTRACE("skel level %g: %lld groups", tag, (long long)gr.size());
    const double t_begin = now_s();
    const int64_t nt = gr.size();
    L.kind = 1;
    L.ngroups = nt;
    std::vector<SkelTask> tasks((size_t)nt);
    std::vector<int32_t> hl;
    size_t smem = 0;
    int max_nc = 0, max_nq = 0;
    scratch.n = 0;
    const int64_t idx_level_start = (int64_t)h_idx.size();
    // exact-order batch index of every group (groups are neighbours when one
    // holds a DOF of the other's neighbour set)
    std::vector<int> batch((size_t)nt, 0);
    std::vector<int32_t> gof_dofs;  // DOFs of this level's groups, to reset
    static thread_local std::vector<int32_t> group_of_tls;
    std::vector<int32_t>& group_of = group_of_tls;  // this thread's; shared with the OpenMP workers
    if ((int64_t)group_of.size() < N) group_of.assign((size_t)N, -1);
#pragma omp parallel for schedule(static) if (nt > 32768)
    for (int64_t t = 0; t < nt; ++t)
      for (int i = 0; i < gr.count(t); ++i) group_of[(size_t)gr.begin(t)[i]] = (int32_t)t;
    int nbatch = 1;
    std::vector<int32_t> preds;          // earlier neighbouring groups (exact order)
    std::vector<int64_t> pred_ptr{0};
    L.lap(nullptr);
    const std::vector<FrontSym> fs = fronts(gr);
    L.lap("fronts");
    // (1) per group, in parallel: workspace mode, arena sizes, earlier
    // neighbouring groups; (2) prefix sums and exact-order batches; (3) fill
    struct Sz {
      size_t scr, fac, smem;
      int64_t pred_off;
      int npred;
    };
    std::vector<Sz> sz((size_t)nt);
    std::vector<uint8_t> promote((size_t)nt, 0);
    const double promote_work = kPromoteWork;
    std::vector<std::vector<int32_t>> tpred((size_t)nthreads);
    const int nthr = nt >= 256 ? nthreads : 1;
#pragma omp parallel num_threads(nthr)
    {
      std::vector<int32_t>& mypred = tpred[(size_t)omp_get_thread_num()];
      mypred.clear();
#pragma omp for schedule(dynamic, 64)
      for (int64_t t = 0; t < nt; ++t) {
        const int nc = gr.count(t);
        const FrontSym& f = fs[(size_t)t];
        const int32_t* q = sym_q(f);
        const int nq = f.nq, nf = nc + nq;
        SkelTask& T = tasks[(size_t)t];
        T.nc = nc;
        T.nq = nq;
        T.nblk = f.nb;
        T.maxnb = f.maxnb;
        T.group = (int32_t)t;
        T.chunk = 0;
        T.pad2 = 0;
        T.scratch_off = -1;
        Sz& z = sz[(size_t)t];
        z.scr = 0;
        z.smem = 0;
        const SkelSizes zz = skel_sizes(nc, nq, T.maxnb);
        (void)nf;
        T.mode = zz.mode;
        T.chunk = zz.chunk;
        z.scr = zz.scr;
        z.smem = zz.smem;
        // one-CTA groups the Gram path can take keep room for the large-group
        // record: they join the large-group pipeline in exact batches
        // (promote[] below), where a one-CTA launch per batch would be exposed
        promote[(size_t)t] = (T.mode == 1 || T.mode == 3) && (double)nq * nc * nc >= promote_work && gram_ok(nc, nq);
        z.fac = zz.fac + ((T.mode == 2 || promote[(size_t)t]) ? zz.fac_big : 0);
        const size_t p0 = mypred.size();
        for (int i = 0; i < nq; ++i) {
          const int32_t go = group_of[(size_t)q[i]];
          if (go >= 0 && go < t) mypred.push_back(go);
        }
        std::sort(mypred.begin() + (int64_t)p0, mypred.end());
        mypred.erase(std::unique(mypred.begin() + (int64_t)p0, mypred.end()), mypred.end());
        z.pred_off = (int64_t)p0 * nthreads + omp_get_thread_num();  // decoded below
        z.npred = (int)(mypred.size() - p0);
      }
    }
    // (2) serial prefix pass
    int64_t idx_tot = 0, hl_tot = 0;
    size_t scr_tot = 0, fac_tot = 0, bv_tot = 0;
    pred_ptr.resize((size_t)nt + 1);
    for (int64_t t = 0; t < nt; ++t) {
      SkelTask& T = tasks[(size_t)t];
      const Sz& z = sz[(size_t)t];
      const int nc = T.nc, nq = T.nq;
      T.dofs_off = idx_tot;
      idx_tot += nc + nq;  // the sk/rd output lists follow all groups' fronts (below)
      T.blk_off = hl_tot;
      hl_tot += T.nblk;
      if (z.scr) { T.scratch_off = (int64_t)scr_tot; scr_tot += z.scr; }
      T.rec_off = (int64_t)fac_tot;
      fac_tot += z.fac;
      T.delta_off = (int64_t)bv_tot;
      bv_tot += (size_t)nc * nc;
      smem = std::max(smem, z.smem);
      max_nc = std::max(max_nc, nc);
      max_nq = std::max(max_nq, nq);
      L.max_front = std::max<int64_t>(L.max_front, nc + nq);
      pred_ptr[(size_t)t + 1] = pred_ptr[(size_t)t] + z.npred;
      const int32_t* pp = tpred[(size_t)(z.pred_off % nthreads)].data() + z.pred_off / nthreads;
      int b = 0;
      for (int i = 0; i < z.npred; ++i) b = std::max(b, batch[(size_t)pp[i]] + 1);
      batch[(size_t)t] = b;
      nbatch = std::max(nbatch, b + 1);
    }
    // output lists of every group, contiguous after the fronts: the level's
    // one readback copies only this tail
    const int64_t out_base = idx_tot;
    for (int64_t t = 0; t < nt; ++t) {
      tasks[(size_t)t].out_off = idx_tot;
      idx_tot += tasks[(size_t)t].nc;
    }
    const int64_t idx_base = (int64_t)h_idx.size();
    h_idx.resize((size_t)(idx_base + idx_tot));
    hl.resize((size_t)hl_tot);
    preds.resize((size_t)pred_ptr[(size_t)nt]);
    const int64_t scr_base = scr_tot ? (int64_t)scratch.bump(scr_tot, s) : 0;
    const int64_t fac_base = (int64_t)F->fac.bump(fac_tot, s);
    fac_grown((size_t)fac_base, fac_tot);
    const size_t bv_old = bvals.n;
    const int64_t bv_base = (int64_t)bvals.bump(bv_tot, s);
    bvals_grown(bv_old);
    // (3) fill, in parallel
#pragma omp parallel for num_threads(nthr) schedule(dynamic, 64)
    for (int64_t t = 0; t < nt; ++t) {
      SkelTask& T = tasks[(size_t)t];
      const Sz& z = sz[(size_t)t];
      const FrontSym& f = fs[(size_t)t];
      const int nc = T.nc, nq = T.nq;
      T.dofs_off += idx_base;
      T.out_off += idx_base;
      if (T.scratch_off >= 0) T.scratch_off += scr_base;
      T.rec_off += fac_base;
      T.delta_off += bv_base;
      int32_t* d = h_idx.data() + T.dofs_off;
      std::copy(gr.begin(t), gr.begin(t) + nc, d);
      std::copy(sym_q(f), sym_q(f) + nq, d + nc);
      std::fill(h_idx.data() + T.out_off, h_idx.data() + T.out_off + nc, 0);
      std::copy(sym_b(f), sym_b(f) + f.nb, hl.data() + T.blk_off);
      const int32_t* pp = tpred[(size_t)(z.pred_off % nthreads)].data() + z.pred_off / nthreads;
      std::copy(pp, pp + z.npred, preds.data() + pred_ptr[(size_t)t]);
    }
#pragma omp parallel for schedule(static) if (nt > 32768)
    for (int64_t t = 0; t < nt; ++t)
      for (int i = 0; i < gr.count(t); ++i) group_of[(size_t)gr.begin(t)[i]] = -1;
    bool exact = opt.order_mode == HIFDE_ORDER_EXACT ||
                 (opt.order_mode == HIFDE_ORDER_AUTO && nbatch <= opt.exact_max_batches);
    if (!exact) {
      std::fill(batch.begin(), batch.end(), 0);
      nbatch = 1;
    }
    L.nbatches = nbatch;
    L.lap("tasks");
    HTRACE("  symbolic done, %d batches", nbatch);
    double tp = now_s();
    L.t_sym = tp - t_begin;
    bool any_huge = false;
    for (const SkelTask& T : tasks) any_huge |= T.mode == 2;
    // 3D: an exact level of medium groups alone also takes the pipeline (its
    // batches beat one chained launch of one-CTA groups: config 4 247 -> 216
    // ms GPU); in 2D the one-launch chain stays faster
    const bool promote_any = g.dim == 3;  // per grid, not per process
    // (a level whose largest medium group is small keeps the one-launch
    // chain: config 5's level 1.333, nq nc^2 <= 1.3e6, is faster chained)
    bool any_promote = false, big_promote = false;
    for (int64_t t = 0; t < nt; ++t)
      if (promote[(size_t)t]) {
        any_promote = true;
        const SkelTask& T = tasks[(size_t)t];
        big_promote = big_promote || (double)T.nq * T.nc * T.nc >= 4e6;
      }
    if (exact && nbatch > 1 && (any_huge || (promote_any && big_promote))) {
      for (int64_t t = 0; t < nt; ++t)
        if (promote[(size_t)t]) tasks[(size_t)t].mode = 2;
      any_huge = any_huge || any_promote;
    }
    const bool one_launch = exact && !any_huge && nt > 1 && opt.order_mode != HIFDE_ORDER_SNAPSHOT;
    // owners: the one-launch exact order runs on rank 0 (its groups wait on
    // one another); otherwise groups go to their subdomain's rank
    own_.assign((size_t)nt, 0);
    if (sharded() && !one_launch)
      for (int64_t t = 0; t < nt; ++t) own_[(size_t)t] = owner_of(gr.begin(t));
    if (sharded()) {
      std::vector<int64_t> bptr((size_t)nt);
      std::vector<int32_t> bcnt((size_t)nt);
      for (int64_t t = 0; t < nt; ++t) {
        bptr[(size_t)t] = tasks[(size_t)t].blk_off;
        bcnt[(size_t)t] = tasks[(size_t)t].nblk;
      }
      exchange_blocks(nt, own_.data(), bptr.data(), bcnt.data(), hl.data());
    }
    if (one_launch) {
      // one launch, per-group dependencies (skel_ordered_kernel)
      upload_idx();
      upload_blocks();
      lists.reserve(std::max<size_t>(hl.size(), 1), s);
      lists.n = hl.size();
      lists.upload(hl.data(), 0, hl.size(), s);
      DBuf<SkelTask> dt;
      DBuf<int64_t> dpp;
      DBuf<int32_t> dpr, dord;
      DBuf<int> ddone;
      dt.reserve(tasks.size(), s);
      dt.upload(tasks.data(), 0, tasks.size(), s);
      dpp.reserve(pred_ptr.size(), s);
      dpp.upload(pred_ptr.data(), 0, pred_ptr.size(), s);
      dpr.reserve(std::max<size_t>(preds.size(), 1), s);
      dpr.upload(preds.data(), 0, preds.size(), s);
      ddone.reserve((size_t)nt + 1, s);
      HCK(cudaMemsetAsync(ddone.p, 0, sizeof(int) * ((size_t)nt + 1), s));
      {  // claim order: by dependency depth, reference order within a depth
        std::vector<int32_t> ord((size_t)nt);
        for (int64_t t = 0; t < nt; ++t) ord[(size_t)t] = (int32_t)t;
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return batch[(size_t)a] < batch[(size_t)b]; });
        dord.reserve((size_t)nt, s);
        dord.upload(ord.data(), 0, ord.size(), s);
      }
      const int64_t st_off = (int64_t)status.bump((size_t)nt, s);
      HCK(cudaMemsetAsync(status.p + st_off, 0, (size_t)nt * sizeof(int), s));
      pending.push_back({st_off, nt, tag, "group"});
      kout.n = 0;
      kout.bump((size_t)nt, s);
      if (real) HCK(cudaMemsetAsync(kout.p, 0, (size_t)nt * sizeof(int32_t), s));
      const bool run_here = rank_lo() == 0;  // rank 0 owns the whole level
      Arenas A = arenas_for(0);
      A.status = status.p + st_off;
      // large groups: a CTA cluster per group (skel_cluster_kernel), 4 or 2 CTAs
      // each, when every group's column slice fits and every group gets a
      // resident cluster of its own (more groups than clusters: the one-CTA
      // kernel's throughput wins)
      size_t smem_cl = 0;
      int cs = 0, ncls = 0;
      bool cluster_ok = max_nc >= kClusterMinNc;
      for (int csz : {4, 2}) {
        if (!cluster_ok) break;
        size_t need_max = 0;
        bool fits = true;
        for (int64_t t = 0; t < nt && fits; ++t) {
          const SkelTask& T = tasks[(size_t)t];
          const size_t need = skel_cluster_need(T.nc, T.nq, T.maxnb, csz);
          need_max = std::max(need_max, need);
          fits = need <= kSmemCap;
        }
        if (!fits) continue;
        const int capc = skel_cluster_capacity(need_max, csz);
        if (capc >= 1 && nt <= capc) {
          cs = csz;
          ncls = (int)std::min<int64_t>(nt, capc);
          smem_cl = need_max;
          break;
        }
      }
      cluster_ok = cluster_ok && cs > 0;
      if (cluster_ok) {
        std::vector<SkelTask> ct(tasks);  // per-group global workspace of the cluster kernel
        size_t tot = 0;
        for (auto& T : ct) {
          T.scratch_off = (int64_t)tot;
          tot += skel_cluster_scratch(T.nc);
        }
        const int64_t base = (int64_t)scratch.bump(tot, s);
        for (auto& T : ct) T.scratch_off += base;
        A.scratch = scratch.p;
        dt.upload(ct.data(), 0, ct.size(), s);
        HCK(cudaEventCreate(&L.ev0));
        HCK(cudaEventCreate(&L.ev1));
        HCK(cudaEventRecord(L.ev0, s));
        if (run_here) {
          const int kl = F->klog.begin("skel_cluster_kernel", tag, 0, 0, 0, s);
          HCK(launch_skel_cluster(dt.p, (int)nt, dpp.p, dpr.p, ddone.p, A, opt.eps, smem_cl, ncls, cs, s));
          F->klog.end(kl, s);
          ++g_launches;
        }
        HCK(cudaEventRecord(L.ev1, s));
        union_level(tasks, nt);
        L.t_launch = now_s() - tp;
        tp = now_s();
        finish_skeleton_level(tasks, idx_level_start + out_base, tag, L, tp);
        dt.release(s);
        dpp.release(s);
        dpr.release(s);
        ddone.release(s);
        return;
      }
      const int nthr = (max_nc > 32 || max_nq > 128) ? 512 : 128;
      const int cap = skel_ordered_capacity(smem, nthr);
      if (cap < 1) throw Fail{HIFDE_CUDA, "ordered skeleton kernel cannot be resident"};
      const int grid = (int)std::min<int64_t>(nt, cap);
      HCK(cudaEventCreate(&L.ev0));
      HCK(cudaEventCreate(&L.ev1));
      HCK(cudaEventRecord(L.ev0, s));
      const char* tlog_dir = getenv("HIFDE_SKEL_TLOG");
      DBuf<unsigned long long> dtl;
      if (tlog_dir) {
        dtl.reserve((size_t)nt * 16, s);
        A.tlog = dtl.p;
      }
      if (run_here) {
        const int kl = F->klog.begin("skel_ordered_kernel", tag, 0, 0, 0, s);
        HCK(launch_skel_ordered(dt.p, (int)nt, dpp.p, dpr.p, dord.p, ddone.p, A, opt.eps, smem, nthr, grid, s));
        F->klog.end(kl, s);
        ++g_launches;
      }
      HCK(cudaEventRecord(L.ev1, s));
      union_level(tasks, nt);
      if (tlog_dir) {  // debug: per-group timestamps + the predecessor CSR
        std::vector<unsigned long long> h((size_t)nt * 16);
        HCK(cudaMemcpyAsync(h.data(), dtl.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
        HCK(cudaStreamSynchronize(s));
        char fn[512];
        snprintf(fn, sizeof fn, "%s/tlog_%.3f_%lld.bin", tlog_dir, tag, (long long)nt);
        if (FILE* fp = fopen(fn, "wb")) {
          const int64_t hdr[3] = {(int64_t)nt, (int64_t)preds.size(), (int64_t)grid};
          fwrite(hdr, 8, 3, fp);
          fwrite(h.data(), 8, h.size(), fp);
          fwrite(pred_ptr.data(), 8, pred_ptr.size(), fp);
          fwrite(preds.data(), 4, preds.size(), fp);
          fclose(fp);
        }
        dtl.release(s);
      }
      L.t_launch = now_s() - tp;
      tp = now_s();
      finish_skeleton_level(tasks, idx_level_start + out_base, tag, L, tp);
      dt.release(s);
      dpp.release(s);
      dpr.release(s);
      dord.release(s);
      ddone.release(s);
      return;
    }
    // order tasks by batch (stable keeps the reference order inside a batch)
    std::vector<int64_t> order((size_t)nt);
    for (int64_t t = 0; t < nt; ++t) order[(size_t)t] = t;
    // (then by owner: a batch's groups are independent, each rank takes a
    // contiguous range)
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
      if (batch[(size_t)a] != batch[(size_t)b]) return batch[(size_t)a] < batch[(size_t)b];
      return own_[(size_t)a] < own_[(size_t)b];
    });
    const int PP = sharded() ? P : 1;
    // per batch and rank: small groups (one CTA each) and large groups
    // (cluster path); ranges indexed by b * PP + r
    std::vector<SkelTask> sorted, hsk;        // small tasks; SkelTask view of large ones
    std::vector<SkelBigTask> huge;
    std::vector<int64_t> bs((size_t)nbatch * PP + 1, 0), bh((size_t)nbatch * PP + 1, 0);
    int huge_max_nq = 0, huge_max_nf = 0, huge_max_nb = 0;
    iscratch.n = 0;
    for (int64_t i = 0; i < nt; ++i) {
      const SkelTask& T = tasks[(size_t)order[(size_t)i]];
      const int b = batch[(size_t)order[(size_t)i]] * PP + own_[(size_t)order[(size_t)i]];
      if (T.mode != 2) {
        sorted.push_back(T);
        bs[(size_t)b + 1]++;
        continue;
      }
      if (T.nc > kMaxBigNc) throw Fail{HIFDE_INTERNAL, "skeleton group larger than kMaxBigNc"};
      SkelBigTask H;
      H.nc = T.nc;
      H.nq = T.nq;
      H.nblk = T.nblk;
      H.maxnb = T.maxnb;
      H.dofs_off = T.dofs_off;
      H.blk_off = T.blk_off;
      const size_t nc = (size_t)T.nc, nq = (size_t)T.nq;
      H.ws_off = (int64_t)scratch.bump(nc * nc + nq * nc + (nc * nc / 4 + nc) + 3 * nc + 4 * kMaxG + 8 +
                                           (gram_ok(T.nc, T.nq) ? nc * nc : 0), s);
      H.iws_off = (int64_t)iscratch.bump(4 * nc + 4, s);
      {
        size_t mtot = 0;
        for (int j = 0; j < T.nblk; ++j) mtot += 2 + 2 * (size_t)blk_n[(size_t)hl[(size_t)(T.blk_off + j)]];
        H.map_off = (int64_t)iscratch.bump(mtot + 1, s);
      }
      H.rec_off = T.rec_off;
      H.delta_off = T.delta_off;
      H.out_off = T.out_off;
      H.group = T.group;
      H.pad = 0;
      huge.push_back(H);
      hsk.push_back(T);
      bh[(size_t)b + 1]++;
      huge_max_nq = std::max(huge_max_nq, T.nq);
      huge_max_nf = std::max(huge_max_nf, T.nc + T.nq);
      huge_max_nb = std::max(huge_max_nb, T.maxnb);
    }
    for (int b = 0; b < nbatch * PP; ++b) {
      bs[(size_t)b + 1] += bs[(size_t)b];
      bh[(size_t)b + 1] += bh[(size_t)b];
    }
    upload_idx();
    upload_blocks();
    lists.reserve(std::max<size_t>(hl.size(), 1), s);
    lists.n = hl.size();
    lists.upload(hl.data(), 0, hl.size(), s);
    DBuf<SkelTask> dt, dth;
    DBuf<SkelBigTask> dhuge;
    DBuf<ElimTask> dinner;
    DBuf<double> ddmin, dscale;
    dt.reserve(sorted.size(), s);
    dt.upload(sorted.data(), 0, sorted.size(), s);
    dth.reserve(hsk.size(), s);
    dth.upload(hsk.data(), 0, hsk.size(), s);
    dhuge.reserve(huge.size(), s);
    dhuge.upload(huge.data(), 0, huge.size(), s);
    dinner.reserve(huge.size(), s);
    ddmin.reserve(huge.size(), s);
    dscale.reserve(huge.size(), s);
    const int64_t st_off = (int64_t)status.bump((size_t)nt, s);
    HCK(cudaMemsetAsync(status.p + st_off, 0, (size_t)nt * sizeof(int), s));
    pending.push_back({st_off, nt, tag, "group"});
    const int64_t st_huge = (int64_t)status.bump(huge.size(), s);
    if (!huge.empty()) {
      HCK(cudaMemsetAsync(status.p + st_huge, 0, huge.size() * sizeof(int), s));
      pending.push_back({st_huge, (int64_t)huge.size(), tag, "large group"});
    }
    kout.n = 0;
    kout.bump((size_t)nt, s);
    if (real) HCK(cudaMemsetAsync(kout.p, 0, (size_t)nt * sizeof(int32_t), s));
    auto arenas_r = [&](int r, bool big_status) {
      Arenas A = arenas_for(r);
      A.status = status.p + (big_status ? st_huge : st_off);
      return A;
    };
    // real ranks: merge the ranks, sk/rd lists and active masks of a batch's
    // groups [lo, hi) of `v` (all ranks' ranges)
    auto merge = [&](const auto& v, int64_t lo, int64_t hi) {
      if (!real || hi <= lo) return;
      std::vector<int64_t> off;
      std::vector<int> len;
      std::vector<int32_t> kid;
      for (int64_t i = lo; i < hi; ++i) {
        off.push_back(v[(size_t)i].out_off);
        len.push_back(v[(size_t)i].nc);
        kid.push_back(v[(size_t)i].group);
      }
      union_state(off.data(), len.data(), kid.data(), (int)off.size(), nt);
    };
    HCK(cudaEventCreate(&L.ev0));
    HCK(cudaEventCreate(&L.ev1));
    HCK(cudaEventRecord(L.ev0, s));
    int kl_huge = -1;  // kernel log: the large-group pipeline of the level, first batch to the joined tails
    for (int b = 0; b < nbatch; ++b) {
      const size_t b0 = (size_t)b * PP, b1 = (size_t)(b + 1) * PP;
      for (int r = rank_lo(); r < rank_hi(); ++r) {
        const int64_t lo = bs[b0 + r], hi = bs[b0 + r + 1];
        if (hi > lo) {
          const int kl = F->klog.begin("skel_kernel", tag, 0, 0, 0, s);
          launch_skel(dt.p + lo, (int)(hi - lo), arenas_r(r, false), opt.eps, smem,
                      (max_nc > 32 || max_nq > 128) ? 512 : 128, (int)max_nc, (int)max_nq, s);
          F->klog.end(kl, s);
          ++g_launches;
        }
      }
      for (int r = rank_lo(); r < rank_hi(); ++r) {
        const int64_t lo = bs[b0 + r], hi = bs[b0 + r + 1];
        if (hi > lo) {
          launch_apply_rd(dt.p + lo, (int)(hi - lo), arenas_r(r, false), s);
          ++g_launches;
        }
      }
      merge(sorted, bs[b0], bs[b1]);
      for (int r = rank_lo(); r < rank_hi(); ++r) {
        const int64_t hlo = bh[b0 + r], hhi = bh[b0 + r + 1];
        if (hhi <= hlo) continue;
        if (kl_huge < 0) kl_huge = F->klog.begin("skel_large_pipeline", tag, 0, 0, 0, s);
        launch_huge_batch(huge, hlo, hhi, dhuge.p, dinner.p, ddmin.p, dscale.p, arenas_r(r, false),
                          arenas_r(r, true), huge_max_nq, huge_max_nf, huge_max_nb, hl);
      }
      // the large groups retire their rd once every rank's pipeline is done
      for (int r = rank_lo(); r < rank_hi(); ++r) {
        const int64_t hlo = bh[b0 + r], hhi = bh[b0 + r + 1];
        if (hhi > hlo) {
          launch_apply_rd(dth.p + hlo, (int)(hhi - hlo), arenas_r(r, false), s);
          ++g_launches;
        }
      }
      merge(huge, bh[b0], bh[b1]);
      if (trace_on()) { HCK(cudaStreamSynchronize(s)); HTRACE("  batch %d done", b); }
    }
    join_tails();  // the delta blocks and records of every tail before the level ends
    F->klog.end(kl_huge, s);
    HCK(cudaEventRecord(L.ev1, s));
    HCK(cudaGetLastError());
    L.t_launch = now_s() - tp;
    tp = now_s();
    dt.release(s);
    dth.release(s);
    dhuge.release(s);
    dinner.release(s);
    ddmin.release(s);
    dscale.release(s);
    finish_skeleton_level(tasks, idx_level_start + out_base, tag, L, tp);
  }

  // Read back ranks and sk/rd lists (the level's one synchronization), then
  // retire rd on the host, register the delta blocks and the solve records.
  void finish_skeleton_level(const std::vector<SkelTask>& tasks, int64_t idx_level_start, double tag, LevelRec& L,
                             double tp) {
    (void)tag;
    const int64_t nt = (int64_t)tasks.size();
    std::vector<int32_t> k((size_t)nt);
    HCK(cudaMemcpyAsync(k.data(), kout.p, nt * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    // read back the sk/rd lists written by the kernels: one copy of this
    // level's slice of the index arena
    if ((int64_t)h_idx.size() > idx_level_start)
      HCK(cudaMemcpyAsync(h_idx.data() + idx_level_start, F->idx.p + idx_level_start,
                          (h_idx.size() - (size_t)idx_level_start) * sizeof(int32_t),
                          cudaMemcpyDeviceToHost, s));
    L.lap("launch");
    check_status();  // synchronizes the stream
    L.lap("wait");
    HTRACE("  readback done");
    L.t_sync = now_s() - tp;
    tp = now_s();
    std::vector<int32_t> newid((size_t)nt, -1);
    size_t nadd = 0;
    L.xrec.reserve((size_t)nt);
    L.recs.reserve((size_t)nt);
    for (int64_t t = 0; t < nt; ++t) {
      const SkelTask& T = tasks[(size_t)t];
      const int kk = k[(size_t)t], r = T.nc - kk;
      const int32_t* out = h_idx.data() + T.out_off;
      L.nskel += kk;
      L.nred += r;
      for (int i = kk; i < T.nc; ++i) active[(size_t)out[i]] = 0;
      if (r > 0 && kk > 0) {
        newid[(size_t)t] = new_block(T.out_off, kk, T.delta_off, own_[(size_t)t]);
        nadd += (size_t)kk;
      }
      {
        hifde_record_t X;
        X.kind = 1;
        X.nc = T.nc;
        X.nq = kk;
        X.nr = r;
        X.cell_off = T.dofs_off;
        X.idx_off = T.out_off;
        X.T_off = T.rec_off;
        X.P_off = T.mode == 2 ? T.rec_off + (int64_t)T.nc * T.nc + 2 * ((int64_t)T.nc * T.nc / 4 + T.nc)
                              : T.rec_off + (int64_t)kk * r;
        X.W_off = T.rec_off + (int64_t)kk * r + (int64_t)r * r;
        L.xrec.push_back(X);
      }
      if (r > 0) {
        SolveRec R;
        R.nc = r;
        R.nq = kk;
        R.idx_off = T.out_off;
        R.T_off = T.rec_off;
        R.C_off = T.rec_off + (int64_t)kk * r;
        R.W_off = R.C_off + (int64_t)r * r;
        if (T.mode == 2)  // large groups keep C and put the packed inverse after the record
          R.C_off = T.rec_off + (int64_t)T.nc * T.nc + 2 * ((int64_t)T.nc * T.nc / 4 + T.nc);
        R.contrib_off = 0;
        R.inv = 1;
        R.pad = 0;
        L.recs.push_back(R);
        if (sharded()) L.rec_own.push_back(own_[(size_t)t]);
        L.max_nc = std::max(L.max_nc, r);
        L.max_nq = std::max(L.max_nq, kk);
        F->m_f_bytes += 8 * ((int64_t)kk * r + (int64_t)r * r + r + (int64_t)r * kk);
      }
      const double dc = T.nc, dq = T.nq, dk = kk, dr = r;
      double fl = 4 * dq * dc * dk - 2 * dk * dk * (dq + dc) + 4 * dk * dk * dk / 3 + 2 * dq * dc +
                  dk * dk * dr + 2 * dk * dk * dr + 4 * dk * dr * dr;
      if (r > 0) fl += dr * dr * dr / 3 + dr * dr * dk + dk * dk * dr;
      const double gb = 8.0 * (dq * dc + dc * dc + dk * dr + dr * dr + dr + dr * dk + 2 * dk * dk) * 1e-9;
      L.gflop += fl * 1e-9;
      L.gbytes += gb;
      L.gf_cls[T.mode == 2] += fl * 1e-9;
      L.gb_cls[T.mode == 2] += gb;
    }
    // kernel log: the level's totals go to its first launch of each class
    {
      bool done[2] = {false, false};
      for (auto& E : F->klog.v) {
        if (E.phase != 0 || E.tag != L.tag) continue;
        const int c = E.name == "skel_large_pipeline" ? 1 : (E.name.rfind("skel_", 0) == 0 ? 0 : -1);
        if (c < 0) continue;
        E.gbytes = done[c] ? 0.0 : L.gb_cls[c];
        E.gflop = done[c] ? 0.0 : L.gf_cls[c];
        done[c] = true;
      }
    }
    // the new delta blocks join the membership lists of their sk DOFs
    member.ensure_room(nadd);
    const int nthu = nt >= 64 ? nthreads : 1;
#pragma omp parallel num_threads(nthu)
    {
      const int tid = omp_get_thread_num(), nth = omp_get_num_threads();
      const int64_t lo = N * tid / nth, hi = N * (tid + 1) / nth;
      for (int64_t t = 0; t < nt; ++t) {
        if (newid[(size_t)t] < 0) continue;
        const int32_t* out = h_idx.data() + tasks[(size_t)t].out_off;
        for (int i = 0; i < k[(size_t)t]; ++i)
          if (out[i] >= lo && out[i] < hi) member.add(out[i], newid[(size_t)t]);
      }
    }
    L.t_upd = now_s() - tp;
    L.lap("retire");
  }

  // Large groups whose ID goes through the Gram matrix (kernels_skelbig.cu):
  // loose tolerances only (u / eps^2 << eps, kGramMinEps), tall fronts, R columns in shared memory
  bool gram_ok(int nc, int nq) const {
    return opt.eps >= kGramMinEps && nq >= 2 * nc && nc <= 1024 && pchol_min_ctas(nc) > 0;
  }

  // Large-group skeletonization pipeline for huge[lo, hi) (one exact-order batch).
  void launch_huge_batch(const std::vector<SkelBigTask>& huge, int64_t lo, int64_t hi, const SkelBigTask* d_all,
                         ElimTask* d_inner_all, double* d_dmin_all, double* d_scale_all,
                         const Arenas& A, const Arenas& AH_all, int max_nq, int max_nf, int max_nb,
                         const std::vector<int32_t>& hlist) {
    const int n = (int)(hi - lo);
    const SkelBigTask* dtk = d_all + lo;
    ElimTask* inner = d_inner_all + lo;
    double* dmin = d_dmin_all + lo;
    double* dscale = d_scale_all + lo;
    Arenas AH = AH_all;
    AH.status = AH_all.status + lo;
    std::vector<int4> wasm, wt, wc0, wc1, wsym, pt, pu, tiles, wrow, wtu;
    InvPlan inv;
    {
      std::vector<int> ncs;
      for (int i = 0; i < n; ++i) ncs.push_back(huge[(size_t)(lo + i)].nc);
      inv.build(ncs);
    }
    std::vector<int32_t> pc;
    int maxnc = 0;
    for (int i = 0; i < n; ++i) maxnc = std::max(maxnc, huge[(size_t)(lo + i)].nc);
    const int npanel = (maxnc + kPanelB - 1) / kPanelB;
    std::vector<int64_t> pco(npanel + 1, 0), pto(npanel + 1, 0), puo(npanel + 1, 0);
    for (int i = 0; i < n; ++i) {
      const SkelBigTask& H = huge[(size_t)(lo + i)];
      const int nc = H.nc, nf = H.nc + H.nq;
      for (int r0 = 0; r0 < nf; r0 += 64) wasm.push_back(make_int4(i, r0, std::min(r0 + 64, nf), 0));
      for (int c0 = 0; c0 < nc; c0 += 128) wt.push_back(make_int4(i, c0, 0, 0));
      for (int r0 = 0; r0 < nc; r0 += 64) wrow.push_back(make_int4(i, r0, 0, 0));
      for (int a0 = 0; a0 < nc; a0 += 64)
        for (int b0 = 0; b0 < nc; b0 += 64) {
          wc0.push_back(make_int4(i, 0, a0, b0));
          wc1.push_back(make_int4(i, 1, a0, b0));
        }
      for (int r0 = 0; r0 < nc; r0 += 64) wsym.push_back(make_int4(i, r0, 0, 0));
      const int ntl = (nc + kSchurTile - 1) / kSchurTile;  // sk <= nc
      for (int a = 0; a < ntl; ++a)
        for (int b = a; b < ntl; ++b) tiles.push_back(make_int4(i, a, b, 0));
    }
    // inner elimination work lists on the size bounds (r <= nc, k <= nc);
    // the kernels skip items beyond the sizes the device actually found
    for (int p = 0; p < npanel; ++p) {
      const int p0 = p * kPanelB;
      for (int i = 0; i < n; ++i) {
        const int nc = huge[(size_t)(lo + i)].nc;
        if (nc <= p0) continue;
        const int p1 = std::min(p0 + kPanelB, nc);
        pc.push_back(i);
        for (int r0 = p1; r0 < nc; r0 += 128) pt.push_back(make_int4(i, 0, r0, 0));
        for (int c0 = 0; c0 < nc; c0 += 128) pt.push_back(make_int4(i, 1, c0, 0));
        for (int a0 = p1; a0 < nc; a0 += 64) {
          for (int b0 = p1; b0 <= a0; b0 += 64) pu.push_back(make_int4(i, 0, a0, b0));
          for (int b0 = 0; b0 < nc; b0 += 64) pu.push_back(make_int4(i, 1, a0, b0));
        }
      }
      pco[(size_t)p + 1] = (int64_t)pc.size();
      pto[(size_t)p + 1] = (int64_t)pt.size();
      puo[(size_t)p + 1] = (int64_t)pu.size();
    }
    // T update tiles per 64-row block b (rows above b0, all rd columns)
    const int ntb = (maxnc + 63) / 64;
    std::vector<int64_t> tuo((size_t)ntb + 1, 0);
    for (int bb = 0; bb < ntb; ++bb) {
      const int b0 = bb * 64;
      for (int i = 0; i < n; ++i) {
        const int nc = huge[(size_t)(lo + i)].nc;
        if (b0 >= nc) continue;
        for (int a0 = 0; a0 < b0; a0 += 64)
          for (int c0 = 0; c0 < nc; c0 += 64) wtu.push_back(make_int4(i, a0, c0, 0));
      }
      tuo[(size_t)bb + 1] = (int64_t)wtu.size();
    }
    DBuf<int4> d1, d2, d3, d4, d5, d6, d7, d8, d10, d11;
    DBuf<int32_t> d9;
    auto up = [&](DBuf<int4>& d, const std::vector<int4>& h) { d.reserve(h.size(), s); d.upload(h.data(), 0, h.size(), s); };
    up(d1, wasm); up(d2, wt); up(d3, wc0); up(d4, wc1); up(d5, wsym); up(d6, pt); up(d7, pu); up(d8, tiles);
    up(d10, wrow); up(d11, wtu);
    inv.upload(s);
    d9.reserve(pc.size(), s);
    d9.upload(pc.data(), 0, pc.size(), s);
    for (int i = 0; i < n; ++i) {
      const SkelBigTask& H = huge[(size_t)(lo + i)];
      HCK(cudaMemsetAsync(A.bvals + H.delta_off, 0, sizeof(double) * (size_t)H.nc * H.nc, s));
    }
    {  // block entry -> front position maps, one CTA per (group, block)
      std::vector<int4> wm;
      for (int i = 0; i < n; ++i) {
        const SkelBigTask& H = huge[(size_t)(lo + i)];
        int off = 0;
        for (int j = 0; j < H.nblk; ++j) {
          wm.push_back(make_int4(i, j, off, 0));
          off += 2 + 2 * blk_n[(size_t)hlist[(size_t)(H.blk_off + j)]];
        }
      }
      DBuf<int4> dm;
      up(dm, wm);
      launch_skelbig_posmap(dtk, dm.p, (int)wm.size(), A, s);
      ++g_launches;
      dm.release(s);
    }
    const size_t smem_asm = align16(sizeof(int32_t) * (size_t)(2 * max_nf));  // front DOFs + alive flags
    launch_skelbig_assemble(dtk, d1.p, (int)wasm.size(), A, smem_asm, s);
    bool gram = true;
    for (int i = 0; i < n && gram; ++i) gram = gram_ok(huge[(size_t)(lo + i)].nc, huge[(size_t)(lo + i)].nq);
    if (gram) {
      // G = Mq^T Mq (DMMA tiles), then pivoted Cholesky of G: cooperative,
      // CTAs per group in proportion to nc^2, at least what keeps its R
      // columns in shared memory; groups beyond one launch's residency go to
      // further launches
      std::vector<int4> wg, wr;  // split tiles; tiles to reduce (several splits)
      for (int i = 0; i < n; ++i) {
        const int nc = huge[(size_t)(lo + i)].nc, nq = huge[(size_t)(lo + i)].nq;
        const int ns = (nq + kGramRows - 1) / kGramRows;
        for (int a0 = 0; a0 < nc; a0 += 64)
          for (int b0 = a0; b0 < nc; b0 += 64) {
            if (ns > 1) wr.push_back(make_int4(i, a0, b0, (int)wg.size()));
            for (int q = 0; q < ns; ++q) wg.push_back(make_int4(i, a0, b0, q));
          }
      }
      DBuf<int4> dg, dr;
      up(dg, wg);
      up(dr, wr);
      if (!wr.empty()) gpart.reserve(wg.size() * 4096, s);
      launch_skelbig_gram(dtk, dg.p, (int)wg.size(), dr.p, (int)wr.size(), gpart.p, A, s);
      g_launches += wr.empty() ? 1 : 2;
      int c0 = 0;
      while (c0 < n) {
        size_t smem0 = 0;
        int cn = 0, need = 0;
        for (int i = c0; i < n; ++i) {
          const int nc = huge[(size_t)(lo + i)].nc;
          const int gm = pchol_min_ctas(nc);
          const size_t sm = std::max(smem0, pchol_smem(nc, gm));
          if (cn > 0 && need + gm > pchol_coop_capacity(sm)) break;
          smem0 = sm;
          need += gm;
          ++cn;
        }
        const int cap = pchol_coop_capacity(smem0);
        double tot = 0;
        for (int i = 0; i < cn; ++i) tot += std::pow((double)huge[(size_t)(lo + c0 + i)].nc, 2);
        std::vector<int> gs((size_t)cn + 1, 0);
        size_t smem = 0;
        for (int i = 0; i < cn; ++i) {
          const int nc = huge[(size_t)(lo + c0 + i)].nc;
          const int gm = pchol_min_ctas(nc);
          const int extra = (int)((double)(cap - need) * ((double)nc * nc) / std::max(tot, 1.0));
          const int g = std::max(gm, std::min({gm + extra, nc, kMaxG}));
          gs[(size_t)i + 1] = gs[(size_t)i] + g;
          smem = std::max(smem, pchol_smem(nc, g));
        }
        DBuf<int> dgs;
        DBuf<unsigned int> dbar;
        dgs.reserve(gs.size(), s);
        dgs.upload(gs.data(), 0, gs.size(), s);
        dbar.reserve((size_t)cn, s);
        HCK(cudaMemsetAsync(dbar.p, 0, sizeof(unsigned int) * (size_t)cn, s));
        HCK(launch_pchol_coop(dtk + c0, cn, dgs.p, gs[(size_t)cn], dbar.p, smem, A, opt.eps, s));
        ++g_launches;
        dgs.release(s);
        dbar.release(s);
        c0 += cn;
      }
      dg.release(s);
      dr.release(s);
    } else {
      // few groups (exact-order batches): all SMs, split over the groups in
      // proportion to their work (nq * nc), at most one CTA per column; more
      // groups than SMs are run in several cooperative launches
      const int cap = std::max(1, cpqr_coop_capacity(sizeof(double) * (size_t)max_nq));
      for (int c0 = 0; c0 < n; c0 += cap) {
        const int cn = std::min(cap, n - c0);
        double tot = 0;
        for (int i = 0; i < cn; ++i) tot += (double)huge[(size_t)(lo + c0 + i)].nq * huge[(size_t)(lo + c0 + i)].nc;
        std::vector<int> gsz((size_t)cn, 1);
        int used = cn;
        for (int i = 0; i < cn; ++i) {  // extra CTAs beyond the one each group gets
          const SkelBigTask& H = huge[(size_t)(lo + c0 + i)];
          const int want = (int)((double)(cap - cn) * ((double)H.nq * H.nc) / std::max(tot, 1.0));
          const int g = std::max(1, std::min({1 + want, H.nc, kMaxG}));
          used += g - 1;
          gsz[(size_t)i] = g;
        }
        (void)used;
        std::vector<int> gs((size_t)cn + 1, 0);
        for (int i = 0; i < cn; ++i) gs[(size_t)i + 1] = gs[(size_t)i] + gsz[(size_t)i];
        DBuf<int> dgs;
        DBuf<unsigned int> dbar;
        dgs.reserve(gs.size(), s);
        dgs.upload(gs.data(), 0, gs.size(), s);
        dbar.reserve((size_t)cn, s);
        HCK(cudaMemsetAsync(dbar.p, 0, sizeof(unsigned int) * (size_t)cn, s));
        HCK(launch_cpqr_coop(dtk + c0, cn, dgs.p, gs[(size_t)cn], dbar.p, max_nq, A, opt.eps, s));
        ++g_launches;
        dgs.release(s);
        dbar.release(s);
      }
    }
    launch_skelbig_sort(dtk, n, AH, inner, dmin, dscale, s);
    // the tail: on the tail stream once the ID, the sort and this batch's
    // uploads (all on the main stream) are done
    const cudaStream_t ts = tail_stream();
    if (ts != s) {
      HCK(cudaEventRecord(ev_id, s));
      HCK(cudaStreamWaitEvent(ts, ev_id, 0));
      tail_pending = true;
    }
    launch_skelbig_tinit(dtk, d10.p, (int)wrow.size(), A, ts);
    for (int bb = ntb - 1; bb >= 0; --bb) {
      launch_skelbig_tsolve(dtk, d2.p, (int)wt.size(), bb * 64, A, ts);
      launch_skelbig_tupdate(dtk, d11.p + tuo[(size_t)bb], (int)(tuo[(size_t)bb + 1] - tuo[(size_t)bb]), bb * 64, A, ts);
      g_launches += 2;
    }
    launch_skelbig_tperm(dtk, d10.p, (int)wrow.size(), A, ts);
    launch_skelbig_congruence(dtk, d3.p, (int)wc0.size(), A, ts);
    launch_skelbig_congruence(dtk, d4.p, (int)wc1.size(), A, ts);
    launch_skelbig_symm(dtk, d5.p, (int)wsym.size(), A, dscale, ts);
    g_launches += 7;
    for (int p = 0; p < npanel; ++p) {
      const int p0 = p * kPanelB;
      launch_panel_chol(inner, d9.p + pco[(size_t)p], (int)(pco[(size_t)p + 1] - pco[(size_t)p]), p0, AH, dmin, ts);
      launch_panel_trsm(inner, d6.p + pto[(size_t)p], (int)(pto[(size_t)p + 1] - pto[(size_t)p]), p0, AH, ts);
      launch_panel_update(inner, d7.p + puo[(size_t)p], (int)(puo[(size_t)p + 1] - puo[(size_t)p]), p0, AH, ts);
      g_launches += 3;
    }
    launch_schur_tiles(inner, d8.p, (int)tiles.size(), AH, ts);
    launch_big_finish(inner, n, AH, dmin, dscale, ts);
    if (trace_on()) {
      HCK(cudaStreamSynchronize(ts));
      HTRACE("    huge: factor done (%d groups)", n);
    }
    g_launches += inv.launch(inner, AH, ts);
    if (trace_on()) { HCK(cudaStreamSynchronize(ts)); HTRACE("    huge: inverse done (%zu loc / %zu diag / %zu tiles)", inv.loc.size(), inv.diag.size(), inv.tiles.size()); }
    g_launches += 2;
    HCK(cudaGetLastError());
    d1.release(s);
    for (auto* d : {&d2, &d3, &d4, &d5, &d6, &d7, &d8, &d10, &d11}) d->release(ts);  // tail-stream order
    inv.release(ts);
    d9.release(ts);
  }

  // Split a level's records: large ones (by size) become tiled product phases
  // (TileOp), the rest stay one-CTA records.
  void build_solve_plan(LevelRec& L) {
    L.nall = (int)L.recs.size();
    for (const SolveRec& R : L.recs) {
      L.all_max_nc = std::max(L.all_max_nc, R.nc);
      L.all_max_nq = std::max(L.all_max_nq, R.nq);
      const double nc = R.nc, nq = R.nq;  // skeleton: r, k (T, P, W); else P, W
      L.solve_fac += nc * (nc + 1) / 2 + nc * nq + (L.kind == 1 ? nc * nq : 0.0);
      L.solve_rows += nc + nq;
    }
    meta.add(&L.d_all, L.recs);
    auto is_large = [](const SolveRec& R) { return R.nc > 96 || R.nq > 192; };
    std::vector<SolveRec> small, large;
    for (const SolveRec& R : L.recs) (is_large(R) ? large : small).push_back(R);
    L.nsmall = (int)small.size();
    L.max_nc = L.max_nq = 0;
    for (const SolveRec& R : small) { L.max_nc = std::max(L.max_nc, R.nc); L.max_nq = std::max(L.max_nq, R.nq); }
    meta.add(&L.d_recs, small);
    if (large.empty()) return;
    auto mk = [](int M, int K, int am, int64_t A_off, int64_t lda, int xm, int64_t xo, int sm, int64_t so, int dm,
                 int64_t dof, double alpha) {
      TileOp o;
      o.M = M; o.K = K; o.amode = am; o.A_off = A_off; o.lda = lda;
      o.xmode = xm; o.x_off = xo; o.smode = sm; o.s_off = so; o.dmode = dm; o.d_off = dof; o.alpha = alpha;
      return o;
    };
    const int nph = L.kind == 1 ? 3 : 2;
    std::vector<std::vector<TileOp>> F(nph), B(nph);
    int64_t rows = 0;
    for (const SolveRec& R : large) {
      if (L.kind != 1) {  // elimination record (and the terminal block): c then q in idx
        const int nc = R.nc, nq = R.nq;
        const int64_t c = R.idx_off, q = R.idx_off + nc, S = rows;
        rows += nc;
        F[0].push_back(mk(nc, nc, 0, R.C_off, 0, 0, c, -1, 0, 1, S, 1.0));               // S = P v_c
        if (nq > 0) F[1].push_back(mk(nq, nc, 3, R.W_off, nq, 1, S, -1, 0, 2, R.contrib_off, 1.0));  // g = W^T S
        F[1].push_back(mk(nc, 0, 2, 0, 0, 1, 0, 1, S, 0, c, 0.0));                        // v_c = S
        B[0].push_back(mk(nc, nq, 2, R.W_off, nq, 0, q, 0, c, 1, S, -1.0));              // T = v_c - W v_q
        B[1].push_back(mk(nc, nc, 1, R.C_off, 0, 1, S, -1, 0, 0, c, 1.0));               // v_c = P^T T
      } else {  // skeleton record: sk[k] then rd[r]; T (k x r), P (r x r), W (r x k)
        const int r = R.nc, k = R.nq;
        const int64_t sk = R.idx_off, rd = R.idx_off + k, X = rows, S = rows + r;
        rows += 2 * r;
        F[0].push_back(mk(r, k, 3, R.T_off, r, 0, sk, 0, rd, 1, X, -1.0));   // X = v_rd - T^T v_sk
        F[1].push_back(mk(r, r, 0, R.C_off, 0, 1, X, -1, 0, 1, S, 1.0));     // S = P X
        F[2].push_back(mk(k, r, 3, R.W_off, k, 1, S, 0, sk, 0, sk, -1.0));   // v_sk -= W^T S
        F[2].push_back(mk(r, 0, 2, 0, 0, 1, 0, 1, S, 0, rd, 0.0));           // v_rd = S
        B[0].push_back(mk(r, k, 2, R.W_off, k, 0, sk, 0, rd, 1, X, -1.0));   // X = v_rd - W v_sk
        B[1].push_back(mk(r, r, 1, R.C_off, 0, 1, X, -1, 0, 0, rd, 1.0));    // v_rd = P^T X
        B[2].push_back(mk(k, r, 2, R.T_off, r, 0, rd, 0, sk, 0, sk, -1.0));  // v_sk -= T v_rd
      }
    }
    F_->tile_rows = std::max(F_->tile_rows, rows);
    auto upload = [&](std::vector<std::vector<TileOp>>& ops, std::vector<LevelRec::Phase>& out) {
      out.reserve(out.size() + ops.size());  // slots registered below stay put
      for (auto& v : ops) {
        std::vector<int2> work;
        for (int i = 0; i < (int)v.size(); ++i)
          for (int i0 = 0; i0 < std::max(v[(size_t)i].M, 1); i0 += 64) work.push_back(make_int2(i, i0));
        out.emplace_back();
        LevelRec::Phase& P = out.back();
        meta.add(&P.d_ops, v);
        meta.add(&P.d_work, work);
        P.nwork = (int)work.size();
      }
    };
    upload(F, L.fwd_ph);
    upload(B, L.bwd_ph);
  }

  // Partitioned solve plans of a sharded factorization (the
  // solve "same partition"): each rank runs the records it owns, and a row
  // of the solve vector moves only when a rank is about to read it while
  // its current value lives elsewhere.  The plan replays both sweeps over
  // the (replicated) record structure with a bitmask of the ranks holding
  // each row's current value:
  //  - forward elimination: a record reads v_c on its owner; the reduction
  //    of a neighbour row q runs on the rank that next reads q in the forward
  //    sweep (its contribution rows from other ranks' records travel there,
  //    and the reduction sums them in record order -- the single-GPU sums);
  //  - forward skeleton / backward: a record reads (and writes) its rows on
  //    its owner; backward eliminations read their neighbour rows too.
  // After the backward sweep each row's holder supplies it to the result.
  void build_shard_solve() {
    const size_t nl = F->levels.size();
    if (P > 32) throw Fail{HIFDE_BADARG, "partitioned solve: more than 32 ranks"};
    std::vector<const Reduction*> red(nl, nullptr);
    for (auto& pr : reductions) red[pr.first] = &pr.second;
    for (const LevelRec& L : F->levels)
      if (L.rec_own.size() != L.recs.size()) throw Fail{HIFDE_INTERNAL, "partitioned solve: record owners missing"};
    // the index arena as the kernels left it (sk / rd lists of every group)
    std::vector<int32_t> hidx(F->idx.n);
    HCK(cudaMemcpyAsync(hidx.data(), F->idx.p, F->idx.n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    const int32_t* hx = hidx.data();
    auto rows_of = [&](const LevelRec& L, const SolveRec& R, bool with_q) {
      // kind 1: sk[k] then rd[r] (all read); else the cell, then its neighbours
      const int64_t n = L.kind == 1 ? (int64_t)R.nc + R.nq : (with_q ? (int64_t)R.nc + R.nq : (int64_t)R.nc);
      return std::make_pair(hx + R.idx_off, n);
    };
    // next forward reader of each row -> the rank reducing it at each level
    std::vector<uint8_t> nxt((size_t)N, 0);
    std::vector<std::vector<uint8_t>> ered(nl);
    for (size_t li = nl; li-- > 0;) {
      const LevelRec& L = F->levels[li];
      if (red[li]) {
        ered[li].resize(red[li]->targets.size());
        for (size_t i = 0; i < red[li]->targets.size(); ++i) ered[li][i] = nxt[(size_t)red[li]->targets[i]];
      }
      for (size_t t = 0; t < L.recs.size(); ++t) {
        const auto rr = rows_of(L, L.recs[t], false);
        for (int64_t j = 0; j < rr.second; ++j) nxt[(size_t)rr.first[j]] = L.rec_own[t];
      }
    }
    const uint32_t all = P == 32 ? 0xFFFFFFFFu : ((1u << P) - 1);
    std::vector<uint32_t> valid((size_t)N, all);
    // ranks receiving a row in the current exchange: not a source before it lands
    std::vector<uint32_t> adding((size_t)N, 0);
    std::vector<int32_t> touched;
    std::vector<std::vector<int32_t>> pend((size_t)P * P);
    auto need = [&](int o, int32_t d) {
      const uint32_t m = valid[(size_t)d];
      uint32_t& a = adding[(size_t)d];
      if ((m | a) >> o & 1u) return;
      pend[(size_t)__builtin_ctz(m) * P + o].push_back(d);
      if (a == 0) touched.push_back(d);
      a |= 1u << o;
    };
    auto flush = [&](LevelRec::XStep& X) {
      for (int32_t d : touched) {
        valid[(size_t)d] |= adding[(size_t)d];
        adding[(size_t)d] = 0;
      }
      touched.clear();
      std::vector<int32_t> rows;
      for (int a = 0; a < P; ++a)
        for (int b = 0; b < P; ++b) {
          std::vector<int32_t>& v = pend[(size_t)a * P + b];
          if (v.empty()) continue;
          X.pairs.push_back(LevelRec::XPair{a, b, (int64_t)rows.size(), (int64_t)v.size()});
          rows.insert(rows.end(), v.begin(), v.end());
          v.clear();
        }
      meta.add(&X.d_rows, rows);
    };
    for (size_t li = 0; li < nl; ++li) {  // forward sweep
      LevelRec& L = F->levels[li];
      for (size_t t = 0; t < L.recs.size(); ++t) {
        const auto rr = rows_of(L, L.recs[t], false);
        for (int64_t j = 0; j < rr.second; ++j) need(L.rec_own[t], rr.first[j]);
      }
      const Reduction* R = red[li];
      if (R)
        for (size_t i = 0; i < R->targets.size(); ++i) need(ered[li][i], R->targets[i]);
      flush(L.xs[0]);
      if (R) {  // contribution rows to the reducing rank
        std::vector<uint8_t> cown((size_t)L.ncontrib, 0);
        for (size_t t = 0; t < L.recs.size(); ++t)
          std::fill_n(cown.begin() + L.recs[t].contrib_off, L.recs[t].nq, L.rec_own[t]);
        for (size_t i = 0; i < R->targets.size(); ++i)
          for (int64_t e = R->ptr[i]; e < R->ptr[i + 1]; ++e) {
            const int64_t row = R->ent[(size_t)e];
            if (cown[(size_t)row] != ered[li][i]) pend[(size_t)cown[(size_t)row] * P + ered[li][i]].push_back((int32_t)row);
          }
      }
      flush(L.xs[1]);
      for (size_t t = 0; t < L.recs.size(); ++t) {
        const auto rr = rows_of(L, L.recs[t], false);
        for (int64_t j = 0; j < rr.second; ++j) valid[(size_t)rr.first[j]] = 1u << L.rec_own[t];
      }
      if (R)
        for (size_t i = 0; i < R->targets.size(); ++i) valid[(size_t)R->targets[i]] = 1u << ered[li][i];
    }
    for (size_t li = nl; li-- > 0;) {  // backward sweep
      LevelRec& L = F->levels[li];
      for (size_t t = 0; t < L.recs.size(); ++t) {
        const auto rr = rows_of(L, L.recs[t], true);
        for (int64_t j = 0; j < rr.second; ++j) need(L.rec_own[t], rr.first[j]);
      }
      flush(L.xs[2]);
      for (size_t t = 0; t < L.recs.size(); ++t) {
        const auto rr = rows_of(L, L.recs[t], false);
        for (int64_t j = 0; j < rr.second; ++j) valid[(size_t)rr.first[j]] = 1u << L.rec_own[t];
      }
    }
    std::vector<uint8_t> holder((size_t)N);
    for (int64_t d = 0; d < N; ++d) {
      holder[(size_t)d] = (uint8_t)__builtin_ctz(valid[(size_t)d]);
      if (emu && holder[(size_t)d] != 0) pend[(size_t)holder[(size_t)d] * P].push_back((int32_t)d);
    }
    meta.add(&F->d_holder, holder);
    flush(F->gather);
    // each rank's records and reduction targets
    for (size_t li = 0; li < nl; ++li) {
      LevelRec& L = F->levels[li];
      L.rank_view.resize((size_t)P);
      for (int r = rank_lo(); r < rank_hi(); ++r) {
        LevelRec& V = L.rank_view[(size_t)r];
        V.kind = L.kind;
        V.tag = L.tag;
        V.ncontrib = L.ncontrib;
        for (size_t t = 0; t < L.recs.size(); ++t)
          if (L.rec_own[t] == r) V.recs.push_back(L.recs[t]);
        build_solve_plan(V);
        // the whole level's kernel choice (the same arithmetic as its single sweep)
        V.max_nc = L.max_nc;
        V.max_nq = L.max_nq;
        V.recs.clear();
        V.recs.shrink_to_fit();
        if (const Reduction* R = red[li]) {
          std::vector<int32_t> tg;
          std::vector<int64_t> ptr{0}, ent;
          for (size_t i = 0; i < R->targets.size(); ++i) {
            if (ered[li][i] != r) continue;
            tg.push_back(R->targets[i]);
            ent.insert(ent.end(), R->ent.begin() + R->ptr[i], R->ent.begin() + R->ptr[i + 1]);
            ptr.push_back((int64_t)ent.size());
          }
          V.ntargets = (int)tg.size();
          meta.add(&V.d_targets, tg);
          meta.add(&V.d_ptr, ptr);
          meta.add(&V.d_ent, ent);
        }
      }
    }
    if (trace_on())
      for (size_t li = 0; li < nl; ++li) {
        const LevelRec& L = F->levels[li];
        std::string o;
        for (int k = 0; k < 3; ++k) {
          o += " |";
          for (const auto& p : L.xs[k].pairs) o += " " + std::to_string(p.src) + ">" + std::to_string(p.dst) + ":" + std::to_string(p.cnt);
        }
        o += " | views";
        for (const LevelRec& V : L.rank_view)
          o += " " + std::to_string(V.nsmall) + "/" + std::to_string(V.nall) + "/" + std::to_string(V.fwd_ph.size()) + "/" + std::to_string(V.ntargets);
        HTRACE("part level %g kind %d recs %zu:%s", L.tag, L.kind, L.recs.size(), o.c_str());
      }
    F->part = true;
    F->emu = emu;
    F->me = me;
    F->comm = comm;
    F->whole = !real;
  }

  // =========================================================================
  // Device symbolic mode (symbolic.cu): the level's partition, fronts, task
  // tables and block-table updates run on the GPU; the host only sizes the
  // arenas (one small readback per level) and launches.  Used from level 0
  // while the levels are interior / interface partitions; dev_to_host()
  // hands the state to the host analysis before the first level it cannot
  // take (adaptive hifde3x cells, large skeleton groups, the terminal block).
  // =========================================================================
  struct SymScalars {
    int64_t nact, nalive, nblk, red_nt, pred_alloc;
    int32_t ng, nretry, fatal, pred_ovf, nretry2, pad_;
  };
  bool dev_mode = false;
  SymWork symw;
  DBuf<int32_t> sy_act, sy_keys, sy_skeys, sy_gmem, sy_head, sy_group_of;
  DBuf<int64_t> sy_goff;
  DBuf<uint8_t> sy_alive;  // block alive flags (device mode)
  DBuf<int32_t> sy_alist, sy_mcnt, sy_mptr, sy_mblk;
  DBuf<int32_t> sy_nq, sy_nb, sy_maxnb, sy_npred, sy_flag, sy_retry, sy_retry2;
  DBuf<int64_t> sy_inc, sy_exc;  // ElimInc / SkelInc storage (8 words per group)
  DBuf<int32_t> sy_preds, sy_b0, sy_b1, sy_changed, sy_depth, sy_depth2, sy_iota, sy_order;
  DBuf<int64_t> sy_pred_ptr, sy_cl_rel, sy_pred_start;
  DBuf<int32_t> sy_pred_tmp;
  DBuf<ElimTask> sy_small, sy_big;
  DBuf<SkelTask> sy_tasks;
  DBuf<int32_t> sy_red_key, sy_red_key2;
  DBuf<int64_t> sy_red_val;
  DBuf<double4> sy_cellstat;
  DBuf<uint8_t> sy_cellcls;
  DBuf<int2> sy_fin;
  DBuf<int> sy_done;
  SymScalars* d_scal = nullptr;
  LevelTotals* d_tot = nullptr;
  LevelStat* d_lstat = nullptr;
  int lstat_cap = 0, nlstat = 0;
  SymScalars* h_scal = nullptr;  // pinned
  LevelTotals* h_tot = nullptr;  // pinned
  int64_t nblk_ub = 0;           // host bound on the device block count
  int64_t nact_ub = 0;           // host bound on the active count
  int last_dev_level = -1;       // LevelRec index of the previous device level (its active_after)
  std::vector<size_t> dev_levels;  // LevelRec indices of the device levels

  void* dev_alloc(size_t bytes) {
    void* q = nullptr;
    HCK(cudaMallocAsync(&q, std::max<size_t>(bytes, 16), s));
    F->dev_allocs.push_back(q);
    return q;
  }

  void dev_init() {
    const int cap = 3 * std::max(g.nlevels, 1) + 8;
    HCK(cudaMallocAsync((void**)&d_scal, sizeof(SymScalars), s));
    HCK(cudaMallocAsync((void**)&d_tot, sizeof(LevelTotals), s));
    HCK(cudaMallocAsync((void**)&d_lstat, sizeof(LevelStat) * (size_t)cap, s));
    HCK(cudaMemsetAsync(d_scal, 0, sizeof(SymScalars), s));
    HCK(cudaMemsetAsync(d_lstat, 0, sizeof(LevelStat) * (size_t)cap, s));
    lstat_cap = cap;
    static SymScalars* hs = nullptr;
    static LevelTotals* ht = nullptr;
    if (!hs) {
      HCK(cudaHostAlloc((void**)&hs, sizeof(SymScalars), cudaHostAllocDefault));
      HCK(cudaHostAlloc((void**)&ht, sizeof(LevelTotals), cudaHostAllocDefault));
    }
    h_scal = hs;
    h_tot = ht;
    sy_group_of.reserve((size_t)N, s);
    HCK(cudaMemsetAsync(sy_group_of.p, 0xFF, sizeof(int32_t) * (size_t)N, s));
    nact_ub = N;
    nblk_ub = 0;
  }

  void dev_release() {
    for (auto* b : {&sy_act, &sy_keys, &sy_skeys, &sy_gmem, &sy_head, &sy_group_of, &sy_alist, &sy_mcnt, &sy_mptr,
                    &sy_mblk, &sy_nq, &sy_nb, &sy_maxnb, &sy_npred, &sy_flag, &sy_retry, &sy_retry2, &sy_preds, &sy_b0, &sy_b1,
                    &sy_changed, &sy_red_key, &sy_red_key2, &sy_depth, &sy_depth2, &sy_iota, &sy_order})
      b->release(s);
    for (auto* b : {&sy_goff, &sy_inc, &sy_exc, &sy_pred_ptr, &sy_cl_rel, &sy_red_val, &sy_pred_start}) b->release(s);
    sy_pred_tmp.release(s);
    sy_alive.release(s);
    sy_cellcls.release(s);
    sy_small.release(s);
    sy_big.release(s);
    sy_tasks.release(s);
    sy_cellstat.release(s);
    sy_fin.release(s);
    sy_done.release(s);
    if (symw.cub_tmp) cudaFreeAsync(symw.cub_tmp, s);
    symw.cub_tmp = nullptr;
    if (symw.stat_part) cudaFreeAsync(symw.stat_part, s);
    symw.stat_part = nullptr;
    symw.cub_bytes = 0;
    for (void** q : {(void**)&d_scal, (void**)&d_tot, (void**)&d_lstat})
      if (*q) {
        cudaFreeAsync(*q, s);
        *q = nullptr;
      }
  }

  // block-table capacity for `ub` blocks (new alive flags zero; growth keeps
  // every existing entry)
  void dev_blocks_reserve(int64_t ub) {
    const size_t old = sy_alive.cap;
    d_blk_dof_off.n = d_blk_dof_off.cap;
    d_blk_n.n = d_blk_n.cap;
    d_blk_val_off.n = d_blk_val_off.cap;
    sy_alive.n = sy_alive.cap;
    d_blk_dof_off.reserve((size_t)ub, s);
    d_blk_n.reserve((size_t)ub, s);
    d_blk_val_off.reserve((size_t)ub, s);
    sy_alive.reserve((size_t)ub, s);
    if (sy_alive.cap > old) HCK(cudaMemsetAsync(sy_alive.p + old, 0, sy_alive.cap - old, s));
  }

  // per-group scratch of the symbolic pass for up to `ng_ub` groups
  void dev_group_reserve(int64_t ng_ub) {
    for (auto* b : {&sy_nq, &sy_nb, &sy_maxnb, &sy_npred, &sy_flag, &sy_retry, &sy_retry2})
      b->reserve((size_t)ng_ub + 1, s);
    sy_inc.reserve((size_t)8 * (ng_ub + 1), s);
    sy_exc.reserve((size_t)8 * (ng_ub + 1), s);
    sy_goff.reserve((size_t)ng_ub + 2, s);
  }

  // pending status words + totals and scalars to the host (the level's sync)
  void dev_sync_totals(bool statuses = true) {
    HCK(cudaMemcpyAsync(h_tot, d_tot, sizeof(LevelTotals), cudaMemcpyDeviceToHost, s));
    HCK(cudaMemcpyAsync(h_scal, d_scal, sizeof(SymScalars), cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    if (statuses) check_status();  // (not while numeric kernels may still run on the other stream)
  }

  // Partition + membership + count pass of a level.  kind 0 interior cells,
  // 1 edges, 2 faces.  Returns false when the level overflowed the device
  // front tiers (the host takes over).
  bool dev_front_count(int ell, int kind, SymFront& P, int64_t& ng_ub) {
    a0_pattern_ready();  // (the values are the numeric kernels' -- arenas())
    // kind 0 cells, 1/2 interfaces, 3 the terminal block (every active DOF, key 0)
    const bool iface = kind == 1 || kind == 2;
    const int w = g.m << std::min(ell, 30), k = kind == 3 ? 0 : g.n / w;
    int64_t nkeys = 1;
    if (kind != 3)
      for (int ax = 0; ax < g.dim; ++ax) nkeys *= k;
    if (iface) nkeys *= g.dim;
    ng_ub = nkeys;
    // active list (its count is the previous device level's active_after)
    sy_act.reserve((size_t)N, s);
    HCK(sym_active_list(d_active, N, sy_act.p, &d_scal->nact, symw, s));
    if (last_dev_level >= 0)
      HCK(sym_copy_count(&d_scal->nact, &d_lstat[F->levels[(size_t)last_dev_level].dev_stat].active_after, s));
    for (auto* b : {&sy_keys, &sy_skeys, &sy_gmem, &sy_head}) b->reserve((size_t)nact_ub + 1, s);
    dev_group_reserve(ng_ub);
    SymPartArgs A;
    A.act = sy_act.p;
    A.nact = &d_scal->nact;
    A.nact_ub = nact_ub;
    A.dim = g.dim;
    A.side = g.n - 1;
    A.w = w;
    A.k = k;
    A.kind = kind;
    A.nkeys = (int32_t)nkeys;
    A.keys = sy_keys.p;
    A.skeys = sy_skeys.p;
    A.gmem = sy_gmem.p;
    A.head = sy_head.p;
    A.goff = sy_goff.p;
    A.ng = &d_scal->ng;
    A.group_of = iface ? sy_group_of.p : nullptr;
    HCK(sym_partition(A, symw, s));
    // membership of the live blocks over the active DOFs
    sy_alist.reserve((size_t)std::max<int64_t>(nblk_ub, 1), s);
    sy_mcnt.reserve((size_t)N + 1, s);
    sy_mptr.reserve((size_t)N + 1, s);
    int64_t ment = 0;  // bound on the membership entries: the live blocks' orders
    ment = std::max<int64_t>(ment, mem_entries_ub);
    sy_mblk.reserve((size_t)std::max<int64_t>(ment, 1), s);
    SymMemberArgs M;
    M.blk_alive = sy_alive.p;
    M.nblk_ub = nblk_ub;
    M.alive_list = sy_alist.p;
    M.nalive = &d_scal->nalive;
    M.blk_n = d_blk_n.p;
    M.blk_dof_off = d_blk_dof_off.p;
    M.idx = F->idx.p;
    M.active = d_active;
    M.N = N;
    M.cnt = sy_mcnt.p;
    M.mptr = sy_mptr.p;
    M.mblk = sy_mblk.p;
    if (nblk_ub > 0) {
      HCK(sym_membership(M, symw, s));
    } else {
      HCK(cudaMemsetAsync(sy_mptr.p, 0, sizeof(int32_t) * ((size_t)N + 1), s));
    }
    std::memset(&P, 0, sizeof P);
    P.goff = sy_goff.p;
    P.gmem = sy_gmem.p;
    P.ng = &d_scal->ng;
    P.mptr = sy_mptr.p;
    P.mblk = sy_mblk.p;
    P.blk_n = d_blk_n.p;
    P.blk_dof_off = d_blk_dof_off.p;
    P.idx = F->idx.p;
    P.indptr = d_indptr;
    P.indices = d_indices;
    P.active = d_active;
    P.group_of = iface ? sy_group_of.p : nullptr;
    P.nq = sy_nq.p;
    P.nb = sy_nb.p;
    P.maxnb = sy_maxnb.p;
    P.npred = sy_npred.p;
    P.flag = sy_flag.p;
    P.retry = sy_retry.p;
    P.nretry = &d_scal->nretry;
    P.retry2 = sy_retry2.p;
    P.nretry2 = &d_scal->nretry2;
    P.fatal = &d_scal->fatal;
    P.pred_tmp = nullptr;
    if (iface && opt.order_mode != HIFDE_ORDER_SNAPSHOT) {  // predecessor lists for the chain
      const int64_t cap = 64 * (ng_ub + 1);
      sy_pred_tmp.reserve((size_t)cap, s);
      sy_pred_start.reserve((size_t)ng_ub + 1, s);
      P.pred_tmp = sy_pred_tmp.p;
      P.pred_start = sy_pred_start.p;
      P.pred_alloc = &d_scal->pred_alloc;
      P.pred_cap = cap;
      P.pred_ovf = &d_scal->pred_ovf;
      HCK(cudaMemsetAsync(&d_scal->pred_alloc, 0, sizeof(int64_t), s));
      HCK(cudaMemsetAsync(&d_scal->pred_ovf, 0, sizeof(int32_t), s));
    }
    HCK(cudaMemsetAsync(sy_npred.p, 0, sizeof(int32_t) * ((size_t)ng_ub + 1), s));
    HCK(sym_fronts_count(P, s));
    return true;
  }
  int64_t mem_entries_ub = 0;  // bound on sum of the live blocks' orders

  // register the level's LevelStat slot
  int dev_stat_slot(LevelRec& L) {
    if (nlstat >= lstat_cap) throw Fail{HIFDE_INTERNAL, "device level statistics overflow"};
    L.dev_stat = nlstat++;
    return L.dev_stat;
  }

  // ---- elimination level ---------------------------------------------------
  // returns false if the host must take this level (state handed over)
  bool dev_elimination_level(int ell, double tag, LevelRec& L, bool top = false) {
    const double t_begin = now_s();
    join_inv();  // its analysis rewrites the big-cell task table
    L.kind = top ? 2 : 0;
    L.lap(nullptr);
    HCK(cudaEventCreate(&L.ev0));
    HCK(cudaEventCreate(&L.ev1));
    HCK(cudaEventRecord(L.ev0, s));
    const int kls = F->klog.begin("symbolic_device", tag, 0, 0, 0, s);
    SymFront P;
    int64_t ng_ub = 0;
    dev_front_count(ell, top ? 3 : 0, P, ng_ub);
    ElimInc* inc = reinterpret_cast<ElimInc*>(sy_inc.p);
    ElimInc* exc = reinterpret_cast<ElimInc*>(sy_exc.p);
    HCK(sym_elim_sizes(P, top ? 1 : 0, (int)ng_ub, inc, exc, d_tot, symw, s));
    dev_sync_totals();
    L.lap("dev-count");
    if (h_scal->fatal) {
      F->klog.end(kls, s);
      HCK(cudaEventRecord(L.ev1, s));
      return false;
    }
    nact_ub = h_scal->nact;
    const LevelTotals T = *h_tot;
    const int64_t ng = T.ng;
    L.ngroups = ng;
    L.max_front = T.max_front;
    const int st = dev_stat_slot(L);
    // arenas
    const int64_t idx_base = (int64_t)F->idx.bump((size_t)T.sum[0], s);
    lists.reserve((size_t)std::max<int64_t>(T.sum[1], 1), s);
    lists.n = (size_t)T.sum[1];
    const int64_t fac_base = (int64_t)F->fac.bump((size_t)T.sum[2], s);
    const int64_t bv_base = T.sum[3] ? (int64_t)bvals.bump((size_t)T.sum[3], s) : 0;
    dev_blocks_reserve(nblk_ub + T.sum[5] + 1);
    sy_small.reserve((size_t)std::max<int64_t>(T.sum[6], 1), s);
    sy_big.reserve((size_t)std::max<int64_t>(T.sum[7], 1), s);
    sy_red_key.reserve((size_t)T.sum[4] + 1, s);
    sy_red_key2.reserve((size_t)T.sum[4] + 1, s);
    sy_red_val.reserve((size_t)T.sum[4] + 1, s);
    sy_cellstat.reserve((size_t)ng + 1, s);
    sy_cellcls.reserve((size_t)ng + 1, s);
    SolveRec* recs = (SolveRec*)dev_alloc(sizeof(SolveRec) * (size_t)ng);
    hifde_record_t* xr = (hifde_record_t*)dev_alloc(sizeof(hifde_record_t) * (size_t)ng);
    int32_t* red_t = (int32_t*)dev_alloc(sizeof(int32_t) * ((size_t)T.sum[4] + 1));
    int64_t* red_ptr = (int64_t*)dev_alloc(sizeof(int64_t) * ((size_t)T.sum[4] + 2));
    int64_t* red_ent = (int64_t*)dev_alloc(sizeof(int64_t) * ((size_t)T.sum[4] + 1));
    int64_t* red_cnt = reinterpret_cast<int64_t*>(sy_inc.p);  // the increments are no longer needed after the fill
    // fronts into the arenas
    P.exc = sy_exc.p;
    P.exc_stride = kElimIncN;
    P.o_nf = 0;
    P.o_nb = 1;
    P.o_pred = 0;
    P.idx_base = idx_base;
    P.idx_out = F->idx.p;
    P.idx = F->idx.p;  // the arenas may have moved since the count pass
    P.blk_n = d_blk_n.p;
    P.blk_dof_off = d_blk_dof_off.p;
    P.lists = lists.p;
    P.preds = nullptr;
    HCK(sym_fronts_fill(P, s));
    ElimFillArgs A;
    A.is_top = top ? 1 : 0;
    A.idx_base = idx_base;
    A.fac_base = fac_base;
    A.bv_base = bv_base;
    A.exc = exc;
    A.small = sy_small.p;
    A.big = sy_big.p;
    A.recs = recs;
    A.xrec = xr;
    A.blk_dof_off = d_blk_dof_off.p;
    A.blk_n = d_blk_n.p;
    A.blk_val_off = d_blk_val_off.p;
    A.blk_alive = sy_alive.p;
    A.nblk = &d_scal->nblk;
    A.newblk_total = &d_tot->sum[5];
    A.lists = lists.p;
    A.idx = F->idx.p;
    A.red_key = sy_red_key.p;
    A.red_val = sy_red_val.p;
    A.red_key2 = sy_red_key2.p;
    A.red_ent = red_ent;
    A.red_targets = red_t;
    A.red_cnt = red_cnt;
    A.red_ptr = red_ptr;
    A.red_nt = &d_scal->red_nt;
    A.N = N;
    A.cellstat = sy_cellstat.p;
    A.cellcls = sy_cellcls.p;
    A.stat = d_lstat + st;
    sy_inc.reserve((size_t)std::max<int64_t>(8 * (ng_ub + 1), T.sum[4] + 2), s);
    red_cnt = reinterpret_cast<int64_t*>(sy_inc.p);
    A.red_cnt = red_cnt;
    HCK(sym_elim_fill(P, A, T.sum[4], symw, s));
    HCK(sym_copy_count(&d_scal->red_nt, &d_lstat[st].ntargets, s));
    HCK(sym_retire_cells(sy_gmem.p, sy_goff.p, &d_scal->ng, d_active, s));
    if (!sharded()) {  // the next skeleton level's analysis may start from here
      sym_stream();
      HCK(cudaEventRecord(ev_symdone, s));
      symdone_ok = true;
    }
    F->klog.end(kls, s);
    nblk_ub += T.sum[5];
    mem_entries_ub += T.sum[4];
    L.t_sym = now_s() - t_begin;
    // numeric launches
    Arenas Ar = arenas();
    const int64_t nsmall = T.sum[6], nbig = T.sum[7];
    if (nsmall) {
      const int64_t st_small = (int64_t)status.bump((size_t)nsmall, s);
      pending.push_back({st_small, nsmall, tag, top ? "top block" : "cell"});
      Ar.status = status.p + st_small;
      const int kl = F->klog.begin(top ? "elim_small_kernel(top)" : "elim_small_kernel", tag, 0, 0, 0, s);
      launch_elim_small(sy_small.p, (int)nsmall, Ar, (size_t)T.smem, T.max_small_nf <= 64 ? 128 : 256, s);
      F->klog.end(kl, s);
      ++g_launches;
    }
    if (nbig) {  // the blocked path builds its work lists from (nc, nq) on the host
      std::vector<ElimTask> big((size_t)nbig);
      HCK(cudaMemcpyAsync(big.data(), sy_big.p, sizeof(ElimTask) * (size_t)nbig, cudaMemcpyDeviceToHost, s));
      HCK(cudaStreamSynchronize(s));
      launch_big_cells(big, sy_big.p, (size_t)T.smem_big, Ar, tag, top, 0, 0, !sharded() && !top);
    }
    HCK(cudaEventRecord(L.ev1, s));
    if (top) F->s_top = nact_ub;
    HCK(cudaGetLastError());
    L.ncontrib = T.sum[4];
    F->max_contrib = std::max(F->max_contrib, L.ncontrib);
    L.d_xrec = xr;
    L.nxrec = ng;
    L.d_recs = recs;
    L.d_all = recs;
    L.d_targets = red_t;
    L.d_ptr = red_ptr;
    L.d_ent = red_ent;
    dev_levels.push_back((size_t)(&L - F->levels.data()));
    last_dev_level = (int)(&L - F->levels.data());
    L.lap("dev-launch");
    return true;
  }

  // ---- skeletonization level -----------------------------------------------
  bool dev_skeleton_level(int ell, int kind, double tag, LevelRec& L) {
    const double t_begin = now_s();
    L.kind = 1;
    L.lap(nullptr);
    HCK(cudaEventCreate(&L.ev0));
    HCK(cudaEventCreate(&L.ev1));
    HCK(cudaEventRecord(L.ev0, s));
    // overlap with the previous elimination's numeric kernels: the analysis
    // below runs on sym_s (swapped into `s`) from ev_symdone on
    const bool ovl = symdone_ok;
    symdone_ok = false;
    if (ovl) {
      if (++sym_overlaps == 1) std::swap(sym_s, sym_hi);
      HCK(cudaStreamWaitEvent(sym_s, ev_symdone, 0));
      std::swap(s, sym_s);
      std::swap(lists, lists_alt);
    }
    auto join = [&]() {  // back to the main stream, after the analysis
      if (!ovl) return;
      HCK(cudaEventRecord(ev_symjoin, s));
      std::swap(s, sym_s);
      HCK(cudaStreamWaitEvent(s, ev_symjoin, 0));
    };
    const int kls = F->klog.begin("symbolic_device", tag, 0, 0, 0, s);
    SymFront P;
    int64_t ng_ub = 0;
    dev_front_count(ell, 1 + kind, P, ng_ub);
    SkelInc* inc = reinterpret_cast<SkelInc*>(sy_inc.p);
    SkelInc* exc = reinterpret_cast<SkelInc*>(sy_exc.p);
    const bool gram_eps = opt.eps >= kGramMinEps;
    HCK(sym_skel_sizes(P, kPromoteWork, gram_eps ? 1 : 0, (int)ng_ub, inc, exc, d_tot, symw, s));
    const int iters = opt.exact_max_batches + 1;
    // AUTO: only whether the chain passes exact_max_batches matters (early exit of the relaxation)
    const int chain_cap = opt.order_mode == HIFDE_ORDER_AUTO ? opt.exact_max_batches : 0;
    const bool chain_early = P.pred_tmp != nullptr;
    if (chain_early) {  // the dependency chain from the count pass's lists: one readback for the level
      sy_b0.reserve((size_t)ng_ub + 1, s);
      sy_b1.reserve((size_t)ng_ub + 1, s);
      sy_changed.reserve((size_t)iters + 1, s);
      HCK(sym_skel_chain(sy_pred_start.p, sy_npred.p, sy_pred_tmp.p, &d_scal->ng, (int)ng_ub, iters, chain_cap,
                         sy_b0.p, sy_b1.p, sy_changed.p, d_tot, s));
    }
    dev_sync_totals(!ovl);
    L.lap("dev-count");
    const LevelTotals T = *h_tot;
    if (h_scal->fatal || T.any_mode2 || (g.dim == 3 && T.any_promote)) {
      HCK(sym_reset_groups(sy_gmem.p, sy_goff.p, &d_scal->ng, sy_group_of.p, s));
      F->klog.end(kls, s);
      join();
      HCK(cudaEventRecord(L.ev1, s));
      return false;
    }
    {  // an arena that must grow moves its contents: not while the elimination
       // (overlapped) or the deferred inverses write them
      const bool grow = F->idx.n + (size_t)(T.sum[0] + T.sum[6]) > F->idx.cap ||
                        F->fac.n + (size_t)T.sum[3] > F->fac.cap || bvals.n + (size_t)T.sum[4] > bvals.cap ||
                        (size_t)T.sum[2] > scratch.cap;
      if (grow && ovl) {
        HCK(cudaEventRecord(ev_symjoin, sym_s));
        HCK(cudaStreamWaitEvent(s, ev_symjoin, 0));
      }
      if (grow) join_inv();
    }
    nact_ub = h_scal->nact;
    const int64_t ng = T.ng;
    L.ngroups = ng;
    L.max_front = T.max_front;
    const int st = dev_stat_slot(L);
    scratch.n = 0;
    const int64_t idx_base = (int64_t)F->idx.bump((size_t)(T.sum[0] + T.sum[6]), s);
    lists.reserve((size_t)std::max<int64_t>(T.sum[1], 1), s);
    lists.n = (size_t)T.sum[1];
    const int64_t scr_base = T.sum[2] ? (int64_t)scratch.bump((size_t)T.sum[2], s) : 0;
    const int64_t fac_base = (int64_t)F->fac.bump((size_t)T.sum[3], s);
    const int64_t bv_base = (int64_t)bvals.bump((size_t)T.sum[4], s);
    sy_preds.reserve((size_t)T.sum[5] + 1, s);
    sy_pred_ptr.reserve((size_t)ng + 2, s);
    sy_cl_rel.reserve((size_t)ng + 1, s);
    sy_tasks.reserve((size_t)ng + 1, s);
    P.exc = sy_exc.p;
    P.exc_stride = kSkelIncN;
    P.o_nf = 0;
    P.o_nb = 1;
    P.o_pred = 5;
    P.idx_base = idx_base;
    P.idx_out = F->idx.p;
    P.idx = F->idx.p;  // the arenas may have moved since the count pass
    P.blk_n = d_blk_n.p;
    P.blk_dof_off = d_blk_dof_off.p;
    P.lists = lists.p;
    P.preds = sy_preds.p;
    HCK(sym_fronts_fill(P, s));
    SkelFillArgs A;
    A.idx_base = idx_base;
    A.scr_base = scr_base;
    A.fac_base = fac_base;
    A.bv_base = bv_base;
    A.tot_nf = T.sum[0];
    A.exc = exc;
    A.tasks = sy_tasks.p;
    A.pred_ptr = sy_pred_ptr.p;
    A.cl_rel = sy_cl_rel.p;
    A.idx = F->idx.p;
    HCK(sym_skel_fill(P, A, s));
    HCK(sym_reset_groups(sy_gmem.p, sy_goff.p, &d_scal->ng, sy_group_of.p, s));
    // exact or snapshot order (the host path's rule)
    bool exact = opt.order_mode == HIFDE_ORDER_EXACT;
    int nbatch = 1;
    if (opt.order_mode != HIFDE_ORDER_SNAPSHOT && ng > 1) {
      if (h_scal->pred_ovf) {  // the early lists overflowed: the chain over the filled CSR (second readback)
        sy_npred.reserve((size_t)ng + 1, s);
        sy_pred_start.reserve((size_t)ng + 1, s);
        HCK(cudaMemcpyAsync(sy_pred_start.p, sy_pred_ptr.p, sizeof(int64_t) * (size_t)ng, cudaMemcpyDeviceToDevice, s));
        HCK(sym_skel_chain(sy_pred_start.p, sy_npred.p, sy_preds.p, &d_scal->ng, (int)ng, iters, chain_cap, sy_b0.p,
                           sy_b1.p, sy_changed.p, d_tot, s));
        HCK(cudaMemcpyAsync(h_tot, d_tot, sizeof(LevelTotals), cudaMemcpyDeviceToHost, s));
        HCK(cudaStreamSynchronize(s));
      }
      nbatch = (int)h_tot->max_chain + 1;
      if (opt.order_mode == HIFDE_ORDER_AUTO) exact = nbatch <= opt.exact_max_batches;
    }
    L.nbatches = exact ? nbatch : 1;
    F->klog.end(kls, s);
    join();
    L.t_sym = now_s() - t_begin;
    L.lap("dev-fill");
    if (status.n + (size_t)ng > status.cap) join_inv();  // (the deferred inverses read their statuses)
    const int64_t st_off = (int64_t)status.bump((size_t)ng, s);
    HCK(cudaMemsetAsync(status.p + st_off, 0, (size_t)ng * sizeof(int), s));
    pending.push_back({st_off, ng, tag, "group"});
    kout.n = 0;
    kout.bump((size_t)ng, s);
    Arenas Ar = arenas();
    Ar.status = status.p + st_off;
    const bool one_launch = exact && ng > 1;
    const int nthr = (T.max_nc > 32 || T.max_nq > 128) ? 512 : 128;
    if (one_launch) {
      sy_done.reserve((size_t)ng + 1, s);
      HCK(cudaMemsetAsync(sy_done.p, 0, sizeof(int) * ((size_t)ng + 1), s));
      int cs = 0, ncls = 0;
      size_t smem_cl = 0;
      if (T.max_nc >= kClusterMinNc) {
        for (int csz : {4, 2}) {
          const size_t need = (size_t)(csz == 4 ? T.cl_need4 : T.cl_need2);
          if (need > kSmemCap) continue;
          const int capc = skel_cluster_capacity(need, csz);
          if (capc >= 1 && ng <= capc) {
            cs = csz;
            ncls = (int)std::min<int64_t>(ng, capc);
            smem_cl = need;
            break;
          }
        }
      }
      if (cs > 0) {
        const int64_t base = (int64_t)scratch.bump((size_t)T.sum[7], s);
        HCK(sym_skel_cluster_tasks(sy_tasks.p, sy_cl_rel.p, base, &d_scal->ng, (int)ng, s));
        Ar.scratch = scratch.p;
        const int kl = F->klog.begin("skel_cluster_kernel", tag, 0, 0, 0, s);
        HCK(launch_skel_cluster(sy_tasks.p, (int)ng, sy_pred_ptr.p, sy_preds.p, sy_done.p, Ar, opt.eps, smem_cl, ncls,
                                cs, s));
        F->klog.end(kl, s);
      } else {
        const int cap = skel_ordered_capacity((size_t)T.smem, nthr);
        if (cap < 1) throw Fail{HIFDE_CUDA, "ordered skeleton kernel cannot be resident"};
        // claim order: stably by dependency depth (the relaxation's result)
        for (auto* b : {&sy_depth, &sy_depth2, &sy_iota, &sy_order}) b->reserve((size_t)ng + 1, s);
        HCK(sym_skel_order(sy_b0.p, sy_b1.p, sy_changed.p, opt.exact_max_batches + 1, &d_scal->ng, (int)ng,
                           sy_depth.p, sy_depth2.p, sy_iota.p, sy_order.p, symw, s));
        const int kl = F->klog.begin("skel_ordered_kernel", tag, 0, 0, 0, s);
        HCK(launch_skel_ordered(sy_tasks.p, (int)ng, sy_pred_ptr.p, sy_preds.p, sy_order.p, sy_done.p, Ar, opt.eps,
                                (size_t)T.smem, nthr, (int)std::min<int64_t>(ng, cap), s));
        F->klog.end(kl, s);
      }
      ++g_launches;
    } else {
      const int kl = F->klog.begin("skel_kernel", tag, 0, 0, 0, s);
      launch_skel(sy_tasks.p, (int)ng, Ar, opt.eps, (size_t)T.smem, nthr, (int)T.max_nc, (int)T.max_nq, s);
      F->klog.end(kl, s);
      launch_apply_rd(sy_tasks.p, (int)ng, Ar, s);
      g_launches += 2;
    }
    // ranks known on the device: delta blocks, solve records, statistics
    SolveRec* recs = (SolveRec*)dev_alloc(sizeof(SolveRec) * (size_t)ng);
    hifde_record_t* xr = (hifde_record_t*)dev_alloc(sizeof(hifde_record_t) * (size_t)ng);
    dev_blocks_reserve(nblk_ub + ng + 1);
    sy_fin.reserve((size_t)2 * ng + 2, s);
    SkelFinishArgs Fa;
    Fa.inc = sy_fin.p;
    Fa.exc = sy_fin.p + ng + 1;
    Fa.recs = recs;
    Fa.xrec = xr;
    Fa.blk_dof_off = d_blk_dof_off.p;
    Fa.blk_n = d_blk_n.p;
    Fa.blk_val_off = d_blk_val_off.p;
    Fa.blk_alive = sy_alive.p;
    Fa.nblk = &d_scal->nblk;
    Fa.stat = d_lstat + st;
    HCK(sym_skel_finish(sy_tasks.p, kout.p, &d_scal->ng, (int)ng, Fa, symw, s));
    HCK(cudaEventRecord(L.ev1, s));
    HCK(cudaGetLastError());
    nblk_ub += ng;
    mem_entries_ub += T.sum[6];  // delta blocks: at most the groups' sizes
    L.d_xrec = xr;
    L.nxrec = ng;
    L.d_recs = recs;
    L.d_all = recs;
    dev_levels.push_back((size_t)(&L - F->levels.data()));
    last_dev_level = (int)(&L - F->levels.data());
    L.lap("dev-launch");
    return true;
  }

  // Hand the device state to the host analysis: block table, index-arena
  // mirror of the live blocks, active mask / list, membership.
  void dev_to_host() {
    if (!dev_mode) return;
    dev_mode = false;
    pat_wait();  // the host analysis reads the pattern
    join_inv();
    // the active list compacted on the device (an O(N) host scan of the mask
    // was ~3 ms at the end of config 3's factorization)
    sy_act.reserve((size_t)N + 1, s);
    HCK(sym_active_list(d_active, N, sy_act.p, &d_scal->nact, symw, s));
    HCK(cudaMemcpyAsync(h_scal, d_scal, sizeof(SymScalars), cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    const int64_t nb = h_scal->nblk;
    act.resize((size_t)h_scal->nact);
    if (!act.empty())
      HCK(cudaMemcpyAsync(act.data(), sy_act.p, sizeof(int32_t) * act.size(), cudaMemcpyDeviceToHost, s));
    blk_dof_off.resize((size_t)nb);
    blk_n.resize((size_t)nb);
    blk_val_off.resize((size_t)nb);
    blk_alive.resize((size_t)nb);
    bf_key.assign((size_t)nb, -2);
    bf_val.assign((size_t)nb, 0);
    if (nb) {
      HCK(cudaMemcpyAsync(blk_dof_off.data(), d_blk_dof_off.p, sizeof(int64_t) * (size_t)nb, cudaMemcpyDeviceToHost, s));
      HCK(cudaMemcpyAsync(blk_n.data(), d_blk_n.p, sizeof(int32_t) * (size_t)nb, cudaMemcpyDeviceToHost, s));
      HCK(cudaMemcpyAsync(blk_val_off.data(), d_blk_val_off.p, sizeof(int64_t) * (size_t)nb, cudaMemcpyDeviceToHost, s));
      HCK(cudaMemcpyAsync(blk_alive.data(), sy_alive.p, (size_t)nb, cudaMemcpyDeviceToHost, s));
    }
    active.resize((size_t)N);
    HCK(cudaMemcpyAsync(active.data(), d_active, (size_t)N, cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    prof.lap("h-tables");
    d_blk_dof_off.n = d_blk_n.n = d_blk_val_off.n = (size_t)nb;
    blk_uploaded = (size_t)nb;
    // index-arena mirror: the DOF lists of the live blocks
    const size_t nidx = F->idx.n;
    h_idx.resize(nidx);
    int64_t lo = (int64_t)nidx;
    for (int64_t b = 0; b < nb; ++b)
      if (blk_alive[(size_t)b]) lo = std::min(lo, blk_dof_off[(size_t)b]);
    if (lo < (int64_t)nidx)
      pinned_xfer().d2h(h_idx.data() + lo, F->idx.p + lo, (nidx - (size_t)lo) * sizeof(int32_t), s);
    idx_uploaded = nidx;
    prof.lap("h-idx");
    // active list and membership (active DOFs only: the host looks up
    // membership of active DOFs alone)
    if (last_dev_level >= 0) F->levels[(size_t)last_dev_level].active_after = (int64_t)act.size();
    prof.lap("h-act");
    member.reset();
    size_t nadd = 0;
    for (int64_t b = 0; b < nb; ++b)
      if (blk_alive[(size_t)b]) nadd += (size_t)blk_n[(size_t)b];
    member.ensure_room(nadd);
    const int nthu = nthreads;
#pragma omp parallel num_threads(nthu)
    {
      const int tid = omp_get_thread_num(), nth = omp_get_num_threads();
      const int64_t dlo = N * tid / nth, dhi = N * (tid + 1) / nth;
      for (int64_t b = 0; b < nb; ++b) {
        if (!blk_alive[(size_t)b]) continue;
        const int32_t* d = h_idx.data() + blk_dof_off[(size_t)b];
        for (int32_t i = 0; i < blk_n[(size_t)b]; ++i)
          if (d[i] >= dlo && d[i] < dhi && active[(size_t)d[i]]) member.add(d[i], (int32_t)b);
      }
    }
    prof.lap("h-member");
    // the upload cursor of the block table continues from here
  }

  // Device levels: statistics to the LevelRecs, solve metadata (device tables
  // when every record is small, else the host plan), kernel-log totals.
  void dev_finalize() {
    if (dev_levels.empty()) return;
    std::vector<LevelStat> st((size_t)nlstat);
    HCK(cudaMemcpyAsync(st.data(), d_lstat, sizeof(LevelStat) * (size_t)nlstat, cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    for (size_t li : dev_levels) {
      LevelRec& L = F->levels[li];
      const LevelStat& S = st[(size_t)L.dev_stat];
      L.ngroups = S.ngroups;
      L.nskel = S.nskel;
      L.nred = S.nred;
      L.max_front = S.max_front;
      L.gflop = S.gflop;
      L.gbytes = S.gbytes;
      for (int c = 0; c < 2; ++c) {
        L.gf_cls[c] = S.gf_cls[c];
        L.gb_cls[c] = S.gb_cls[c];
      }
      L.solve_fac = S.solve_fac;
      L.solve_rows = S.solve_rows;
      if (L.active_after == 0 && (int)li != last_dev_level) L.active_after = S.active_after;
      F->m_f_bytes += S.mf_bytes;
      L.nall = (int)S.nrecs;
      L.all_max_nc = (int)S.max_nc;
      L.all_max_nq = (int)S.max_nq;
      if (L.kind == 0) L.ntargets = (int)S.ntargets;
      const bool all_small = S.max_nc <= 96 && S.max_nq <= 192;
      if (all_small) {
        L.nsmall = (int)S.nrecs;
        L.max_nc = (int)S.max_nc;
        L.max_nq = (int)S.max_nq;
      } else {  // large records: the host plan (tiled phases)
        L.recs.resize((size_t)S.nrecs);
        HCK(cudaMemcpy(L.recs.data(), L.d_recs, sizeof(SolveRec) * (size_t)S.nrecs, cudaMemcpyDeviceToHost));
        L.d_recs = nullptr;
        L.d_all = nullptr;
        L.nall = 0;
        L.all_max_nc = L.all_max_nq = 0;
        L.solve_fac = L.solve_rows = 0;
        build_solve_plan(L);
      }
      for (auto& E : F->klog.v) {  // kernel log: the level's totals to its main launch
        if (E.phase != 0 || E.tag != L.tag) continue;
        if (E.name == "elim_small_kernel" || E.name == "elim_small_kernel(top)") {
          E.gbytes = L.gb_cls[0];
          E.gflop = L.gf_cls[0];
        }
        if (E.name == "elim_blocked_pipeline" || E.name == "elim_blocked_pipeline(top)") {
          E.gbytes = L.gb_cls[1];
          E.gflop = L.gf_cls[1];
        }
        if (E.name == "skel_kernel" || E.name == "skel_ordered_kernel" || E.name == "skel_cluster_kernel") {
          E.gbytes = L.gbytes;
          E.gflop = L.gflop;
        }
      }
    }
  }

  // -------------------------------------------------------------------------
  // Thread-safe variant for the wavefront partition: the block verdicts are
  // cached per thread for the cell being processed (owners do not change
  // while one cell decides).
  struct AfCache {
    int64_t key = -1;
    std::vector<std::pair<int32_t, uint8_t>> v;
  };
  std::vector<AfCache> afc;
  bool adaptive_foreign_tid(int32_t d, int64_t key, const int64_t* owner, int tid) {
    for (int64_t k = indptr[(size_t)d]; k < indptr[(size_t)d + 1]; ++k) {
      const int64_t o = owner[indices[(size_t)k]];
      if (o != -1 && o != key) return true;
    }
    AfCache& c = afc[(size_t)tid];
    if (c.key != key) {
      c.key = key;
      c.v.clear();
    }
    bool found = false;
    member.for_each(d, [&](int32_t b) {
      if (found) return;
      int f = -1;
      for (const auto& e : c.v)
        if (e.first == b) {
          f = e.second;
          break;
        }
      if (f < 0) {
        f = 0;
        const int32_t* dd = h_idx.data() + blk_dof_off[(size_t)b];
        for (int32_t i = 0; i < blk_n[(size_t)b] && !f; ++i) {
          const int32_t e = dd[i];
          if (!active[(size_t)e]) continue;
          const int64_t o = owner[e];
          if (o != -1 && o != key) f = 1;
        }
        c.v.emplace_back(b, (uint8_t)f);
      }
      if (f) found = true;
    });
    return found;
  }

  bool adaptive_foreign(int32_t d, int64_t key, const int64_t* owner) {
    for (int64_t k = indptr[(size_t)d]; k < indptr[(size_t)d + 1]; ++k) {
      const int64_t o = owner[indices[(size_t)k]];
      if (o != -1 && o != key) return true;
    }
    const int64_t tag = (bf_epoch << 32) + key;
    bool found = false;
    member.for_each(d, [&](int32_t b) {
      if (found) return;
      if (bf_key[(size_t)b] != tag) {
        bf_key[(size_t)b] = tag;
        uint8_t f = 0;
        const int32_t* dd = h_idx.data() + blk_dof_off[(size_t)b];
        for (int32_t i = 0; i < blk_n[(size_t)b] && !f; ++i) {
          const int32_t e = dd[i];
          if (!active[(size_t)e]) continue;
          const int64_t o = owner[e];
          if (o != -1 && o != key) f = 1;
        }
        bf_val[(size_t)b] = f;
      }
      if (bf_val[(size_t)b]) found = true;
    });
    return found;
  }

  // Rebuild a factor from exported records (hifde_import): arenas to the
  // device, solve records, reductions and the solve plan as after run().
  void import_records(int nlevels, const double* tags, const int32_t* kinds, const int64_t* rec_ptr,
                      const hifde_record_t* recs, const double* fac, int64_t fac_len, const int32_t* idx,
                      int64_t idx_len) {
    N = F->n;
    pinned_stage().begin(s);
    g_stage = &pinned_stage();
    struct StageOff {
      ~StageOff() { g_stage = nullptr; }
    } stage_off;
    h_idx.assign(idx, idx + idx_len);
    F->fac.reserve((size_t)std::max<int64_t>(fac_len, 1), s);
    F->fac.n = (size_t)fac_len;
    F->fac.upload(fac, 0, (size_t)fac_len, s);
    F->idx.reserve((size_t)std::max<int64_t>(idx_len, 1), s);
    F->idx.n = (size_t)idx_len;
    F->idx.upload(idx, 0, (size_t)idx_len, s);
    for (int li = 0; li < nlevels; ++li) {
      F->levels.emplace_back();
      LevelRec& L = F->levels.back();
      L.tag = tags[li];
      L.kind = kinds[li];
      const hifde_record_t* r0 = recs + rec_ptr[li];
      const int64_t nr = rec_ptr[li + 1] - rec_ptr[li];
      L.ngroups = nr;
      L.xrec.assign(r0, r0 + nr);
      for (int64_t t = 0; t < nr; ++t) {
        const hifde_record_t& X = r0[t];
        if ((X.kind == 1) != (L.kind == 1)) throw Fail{HIFDE_BADARG, "record kind does not match its level"};
        SolveRec R;
        R.T_off = 0;
        R.inv = 1;
        R.pad = 0;
        R.contrib_off = 0;
        if (X.kind == 1) {
          L.nskel += X.nq;
          L.nred += X.nr;
          if (X.nr == 0) continue;
          R.nc = X.nr;
          R.nq = X.nq;
          R.idx_off = X.idx_off;
          R.T_off = X.T_off;
        } else {
          R.nc = X.nc;
          R.nq = X.nq;
          R.idx_off = X.idx_off;
          R.contrib_off = L.ncontrib;
          L.ncontrib += X.nq;
          if (X.kind == 2) F->s_top = X.nc;
        }
        R.C_off = X.P_off;
        R.W_off = X.W_off;
        L.recs.push_back(R);
        L.max_nc = std::max(L.max_nc, R.nc);
        L.max_nq = std::max(L.max_nq, R.nq);
        F->m_f_bytes += X.kind == 1 ? 8 * ((int64_t)X.nq * X.nr + (int64_t)X.nr * X.nr + X.nr + (int64_t)X.nr * X.nq)
                                    : 8 * ((int64_t)X.nc * X.nc + X.nc + (int64_t)X.nc * X.nq);
      }
      if (L.kind == 0) build_reduction((size_t)li, L);
    }
    helper.drain();
    finish_reductions();
    for (auto& L : F->levels) build_solve_plan(L);
    F->meta = meta.commit(s, [&](void* d, const void* h, size_t n) {
      if (!pinned_stage().copy(d, h, n)) HCK(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s));
    });
    HCK(cudaStreamSynchronize(s));
  }

  // Starts the device-to-host copy of a device-resident pattern on pat_s;
  // false (nothing started) when the pinned cache buffers are not available.
  bool pat_async(const int64_t* ip, const int32_t* ix, const double* va, int64_t& nnz_out) {
    HostCache& hc = host_cache();
    int64_t* hip = (int64_t*)hc.pat_ip.get((N + 1) * sizeof(int64_t));
    if (!hip) return false;
    int64_t nz = 0;
    HCK(cudaMemcpyAsync(&nz, ip + N, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));  // (also: the caller's arrays are complete on s)
    int32_t* hix = (int32_t*)hc.pat_ix.get((size_t)std::max<int64_t>(nz, 1) * sizeof(int32_t));
    if (!hix) return false;
    if (!pat_s) {
      HCK(cudaStreamCreateWithFlags(&pat_s, cudaStreamNonBlocking));
      HCK(cudaEventCreateWithFlags(&ev_pat, cudaEventDisableTiming));
    }
    HCK(cudaMemcpyAsync(hip, ip, (N + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, pat_s));
    HCK(cudaMemcpyAsync(hix, ix, nz * sizeof(int32_t), cudaMemcpyDeviceToHost, pat_s));
    HCK(cudaEventRecord(ev_pat, pat_s));
    pat_pending = true;
    nnz_out = nz;
    indptr = hip;
    indices = hix;
    d_indptr = const_cast<int64_t*>(ip);
    d_indices = const_cast<int32_t*>(ix);
    d_a0 = const_cast<double*>(va);
    return true;
  }

  void run(const int64_t* ip, const int32_t* ix, const double* va, int64_t nnz) {
    const double t0 = now_s();
    N = g.ndof();
    comm = opt.comm;
    if (comm && comm->P > 1) {
      P = comm->P;
      me = comm->rank;
      emu = comm->emulated;
      real = !emu;
      geom = shard_geom(P, g.dim, g.n);
      ledger.reset(P);
      if (emu) lanes.resize((size_t)P - 1);
    } else {
      comm = nullptr;
    }
    HTRACE("factor start N=%lld", (long long)N);
    LevelRec& PR = prof;  // setup / finish sub-phases (HIFDE_PROFILE)
    PR.lap(nullptr);
    pinned_stage().begin(s);
    PR.lap("stage");
    g_stage = &pinned_stage();
    struct StageOff {
      ~StageOff() { g_stage = nullptr; }
    } stage_off;
    // A0: the symbolic analysis needs the pattern on the host
    const bool dev_first = opt.symbolic == HIFDE_SYMBOLIC_AUTO && !sharded() && !opt.verify && N > 0;
    if (opt.input_on_device && dev_first && pat_async(ip, ix, va, nnz)) {
      // (pattern copy in flight on pat_s)
    } else if (opt.input_on_device) {
      HostCache& hc = host_cache();
      int64_t* hip = (int64_t*)hc.pat_ip.get((N + 1) * sizeof(int64_t));
      if (hip) {
        HCK(cudaMemcpyAsync(hip, ip, (N + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        HCK(cudaStreamSynchronize(s));
        nnz = hip[N];
      } else {
        indptr_own.resize((size_t)N + 1);
        pinned_xfer().d2h(indptr_own.data(), ip, (N + 1) * sizeof(int64_t), s);
        hip = indptr_own.data();
        nnz = indptr_own.back();
      }
      int32_t* hix = (int32_t*)hc.pat_ix.get((size_t)std::max<int64_t>(nnz, 1) * sizeof(int32_t));
      if (hix) {
        HCK(cudaMemcpyAsync(hix, ix, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        HCK(cudaStreamSynchronize(s));
      } else {
        indices_own.resize((size_t)nnz);
        pinned_xfer().d2h(indices_own.data(), ix, nnz * sizeof(int32_t), s);
        hix = indices_own.data();
      }
      indptr = hip;
      indices = hix;
      d_indptr = const_cast<int64_t*>(ip);
      d_indices = const_cast<int32_t*>(ix);
      d_a0 = const_cast<double*>(va);
    } else {
      indptr = ip;
      indices = ix;
      HCK(cudaMallocAsync((void**)&d_indptr, (N + 1) * sizeof(int64_t), s));
      HCK(cudaMallocAsync((void**)&d_indices, std::max<int64_t>(nnz, 1) * sizeof(int32_t), s));
      HCK(cudaMallocAsync((void**)&d_a0, std::max<int64_t>(nnz, 1) * sizeof(double), s));
      own_a0 = true;
      // pageable H2D copies block the calling thread: a helper thread issues
      // them while this one runs the level-0 symbolic analysis (joined before
      // the first kernel launch, a0_ready())
      int dev = 0;
      HCK(cudaGetDevice(&dev));
      const size_t pin_min = (size_t)1 << 20;
      const bool big = (size_t)nnz * 12 > pin_min;  // large inputs: pinned staging
      HCK(cudaStreamCreateWithFlags(&a0_s, cudaStreamNonBlocking));
      {  // the values' copy follows the allocations
        cudaEvent_t e0;
        HCK(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
        HCK(cudaEventRecord(e0, s));
        HCK(cudaStreamWaitEvent(a0_s, e0, 0));
        HCK(cudaEventDestroy(e0));
      }
      HCK(cudaEventCreateWithFlags(&ev_a0, cudaEventDisableTiming));
      const cudaStream_t vs = a0_s;
      const cudaEvent_t ev_v = ev_a0;
      a0_pat_job = helper.post([=]() {
        cudaError_t e = cudaSetDevice(dev);
        if (e == cudaSuccess && big) {
          try {
            pinned_xfer().h2d(d_indptr, ip, (N + 1) * sizeof(int64_t), s);
            pinned_xfer().h2d(d_indices, ix, nnz * sizeof(int32_t), s);
          } catch (const Fail&) {
            e = cudaErrorUnknown;
          }
        } else {
          if (e == cudaSuccess) e = cudaMemcpyAsync(d_indptr, ip, (N + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
          if (e == cudaSuccess) e = cudaMemcpyAsync(d_indices, ix, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s);
          if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        }
        if (e != cudaSuccess) a0_err = e;
      });
      hifde_factor_t* const Fq = F;
      a0_job = helper.post([=]() {
        cudaError_t e = cudaSetDevice(dev);
        if (e == cudaSuccess && big) {
          try {
            pinned_xfer().h2d(d_a0, va, nnz * sizeof(double), vs);
          } catch (const Fail&) {
            e = cudaErrorUnknown;
          }
        } else {
          if (e == cudaSuccess) e = cudaMemcpyAsync(d_a0, va, nnz * sizeof(double), cudaMemcpyHostToDevice, vs);
        }
        // page-locked values: only issued here, the numeric launches' stream
        // waits for ev_a0 on the device (the host runs on into the next
        // level's analysis meanwhile)
        if (e == cudaSuccess) e = cudaEventRecord(ev_v, vs);
        if (e != cudaSuccess) a0_err = e;
        // (an asynchronous factorization: a waiting solve may queue its own
        // uploads behind the matrix's now)
        {
          std::lock_guard<std::mutex> lk(Fq->ev_m);
          Fq->ev_inputs = e == cudaSuccess ? ev_v : nullptr;
        }
        Fq->inputs_issued.store(1);
      });
    }
    PR.lap("A0");
    if (!own_a0) F->inputs_issued.store(1);
    {  // borrow the persistent host buffers (returned at the end of run)
      HostCache& hc = host_cache();
      h_idx.swap(hc.idx_buf);
      h_idx.resize(0);
      meta.h.swap(hc.meta_buf);
      meta.h.resize(0);
      borrowed = true;
    }
    // the host's active mask, active list and block membership: filled here
    // for the host analysis, or by dev_to_host when the device symbolic pass
    // runs the first levels (config 3: 3.7 ms of O(N) host fills saved)
    if (!dev_first) {
      active.resize((size_t)N);
      act.resize((size_t)N);
#pragma omp parallel for schedule(static) if (N > (1 << 16))
      for (int64_t i = 0; i < N; ++i) {
        active[(size_t)i] = 1;
        act[(size_t)i] = (int32_t)i;
      }
    }
    HCK(cudaMallocAsync((void**)&d_active, std::max<int64_t>(N, 1), s));
    HCK(cudaMemsetAsync(d_active, 1, (size_t)N, s));
    {
      const char* env = getenv("HIFDE_HOST_THREADS");
      nthreads = env ? std::max(1, atoi(env)) : std::min(15, std::max(1, omp_get_max_threads() - 1));
      HostCache& hc = host_cache();
      const bool same = hc.valid && hc.g.dim == g.dim && hc.g.n == g.n;
      if (!same) {
        X.build(g);
        member.init(N);
        ctx.clear();
        hc.g = g;
        hc.valid = true;
        hc.variant = -1;  // arena hints belong to the previous grid
      } else if (!dev_first) {
        member.reset();  // (dev_to_host resets it before rebuilding)
      }
      if ((int)ctx.size() < nthreads) ctx.resize((size_t)nthreads);
      for (auto& x : ctx)
        if ((int64_t)x.dstamp.size() != N) {
          x.dstamp.assign((size_t)N, 0);
          x.bstamp.clear();
          x.stamp = 0;
        }
    }
    PR.lap("host-state");
    {
      HostCache& hc = host_cache();
      const bool hint = hc.variant == opt.variant;
      auto want = [&](size_t h, int64_t dflt) { return std::max<size_t>(hint ? h + h / 16 : 0, (size_t)dflt); };
      F->fac.reserve(want(hc.hint_fac, std::max<int64_t>(64 * N, 1 << 16)), s);
      F->idx.reserve(want(hc.hint_idx, std::max<int64_t>(16 * N, 1 << 16)), s);
      bvals.reserve(want(hc.hint_bv, std::max<int64_t>(64 * N, 1 << 16)), s);
      h_idx.reserve(want(hc.hint_idx, std::max<int64_t>(16 * N, 1 << 16)));
      if (hint && hc.hint_scr) scratch.reserve(hc.hint_scr, s);
      if (hint && hc.hint_meta) meta.h.reserve(hc.hint_meta + hc.hint_meta / 8);
    }

    PR.lap("reserve");
    const int Lv = g.nlevels;
    F->levels.reserve((size_t)3 * std::max(Lv, 1) + 4);  // stable LevelRec addresses for the helper
    const double t_setup = now_s() - t0;
    HTRACE("setup done");
    std::vector<int32_t> act_tmp;
    auto record_trace = [&](LevelRec& L, double tl) {
      size_t w = 0;
      const int64_t na = (int64_t)act.size();
      if (na < 16384) {
        for (size_t i = 0; i < act.size(); ++i)
          if (active[(size_t)act[i]]) act[w++] = act[i];
        act.resize(w);
      } else {  // parallel stable compaction: chunk counts, prefix, scatter
        const int nth = nthreads;
        std::vector<int64_t> cnt((size_t)nth + 1, 0);
        act_tmp.resize(act.size());
#pragma omp parallel num_threads(nth)
        {
          const int tid = omp_get_thread_num();
          const int64_t lo = na * tid / nth, hi = na * (tid + 1) / nth;
          int64_t c = 0;
          for (int64_t i = lo; i < hi; ++i) c += active[(size_t)act[(size_t)i]] ? 1 : 0;
          cnt[(size_t)tid + 1] = c;
#pragma omp barrier
#pragma omp single
          for (int t = 0; t < nth; ++t) cnt[(size_t)t + 1] += cnt[(size_t)t];
          int64_t o = cnt[(size_t)tid];
          for (int64_t i = lo; i < hi; ++i)
            if (active[(size_t)act[(size_t)i]]) act_tmp[(size_t)o++] = act[(size_t)i];
        }
        w = (size_t)cnt[(size_t)nth];
        act_tmp.resize(w);
        act.swap(act_tmp);
      }
      L.active_after = (int64_t)w;
      L.seconds = now_s() - tl;
    };
    // device symbolic mode from level 0 (not for the sharded sweep, whose
    // ranks keep the host analysis, nor for verify runs)
    dev_mode = dev_first;
    if (dev_mode) dev_init();
    // a device level that cannot run on the device hands over and is redone on the host
    auto dev_fallback = [&](LevelRec& L, double tag) {
      if (L.ev0) cudaEventDestroy(L.ev0);
      if (L.ev1) cudaEventDestroy(L.ev1);
      L = LevelRec();
      L.tag = tag;
      dev_to_host();
    };
    for (int ell = 0; ell < Lv; ++ell) {
      if (dev_mode && opt.variant == HIFDE_VARIANT_HIFDE3X && ell > 0) dev_to_host();  // adaptive cells: host
      if (dev_mode) {
        const double tl = now_s();
        F->levels.emplace_back();
        LevelRec& L = F->levels.back();
        L.tag = (double)ell;
        if (dev_elimination_level(ell, L.tag, L)) {
          L.seconds = now_s() - tl;
        } else {
          dev_fallback(L, (double)ell);
          F->levels.pop_back();
        }
      }
      if (!dev_mode || F->levels.empty() || F->levels.back().tag != (double)ell) {
        const double tl = now_s();
        Groups gr;
        if (opt.variant == HIFDE_VARIANT_HIFDE3X && ell > 0) {
          // few (large) cells: the sequential pass with its per-block cache;
          // many: wavefronts of cells on the host threads
          const int64_t ncell_est = [&] {
            int64_t c = 1;
            for (int ax = 0; ax < g.dim; ++ax) c *= g.n / (g.m << ell);
            return c;
          }();
          afc.resize((size_t)std::max(nthreads, 1));
          for (auto& c : afc) c.key = -1;
          if (ncell_est < 256 || nthreads < 2) {
            ++bf_epoch;
            gr = adaptive_groups(g, X, ell, act, N, [&](int32_t d, int64_t key, const int64_t* owner) {
              return adaptive_foreign(d, key, owner);
            });
          } else
          gr = adaptive_groups_par(
              g, X, ell, act, N,
              [&](int32_t d, int64_t key, const int64_t* owner, int tid) {
                return adaptive_foreign_tid(d, key, owner, tid);
              },
              nthreads);
          static const bool check = getenv("HIFDE_CHECK_ADAPTIVE") != nullptr;  // debug: sequential cross-check
          if (check) {
            ++bf_epoch;
            Groups ref = adaptive_groups(g, X, ell, act, N, [&](int32_t d, int64_t key, const int64_t* owner) {
              return adaptive_foreign(d, key, owner);
            });
            if (ref.members != gr.members || ref.offsets != gr.offsets)
              throw Fail{HIFDE_INTERNAL, "wavefront adaptive partition differs from the sequential one"};
          }
        } else {
          gr = interior_groups(g, X, ell, act);
        }
        if (opt.verify) check_noninteracting(gr, (double)ell);
        F->levels.emplace_back();
        LevelRec& L = F->levels.back();
        L.t_part = now_s() - tl;
        L.tag = (double)ell;
        elimination_level(gr, L.tag, L, false);
        record_trace(L, tl);
        helper.post([this, &L]() { build_solve_plan(L); });
      }
      auto skel = [&](double tag, int kind) {
        if (dev_mode) {
          const double tl = now_s();
          F->levels.emplace_back();
          LevelRec& L = F->levels.back();
          L.tag = tag;
          if (dev_skeleton_level(ell, kind, tag, L)) {
            L.seconds = now_s() - tl;
            return;
          }
          dev_fallback(L, tag);
          F->levels.pop_back();
        }
        const double tl = now_s();
        Groups gr = interface_groups(g, X, ell, act, kind);
        F->levels.emplace_back();
        LevelRec& L = F->levels.back();
        L.t_part = now_s() - tl;
        L.tag = tag;
        skeleton_level(gr, tag, L);
        record_trace(L, tl);
        helper.post([this, &L]() { build_solve_plan(L); });
      };
      if (opt.variant == HIFDE_VARIANT_HIFDE) {
        if (ell >= opt.skip_levels) skel(ell + 0.5, g.dim == 2 ? 0 : 1);
      } else if (opt.variant == HIFDE_VARIANT_HIFDE3X) {
        skel(ell + 1.0 / 3.0, 1);
        if (ell >= opt.skip_levels) skel(ell + 2.0 / 3.0, 0);
      }
    }
    prof.lap("levels");
    // terminal block: every DOF still active (src/driver.py:152-157); on the
    // device path when the levels ran there (one cell of every active DOF,
    // no neighbours), else on the host path after the hand-over
    bool top_dev = false;
    if (dev_mode) {
      const double tl = now_s();
      F->levels.emplace_back();
      LevelRec& L = F->levels.back();
      L.tag = (double)Lv;
      if (dev_elimination_level(Lv, L.tag, L, true)) {
        check_status();
        L.seconds = now_s() - tl;
        top_dev = true;
      } else {
        dev_fallback(L, (double)Lv);
        F->levels.pop_back();
      }
    }
    if (!top_dev) {
      dev_to_host();
      {
        const double tl = now_s();
        Groups top;
        top.members = act;
        F->s_top = (int64_t)top.members.size();
        F->levels.emplace_back();
        LevelRec& L = F->levels.back();
        L.tag = (double)Lv;
        if (!top.members.empty()) {
          top.offsets.push_back((int64_t)top.members.size());
          elimination_level(top, L.tag, L, true);
          L.gflop = std::pow((double)F->s_top, 3) / 3 * 1e-9;
          L.gbytes = 16.0 * F->s_top * F->s_top * 1e-9;
        }
        L.kind = 2;
        record_trace(L, tl);
      }
    }
    PR.lap("top");
    // real ranks: every record lives on its owner (zeros elsewhere) -- the
    // partitioned solve needs nothing else; ensure_whole() sums the arenas
    // the first time an operation needs every record
    F->nranks = sharded() ? P : 1;
    F->xfer_bytes = xfer_bytes;
    helper.drain();
    if (!top_dev) build_solve_plan(F->levels.back());  // the terminal block
    dev_finalize();
    if (sharded()) build_shard_solve();
    finish_reductions();
    PR.lap("reductions");
    // solve metadata to the device: small records one CTA each, large ones as
    // tiled product phases (built level by level on the helper thread)
    meta_bytes = meta.h.size();
    F->meta = meta.commit(s, [&](void* d, const void* h, size_t n) {
      if (!pinned_stage().copy(d, h, n)) HCK(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s));
    });
    PR.lap("solve-plan");
    HCK(cudaStreamSynchronize(s));
    PR.lap("sync");
    for (auto& L : F->levels) {
      if (L.ev0 && L.ev1) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, L.ev0, L.ev1) == cudaSuccess) L.gpu_seconds = ms * 1e-3;
        cudaEventDestroy(L.ev0);
        cudaEventDestroy(L.ev1);
        L.ev0 = L.ev1 = nullptr;
      }
    }
    {
      HostCache& hc = host_cache();
      hc.variant = opt.variant;
      hc.hint_fac = F->fac.n;
      hc.hint_bv = bvals.n;
      hc.hint_idx = h_idx.size();
      hc.hint_scr = scratch.cap;
      hc.hint_meta = meta_bytes;
    }
    release_all();
    HCK(cudaStreamSynchronize(s));
    PR.lap("release");
    F->t_f = now_s() - t0;
    if (getenv("HIFDE_PROFILE")) {
      fprintf(stderr, "[hifde] setup/finish:");
      for (const auto& p : PR.sub) fprintf(stderr, " %s %.3f", p.first, p.second * 1e3);
      fprintf(stderr, "\n");
      fprintf(stderr, "[hifde] factor %.3f ms (setup %.3f ms)\n", F->t_f * 1e3, t_setup * 1e3);
      for (const auto& L : F->levels)
        fprintf(stderr,
                "[hifde] tag %6.3f kind %d groups %7lld batches %3d maxfront %5lld | host ms: part %.3f sym %.3f "
                "upd %.3f launch %.3f sync %.3f total %.3f | gpu ms %.3f\n",
                L.tag, L.kind, (long long)L.ngroups, L.nbatches, (long long)L.max_front, L.t_part * 1e3,
                L.t_sym * 1e3, L.t_upd * 1e3, L.t_launch * 1e3, L.t_sync * 1e3, L.seconds * 1e3,
                L.gpu_seconds * 1e3);
      for (const auto& L : F->levels) {
        fprintf(stderr, "[hifde]   tag %6.3f sub:", L.tag);
        for (const auto& p : L.sub) fprintf(stderr, " %s %.3f", p.first, p.second * 1e3);
        fprintf(stderr, "\n");
      }
      if (F->klog.on && !F->klog.v.empty()) {  // device timeline of the logged launches (ms from the first)
        HCK(cudaDeviceSynchronize());
        const cudaEvent_t t0e = F->klog.v.front().e0;
        for (const auto& E : F->klog.v) {
          if (E.phase != 0) continue;
          float a = 0.f, b = 0.f;
          cudaEventElapsedTime(&a, t0e, E.e0);
          cudaEventElapsedTime(&b, t0e, E.e1);
          fprintf(stderr, "[hifde] tl %8.3f %8.3f %7.3f  %-28s tag %.3f\n", a, b, b - a, E.name.c_str(), E.tag);
        }
      }
    }
  }
};

// ---------------------------------------------------------------------------
// Solve sweep
// ---------------------------------------------------------------------------
// The up/down sweep on the device block v (N x nrhs row-major, in place).
// Level 0 of the sweep in record bands (solve_pipelined): the forward band
// b waits on fwd_wait[b] (the upload of the rows it reads), the backward
// band b records bwd_done[b] (its rows may leave).
struct SweepBands {
  std::vector<std::pair<int, int>> fwd, bwd;
  std::vector<cudaEvent_t> fwd_wait, bwd_done;
};

// Whether level 0 can run banded: every record on the one-CTA kernels.
bool level0_bandable(const hifde_factor_t* F) {
  if (F->levels.empty()) return false;
  const LevelRec& L = F->levels[0];
  return L.kind == 0 && L.d_recs && L.nsmall > 0 && L.nsmall == L.nall && L.fwd_ph.empty() && L.bwd_ph.empty() &&
         L.max_nc <= 96 && L.max_nq <= 192;
}

// Sums the real ranks' factor arenas once (each holds its own records, zeros
// elsewhere) before an operation that reads every record.
void ensure_whole(const hifde_factor_t* F, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(F->whole_m);
  if (F->whole) return;
  try {
    comm_allreduce(F->comm, F->fac.p, F->fac.n, kF64, kSum, s);
  } catch (const std::exception& e) {
    throw Fail{HIFDE_CUDA, e.what()};
  }
  F->whole = true;
}

void solve_sweep(const hifde_factor_t* F, double* v, int nrhs, cudaStream_t s, const SweepBands* bands = nullptr) {
  double* contrib = nullptr;
  HCK(cudaMallocAsync((void**)&contrib, std::max<size_t>(F->max_contrib * nrhs * sizeof(double), 8), s));
  double* tscr = nullptr;
  HCK(cudaMallocAsync((void**)&tscr, std::max<size_t>(F->tile_rows * nrhs * sizeof(double), 8), s));
  // global workspace for one-CTA records too large for shared memory
  size_t scratch_need = 0;
  auto ws_plan = [&](const LevelRec& L, int64_t per_rec_doubles, size_t& smem, int64_t& per_rec) {
    const size_t need = (size_t)per_rec_doubles * sizeof(double);
    if (need <= kSolveDynSmem) { smem = need; per_rec = 0; }
    else { smem = 0; per_rec = per_rec_doubles; scratch_need = std::max(scratch_need, (size_t)per_rec * L.nsmall); }
  };
  auto ws_of = [&](const LevelRec& L) {
    return (int64_t)(2 * L.max_nc + L.max_nq) * nrhs;  // two nc blocks + the neighbour block
  };
  for (const auto& L : F->levels) {
    size_t sm; int64_t pr;
    ws_plan(L, ws_of(L), sm, pr);
    for (const auto& V : L.rank_view) ws_plan(V, ws_of(V), sm, pr);
  }
  double* scratch = nullptr;
  HCK(cudaMallocAsync((void**)&scratch, std::max<size_t>(scratch_need * sizeof(double), 8), s));
  // fine elimination levels: the single-load-phase kernels
  constexpr int small_max_rhs = 64, small_max_n = 96;
  constexpr size_t small_max_smem = kSmemCapBytes;  // (200 KB kept config 3 level 3, 208 KB, on the streaming kernels: 2x slower)
  // (HIFDE_NO_SOLVE_SMALL: the general record kernels instead -- the tests' A/B of the two)
  static const bool no_small = getenv("HIFDE_NO_SOLVE_SMALL") != nullptr;
  auto small_path = [&](const LevelRec& L) {
    return !no_small && L.kind == 0 && nrhs >= 2 && nrhs <= small_max_rhs && L.max_nc <= small_max_n &&
           L.max_nq <= 2 * small_max_n && solve_small_smem(L.max_nc, L.max_nq, nrhs) <= small_max_smem;
  };
  auto small_skel = [&](const LevelRec& L) {
    return !no_small && L.kind == 1 && nrhs >= 2 && nrhs <= small_max_rhs && L.max_nc <= small_max_n &&
           L.max_nq <= 2 * small_max_n && solve_skel_small_smem(L.max_nc, L.max_nq, nrhs) <= small_max_smem;
  };
  const int32_t* idx = F->idx.p;
  const double* fac = F->fac.p;
  auto phases = [&](const std::vector<LevelRec::Phase>& ph, double* vv, double* cc) {
    for (const auto& P : ph) {
      launch_solve_tiles(P.d_ops, P.d_work, P.nwork, idx, fac, vv, nrhs, tscr, cc, s);
      ++g_launches;
    }
  };
  // Forward records of a level (or of one rank's share of it): v_c = P v_c
  // and the contribution rows W^T v_c (elimination), or the skeleton record
  // in place.  `band0`: level 0 of the banded host solve.
  auto fwd_records = [&](const LevelRec& L, double* vv, double* cc, bool band0) {
    const int nr = L.nsmall;
    size_t sm; int64_t pr;
    ws_plan(L, ws_of(L), sm, pr);
    if (L.kind == 1) {
      if (nr && small_skel(L)) {
        launch_solve_skel_small(L.d_recs, nr, idx, fac, vv, nrhs, solve_skel_small_smem(L.max_nc, L.max_nq, nrhs), 1,
                                s);
        ++g_launches;
      } else if (nr) {
        launch_solve_skel(L.d_recs, nr, idx, fac, vv, nrhs, 1, scratch, pr, sm, s);
        ++g_launches;
      }
      phases(L.fwd_ph, vv, cc);
      return;
    }
    if (band0 && !(nr && small_path(L)))  // (not banded after all: wait for the whole upload)
      for (cudaEvent_t e : bands->fwd_wait) HCK(cudaStreamWaitEvent(s, e, 0));
    if (band0 && nr && small_path(L)) {  // upload bands as they land
      for (size_t b = 0; b < bands->fwd.size(); ++b) {
        HCK(cudaStreamWaitEvent(s, bands->fwd_wait[b], 0));
        const int lo = bands->fwd[b].first, hi = bands->fwd[b].second;
        if (hi > lo) {
          launch_solve_elim_small(L.d_recs + lo, hi - lo, idx, fac, (int64_t)F->fac.cap, vv, nrhs, cc, L.max_nc,
                                  L.max_nq, solve_small_smem(L.max_nc, L.max_nq, nrhs), 1, s);
          ++g_launches;
        }
      }
    } else if (nr && small_path(L)) {
      launch_solve_elim_small(L.d_recs, nr, idx, fac, (int64_t)F->fac.cap, vv, nrhs, cc, L.max_nc, L.max_nq,
                              solve_small_smem(L.max_nc, L.max_nq, nrhs), 1, s);
      ++g_launches;
    } else if (nr) {
      launch_solve_elim_fwd(L.d_recs, nr, idx, fac, vv, nrhs, cc, scratch, pr, sm, s);
      ++g_launches;
    }
    phases(L.fwd_ph, vv, cc);
  };
  // the elimination's neighbour rows: v_q -= the contribution rows, summed in record order
  auto fwd_reduce = [&](const LevelRec& L, double* vv, double* cc) {
    if (L.kind == 0 && L.ntargets) {
      launch_solve_reduce(L.d_targets, L.d_ptr, L.d_ent, L.ntargets, cc, vv, nrhs, s);
      ++g_launches;
    }
  };
  auto bwd_records = [&](const LevelRec& L, double* vv, bool band0) {
    const int nr = L.nsmall;
    size_t sm; int64_t pr;
    ws_plan(L, ws_of(L), sm, pr);
    if (L.kind == 1) {
      if (nr && small_skel(L)) {
        launch_solve_skel_small(L.d_recs, nr, idx, fac, vv, nrhs, solve_skel_small_smem(L.max_nc, L.max_nq, nrhs), 0,
                                s);
        ++g_launches;
      } else if (nr) {
        launch_solve_skel(L.d_recs, nr, idx, fac, vv, nrhs, 0, scratch, pr, sm, s);
        ++g_launches;
      }
    } else {
      if (band0 && nr && small_path(L)) {  // rows leave as their bands finish
        for (size_t b = 0; b < bands->bwd.size(); ++b) {
          const int lo = bands->bwd[b].first, hi = bands->bwd[b].second;
          if (hi > lo) {
            launch_solve_elim_small(L.d_recs + lo, hi - lo, idx, fac, (int64_t)F->fac.cap, vv, nrhs, nullptr,
                                    L.max_nc, L.max_nq, solve_small_smem(L.max_nc, L.max_nq, nrhs), 0, s);
            ++g_launches;
          }
          HCK(cudaEventRecord(bands->bwd_done[b], s));
        }
      } else if (nr && small_path(L)) {
        launch_solve_elim_small(L.d_recs, nr, idx, fac, (int64_t)F->fac.cap, vv, nrhs, nullptr, L.max_nc, L.max_nq,
                                solve_small_smem(L.max_nc, L.max_nq, nrhs), 0, s);
        ++g_launches;
      } else if (nr) {
        launch_solve_elim_bwd(L.d_recs, nr, idx, fac, vv, nrhs, scratch, pr, sm, s);
        ++g_launches;
      }
    }
    phases(L.bwd_ph, vv, nullptr);
    if (band0 && !(nr && small_path(L)))  // (not banded after all: every band done here)
      for (cudaEvent_t e : bands->bwd_done) HCK(cudaEventRecord(e, s));
  };
  const size_t nl = F->levels.size();
  if (F->part) {
    // Partitioned sweep (build_shard_solve): this process's ranks run their
    // own records on their own copy of v; the planned rows move in between.
    const int P = F->nranks;
    const int lo = F->emu ? 0 : F->me, hi = F->emu ? P : F->me + 1;
    std::vector<double*> vr((size_t)P, nullptr), cr((size_t)P, nullptr);
    std::vector<void*> owned;
    const size_t vbytes = (size_t)F->n * nrhs * sizeof(double);
    for (int r = lo; r < hi; ++r) {
      if (r == lo) {
        vr[(size_t)r] = v;
        cr[(size_t)r] = contrib;
        continue;
      }
      HCK(cudaMallocAsync((void**)&vr[(size_t)r], std::max<size_t>(vbytes, 8), s));
      HCK(cudaMemcpyAsync(vr[(size_t)r], v, vbytes, cudaMemcpyDeviceToDevice, s));
      HCK(cudaMallocAsync((void**)&cr[(size_t)r], std::max<size_t>(F->max_contrib * nrhs * sizeof(double), 8), s));
      owned.push_back(vr[(size_t)r]);
      owned.push_back(cr[(size_t)r]);
    }
    int64_t xmax = 0;
    auto step_rows = [&](const LevelRec::XStep& X, bool mine_only) {
      int64_t sn = 0, rn = 0;
      for (const auto& p : X.pairs) {
        if (!F->emu && mine_only) {
          if (p.src == F->me) sn += p.cnt;
          if (p.dst == F->me) rn += p.cnt;
        } else {
          sn = std::max(sn, p.cnt);
        }
      }
      return F->emu ? sn : sn + rn;
    };
    for (const auto& L : F->levels)
      for (const auto& X : L.xs) xmax = std::max(xmax, step_rows(X, true));
    xmax = std::max(xmax, step_rows(F->gather, true));
    double* xbuf = nullptr;
    HCK(cudaMallocAsync((void**)&xbuf, std::max<size_t>((size_t)xmax * nrhs * sizeof(double), 8), s));
    owned.push_back(xbuf);
    int64_t moved = 0;
    // rows listed by X from bufs[src] to bufs[dst] (vector rows or contribution rows)
    auto exchange = [&](const LevelRec::XStep& X, std::vector<double*>& bufs) {
      if (X.pairs.empty()) return;
      if (F->emu) {
        for (const auto& p : X.pairs) {
          launch_rows_gather(bufs[(size_t)p.src], X.d_rows + p.off, p.cnt, nrhs, xbuf, s);
          launch_rows_scatter(xbuf, X.d_rows + p.off, p.cnt, nrhs, bufs[(size_t)p.dst], s);
          g_launches += 2;
          moved += p.cnt;
        }
        return;
      }
      std::vector<P2P> sends, recvs;
      std::vector<const LevelRec::XPair*> unpack;
      int64_t o = 0;
      for (const auto& p : X.pairs) {
        if (p.src == F->me) {
          launch_rows_gather(bufs[(size_t)F->me], X.d_rows + p.off, p.cnt, nrhs, xbuf + o * nrhs, s);
          ++g_launches;
          sends.push_back(P2P{p.dst, xbuf + o * nrhs, (size_t)p.cnt * nrhs * sizeof(double)});
          o += p.cnt;
          moved += p.cnt;
        }
      }
      const int64_t rbase = o;
      for (const auto& p : X.pairs) {
        if (p.dst == F->me) {
          recvs.push_back(P2P{p.src, xbuf + o * nrhs, (size_t)p.cnt * nrhs * sizeof(double)});
          unpack.push_back(&p);
          o += p.cnt;
          moved += p.cnt;
        }
      }
      if (sends.empty() && recvs.empty()) return;
      try {
        comm_sendrecv(F->comm, sends.data(), (int)sends.size(), recvs.data(), (int)recvs.size(), s);
      } catch (const std::exception& e) {
        throw Fail{HIFDE_CUDA, e.what()};
      }
      o = rbase;
      for (const auto* p : unpack) {
        launch_rows_scatter(xbuf + o * nrhs, X.d_rows + p->off, p->cnt, nrhs, bufs[(size_t)F->me], s);
        ++g_launches;
        o += p->cnt;
      }
    };
    for (size_t li = 0; li < nl; ++li) {
      const LevelRec& L = F->levels[li];
      exchange(L.xs[0], vr);
      for (int r = lo; r < hi; ++r) fwd_records(L.rank_view[(size_t)r], vr[(size_t)r], cr[(size_t)r], false);
      exchange(L.xs[1], cr);
      for (int r = lo; r < hi; ++r) fwd_reduce(L.rank_view[(size_t)r], vr[(size_t)r], cr[(size_t)r]);
    }
    for (size_t li = nl; li-- > 0;) {
      const LevelRec& L = F->levels[li];
      exchange(L.xs[2], vr);
      for (int r = lo; r < hi; ++r) bwd_records(L.rank_view[(size_t)r], vr[(size_t)r], false);
    }
    if (F->emu) {  // rows held by virtual ranks 1.. into rank 0's vector
      exchange(F->gather, vr);
    } else {  // every rank returns the whole solution: zeros where another rank holds the row, summed
      launch_rows_zero_unheld(v, F->d_holder, F->me, F->n, nrhs, s);
      ++g_launches;
      try {
        comm_allreduce(F->comm, v, (size_t)F->n * nrhs, kF64, kSum, s);
      } catch (const std::exception& e) {
        throw Fail{HIFDE_CUDA, e.what()};
      }
    }
    F->solve_xfer_bytes += moved * nrhs * (int64_t)sizeof(double);
    for (void* q : owned) HCK(cudaFreeAsync(q, s));
  } else {
    // kernel log: one entry per level and direction; algorithmic bytes = the
    // level's factor entries + one read and one write of every touched row
    auto kbegin = [&](const LevelRec& L, bool fwd) {
      if (!F->klog.on || (L.nall == 0 && L.recs.empty())) return -1;
      const char* nm = L.kind == 1 ? (fwd ? "solve_skel_fwd" : "solve_skel_bwd")
                                   : (fwd ? "solve_elim_fwd" : "solve_elim_bwd");
      return F->klog.begin(nm, L.tag, 1, 8.0 * (L.solve_fac + 2.0 * L.solve_rows * nrhs) * 1e-9,
                           2.0 * L.solve_fac * nrhs * 1e-9, s);
    };
    struct KEnd {
      const hifde_factor_t* F; int kl; cudaStream_t s;
      ~KEnd() { F->klog.end(kl, s); }
    };
    for (size_t li = 0; li < nl; ++li) {
      const LevelRec& L = F->levels[li];
      KEnd kend{F, kbegin(L, true), s};
      fwd_records(L, v, contrib, li == 0 && bands);
      fwd_reduce(L, v, contrib);
    }
    for (size_t li = nl; li-- > 0;) {
      const LevelRec& L = F->levels[li];
      KEnd kend{F, kbegin(L, false), s};
      bwd_records(L, v, li == 0 && bands);
    }
  }
  HCK(cudaGetLastError());
  HCK(cudaFreeAsync(contrib, s));
  HCK(cudaFreeAsync(tscr, s));
  HCK(cudaFreeAsync(scratch, s));
}

// The level-0 record bounds of the banded host solve, computed once per
// factor: prefix max of the records' largest cell DOF (pmax[j] = over
// records < j) and suffix min of their smallest (smin[j] = over records >= j).
bool level0_bands(const hifde_factor_t* F, cudaStream_t s) {
  if (!level0_bandable(F)) return false;
  std::lock_guard<std::mutex> lk(F->band_m);
  if (!F->band_done) {
    const LevelRec& L = F->levels[0];
    const int nrec = L.nsmall;
    int32_t* d = nullptr;
    HCK(cudaMallocAsync((void**)&d, sizeof(int32_t) * 2 * (size_t)nrec, s));
    launch_solve_rec_rows(L.d_recs, nrec, F->idx.p, d, d + nrec, s);
    std::vector<int32_t> h((size_t)2 * nrec);
    HCK(cudaMemcpyAsync(h.data(), d, sizeof(int32_t) * h.size(), cudaMemcpyDeviceToHost, s));
    HCK(cudaFreeAsync(d, s));
    HCK(cudaStreamSynchronize(s));
    F->band_pmax.assign((size_t)nrec + 1, -1);
    F->band_smin.assign((size_t)nrec + 1, (int32_t)F->n);
    for (int j = 0; j < nrec; ++j) F->band_pmax[(size_t)j + 1] = std::max(F->band_pmax[(size_t)j], h[(size_t)nrec + j]);
    for (int j = nrec; j-- > 0;) F->band_smin[(size_t)j] = std::min(F->band_smin[(size_t)j + 1], h[(size_t)j]);
    F->band_done = true;
  }
  return true;
}

// Host right-hand sides already page-locked (a pinned torch tensor, ...) and a
// large block: column chunks flow through three engines at once -- the H2D
// copy engine uploads chunk c + 1 (a strided 2D DMA straight from the
// caller's rows) while the SMs sweep chunk c and the D2H engine returns chunk
// c - 1, by a strided DMA straight into the caller's columns when the output
// is page-locked too (hifde_host_alloc blocks), else through pinned pieces
// that host threads scatter.  Same result as one sweep of the whole block,
// column by column.
// `ready` (may be empty) runs once every upload is queued and before the
// factor is read: an options.async_factor factorization is waited for there,
// so the right-hand sides cross PCIe while it still runs.
void solve_pipelined(const hifde_factor_t* F, const double* b, double* x, int nrhs, cudaStream_t s,
                     const std::function<void()>& ready = {}) {
  const int64_t N = F->n;
  const bool early = (bool)ready;
  // Two column chunks (one below 32 RHS): strided DMAs of 8-column (64 B)
  // row pieces run at 24-28 GB/s, 16-column pieces at 47-51 GB/s alone and
  // 71 GB/s both directions at once, 32-column pieces at 56-57 and 101 GB/s
  // (tools/dma2d_probe.py).  Config 3, 64 RHS: 4 chunks of 16 columns 83 ms,
  // 2 of 32 71 ms (H2D 2 x 19.3 + last sweep 10 + last D2H 21).
  const int nch = nrhs >= 32 ? 2 : 1;
  std::vector<int> c0((size_t)nch + 1, 0);
  for (int c = 0; c < nch; ++c) c0[(size_t)c + 1] = (int)((int64_t)nrhs * (c + 1) / nch / 8 * 8);
  c0[(size_t)nch] = nrhs;
  int wmax = 0;
  for (int c = 0; c < nch; ++c) wmax = std::max(wmax, c0[(size_t)c + 1] - c0[(size_t)c]);
  cudaStream_t sh = nullptr, sd = nullptr;
  HCK(cudaStreamCreateWithFlags(&sh, cudaStreamNonBlocking));
  HCK(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
  std::vector<cudaEvent_t> eh((size_t)nch), es((size_t)nch);
  for (int c = 0; c < nch; ++c) {
    HCK(cudaEventCreateWithFlags(&eh[(size_t)c], cudaEventDisableTiming));
    HCK(cudaEventCreateWithFlags(&es[(size_t)c], cudaEventDisableTiming));
  }
  std::vector<double*> vb((size_t)nch, nullptr);
  // (early: on the upload stream -- `s` is busy with the factorization, and an
  // allocation ordered on it would hold the uploads back until it ends)
  for (int c = 0; c < nch; ++c)
    HCK(cudaMallocAsync((void**)&vb[(size_t)c], (size_t)N * (c0[(size_t)c + 1] - c0[(size_t)c]) * sizeof(double),
                        early ? sh : s));
  cudaEvent_t ealloc = nullptr;
  HCK(cudaEventCreateWithFlags(&ealloc, cudaEventDisableTiming));
  if (!early) {
    HCK(cudaEventRecord(ealloc, s));
    HCK(cudaStreamWaitEvent(sh, ealloc, 0));
  }
  // every chunk's upload in kBands row bands, an event per band
  constexpr int kBands = 8;
  std::vector<cudaEvent_t> band_events;
  auto new_event = [&]() {
    cudaEvent_t e;
    HCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    band_events.push_back(e);
    return e;
  };
  std::vector<std::vector<cudaEvent_t>> up_ev((size_t)nch);
  if (early) {  // the factorization's own uploads (the CSR) go first
    while (!F->inputs_issued.load()) std::this_thread::sleep_for(std::chrono::microseconds(20));
    hifde_factor_t* Fm = const_cast<hifde_factor_t*>(F);
    std::lock_guard<std::mutex> lk(Fm->ev_m);
    if (Fm->ev_inputs) HCK(cudaStreamWaitEvent(sh, Fm->ev_inputs, 0));
  }
  // early: the factorization's own host-to-device copies (the task tables of
  // the blocked levels) share the copy engine with these uploads, and with
  // upload work always queued they were starved until the last band had
  // gone (config 3: level 2's blocked elimination began 27 ms late; three
  // 4 MB pieces in flight did the same).  So the bands go in 8 MB pieces,
  // ONE in flight: this thread waits for a piece before it queues the next
  // (it has nothing else to do until the factor is complete), and the gap
  // lets the other stream's copy in.  Piece sizes from 4 to 64 MB measure
  // the same step time.
  cudaEvent_t fc[4] = {nullptr, nullptr, nullptr, nullptr};
  if (early)
    for (auto& e : fc) e = new_event();
  int64_t issued = 0;
  for (int c = 0; c < nch; ++c) {
    const int w = c0[(size_t)c + 1] - c0[(size_t)c];
    const int64_t piece = early ? std::max<int64_t>(1024, ((int64_t)8 << 20) / ((int64_t)w * 8)) : N;
    for (int k = 0; k < kBands; ++k) {
      const int64_t r0 = N * k / kBands, r1 = k + 1 == kBands ? N : N * (k + 1) / kBands;
      for (int64_t q0 = r0; q0 < r1; q0 += piece) {
        const int64_t q1 = std::min(r1, q0 + piece);
        if (early && issued >= 1) HCK(cudaEventSynchronize(fc[(issued - 1) & 3]));
        HCK(cudaMemcpy2DAsync(vb[(size_t)c] + (size_t)q0 * w, (size_t)w * sizeof(double),
                              b + (size_t)q0 * nrhs + c0[(size_t)c], (size_t)nrhs * sizeof(double),
                              (size_t)w * sizeof(double), (size_t)(q1 - q0), cudaMemcpyHostToDevice, sh));
        if (early) HCK(cudaEventRecord(fc[issued & 3], sh));
        ++issued;
      }
      up_ev[(size_t)c].push_back(new_event());
      HCK(cudaEventRecord(up_ev[(size_t)c].back(), sh));
    }
    HCK(cudaEventRecord(eh[(size_t)c], sh));
  }
  if (early) {
    try {
      ready();
    } catch (...) {  // the factorization failed: nothing of it may be read
      for (int c = 0; c < nch; ++c) cudaFreeAsync(vb[(size_t)c], sh);
      cudaStreamSynchronize(sh);
      for (cudaEvent_t e : band_events) cudaEventDestroy(e);
      for (int c = 0; c < nch; ++c) {
        cudaEventDestroy(eh[(size_t)c]);
        cudaEventDestroy(es[(size_t)c]);
      }
      cudaEventDestroy(ealloc);
      cudaStreamDestroy(sh);
      cudaStreamDestroy(sd);
      throw;
    }
  }
  // Banded level 0 (page-locked output, a level 0 of one-CTA records): each
  // chunk uploads in row bands and its level-0 forward records run as the
  // rows they read land; its level-0 backward runs in record bands and the
  // rows they finish leave at once -- the first and last level of every
  // chunk's sweep overlap its own transfers (config 3, 64 RHS: the last
  // chunk's tail was sweep 8 + D2H 19 ms after its upload).
  const bool banded = PinnedXfer::page_locked(x) && level0_bands(F, s);
  std::vector<SweepBands> sb((size_t)nch);
  std::vector<std::vector<std::pair<int64_t, int64_t>>> d2h_rows((size_t)nch);
  if (banded) {
    const int nrec = (int)F->band_pmax.size() - 1;
    for (int c = 0; c < nch; ++c) {
      SweepBands& B = sb[(size_t)c];
      // forward: band k = records whose cells lie below upload row bound k + 1
      int j = 0;
      for (int k = 0; k < kBands; ++k) {
        const int64_t ub = k + 1 == kBands ? N : N * (k + 1) / kBands;
        int j1 = j;
        if (k + 1 == kBands) j1 = nrec;
        else
          while (j1 < nrec && F->band_pmax[(size_t)j1 + 1] < ub) ++j1;  // pmax[j1+1]: max cell DOF of records < j1+1
        B.fwd.emplace_back(j, j1);
        B.fwd_wait.push_back(up_ev[(size_t)c][(size_t)k]);
        j = j1;
      }
      // backward: equal record bands; rows below the smallest cell DOF of the
      // records still to come are final
      int64_t done = 0;
      for (int k = 0; k < kBands; ++k) {
        const int lo = (int)((int64_t)nrec * k / kBands), hi = (int)((int64_t)nrec * (k + 1) / kBands);
        B.bwd.emplace_back(lo, hi);
        B.bwd_done.push_back(new_event());
        const int64_t fin = hi >= nrec ? N : std::min<int64_t>(N, F->band_smin[(size_t)hi]);
        d2h_rows[(size_t)c].emplace_back(done, std::max(done, fin));
        done = std::max(done, fin);
      }
    }
  }
  for (int c = 0; c < nch; ++c) {  // every sweep queued at once (the uploads are)
    const int w = c0[(size_t)c + 1] - c0[(size_t)c];
    if (banded) {
      solve_sweep(F, vb[(size_t)c], w, s, &sb[(size_t)c]);
    } else {
      HCK(cudaStreamWaitEvent(s, eh[(size_t)c], 0));
      solve_sweep(F, vb[(size_t)c], w, s);
    }
    HCK(cudaEventRecord(es[(size_t)c], s));
  }
  if (banded) {  // each chunk's finished row bands straight into the caller's columns
    for (int c = 0; c < nch; ++c) {
      const int w = c0[(size_t)c + 1] - c0[(size_t)c];
      for (int k = 0; k < kBands; ++k) {
        HCK(cudaStreamWaitEvent(sd, sb[(size_t)c].bwd_done[(size_t)k], 0));
        const int64_t r0 = d2h_rows[(size_t)c][(size_t)k].first, r1 = d2h_rows[(size_t)c][(size_t)k].second;
        if (r1 > r0)
          HCK(cudaMemcpy2DAsync(x + (size_t)r0 * nrhs + c0[(size_t)c], (size_t)nrhs * sizeof(double),
                                vb[(size_t)c] + (size_t)r0 * w, (size_t)w * sizeof(double), (size_t)w * sizeof(double),
                                (size_t)(r1 - r0), cudaMemcpyDeviceToHost, sd));
      }
      HCK(cudaStreamWaitEvent(sd, es[(size_t)c], 0));  // (rows past the last band bound: none; the sweep's end)
      const int64_t rdone = d2h_rows[(size_t)c].back().second;
      if (rdone < N)
        HCK(cudaMemcpy2DAsync(x + (size_t)rdone * nrhs + c0[(size_t)c], (size_t)nrhs * sizeof(double),
                              vb[(size_t)c] + (size_t)rdone * w, (size_t)w * sizeof(double), (size_t)w * sizeof(double),
                              (size_t)(N - rdone), cudaMemcpyDeviceToHost, sd));
    }
    for (int c = 0; c < nch; ++c) HCK(cudaFreeAsync(vb[(size_t)c], sd));
    HCK(cudaStreamSynchronize(sd));
    for (cudaEvent_t e : band_events) cudaEventDestroy(e);
    for (int c = 0; c < nch; ++c) {
      cudaEventDestroy(eh[(size_t)c]);
      cudaEventDestroy(es[(size_t)c]);
    }
    cudaEventDestroy(ealloc);
    HCK(cudaStreamSynchronize(s));
    cudaStreamDestroy(sh);
    cudaStreamDestroy(sd);
    return;
  }
  const size_t total = (size_t)N * nrhs * sizeof(double);
  PinnedXfer::prefault(x, total);  // while the first chunks upload and sweep
  pinned_xfer().d2h_columns(x, nrhs, vb, c0, N, es, sd);
  for (int c = 0; c < nch; ++c) HCK(cudaFreeAsync(vb[(size_t)c], sd));
  HCK(cudaStreamSynchronize(sd));
  for (cudaEvent_t e : band_events) cudaEventDestroy(e);
  for (int c = 0; c < nch; ++c) {
    cudaEventDestroy(eh[(size_t)c]);
    cudaEventDestroy(es[(size_t)c]);
  }
  cudaEventDestroy(ealloc);
  HCK(cudaStreamSynchronize(s));
  cudaStreamDestroy(sh);
  cudaStreamDestroy(sd);
}

// Joins an options.async_factor factorization; its status (and message).
int async_done(const hifde_factor_t* f) {
  std::lock_guard<std::mutex> lk(f->async_m);
  if (f->worker.joinable()) f->worker.join();
  f->async_pending.store(0);
  if (f->async_status != HIFDE_OK) g_err = f->async_err;
  return f->async_status;
}

void do_solve(const hifde_factor_t* F, const double* b, double* x, int nrhs, bool dev, cudaStream_t s) {
  const int64_t N = F->n;
  const size_t bytes = (size_t)N * nrhs * sizeof(double);
  std::unique_lock<std::mutex> klk(F->klog_m, std::defer_lock);
  const bool disjoint = (const char*)x >= (const char*)b + bytes || (const char*)x + bytes <= (const char*)b;
  const bool pipe_ok = !dev && nrhs >= 16 && bytes >= ((size_t)64 << 20) && disjoint && PinnedXfer::page_locked(b);
  auto wait_factor = [&]() {  // an options.async_factor factorization (never sharded)
    if (const int st = async_done(F)) throw Fail{st, F->async_err};
  };
  auto klog_begin = [&]() {
    if (F->klog.on) {
      klk.lock();
      F->klog.clear(1);
    }
  };
  auto solve_timeline = [&]() {  // HIFDE_PROFILE: the solve's logged launches on the factorization's clock
    if (!getenv("HIFDE_PROFILE") || !F->klog.on || F->klog.v.empty()) return;
    cudaDeviceSynchronize();
    const cudaEvent_t t0e = F->klog.v.front().e0;
    for (const auto& E : F->klog.v) {
      if (E.phase != 1) continue;
      float a = 0.f, c = 0.f;
      cudaEventElapsedTime(&a, t0e, E.e0);
      cudaEventElapsedTime(&c, t0e, E.e1);
      fprintf(stderr, "[hifde] tl1 %8.3f %8.3f %7.3f  %-24s tag %.3f\n", a, c, c - a, E.name.c_str(), E.tag);
    }
  };
  if (pipe_ok && F->async_pending.load()) {  // uploads first, then wait for the factor
    solve_pipelined(F, b, x, nrhs, s, [&]() {
      wait_factor();
      klog_begin();
    });
    solve_timeline();
    return;
  }
  wait_factor();
  klog_begin();
  if (pipe_ok && !F->part) {
    solve_pipelined(F, b, x, nrhs, s);
    solve_timeline();
    return;
  }
  double* v = nullptr;
  HCK(cudaMallocAsync((void**)&v, std::max<size_t>(bytes, 8), s));
  if (dev) HCK(cudaMemcpyAsync(v, b, bytes, cudaMemcpyDeviceToDevice, s));
  else pinned_xfer().h2d(v, b, bytes, s);
  solve_sweep(F, v, nrhs, s);
  // host output that is not the input: fault its pages in while the sweep runs
  if (!dev && disjoint) PinnedXfer::prefault(x, bytes);
  if (dev) HCK(cudaMemcpyAsync(x, v, bytes, cudaMemcpyDeviceToDevice, s));
  else pinned_xfer().d2h(x, v, bytes, s);
  HCK(cudaFreeAsync(v, s));
  if (!dev) HCK(cudaStreamSynchronize(s));
}


// y = F x: the solve sweep inverted record by record (kernels_solve.cu).
void do_apply(const hifde_factor_t* F, const double* x, double* y, int nrhs, bool dev, cudaStream_t s) {
  ensure_whole(F, s);
  const int64_t N = F->n;
  const size_t bytes = (size_t)N * nrhs * sizeof(double);
  double* v = nullptr;
  HCK(cudaMallocAsync((void**)&v, std::max<size_t>(bytes, 8), s));
  if (dev) HCK(cudaMemcpyAsync(v, x, bytes, cudaMemcpyDeviceToDevice, s));
  else pinned_xfer().h2d(v, x, bytes, s);
  double* contrib = nullptr;
  HCK(cudaMallocAsync((void**)&contrib, std::max<size_t>(F->max_contrib * nrhs * sizeof(double), 8), s));
  size_t scratch_need = 0;
  auto plan = [&](const LevelRec& L, size_t& smem, int64_t& per_rec) {
    const int64_t d = (int64_t)(L.all_max_nc + L.all_max_nq) * nrhs;
    const size_t need = (size_t)d * sizeof(double);
    if (need <= kSolveDynSmem) { smem = need; per_rec = 0; }
    else { smem = 0; per_rec = d; scratch_need = std::max(scratch_need, (size_t)d * L.nall); }
  };
  for (const auto& L : F->levels) { size_t a; int64_t b; plan(L, a, b); }
  double* scratch = nullptr;
  HCK(cudaMallocAsync((void**)&scratch, std::max<size_t>(scratch_need * sizeof(double), 8), s));
  const int32_t* idx = F->idx.p;
  const double* fac = F->fac.p;
  const size_t nl = F->levels.size();
  for (size_t li = 0; li < nl; ++li) {  // inverse of the backward sweep, level 0 first
    const LevelRec& L = F->levels[li];
    size_t sm; int64_t pr;
    plan(L, sm, pr);
    if (L.kind == 1) launch_apply_skel(L.d_all, L.nall, idx, fac, v, nrhs, scratch, pr, sm, 0, s);
    else launch_apply_elim(L.d_all, L.nall, idx, fac, v, nrhs, contrib, scratch, pr, sm, 0, s);
    if (L.nall) ++g_launches;
  }
  for (size_t li = nl; li-- > 0;) {  // inverse of the forward sweep, top first
    const LevelRec& L = F->levels[li];
    size_t sm; int64_t pr;
    plan(L, sm, pr);
    if (L.kind == 1) {
      launch_apply_skel(L.d_all, L.nall, idx, fac, v, nrhs, scratch, pr, sm, 1, s);
    } else {
      launch_apply_elim(L.d_all, L.nall, idx, fac, v, nrhs, contrib, scratch, pr, sm, 1, s);
      if (L.kind == 0 && L.ntargets) {
        launch_solve_reduce(L.d_targets, L.d_ptr, L.d_ent, L.ntargets, contrib, v, nrhs, s, 1.0);
        ++g_launches;
      }
    }
    if (L.nall) ++g_launches;
  }
  HCK(cudaGetLastError());
  if (dev) HCK(cudaMemcpyAsync(y, v, bytes, cudaMemcpyDeviceToDevice, s));
  else pinned_xfer().d2h(y, v, bytes, s);
  HCK(cudaFreeAsync(v, s));
  HCK(cudaFreeAsync(contrib, s));
  HCK(cudaFreeAsync(scratch, s));
  if (!dev) HCK(cudaStreamSynchronize(s));
}

// Preconditioned CG with A (CSR) and the factor as preconditioner, all on the
// device (src/krylov.py:48-77): the host only reads ||r|| each iteration.
void do_pcg(const hifde_factor_t* F, const int64_t* ip, const int32_t* ix, const double* va, int64_t nnz,
            const double* b, double* x, double tol, int max_iter, bool dev, cudaStream_t s, int* iters,
            double* resid, int* converged) {
  const int64_t N = F->n;
  const size_t vb = (size_t)std::max<int64_t>(N, 1) * sizeof(double);
  const int64_t *d_ip = ip;
  const int32_t* d_ix = ix;
  const double* d_va = va;
  std::vector<void*> owned;
  auto dalloc = [&](size_t bytes) {
    void* p = nullptr;
    HCK(cudaMallocAsync(&p, std::max<size_t>(bytes, 8), s));
    owned.push_back(p);
    return p;
  };
  if (!dev) {
    int64_t* a = (int64_t*)dalloc((N + 1) * sizeof(int64_t));
    int32_t* c = (int32_t*)dalloc(nnz * sizeof(int32_t));
    double* v = (double*)dalloc(nnz * sizeof(double));
    HCK(cudaMemcpyAsync(a, ip, (N + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    HCK(cudaMemcpyAsync(c, ix, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    HCK(cudaMemcpyAsync(v, va, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
    d_ip = a; d_ix = c; d_va = v;
  }
  double* xv = (double*)dalloc(vb);
  double* r = (double*)dalloc(vb);
  double* z = (double*)dalloc(vb);
  double* p = (double*)dalloc(vb);
  double* ap = (double*)dalloc(vb);
  double* part = (double*)dalloc(sizeof(double) * dot_partials());
  double* sc = (double*)dalloc(sizeof(double) * 8);  // rz, pAp, rr, rz_new, bb
  HCK(cudaMemcpyAsync(r, b, vb, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  HCK(cudaMemsetAsync(xv, 0, vb, s));
  double* hs = nullptr;  // pinned readback of the residual
  HCK(cudaMallocHost((void**)&hs, 2 * sizeof(double)));
  struct Free {
    std::vector<void*>& o; double* h; cudaStream_t s;
    ~Free() { for (void* q : o) cudaFreeAsync(q, s); if (h) cudaFreeHost(h); }
  } fr{owned, hs, s};
  launch_dot(r, r, N, part, sc + 4, s);
  HCK(cudaMemcpyAsync(hs, sc + 4, sizeof(double), cudaMemcpyDeviceToHost, s));
  HCK(cudaStreamSynchronize(s));
  const double bnorm = std::sqrt(hs[0]);
  *iters = 0; *resid = 0.0; *converged = 1;
  if (bnorm == 0.0) {
    HCK(cudaMemcpyAsync(x, xv, vb, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    return;
  }
  do_solve(F, r, z, 1, true, s);
  HCK(cudaMemcpyAsync(p, z, vb, cudaMemcpyDeviceToDevice, s));
  launch_dot(r, z, N, part, sc + 0, s);
  double res = 1.0;
  *converged = 0;
  int it = 1;
  for (; it <= max_iter; ++it) {
    launch_spmv(d_ip, d_ix, d_va, p, ap, N, s);
    launch_dot(p, ap, N, part, sc + 1, s);
    launch_cg_xr(xv, r, p, ap, sc, N, s);
    launch_dot(r, r, N, part, sc + 2, s);
    HCK(cudaMemcpyAsync(hs, sc + 2, sizeof(double), cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    res = std::sqrt(hs[0]) / bnorm;
    if (res <= tol) { *converged = 1; break; }
    do_solve(F, r, z, 1, true, s);
    launch_dot(r, z, N, part, sc + 3, s);
    launch_cg_p(p, z, sc, N, s);
  }
  *iters = std::min(it, max_iter);
  *resid = res;
  HCK(cudaMemcpyAsync(x, xv, vb, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  HCK(cudaStreamSynchronize(s));
}

// sqrt of the dominant eigenvalue of G^T G by power iteration (src/krylov.py:
// 153-170), on the device.  kind 0: G = G^T = A - F; 1: G = G^T = A;
// 2: G = I - A F^-1, G^T = I - F^-1 A.  x0 = the reference's start vector.
void do_power(const hifde_factor_t* F, const int64_t* ip, const int32_t* ix, const double* va, int64_t nnz,
              int kind, const double* x0, double rtol, int max_iter, cudaStream_t s, double* value, int* conv,
              int* iters) {
  const int64_t N = F->n;
  const size_t vb = (size_t)std::max<int64_t>(N, 1) * sizeof(double);
  std::vector<void*> owned;
  auto dalloc = [&](size_t bytes) {
    void* p = nullptr;
    HCK(cudaMallocAsync(&p, std::max<size_t>(bytes, 8), s));
    owned.push_back(p);
    return p;
  };
  int64_t* d_ip = (int64_t*)dalloc((N + 1) * sizeof(int64_t));
  int32_t* d_ix = (int32_t*)dalloc(nnz * sizeof(int32_t));
  double* d_va = (double*)dalloc(nnz * sizeof(double));
  HCK(cudaMemcpyAsync(d_ip, ip, (N + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  HCK(cudaMemcpyAsync(d_ix, ix, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  HCK(cudaMemcpyAsync(d_va, va, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
  double* x = (double*)dalloc(vb);
  double* t = (double*)dalloc(vb);
  double* u = (double*)dalloc(vb);
  double* y = (double*)dalloc(vb);
  double* z = (double*)dalloc(vb);
  double* part = (double*)dalloc(sizeof(double) * dot_partials());
  double* nn = (double*)dalloc(sizeof(double));
  double* hs = nullptr;
  HCK(cudaMallocHost((void**)&hs, sizeof(double)));
  struct Free {
    std::vector<void*>& o; double* h; cudaStream_t s;
    ~Free() { for (void* q : o) cudaFreeAsync(q, s); if (h) cudaFreeHost(h); }
  } fr{owned, hs, s};
  HCK(cudaMemcpyAsync(x, x0, vb, cudaMemcpyHostToDevice, s));
  // out = G v  (or G^T v when trans), using t as scratch
  auto gapply = [&](const double* v, double* out, bool trans) {
    if (kind == 1) {
      launch_spmv(d_ip, d_ix, d_va, v, out, N, s);
    } else if (kind == 0) {
      launch_spmv(d_ip, d_ix, d_va, v, t, N, s);
      do_apply(F, v, u, 1, true, s);
      launch_sub(out, t, u, N, s);
    } else if (!trans) {  // v - A F^-1 v
      do_solve(F, v, u, 1, true, s);
      launch_spmv(d_ip, d_ix, d_va, u, t, N, s);
      launch_sub(out, v, t, N, s);
    } else {              // v - F^-1 A v
      launch_spmv(d_ip, d_ix, d_va, v, t, N, s);
      do_solve(F, t, u, 1, true, s);
      launch_sub(out, v, u, N, s);
    }
  };
  double est = 0.0;
  *conv = 0;
  *iters = max_iter;
  *value = 0.0;
  for (int it = 1; it <= max_iter; ++it) {
    gapply(x, y, false);
    gapply(y, z, true);  // z = G^T (G x)
    launch_dot(z, z, N, part, nn, s);
    HCK(cudaMemcpyAsync(hs, nn, sizeof(double), cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    const double lam = std::sqrt(hs[0]);
    const double new_est = std::sqrt(lam);
    if (lam == 0.0 || !std::isfinite(lam)) {
      *value = std::isfinite(lam) ? new_est : INFINITY;
      *conv = 1;
      *iters = it;
      return;
    }
    launch_scale(x, z, nn, N, s);
    if (it > 1 && std::fabs(new_est - est) <= rtol * new_est) {
      *value = new_est;
      *conv = 1;
      *iters = it;
      HCK(cudaStreamSynchronize(s));
      return;
    }
    est = new_est;
  }
  *value = est;
  HCK(cudaStreamSynchronize(s));
}

int fail_to_status(const Fail& f) {
  g_err = f.msg;
  return f.code;
}

void set_pool_threshold(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

}  // namespace
}  // namespace hifde

// ===========================================================================
// C ABI
// ===========================================================================
using namespace hifde;

extern "C" {

const char* hifde_version(void) { return "hifde-b200 0.1.0 (sm_100a)"; }

int hifde_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void hifde_default_options(hifde_options_t* o, int variant) {
  std::memset(o, 0, sizeof *o);
  o->variant = variant;
  o->skip_levels = variant == HIFDE_VARIANT_HIFDE3X ? 1 : 0;
  o->spd = 1;
  o->order_mode = HIFDE_ORDER_AUTO;
  o->exact_max_batches = 64;
  o->device = 0;
  o->eps = 0.0;
}

const char* hifde_last_error(void) { return g_err.c_str(); }

int64_t hifde_last_launch_count(void) { return g_launches; }

// The factorization proper (the calling thread's device is opt.device).
static int factor_run(hifde_factor_t* F, const GridDesc& g, const hifde_options_t& o, const int64_t* indptr,
                      const int32_t* indices, const double* vals, int64_t n, int nlevels) {
  const hifde_options_t* opt = &o;
  try {
    std::lock_guard<std::mutex> lock(g_host_mutex);
    HTRACE("locked");
    Factorizer fz;
    HTRACE("factorizer constructed");
    fz.g = g;
    fz.opt = *opt;
    if (opt->variant == HIFDE_VARIANT_MF) {
      fz.opt.variant = HIFDE_VARIANT_HIFDE;
      fz.opt.skip_levels = nlevels;  // factor_mf == factor_hifde(skip_levels=L)
      fz.opt.eps = 0.0;
    }
    if (fz.opt.exact_max_batches <= 0) fz.opt.exact_max_batches = 64;
    fz.F = F;
    fz.F_ = F;
    fz.s = F->stream;
    F->klog.on = opt->kernel_log != 0;
    // int32 offsets from the caller: widened here on the host threads into
    // a cached buffer (its pages stay mapped across factorizations)
    const int64_t* ip64 = indptr;
    if (opt->indptr_int32) {
      if (opt->input_on_device) throw Fail{HIFDE_BADARG, "indptr_int32 needs host arrays"};
      const int32_t* ip32 = reinterpret_cast<const int32_t*>(indptr);
      int64_t* w = (int64_t*)host_cache().wide_ip.get((size_t)(n + 1) * sizeof(int64_t));
      if (!w) throw Fail{HIFDE_CUDA, "page-locked host allocation failed"};
      const int nth = n > (1 << 20) ? PinnedXfer::copy_threads() : 1;
#pragma omp parallel for num_threads(nth) schedule(static)
      for (int64_t i = 0; i <= n; ++i) w[i] = ip32[i];
      ip64 = w;
    }
    const int64_t nnz = opt->input_on_device ? 0 : ip64[n];
    const char* sample = getenv("HIFDE_SAMPLE");  // host sampling profile (diagnostics)
    if (sample) host_sampler_start();
    fz.run(ip64, indices, vals, nnz);
    if (sample) host_sampler_stop(sample);
  } catch (const Fail& f) {
    return fail_to_status(f);
  } catch (const std::exception& e) {
    g_err = e.what();
    return HIFDE_INTERNAL;
  }
  return HIFDE_OK;
}

int hifde_factor(const int64_t* indptr, const int32_t* indices, const double* vals, int64_t n,
                 int dim, int n_grid, int m_leaf, int nlevels, const hifde_options_t* opt,
                 hifde_factor_t** out) {
  g_err.clear();
  g_launches = 0;
  if (!out || !opt) { g_err = "null argument"; return HIFDE_BADARG; }
  *out = nullptr;
  if (dim != 2 && dim != 3) { g_err = "dim must be 2 or 3"; return HIFDE_BADARG; }
  if (opt->variant == HIFDE_VARIANT_HIFDE3X && dim != 3) {
    g_err = "factor_hifde3x requires a 3D grid";
    return HIFDE_BADARG;
  }
  if (!opt->spd) {
    g_err = "indefinite (Bunch-Kaufman) factorization is not implemented on the GPU path";
    return HIFDE_BADARG;
  }
  if (opt->comm && !opt->comm->emulated && opt->comm->P > 1 && opt->comm->device != opt->device) {
    g_err = "options.device differs from the communicator's device";
    return HIFDE_BADARG;
  }
  GridDesc g;
  g.dim = dim;
  g.n = n_grid;
  g.m = m_leaf;
  g.nlevels = nlevels;
  if (n_grid < 2 || m_leaf < 2 || nlevels < 0 || g.ndof() != n) {
    g_err = "grid does not match the matrix order";
    return HIFDE_BADARG;
  }
  if (nlevels > 0 && ((int64_t)m_leaf << nlevels) != n_grid) {
    g_err = "n must equal m * 2^nlevels";
    return HIFDE_BADARG;
  }
  std::unique_ptr<hifde_factor_t> F(new hifde_factor_t);
  HTRACE("hifde_factor entry");
  try {
    HCK(cudaSetDevice(opt->device));
    HTRACE("device set");
    set_pool_threshold(opt->device);
    F->device = opt->device;
    F->n = n;
    F->dim = dim;
    F->variant = opt->variant;
    F->spd = 1;
    F->eps = opt->variant == HIFDE_VARIANT_MF ? 0.0 : opt->eps;
    if (opt->stream) {
      F->stream = (cudaStream_t)opt->stream;
    } else {
      HCK(cudaStreamCreateWithFlags(&F->stream, cudaStreamNonBlocking));
      F->own_stream = true;
    }
    HTRACE("stream ready");
  } catch (const Fail& f) {
    return fail_to_status(f);
  } catch (const std::exception& e) {
    g_err = e.what();
    return HIFDE_INTERNAL;
  }
  // options.async_factor (one GPU): the factorization on a library thread;
  // the handle goes back at once, async_done() joins
  if (opt->async_factor && !(opt->comm && opt->comm->P > 1)) {
    hifde_factor_t* Fp = F.get();
    const hifde_options_t o = *opt;
    Fp->inputs_issued.store(0);
    Fp->async_pending.store(1);
    Fp->worker = std::thread([=]() {
      g_err.clear();
      g_launches = 0;
      int st = HIFDE_OK;
      if (cudaSetDevice(o.device) != cudaSuccess) {
        st = HIFDE_CUDA;
        g_err = "cudaSetDevice failed";
      } else {
        st = factor_run(Fp, g, o, indptr, indices, vals, n, nlevels);
      }
      Fp->async_status = st;
      Fp->async_err = g_err;
      Fp->inputs_issued.store(1);
    });
    *out = F.release();
    return HIFDE_OK;
  }
  const int st = factor_run(F.get(), g, *opt, indptr, indices, vals, n, nlevels);
  if (st != HIFDE_OK) return st;
  *out = F.release();
  return HIFDE_OK;
}

int hifde_wait(const hifde_factor_t* f) {
  if (!f) { g_err = "null argument"; return HIFDE_BADARG; }
  return async_done(f);
}

int hifde_import(int64_t n, int dim, double eps, int nlevels, const double* tags, const int32_t* kinds,
                 const int64_t* rec_ptr, const hifde_record_t* recs, const double* fac, int64_t fac_len,
                 const int32_t* idx, int64_t idx_len, int device, hifde_factor_t** out) {
  g_err.clear();
  g_launches = 0;
  if (!out || !tags || !kinds || !rec_ptr || (!recs && rec_ptr[nlevels] > 0) || (!fac && fac_len) ||
      (!idx && idx_len) || n < 1 || nlevels < 1 || kinds[nlevels - 1] != 2) {
    g_err = "bad import arguments (the last level must be the terminal block)";
    return HIFDE_BADARG;
  }
  *out = nullptr;
  std::unique_ptr<hifde_factor_t> F(new hifde_factor_t);
  try {
    HCK(cudaSetDevice(device));
    set_pool_threshold(device);
    F->device = device;
    F->n = n;
    F->dim = dim;
    F->variant = 0;
    F->spd = 1;
    F->eps = eps;
    HCK(cudaStreamCreateWithFlags(&F->stream, cudaStreamNonBlocking));
    F->own_stream = true;
    std::lock_guard<std::mutex> lock(g_host_mutex);
    Factorizer fz;
    fz.F = F.get();
    fz.F_ = F.get();
    fz.s = F->stream;
    fz.import_records(nlevels, tags, kinds, rec_ptr, recs, fac, fac_len, idx, idx_len);
  } catch (const Fail& f) {
    return fail_to_status(f);
  } catch (const std::exception& e) {
    g_err = e.what();
    return HIFDE_INTERNAL;
  }
  *out = F.release();
  return HIFDE_OK;
}

int hifde_host_alloc(size_t bytes, void** out) {
  g_err.clear();
  if (!out) { g_err = "null argument"; return HIFDE_BADARG; }
  *out = nullptr;
  try {
    *out = host_pool().alloc(bytes);
  } catch (const std::exception& e) {
    g_err = e.what();
    return HIFDE_INTERNAL;
  }
  if (!*out) { g_err = "page-locked host allocation failed"; return HIFDE_CUDA; }
  return HIFDE_OK;
}

int hifde_host_free(void* p) {
  g_err.clear();
  if (!p) return HIFDE_OK;
  try {
    if (!host_pool().release(p)) { g_err = "not a block of hifde_host_alloc"; return HIFDE_BADARG; }
  } catch (const std::exception& e) {
    g_err = e.what();
    return HIFDE_INTERNAL;
  }
  return HIFDE_OK;
}

int hifde_solve(const hifde_factor_t* f, const double* b, double* x, int64_t n, int nrhs,
                int device_ptrs, void* stream) {
  g_err.clear();
  g_launches = 0;
  if (!f || !b || !x) { g_err = "null argument"; return HIFDE_BADARG; }
  if (n != f->n || nrhs < 1) { g_err = "right-hand side shape mismatch"; return HIFDE_BADARG; }
  try {
    HCK(cudaSetDevice(f->device));
    cudaStream_t s = stream ? (cudaStream_t)stream : f->stream;
    do_solve(f, b, x, nrhs, device_ptrs != 0, s);  // (waits for an asynchronous factorization itself)
  } catch (const Fail& e) {
    return fail_to_status(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return HIFDE_INTERNAL;
  }
  return HIFDE_OK;
}

int hifde_apply(const hifde_factor_t* f, const double* x, double* y, int64_t n, int nrhs,
                int device_ptrs, void* stream) {
  g_err.clear();
  g_launches = 0;
  if (!f || !x || !y) { g_err = "null argument"; return HIFDE_BADARG; }
  if (const int st = async_done(f)) return st;
  if (n != f->n || nrhs < 1) { g_err = "vector shape mismatch"; return HIFDE_BADARG; }
  try {
    HCK(cudaSetDevice(f->device));
    cudaStream_t s = stream ? (cudaStream_t)stream : f->stream;
    do_apply(f, x, y, nrhs, device_ptrs != 0, s);
  } catch (const Fail& e) {
    return fail_to_status(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return HIFDE_INTERNAL;
  }
  return HIFDE_OK;
}

int hifde_pcg(const hifde_factor_t* f, const int64_t* indptr, const int32_t* indices, const double* vals,
              const double* b, double* x, int64_t n, double tol, int max_iter, int device_ptrs, void* stream,
              int* iters, double* residual, int* converged) {
  g_err.clear();
  g_launches = 0;
  if (f)
    if (const int st = async_done(f)) return st;
  if (!f || !indptr || !indices || !vals || !b || !x || !iters || !residual || !converged) {
    g_err = "null argument";
    return HIFDE_BADARG;
  }
  if (n != f->n || max_iter < 1 || !(tol >= 0.0)) { g_err = "bad pcg arguments"; return HIFDE_BADARG; }
  try {
    HCK(cudaSetDevice(f->device));
    cudaStream_t s = stream ? (cudaStream_t)stream : f->stream;
    int64_t nnz = 0;
    if (device_ptrs) HCK(cudaMemcpy(&nnz, indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
    else nnz = indptr[n];
    do_pcg(f, indptr, indices, vals, nnz, b, x, tol, max_iter, device_ptrs != 0, s, iters, residual, converged);
  } catch (const Fail& e) {
    return fail_to_status(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return HIFDE_INTERNAL;
  }
  return HIFDE_OK;
}

int hifde_level_records(const hifde_factor_t* f, int level, hifde_record_t* out, int64_t cap,
                        int64_t* count) {
  g_err.clear();
  if (f)
    if (const int st = async_done(f)) return st;
  if (!f || !count || level < 0 || level >= (int)f->levels.size()) { g_err = "bad level"; return HIFDE_BADARG; }
  auto& L = const_cast<hifde::LevelRec&>(f->levels[(size_t)level]);
  if (L.d_xrec && L.xrec.empty() && L.nxrec > 0) {  // device-symbolic level: copy its export view once
    L.xrec.resize((size_t)L.nxrec);
    if (cudaSetDevice(f->device) != cudaSuccess ||
        cudaMemcpy(L.xrec.data(), L.d_xrec, L.nxrec * sizeof(hifde_record_t), cudaMemcpyDeviceToHost) != cudaSuccess) {
      L.xrec.clear();
      g_err = "record copy failed";
      return HIFDE_CUDA;
    }
  }
  const auto& X = L.xrec;
  *count = (int64_t)X.size();
  if (out) {
    if (cap < (int64_t)X.size()) { g_err = "record buffer too small"; return HIFDE_BADARG; }
    std::memcpy(out, X.data(), X.size() * sizeof(hifde_record_t));
  }
  return HIFDE_OK;
}

int hifde_copy_arenas(const hifde_factor_t* f, double* fac, int64_t fac_len, int32_t* idx, int64_t idx_len) {
  g_err.clear();
  if (!f) { g_err = "null factor"; return HIFDE_BADARG; }
  if (const int st = async_done(f)) return st;
  if ((fac && fac_len != (int64_t)f->fac.n) || (idx && idx_len != (int64_t)f->idx.n)) {
    g_err = "arena length mismatch";
    return HIFDE_BADARG;
  }
  try {
    HCK(cudaSetDevice(f->device));
    if (fac && fac_len && !f->whole) {  // sharded over real ranks: every rank calls this (a collective)
      ensure_whole(f, f->stream);
      HCK(cudaStreamSynchronize(f->stream));
    }
    if (fac && fac_len) HCK(cudaMemcpy(fac, f->fac.p, (size_t)fac_len * sizeof(double), cudaMemcpyDeviceToHost));
    if (idx && idx_len) HCK(cudaMemcpy(idx, f->idx.p, (size_t)idx_len * sizeof(int32_t), cudaMemcpyDeviceToHost));
  } catch (const Fail& e) {
    return fail_to_status(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return HIFDE_INTERNAL;
  }
  return HIFDE_OK;
}

int hifde_power_norm(const hifde_factor_t* f, const int64_t* indptr, const int32_t* indices, const double* vals,
                     int64_t n, int kind, const double* x0, double rtol, int max_iter, double* value,
                     int* converged, int* iters) {
  g_err.clear();
  g_launches = 0;
  if (f)
    if (const int st = async_done(f)) return st;
  if (!f || !indptr || !indices || !vals || !x0 || !value || !converged || !iters || n != f->n || kind < 0 ||
      kind > 2 || max_iter < 1) {
    g_err = "bad power-iteration arguments";
    return HIFDE_BADARG;
  }
  try {
    HCK(cudaSetDevice(f->device));
    do_power(f, indptr, indices, vals, indptr[n], kind, x0, rtol, max_iter, f->stream, value, converged, iters);
  } catch (const Fail& e) {
    return fail_to_status(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return HIFDE_INTERNAL;
  }
  return HIFDE_OK;
}

int hifde_get_info(const hifde_factor_t* f, hifde_info_t* info) {
  if (!f || !info) return HIFDE_BADARG;
  if (const int st = async_done(f)) return st;
  std::memset(info, 0, sizeof *info);
  info->n = f->n;
  info->dim = f->dim;
  info->nlevels = (int32_t)f->levels.size() - 1;
  info->s_top = f->s_top;
  info->m_f_bytes = f->m_f_bytes;
  info->device_bytes = (int64_t)(f->fac.n * sizeof(double) + f->idx.n * sizeof(int32_t));
  info->t_f_seconds = f->t_f;
  info->eps = f->eps;
  info->spd = f->spd;
  info->variant = f->variant;
  info->fac_len = (int64_t)f->fac.n;
  info->idx_len = (int64_t)f->idx.n;
  info->nranks = f->nranks;
  info->xfer_bytes = f->xfer_bytes;
  info->factor_whole = f->whole ? 1 : 0;
  info->solve_xfer_bytes = f->solve_xfer_bytes.load();
  return HIFDE_OK;
}

int hifde_get_level(const hifde_factor_t* f, int level, hifde_level_info_t* info) {
  if (!f || !info) return HIFDE_BADARG;
  if (const int st = async_done(f)) return st;
  if (level < 0 || level >= (int)f->levels.size()) return HIFDE_BADARG;
  const auto& L = f->levels[(size_t)level];
  info->tag = L.tag;
  info->kind = L.kind;
  info->nbatches = L.nbatches;
  info->ngroups = L.ngroups;
  info->nskel = L.nskel;
  info->nredundant = L.nred;
  info->active_after = L.active_after;
  info->max_front = L.max_front;
  info->seconds = L.seconds;
  info->gflop = L.gflop;
  info->gbytes = L.gbytes;
  info->gpu_seconds = L.gpu_seconds;
  return HIFDE_OK;
}

int hifde_kernel_stats(const hifde_factor_t* f, int phase, hifde_kernel_stat_t* out, int64_t cap, int64_t* count) {
  g_err.clear();
  if (!f || !count || phase < 0 || phase > 1) { g_err = "bad arguments"; return HIFDE_BADARG; }
  if (const int st = async_done(f)) return st;
  try {
    HCK(cudaSetDevice(f->device));
    std::lock_guard<std::mutex> lk(f->klog_m);
    // aggregate by (name, tag) in first-launch order
    std::vector<hifde_kernel_stat_t> agg;
    for (const auto& E : f->klog.v) {
      if (E.phase != phase) continue;
      HCK(cudaEventSynchronize(E.e1));
      float ms = 0.f;
      HCK(cudaEventElapsedTime(&ms, E.e0, E.e1));
      hifde_kernel_stat_t* a = nullptr;
      for (auto& x : agg)
        if (x.tag == E.tag && E.name == x.name) a = &x;
      if (!a) {
        agg.emplace_back();
        a = &agg.back();
        std::memset(a, 0, sizeof *a);
        std::snprintf(a->name, sizeof a->name, "%s", E.name.c_str());
        a->tag = E.tag;
        a->phase = phase;
      }
      a->launches += 1;
      a->seconds += ms * 1e-3;
      a->gbytes += E.gbytes;
      a->gflop += E.gflop;
    }
    *count = (int64_t)agg.size();
    if (out) {
      if (cap < (int64_t)agg.size()) { g_err = "stat buffer too small"; return HIFDE_BADARG; }
      std::memcpy(out, agg.data(), agg.size() * sizeof(hifde_kernel_stat_t));
    }
  } catch (const Fail& e) {
    return fail_to_status(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return HIFDE_INTERNAL;
  }
  return HIFDE_OK;
}

void hifde_free(hifde_factor_t* f) { delete f; }

int64_t hifde_partition(int dim, int n_grid, int m_leaf, int ell, int level_kind,
                        const uint8_t* active, int32_t* members, int64_t members_cap,
                        int64_t* offsets, int64_t offsets_cap) {
  try {
    GridDesc g;
    g.dim = dim;
    g.n = n_grid;
    g.m = m_leaf;
    int L = 0;
    while (((int64_t)m_leaf << (L + 1)) <= n_grid) ++L;
    g.nlevels = L;
    Coords X;
    X.build(g);
    std::vector<int32_t> act;
    for (int64_t i = 0; i < g.ndof(); ++i)
      if (active[i]) act.push_back((int32_t)i);
    Groups gr = level_kind == 0 ? interior_groups(g, X, ell, act)
                                : interface_groups(g, X, ell, act, level_kind == 2 ? 1 : 0);
    if ((int64_t)gr.members.size() > members_cap || gr.size() + 1 > offsets_cap) return -1;
    std::memcpy(members, gr.members.data(), gr.members.size() * sizeof(int32_t));
    std::memcpy(offsets, gr.offsets.data(), gr.offsets.size() * sizeof(int64_t));
    return gr.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
