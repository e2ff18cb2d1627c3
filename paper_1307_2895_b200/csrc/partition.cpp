// Level partitioning on the host.  Exact integer geometry in doubled grid
// units, mirroring the reference's semantics (src/partition.py):
//   * interior cells: active DOFs with no coordinate on a separator plane,
//     keyed by cell index with the first axis fastest (:68-92);
//   * interface groups: Voronoi assignment to edge / face centres with the
//     multi-plane exclusions, lowest family winning distance ties and ties
//     within a family rounding down (:95-181);
//   * adaptive cells: Voronoi to cell centres, then in ascending key order
//     each cell sheds members still coupled to another current cell (:184-227).
// Groups come out in the reference's order: ascending key (family-major for
// interfaces), members ascending.
#include "partition.h"
#include "keys.h"

#include <algorithm>
#include <stdexcept>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace hifde {

void Coords::build(const GridDesc& g) {
  dim = g.dim;
  const int64_t N = g.ndof();
  const int s = g.side();
  for (int ax = 0; ax < g.dim; ++ax) x[ax].resize((size_t)N);
  int c[3] = {1, 1, 1};
  for (int64_t d = 0; d < N; ++d) {
    for (int ax = 0; ax < g.dim; ++ax) x[ax][(size_t)d] = (int16_t)c[ax];
    for (int ax = 0; ax < g.dim; ++ax) {  // odometer, first axis fastest
      if (++c[ax] <= s) break;
      c[ax] = 1;
    }
  }
}

namespace {

// Bucket the selected DOFs (ascending) by key in [0, nkeys): counting sort,
// which keeps members ascending inside each bucket.  Empty buckets dropped.
Groups bucket(const std::vector<int32_t>& dofs, const std::vector<int32_t>& keys, int64_t nkeys) {
  Groups out;
  std::vector<int64_t> cnt((size_t)nkeys + 1, 0);
  for (int32_t k : keys) cnt[(size_t)k + 1]++;
  for (int64_t i = 0; i < nkeys; ++i) cnt[(size_t)i + 1] += cnt[(size_t)i];
  out.members.resize(dofs.size());
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  for (size_t i = 0; i < dofs.size(); ++i) out.members[(size_t)pos[(size_t)keys[i]]++] = dofs[i];
  out.offsets.clear();
  out.offsets.push_back(0);
  for (int64_t k = 0; k < nkeys; ++k)
    if (cnt[(size_t)k + 1] > cnt[(size_t)k]) out.offsets.push_back(cnt[(size_t)k + 1]);
  return out;
}

// Bucket act[i] by kall[i] (>= 0; -1 = not selected) into nkeys groups,
// members ascending, empty buckets dropped.  Per-thread counts over
// contiguous chunks, a prefix over (key, thread), then a parallel scatter:
// the thread chunks are in ascending order, so members stay ascending.
Groups bucket_keys(const std::vector<int32_t>& act, const std::vector<int32_t>& kall, int64_t nkeys) {
  const int64_t na = (int64_t)act.size();
  int nth = 1;
#ifdef _OPENMP
  nth = std::min(omp_get_max_threads(), 16);
#endif
  if (na < 16384 || nkeys * nth > 4 * na) {  // small: the serial counting sort
    std::vector<int32_t> dofs, keys;
    dofs.reserve(act.size());
    keys.reserve(act.size());
    for (int64_t i = 0; i < na; ++i)
      if (kall[(size_t)i] >= 0) {
        dofs.push_back(act[(size_t)i]);
        keys.push_back(kall[(size_t)i]);
      }
    return bucket(dofs, keys, nkeys);
  }
  // counts and then write positions, [key][thread] so the prefix walks memory in order
  std::vector<int64_t> cnt((size_t)nth * (size_t)nkeys);
#pragma omp parallel num_threads(nth)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    for (int64_t k = tid; k < nkeys; k += nth)
      for (int t = 0; t < nth; ++t) cnt[(size_t)k * nth + t] = 0;
#pragma omp barrier
    const int64_t lo = na * tid / nth, hi = na * (tid + 1) / nth;
    for (int64_t i = lo; i < hi; ++i)
      if (kall[(size_t)i] >= 0) ++cnt[(size_t)kall[(size_t)i] * nth + tid];
  }
  Groups out;
  out.offsets.clear();
  out.offsets.reserve((size_t)nkeys + 1);
  out.offsets.push_back(0);
  int64_t run = 0;
  for (int64_t k = 0; k < nkeys; ++k) {
    const int64_t start = run;
    int64_t* c = cnt.data() + (size_t)k * nth;
    for (int t = 0; t < nth; ++t) {
      const int64_t v = c[t];
      c[t] = run;  // becomes the thread's write position for key k
      run += v;
    }
    if (run > start) out.offsets.push_back(run);
  }
  out.members.resize((size_t)run);
#pragma omp parallel num_threads(nth)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    const int64_t lo = na * tid / nth, hi = na * (tid + 1) / nth;
    for (int64_t i = lo; i < hi; ++i) {
      const int32_t k = kall[(size_t)i];
      if (k >= 0) out.members[(size_t)cnt[(size_t)k * nth + tid]++] = act[(size_t)i];
    }
  }
  return out;
}

inline int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

inline int near_half(int x2, int w, int top) { return key_near_half(x2, w, top); }

}  // namespace

Groups interior_groups(const GridDesc& g, const Coords& X, int ell, const std::vector<int32_t>& act) {
  if (ell < 0 || ell >= std::max(g.nlevels, 1)) throw std::invalid_argument("level out of range");
  const int w = g.m << ell;
  const int k = g.n / w;
  const int64_t na = (int64_t)act.size();
  std::vector<int32_t> kall((size_t)na);
#pragma omp parallel for schedule(static) if (na > 16384)
  for (int64_t i = 0; i < na; ++i) {
    const int32_t d = act[(size_t)i];
    int x[3] = {0, 0, 0};
    for (int ax = 0; ax < g.dim; ++ax) x[ax] = X.x[ax][(size_t)d];
    kall[(size_t)i] = interior_key(x, g.dim, w, k);
  }
  return bucket_keys(act, kall, ipow(k, g.dim));
}

Groups interface_groups(const GridDesc& g, const Coords& X, int ell, const std::vector<int32_t>& act,
                        int kind) {
  const bool face = kind == 1;
  if (g.dim == 2 && face) throw std::invalid_argument("faces need a 3D grid");
  const int w = g.m << ell;
  const int k = g.n / w;
  const int span = (int)ipow(k, g.dim);
  const int64_t na = (int64_t)act.size();
  std::vector<int32_t> kall((size_t)na);
#pragma omp parallel for schedule(static) if (na > 16384)
  for (int64_t i = 0; i < na; ++i) {
    const int32_t d = act[(size_t)i];
    int x[3] = {0, 0, 0};
    for (int ax = 0; ax < g.dim; ++ax) x[ax] = X.x[ax][(size_t)d];
    kall[(size_t)i] = interface_key(x, g.dim, w, k, face);
  }
  return bucket_keys(act, kall, (int64_t)span * g.dim);
}

Groups adaptive_groups(const GridDesc& g, const Coords& X, int ell, const std::vector<int32_t>& act,
                       int64_t ndof, const CouplingTest& foreign) {
  const int w = g.m << ell;
  const int k = g.n / w;
  std::vector<int32_t> dofs, keys;
  std::vector<int64_t> owner((size_t)ndof, -1);
  for (int32_t d : act) {
    int key = 0, stride = 1;
    for (int ax = 0; ax < g.dim; ++ax) {
      key += (near_half(2 * X.x[ax][(size_t)d], w, k) - 1) * stride;
      stride *= k;
    }
    owner[(size_t)d] = key;
    dofs.push_back(d);
    keys.push_back(key);
  }
  Groups vor = bucket(dofs, keys, ipow(k, g.dim));
  Groups out;
  std::vector<char> shed;
  for (int64_t gi = 0; gi < vor.size(); ++gi) {
    const int32_t* mem = vor.begin(gi);
    const int cnt = vor.count(gi);
    const int64_t key = owner[(size_t)mem[0]];
    shed.assign((size_t)cnt, 0);
    for (int i = 0; i < cnt; ++i) shed[(size_t)i] = foreign(mem[i], key, owner.data()) ? 1 : 0;
    int kept = 0;
    for (int i = 0; i < cnt; ++i) {
      if (shed[(size_t)i]) owner[(size_t)mem[i]] = -1;
      else { out.members.push_back(mem[i]); ++kept; }
    }
    if (kept) out.offsets.push_back((int64_t)out.members.size());
  }
  return out;
}

Groups adaptive_groups_par(const GridDesc& g, const Coords& X, int ell, const std::vector<int32_t>& act,
                           int64_t ndof, const CouplingTestTid& foreign, int nthreads) {
  const int w = g.m << ell;
  const int k = g.n / w;
  std::vector<int32_t> dofs(act.size()), keys(act.size());
  std::vector<int64_t> owner((size_t)ndof, -1);
#pragma omp parallel for num_threads(nthreads) schedule(static) if (act.size() > 65536)
  for (int64_t i = 0; i < (int64_t)act.size(); ++i) {
    const int32_t d = act[(size_t)i];
    int key = 0, stride = 1;
    for (int ax = 0; ax < g.dim; ++ax) {
      key += (near_half(2 * X.x[ax][(size_t)d], w, k) - 1) * stride;
      stride *= k;
    }
    owner[(size_t)d] = key;
    dofs[(size_t)i] = d;
    keys[(size_t)i] = key;
  }
  Groups vor = bucket(dofs, keys, ipow(k, g.dim));
  const int64_t ng = vor.size();
  // waves of mutually non-adjacent cells (cell coordinates from the key)
  std::vector<int> wave((size_t)ng);
  int nwave = 0;
  for (int64_t gi = 0; gi < ng; ++gi) {
    int64_t key = owner[(size_t)vor.begin(gi)[0]];
    int wv = 0, mul = 1;
    for (int ax = 0; ax < g.dim; ++ax) {
      wv += (int)(key % k) * mul;
      key /= k;
      mul *= 2;
    }
    wave[(size_t)gi] = wv;
    nwave = std::max(nwave, wv + 1);
  }
  std::vector<int64_t> wptr((size_t)nwave + 1, 0), worder((size_t)ng);
  for (int64_t gi = 0; gi < ng; ++gi) ++wptr[(size_t)wave[(size_t)gi] + 1];
  for (int v = 0; v < nwave; ++v) wptr[(size_t)v + 1] += wptr[(size_t)v];
  {
    std::vector<int64_t> fill(wptr.begin(), wptr.end() - 1);
    for (int64_t gi = 0; gi < ng; ++gi) worder[(size_t)fill[(size_t)wave[(size_t)gi]]++] = gi;
  }
  std::vector<char> shed(vor.members.size(), 0);
#pragma omp parallel num_threads(nthreads)
  {
    const int tid = omp_get_thread_num();
    for (int v = 0; v < nwave; ++v) {
#pragma omp for schedule(dynamic, 2)
      for (int64_t j = wptr[(size_t)v]; j < wptr[(size_t)v + 1]; ++j) {
        const int64_t gi = worder[(size_t)j];
        const int32_t* mem = vor.begin(gi);
        const int cnt = vor.count(gi);
        const int64_t key = owner[(size_t)mem[0]];
        char* sh = shed.data() + vor.offsets[(size_t)gi];
        for (int i = 0; i < cnt; ++i) sh[i] = foreign(mem[i], key, owner.data(), tid) ? 1 : 0;
        for (int i = 0; i < cnt; ++i)
          if (sh[i]) owner[(size_t)mem[i]] = -1;
      }  // implicit barrier: the next wave sees this wave's owners
    }
  }
  Groups out;
  out.members.reserve(vor.members.size());
  for (int64_t gi = 0; gi < ng; ++gi) {
    const int32_t* mem = vor.begin(gi);
    const char* sh = shed.data() + vor.offsets[(size_t)gi];
    int kept = 0;
    for (int i = 0; i < vor.count(gi); ++i)
      if (!sh[i]) {
        out.members.push_back(mem[i]);
        ++kept;
      }
    if (kept) out.offsets.push_back((int64_t)out.members.size());
  }
  return out;
}

}  // namespace hifde
