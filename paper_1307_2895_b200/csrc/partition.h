// Host-side level partitioning (src/partition.py restated in C++).
#pragma once
#include <cstdint>
#include <functional>
#include <vector>

namespace hifde {

struct GridDesc {
  int dim = 2, n = 2, m = 2, nlevels = 0;
  int side() const { return n - 1; }
  int64_t ndof() const {
    int64_t s = 1;
    for (int i = 0; i < dim; ++i) s *= side();
    return s;
  }
};

// 1-based integer grid coordinates of every DOF (first axis fastest),
// precomputed once per factorization.
struct Coords {
  int dim = 0;
  std::vector<int16_t> x[3];
  void build(const GridDesc& g);
};

// Groups in CSR form: members[offsets[g] .. offsets[g+1]), ascending members.
struct Groups {
  std::vector<int32_t> members;
  std::vector<int64_t> offsets{0};
  int64_t size() const { return (int64_t)offsets.size() - 1; }
  const int32_t* begin(int64_t g) const { return members.data() + offsets[g]; }
  int count(int64_t g) const { return (int)(offsets[g + 1] - offsets[g]); }
};

// `act` is the ascending list of active DOFs.
// interior_cells (src/partition.py:68-92)
Groups interior_groups(const GridDesc& g, const Coords& X, int ell, const std::vector<int32_t>& act);

// interface_cells (src/partition.py:108-181); kind: 0 = edge, 1 = face
Groups interface_groups(const GridDesc& g, const Coords& X, int ell, const std::vector<int32_t>& act,
                        int kind);

// adaptive_interior_cells (src/partition.py:184-227).  `foreign(d, key, owner)`
// must report whether DOF d (active, owned by cell `key`) couples to an active
// DOF whose current owner is neither -1 nor `key`.
using CouplingTest = std::function<bool(int32_t d, int64_t key, const int64_t* owner)>;
Groups adaptive_groups(const GridDesc& g, const Coords& X, int ell, const std::vector<int32_t>& act,
                       int64_t ndof, const CouplingTest& foreign);

// The same partition with the shedding pass run in wavefronts of cells on
// nthreads threads.  A cell's decisions read the current owners of DOFs in
// adjacent cells only; with wave = cx + 2 cy + 4 cz every earlier adjacent
// cell (ascending key order) lies in an earlier wave and no two cells of one
// wave are adjacent, so the result is the sequential one.  foreign(d, key,
// owner, tid) must be safe to call concurrently for different cells.
using CouplingTestTid = std::function<bool(int32_t d, int64_t key, const int64_t* owner, int tid)>;
Groups adaptive_groups_par(const GridDesc& g, const Coords& X, int ell, const std::vector<int32_t>& act,
                           int64_t ndof, const CouplingTestTid& foreign, int nthreads);

}  // namespace hifde
