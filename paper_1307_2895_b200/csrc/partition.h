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
  // 1-based grid coordinate of DOF d along axis ax (first axis fastest).
  int coord(int64_t d, int ax) const {
    const int64_t s = side();
    for (int i = 0; i < ax; ++i) d /= s;
    return (int)(d % s) + 1;
  }
};

// Groups in CSR form: members[offsets[g] .. offsets[g+1]), ascending members.
struct Groups {
  std::vector<int32_t> members;
  std::vector<int64_t> offsets{0};
  int64_t size() const { return (int64_t)offsets.size() - 1; }
  const int32_t* begin(int64_t g) const { return members.data() + offsets[g]; }
  int count(int64_t g) const { return (int)(offsets[g + 1] - offsets[g]); }
};

// interior_cells (src/partition.py:68-92)
Groups interior_groups(const GridDesc& g, int ell, const uint8_t* active);

// interface_cells (src/partition.py:108-181); kind: 0 = edge, 1 = face
Groups interface_groups(const GridDesc& g, int ell, const uint8_t* active, int kind);

// adaptive_interior_cells (src/partition.py:184-227).  `foreign(d, key, owner)`
// must report whether DOF d (active, owned by cell `key`) couples to an active
// DOF whose current owner is neither -1 nor `key`.
using CouplingTest = std::function<bool(int32_t d, int64_t key, const int64_t* owner)>;
Groups adaptive_groups(const GridDesc& g, int ell, const uint8_t* active, const CouplingTest& foreign);

}  // namespace hifde
