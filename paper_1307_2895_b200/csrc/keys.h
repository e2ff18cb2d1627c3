// Level-partition keys of one DOF, shared by the host partition
// (partition.cpp) and the device symbolic pass (symbolic.cu), so both give
// the reference's groups (src/partition.py:68-181) by construction.
// Coordinates are 1-based integer grid positions; w = m 2^ell is the cell
// width and k = n / w the number of cells per axis.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define HIFDE_HD __host__ __device__ __forceinline__
#else
#define HIFDE_HD inline
#endif

namespace hifde {

// nearest centre w*j, j in [1, top], ties to the lower j (doubled coords x2)
HIFDE_HD int key_near_mult(int x2, int w, int top) {
  int j = (x2 + w - 1) / (2 * w);
  return j < 1 ? 1 : (j > top ? top : j);
}
// nearest centre w*(j - 1/2), j in [1, top], ties to the lower j
HIFDE_HD int key_near_half(int x2, int w, int top) {
  int j = (x2 + 2 * w - 1) / (2 * w);
  return j < 1 ? 1 : (j > top ? top : j);
}

// interior_cells (src/partition.py:68-92): cell index with the first axis
// fastest, or -1 for a DOF on a separator plane (a coordinate = 0 mod w)
HIFDE_HD int interior_key(const int* x, int dim, int w, int k) {
  int key = 0, stride = 1;
  for (int ax = 0; ax < dim; ++ax) {
    const int q = x[ax] / w;
    if (x[ax] - q * w == 0) return -1;
    key += q * stride;
    stride *= k;
  }
  return key;
}

// interface_cells (src/partition.py:108-181): Voronoi assignment to the edge
// (face = false) or face (face = true) centres in doubled coordinates, the
// multi-plane exclusions (:122-129), lowest family on distance ties (:162)
// and ties within a family rounding down (:95-105); -1 if excluded.  Keys
// are family-major: fam * k^dim + the centre's index.
HIFDE_HD int interface_key(const int* x, int dim, int w, int k, bool face) {
  int span = 1;
  for (int ax = 0; ax < dim; ++ax) span *= k;
  int x2[3] = {0, 0, 0};
  int planes = 0;
  for (int ax = 0; ax < dim; ++ax) {
    x2[ax] = 2 * x[ax];
    planes += (x[ax] % w == 0);
  }
  bool excluded;
  if (dim == 2) excluded = planes == 2;
  else if (face) excluded = planes >= 2;
  else excluded = planes == 3;
  if (excluded) return -1;
  int64_t best_d = INT64_MAX;
  int best_key = 0;
  for (int fam = 0; fam < dim; ++fam) {
    int64_t dist = 0;
    int key = 0, stride = 1;
    for (int ax = 0; ax < dim; ++ax) {
      const bool on_plane = face ? (ax == fam) : (ax != fam);
      int j, c2, sp;
      if (on_plane) { j = key_near_mult(x2[ax], w, k - 1); c2 = 2 * w * j; sp = k - 1; }
      else { j = key_near_half(x2[ax], w, k); c2 = w * (2 * j - 1); sp = k; }
      dist += (int64_t)(x2[ax] - c2) * (x2[ax] - c2);
      key += (j - 1) * stride;
      stride *= sp;
    }
    if (dist < best_d) { best_d = dist; best_key = fam * span + key; }
  }
  return best_key;
}

}  // namespace hifde
