// Host side of the sharded level sweep: subdomain ownership and the block
// transfer ledger (shard.h).  No CUDA here: the CPU tests drive these through
// the C ABI hooks hifde_shard_owner / hifde_shard_plan.
#include "shard.h"

#include <algorithm>
#include <stdexcept>

#include "../../include/hifde_gpu.h"

namespace hifde {

ShardGeom shard_geom(int P, int dim, int n_grid) {
  if (P < 1 || P > kMaxRanks) throw std::invalid_argument("shard: rank count out of range");
  ShardGeom G;
  G.P = P;
  G.dim = dim;
  G.n = n_grid;
  if ((P & (P - 1)) == 0) {
    int ax = 0;
    for (int p = P; p > 1; p >>= 1) {
      G.parts[ax] *= 2;
      ax = (ax + 1) % dim;
    }
  } else {
    G.parts[0] = P;
  }
  return G;
}

int shard_owner_xyz(const ShardGeom& G, const int* x) {
  int r = 0, stride = 1;
  for (int ax = 0; ax < G.dim; ++ax) {
    const int p = G.parts[ax];
    int b = (int)((int64_t)x[ax] * p / G.n);
    b = std::min(std::max(b, 0), p - 1);
    r += b * stride;
    stride *= p;
  }
  return r;
}

int shard_owner(const ShardGeom& G, const Coords& X, int32_t dof) {
  int x[3] = {0, 0, 0};
  for (int ax = 0; ax < G.dim; ++ax) x[ax] = X.x[ax][(size_t)dof];
  return shard_owner_xyz(G, x);
}

void BlockLedger::add(int32_t id, int producer) {
  if ((size_t)id != src.size()) throw std::logic_error("shard ledger: block ids must be dense");
  src.push_back((uint8_t)producer);
  have.push_back(1u << producer);
}

void BlockLedger::plan(int64_t ntasks, const uint8_t* owner, const int64_t* ptr, const int32_t* cnt,
                       const int32_t* lists, std::vector<Xfer>& out) {
  const size_t base = out.size();
  for (int64_t t = 0; t < ntasks; ++t) {
    const int r = owner[t];
    const uint32_t bit = 1u << r;
    const int32_t* l = lists + ptr[t];
    for (int j = 0; j < cnt[t]; ++j) {
      const int32_t b = l[j];
      if (b < 0 || (size_t)b >= have.size()) throw std::logic_error("shard ledger: unknown block");
      if (have[(size_t)b] & bit) continue;
      have[(size_t)b] |= bit;
      out.push_back(Xfer{(int32_t)src[(size_t)b], (int32_t)r, b});
    }
  }
  std::sort(out.begin() + (int64_t)base, out.end(), [](const Xfer& a, const Xfer& b) {
    if (a.src != b.src) return a.src < b.src;
    if (a.dst != b.dst) return a.dst < b.dst;
    return a.blk < b.blk;
  });
}

}  // namespace hifde

using namespace hifde;

extern "C" {

int hifde_shard_owner(int nranks, int dim, int n_grid, const int32_t* dofs, int64_t count, int32_t* owner) {
  if (dim != 2 && dim != 3) return HIFDE_BADARG;
  if (nranks < 1 || nranks > kMaxRanks || n_grid < 2 || (count > 0 && (!dofs || !owner))) return HIFDE_BADARG;
  const ShardGeom G = shard_geom(nranks, dim, n_grid);
  const int64_t s = n_grid - 1;
  int64_t ndof = 1;
  for (int ax = 0; ax < dim; ++ax) ndof *= s;
  for (int64_t i = 0; i < count; ++i) {
    int64_t d = dofs[i];
    if (d < 0 || d >= ndof) return HIFDE_BADARG;
    int x[3] = {0, 0, 0};
    for (int ax = 0; ax < dim; ++ax) {  // first axis fastest, 1-based (Coords::build)
      x[ax] = (int)(d % s) + 1;
      d /= s;
    }
    owner[i] = shard_owner_xyz(G, x);
  }
  return HIFDE_OK;
}

int64_t hifde_shard_plan(int nranks, int64_t nblocks, const int32_t* producer, uint32_t* have, int64_t ntasks,
                         const int32_t* owner, const int64_t* list_ptr, const int32_t* lists, int32_t* out,
                         int64_t cap) {
  if (nranks < 1 || nranks > kMaxRanks || nblocks < 0 || ntasks < 0) return -1;
  try {
    BlockLedger L;
    L.reset(nranks);
    for (int64_t b = 0; b < nblocks; ++b) {
      if (producer[b] < 0 || producer[b] >= nranks) return -1;
      L.add((int32_t)b, producer[b]);
      if (have) L.have[(size_t)b] |= have[b];
    }
    std::vector<uint8_t> own((size_t)ntasks);
    std::vector<int32_t> cnt((size_t)ntasks);
    for (int64_t t = 0; t < ntasks; ++t) {
      if (owner[t] < 0 || owner[t] >= nranks) return -1;
      own[(size_t)t] = (uint8_t)owner[t];
      cnt[(size_t)t] = (int32_t)(list_ptr[t + 1] - list_ptr[t]);
    }
    std::vector<Xfer> x;
    L.plan(ntasks, own.data(), list_ptr, cnt.data(), lists, x);
    if (!out) return (int64_t)x.size();  // size query (have[] untouched)
    if ((int64_t)x.size() > cap) return -2 - (int64_t)x.size();
    if (have)
      for (int64_t b = 0; b < nblocks; ++b) have[b] = L.have[(size_t)b];
    for (size_t i = 0; i < x.size(); ++i) {
      out[3 * i] = x[i].src;
      out[3 * i + 1] = x[i].dst;
      out[3 * i + 2] = x[i].blk;
    }
    return (int64_t)x.size();
  } catch (...) {
    return -1;
  }
}

}  // extern "C"
