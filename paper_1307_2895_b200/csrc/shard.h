// Spatial sharding of the level sweep over P ranks (DESIGN (e)).
//
// Every rank runs the same host symbolic analysis (replicated, integer-only),
// so block ids and arena offsets agree everywhere.  Each group of a level has
// one owner rank, which launches its kernels; blocks are immutable once
// written, so the only data a rank needs from its peers are the blocks its own
// groups consume that another rank produced.  The ledger below tracks, per
// block, the producer and the ranks already holding it, and turns a level's
// consumption lists into a deterministic transfer list that every rank
// computes identically (sends and receives match without any negotiation).
#pragma once
#include <cstdint>
#include <vector>

#include "partition.h"

namespace hifde {

constexpr int kMaxRanks = 32;

// Subdomain boxes: P is split over the axes round-robin by factors of two
// (2: 2x1, 4: 2x2, 8: 2x2x2 in 3D, 4x2 in 2D); a P that is not a power of two
// splits the first axis P ways.  Box of a DOF with 1-based coordinate x along
// an axis of `parts` slabs: x * parts / n (the middle separator plane of an
// even split belongs to the upper slab).
struct ShardGeom {
  int P = 1, dim = 2, n = 2;
  int parts[3] = {1, 1, 1};
};
ShardGeom shard_geom(int P, int dim, int n_grid);
int shard_owner_xyz(const ShardGeom& G, const int* x);
int shard_owner(const ShardGeom& G, const Coords& X, int32_t dof);

struct Xfer {
  int32_t src, dst, blk;
};

struct BlockLedger {
  int P = 1;
  std::vector<uint8_t> src;    // producer rank per block id
  std::vector<uint32_t> have;  // bit r: rank r holds the block's values
  void reset(int nranks) {
    P = nranks;
    src.clear();
    have.clear();
  }
  void add(int32_t id, int producer);
  // Transfers that make every block listed by a task resident on the task's
  // owner: task t owns lists[ptr[t] .. ptr[t] + cnt[t]).  Appends to `out`
  // sorted by (src, dst, blk) and marks the receivers as holders.
  void plan(int64_t ntasks, const uint8_t* owner, const int64_t* ptr, const int32_t* cnt, const int32_t* lists,
            std::vector<Xfer>& out);
};

}  // namespace hifde
