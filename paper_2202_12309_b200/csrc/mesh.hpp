// mesh.hpp -- host-side block tree, Morton order, partition, neighbour lists and the
// fill-in-one exchange plan of the B200 path.  Independent of oracle/ (shares no code).
//
// Paper: blocks are leaves of an oct-tree; Z-order distribution
// (P:197); whole-tree rebuild on remesh; 2:1 balance over faces,
// edges and corners (implied; pinned by the paper mesh counts P:857-860, reading A15).
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace ph {

// packed logical location: level(6) | x3(19) | x2(19) | x1(19)
using LocKey = uint64_t;
struct Loc {
  int level;
  int64_t x[3];
};
inline LocKey pack(const Loc& l) {
  return ((uint64_t)l.level << 57) | ((uint64_t)l.x[2] << 38) | ((uint64_t)l.x[1] << 19) | (uint64_t)l.x[0];
}
inline Loc unpack(LocKey k) {
  Loc l;
  l.level = (int)(k >> 57);
  l.x[2] = (int64_t)((k >> 38) & 0x7FFFF);
  l.x[1] = (int64_t)((k >> 19) & 0x7FFFF);
  l.x[0] = (int64_t)(k & 0x7FFFF);
  return l;
}
inline Loc parent(const Loc& l) { return Loc{l.level - 1, {l.x[0] >> 1, l.x[1] >> 1, l.x[2] >> 1}}; }
inline Loc child(const Loc& l, int c) {
  return Loc{l.level + 1, {2 * l.x[0] + (c & 1), 2 * l.x[1] + ((c >> 1) & 1), 2 * l.x[2] + ((c >> 2) & 1)}};
}

uint64_t morton3(int level, const int64_t x[3], int max_level);  // x1 least significant (A17)

struct MeshCfg {
  int64_t n[3];        // block cells
  int64_t nrb[3];      // root blocks
  int max_level;
  bool periodic[3];
  int bc_in[3], bc_out[3];
  double xmin[3], xmax[3];
};

struct Neighbor {
  int64_t gid;
  int rank;
  int8_t off[3];
  int8_t dlevel;
  int8_t fine[2];
};

struct BlockInfo {
  Loc loc;
  int64_t gid;
  int rank;
  int64_t local;       // slot on its rank
  double xmin[3], xmax[3], dx[3];
  bool phys_lo[3], phys_hi[3];  // touches a non-periodic domain face
  std::vector<Neighbor> nbrs;
  bool has_coarser = false;
  bool has_finer_face = false;
};

class Tree {
 public:
  explicit Tree(const MeshCfg& c);
  // 0: leaf at l; -k: covered by a leaf k levels coarser (*out); +1: refined
  int find(const Loc& l, Loc* out) const;
  bool wrap(Loc& l) const;
  void refine_leaf(const Loc& l);
  void balance();  // refine-only 2:1 closure (faces, edges, corners)
  void refine_regions(const std::vector<double>& regions);  // [7*r]: level, box
  void box(const Loc& l, double* bmin, double* bmax) const;
  std::vector<Loc> leaves_sorted() const;  // Morton order
  const std::unordered_set<LocKey>& leaves() const { return leaves_; }
  void set_leaves(const std::unordered_set<LocKey>& s);
  const MeshCfg& cfg() const { return c_; }
  bool is_leaf(const Loc& l) const { return leaves_.count(pack(l)) != 0; }
  bool is_internal(const Loc& l) const { return internal_.count(pack(l)) != 0; }

 private:
  void rebuild_internal();
  MeshCfg c_;
  std::unordered_set<LocKey> leaves_;
  std::unordered_set<LocKey> internal_;  // refined (non-leaf) nodes
};

// Build gid-ordered block list with partition and canonical neighbour lists (O2, O3).
void build_blocks(const Tree& t, int nranks, int rank, std::vector<BlockInfo>& out,
                  std::unordered_map<LocKey, int64_t>& gid_of);

void partition_range(int64_t nb, int R, int r, int64_t* lo, int64_t* hi);

// AMR flag normalisation: refine flagged leaves, restore 2:1
// (refine-only closure), then accept a derefinement of 8 siblings only if the gate is open, all
// 8 are leaves flagged -1 and the parent keeps 2:1 against the post-refinement tree.
// flags: +1 refine, -1 derefine, 0 keep, per entry of `locs`.  Returns the new leaf set.
std::unordered_set<LocKey> normalize_flags(const Tree& t, const std::vector<Loc>& locs,
                                           const std::vector<int8_t>& flags, bool allow_deref);

}  // namespace ph
