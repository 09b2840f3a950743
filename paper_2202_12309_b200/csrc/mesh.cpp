// mesh.cpp -- see mesh.hpp.  Worklist 2:1 closure, magic-number Morton keys, hashed tree.
#include "mesh.hpp"

#include <algorithm>
#include <stdexcept>

namespace ph {

static uint64_t spread3(uint64_t x) {
  x &= 0x1fffffull;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

uint64_t morton3(int level, const int64_t x[3], int max_level) {
  int s = max_level - level;
  return spread3((uint64_t)x[0] << s) | (spread3((uint64_t)x[1] << s) << 1) | (spread3((uint64_t)x[2] << s) << 2);
}

void partition_range(int64_t nb, int R, int r, int64_t* lo, int64_t* hi) {
  int64_t q = nb / R, e = nb % R;
  *lo = r * q + (r < e ? r : e);
  *hi = *lo + q + (r < e ? 1 : 0);
}

Tree::Tree(const MeshCfg& c) : c_(c) {
  for (int64_t z = 0; z < c.nrb[2]; ++z)
    for (int64_t y = 0; y < c.nrb[1]; ++y)
      for (int64_t x = 0; x < c.nrb[0]; ++x) leaves_.insert(pack(Loc{0, {x, y, z}}));
}

bool Tree::wrap(Loc& l) const {
  for (int d = 0; d < 3; ++d) {
    int64_t nb = c_.nrb[d] << l.level;
    if (l.x[d] >= 0 && l.x[d] < nb) continue;
    if (!c_.periodic[d]) return false;
    l.x[d] = (l.x[d] + nb) % nb;  // offsets are within one block, so one wrap suffices
  }
  return true;
}

int Tree::find(const Loc& l, Loc* out) const {
  if (leaves_.count(pack(l))) {
    if (out) *out = l;
    return 0;
  }
  if (internal_.count(pack(l))) return 1;
  Loc p = l;
  while (p.level > 0) {
    p = parent(p);
    if (leaves_.count(pack(p))) {
      if (out) *out = p;
      return p.level - l.level;
    }
  }
  throw std::runtime_error("location outside the tree");
}

void Tree::refine_leaf(const Loc& l) {
  LocKey k = pack(l);
  leaves_.erase(k);
  internal_.insert(k);
  for (int c = 0; c < 8; ++c) leaves_.insert(pack(child(l, c)));
}

void Tree::balance() {
  std::vector<Loc> work;
  for (LocKey k : leaves_) {
    Loc l = unpack(k);
    if (l.level >= 2) work.push_back(l);
  }
  while (!work.empty()) {
    Loc l = work.back();
    work.pop_back();
    if (!is_leaf(l)) continue;
    bool again = false;
    for (int o = 0; o < 27 && !again; ++o) {
      if (o == 13) continue;
      Loc q{l.level, {l.x[0] + o % 3 - 1, l.x[1] + (o / 3) % 3 - 1, l.x[2] + o / 9 - 1}};
      if (!wrap(q)) continue;
      Loc c;
      if (find(q, &c) < -1) {
        refine_leaf(c);
        for (int ch = 0; ch < 8; ++ch) {
          Loc cl = child(c, ch);
          if (cl.level >= 2) work.push_back(cl);
        }
        again = true;
      }
    }
    if (again) work.push_back(l);
  }
}

void Tree::box(const Loc& l, double* bmin, double* bmax) const {
  for (int d = 0; d < 3; ++d) {
    double w = (c_.xmax[d] - c_.xmin[d]) / (double)(c_.nrb[d] << l.level);
    bmin[d] = c_.xmin[d] + (double)l.x[d] * w;
    bmax[d] = c_.xmin[d] + (double)(l.x[d] + 1) * w;
  }
}

void Tree::refine_regions(const std::vector<double>& regions) {
  int nr = (int)regions.size() / 7;
  for (int lev = 0; lev < c_.max_level; ++lev) {
    std::vector<Loc> todo;
    for (LocKey k : leaves_) {
      Loc l = unpack(k);
      if (l.level != lev) continue;
      double lo[3], hi[3];
      box(l, lo, hi);
      for (int r = 0; r < nr; ++r) {
        const double* R = &regions[7 * r];
        if ((int)R[0] <= lev) continue;
        if (lo[0] < R[2] && hi[0] > R[1] && lo[1] < R[4] && hi[1] > R[3] && lo[2] < R[6] && hi[2] > R[5]) {
          todo.push_back(l);
          break;
        }
      }
    }
    for (const Loc& l : todo) refine_leaf(l);
    balance();
  }
}

void Tree::rebuild_internal() {
  internal_.clear();
  for (LocKey k : leaves_) {
    Loc l = unpack(k);
    while (l.level > 0) {
      l = parent(l);
      if (!internal_.insert(pack(l)).second) break;
    }
  }
}

void Tree::set_leaves(const std::unordered_set<LocKey>& s) {
  leaves_ = s;
  rebuild_internal();
}

std::vector<Loc> Tree::leaves_sorted() const {
  std::vector<std::pair<uint64_t, LocKey>> v;
  v.reserve(leaves_.size());
  for (LocKey k : leaves_) {
    Loc l = unpack(k);
    v.push_back({morton3(l.level, l.x, c_.max_level), k});
  }
  std::sort(v.begin(), v.end());
  std::vector<Loc> out;
  out.reserve(v.size());
  for (auto& p : v) out.push_back(unpack(p.second));
  return out;
}

void build_blocks(const Tree& t, int nranks, int rank, std::vector<BlockInfo>& out,
                  std::unordered_map<LocKey, int64_t>& gid_of) {
  const MeshCfg& c = t.cfg();
  std::vector<Loc> ls = t.leaves_sorted();
  int64_t nb = (int64_t)ls.size();
  out.assign(nb, BlockInfo());
  gid_of.clear();
  gid_of.reserve(nb * 2);
  std::vector<int64_t> lo(nranks), hi(nranks);
  for (int r = 0; r < nranks; ++r) partition_range(nb, nranks, r, &lo[r], &hi[r]);
  int r = 0;
  for (int64_t g = 0; g < nb; ++g) {
    while (g >= hi[r]) ++r;
    BlockInfo& b = out[g];
    b.loc = ls[g];
    b.gid = g;
    b.rank = r;
    b.local = g - lo[r];
    gid_of[pack(ls[g])] = g;
    t.box(b.loc, b.xmin, b.xmax);
    for (int d = 0; d < 3; ++d) {
      double w = (c.xmax[d] - c.xmin[d]) / (double)(c.nrb[d] << b.loc.level);
      b.dx[d] = w / (double)c.n[d];
      b.phys_lo[d] = !c.periodic[d] && b.loc.x[d] == 0;
      b.phys_hi[d] = !c.periodic[d] && b.loc.x[d] == (c.nrb[d] << b.loc.level) - 1;
    }
  }
  (void)rank;
  for (int64_t g = 0; g < nb; ++g) {
    BlockInfo& b = out[g];
    b.nbrs.clear();
    for (int o3 = -1; o3 <= 1; ++o3)
      for (int o2 = -1; o2 <= 1; ++o2)
        for (int o1 = -1; o1 <= 1; ++o1) {
          if (!o1 && !o2 && !o3) continue;
          int o[3] = {o1, o2, o3};
          Loc q{b.loc.level, {b.loc.x[0] + o1, b.loc.x[1] + o2, b.loc.x[2] + o3}};
          if (!t.wrap(q)) continue;
          Loc cv;
          int rel = t.find(q, &cv);
          if (rel == 0 || rel == -1) {
            Neighbor e{};
            e.gid = gid_of.at(pack(cv));
            for (int d = 0; d < 3; ++d) e.off[d] = (int8_t)o[d];
            e.dlevel = (int8_t)rel;
            b.nbrs.push_back(e);
            if (rel == -1) b.has_coarser = true;
          } else if (rel == 1) {
            int freed[3], nf = 0;
            for (int d = 0; d < 3; ++d)
              if (!o[d]) freed[nf++] = d;
            for (int cc = 0; cc < (1 << nf); ++cc) {
              int64_t ch[3];
              int8_t fi[2] = {0, 0};
              for (int d = 0; d < 3; ++d) ch[d] = (o[d] == 1) ? 0 : 1;
              for (int f = 0; f < nf; ++f) {
                ch[freed[f]] = (cc >> f) & 1;
                fi[f] = (int8_t)((cc >> f) & 1);
              }
              Loc fl{q.level + 1, {2 * q.x[0] + ch[0], 2 * q.x[1] + ch[1], 2 * q.x[2] + ch[2]}};
              auto it = gid_of.find(pack(fl));
              if (it == gid_of.end()) throw std::runtime_error("2:1 balance violated");
              Neighbor e{};
              e.gid = it->second;
              for (int d = 0; d < 3; ++d) e.off[d] = (int8_t)o[d];
              e.dlevel = 1;
              e.fine[0] = fi[0];
              e.fine[1] = fi[1];
              b.nbrs.push_back(e);
              if ((o[0] != 0) + (o[1] != 0) + (o[2] != 0) == 1) b.has_finer_face = true;
            }
          } else {
            throw std::runtime_error("2:1 balance violated");
          }
        }
  }
  for (auto& b : out)
    for (auto& e : b.nbrs) e.rank = out[e.gid].rank;
}

std::unordered_set<LocKey> normalize_flags(const Tree& t, const std::vector<Loc>& locs,
                                           const std::vector<int8_t>& flags, bool allow_deref) {
  Tree nt = t;
  for (size_t i = 0; i < locs.size(); ++i)
    if (flags[i] == 1 && nt.is_leaf(locs[i]) && locs[i].level < nt.cfg().max_level) nt.refine_leaf(locs[i]);
  nt.balance();
  if (!allow_deref) return nt.leaves();
  std::unordered_map<LocKey, int> cnt;
  for (size_t i = 0; i < locs.size(); ++i)
    if (flags[i] == -1 && locs[i].level > 0 && nt.is_leaf(locs[i])) cnt[pack(parent(locs[i]))]++;
  std::vector<Loc> accept;
  for (auto& kv : cnt) {
    if (kv.second != 8) continue;
    const Loc P = unpack(kv.first);
    bool ok = true;
    // every leaf touching P must be at most one level finer than P: a refined same-level
    // neighbour region may not have refined children on the side facing P
    for (int o = 0; o < 27 && ok; ++o) {
      if (o == 13) continue;
      const int od[3] = {o % 3 - 1, (o / 3) % 3 - 1, o / 9 - 1};
      Loc q{P.level, {P.x[0] + od[0], P.x[1] + od[1], P.x[2] + od[2]}};
      if (!nt.wrap(q) || !nt.is_internal(q)) continue;
      for (int ch = 0; ch < 8 && ok; ++ch) {
        const int cd[3] = {ch & 1, (ch >> 1) & 1, (ch >> 2) & 1};
        bool adj = true;
        for (int d = 0; d < 3; ++d)
          if ((od[d] == 1 && cd[d] != 0) || (od[d] == -1 && cd[d] != 1)) adj = false;
        if (adj && nt.is_internal(child(q, ch))) ok = false;
      }
    }
    if (ok) accept.push_back(P);
  }
  std::unordered_set<LocKey> leaves = nt.leaves();
  for (const Loc& P : accept) {
    for (int ch = 0; ch < 8; ++ch) leaves.erase(pack(child(P, ch)));
    leaves.insert(pack(P));
  }
  return leaves;
}

}  // namespace ph
