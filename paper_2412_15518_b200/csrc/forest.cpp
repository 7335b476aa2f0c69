// Host forest: see forest.h. Everything here is integer indexing that must be
// bit-exact with the reference (tests/test_forest.py compares it against the
// reference Tree on random AMR topologies).
#include "forest.h"

#include <algorithm>

namespace tmgpu {

uint64_t morton_encode(int level, uint64_t i, uint64_t j, uint64_t k) {
  if (level < 0 || level > kMaxMortonLevel) throw AmrError("morton_encode: level out of range");
  const uint64_t lim = 1ull << level;
  if (i >= lim || j >= lim || k >= lim)
    throw AmrError("morton_encode: coordinate out of range for level");
  uint64_t idx = 0;
  for (int b = 0; b < level; ++b)
    idx |= (((i >> b) & 1ull) | (((j >> b) & 1ull) << 1) | (((k >> b) & 1ull) << 2)) << (3 * b);
  return idx;
}

void morton_decode(int level, uint64_t index, uint64_t& i, uint64_t& j, uint64_t& k) {
  if (level < 0 || level > kMaxMortonLevel) throw AmrError("morton_decode: level out of range");
  if ((index >> (3 * level)) != 0) throw AmrError("morton_decode: index has bits above the level");
  i = j = k = 0;
  for (int b = 0; b < level; ++b) {
    const uint64_t t = index >> (3 * b);
    i |= (t & 1ull) << b;
    j |= ((t >> 1) & 1ull) << b;
    k |= ((t >> 2) & 1ull) << b;
  }
}

Forest::Forest(const ForestConfig& cfg) : cfg_(cfg) {
  if (cfg_.edge < 4 || cfg_.edge % 2 != 0) throw AmrError("subgrid edge must be even and at least 4");
  if (cfg_.ghost < 2) throw AmrError("ghost width must be at least 2");
  const int maxdim = std::max({cfg_.root_dims[0], cfg_.root_dims[1], cfg_.root_dims[2]});
  if (maxdim < 1) throw AmrError("root_dims must be positive");
  root_extent_ = 1.0 / maxdim;
  for (int rk = 0; rk < cfg_.root_dims[2]; ++rk)
    for (int rj = 0; rj < cfg_.root_dims[1]; ++rj)
      for (int ri = 0; ri < cfg_.root_dims[0]; ++ri)
        nodes_[NodeId{0, uint32_t(ri), uint32_t(rj), uint32_t(rk)}.packed()] = Node{};
}

bool Forest::is_leaf(const NodeId& id) const {
  auto it = nodes_.find(id.packed());
  return it != nodes_.end() && it->second.children_mask == 0;
}

std::array<double, 3> Forest::cell_center(const NodeId& id, int i, int j, int k) const {
  const double dx = cell_size(id.level);
  auto coord = [&](uint32_t c, int s) {
    const long long g = (long long)c * cfg_.edge + (s - cfg_.ghost);
    return ((double)g + 0.5) * dx;
  };
  return {coord(id.ci, i), coord(id.cj, j), coord(id.ck, k)};
}

const std::vector<NodeId>& Forest::leaves() const {
  if (cache_valid_) return leaf_cache_;
  struct Keyed {
    uint64_t root, rank;
    NodeId id;
  };
  std::vector<Keyed> keyed;
  keyed.reserve(nodes_.size());
  for (const auto& [bits, node] : nodes_) {
    if (node.children_mask) continue;
    const NodeId id = NodeId::unpack(bits);
    const uint32_t ri = id.ci >> id.level, rj = id.cj >> id.level, rk = id.ck >> id.level;
    const uint64_t root = ((uint64_t)rk * cfg_.root_dims[1] + rj) * cfg_.root_dims[0] + ri;
    const uint64_t mask = (1u << id.level) - 1;
    const uint64_t m = morton_encode(id.level, id.ci & mask, id.cj & mask, id.ck & mask);
    keyed.push_back({root, morton_dfs_rank(id.level, m), id});
  }
  std::sort(keyed.begin(), keyed.end(), [](const Keyed& a, const Keyed& b) {
    return a.root != b.root ? a.root < b.root : a.rank < b.rank;
  });
  leaf_cache_.clear();
  slot_cache_.clear();
  for (size_t s = 0; s < keyed.size(); ++s) {
    leaf_cache_.push_back(keyed[s].id);
    slot_cache_[keyed[s].id.packed()] = int(s);
  }
  cache_valid_ = true;
  return leaf_cache_;
}

int Forest::slot_of(const NodeId& leaf) const {
  leaves();
  auto it = slot_cache_.find(leaf.packed());
  return it == slot_cache_.end() ? -1 : it->second;
}

std::optional<NodeId> Forest::covering_leaf(const NodeId& cell) const {
  for (int lvl = cell.level; lvl >= 0; --lvl) {
    const int sh = cell.level - lvl;
    const NodeId probe{lvl, cell.ci >> sh, cell.cj >> sh, cell.ck >> sh};
    auto it = nodes_.find(probe.packed());
    if (it != nodes_.end()) {
      if (it->second.children_mask == 0) return probe;
      return std::nullopt;
    }
  }
  return std::nullopt;
}

// Neighbour cell across (axis, dir) at the same level; false at a reflective wall.
static bool step_cell(const Forest& f, const NodeId& id, int axis, int dir, NodeId& cell) {
  int64_t c[3] = {id.ci, id.cj, id.ck};
  c[axis] += dir > 0 ? 1 : -1;
  const int64_t ext = (int64_t)f.cells_per_axis(id.level, axis);
  if (c[axis] < 0 || c[axis] >= ext) {
    if (f.config().bc[axis]) return false;
    c[axis] = (c[axis] + ext) % ext;
  }
  cell = NodeId{id.level, uint32_t(c[0]), uint32_t(c[1]), uint32_t(c[2])};
  return true;
}

// The four children of `cell` on the face looking back along -dir, ordered
// (t2 outer, t1 inner) (octree.cpp:110-121).
static std::array<NodeId, 4> face_children(const NodeId& cell, int axis, int dir) {
  std::array<NodeId, 4> out;
  const int face_bit = dir > 0 ? 0 : 1, t1 = (axis + 1) % 3, t2 = (axis + 2) % 3;
  int n = 0;
  for (int b2 = 0; b2 < 2; ++b2)
    for (int b1 = 0; b1 < 2; ++b1) {
      int bits[3];
      bits[axis] = face_bit;
      bits[t1] = b1;
      bits[t2] = b2;
      out[n++] = cell.child(bits[0], bits[1], bits[2]);
    }
  return out;
}

FaceNeighbors Forest::face_neighbor(const NodeId& leaf, int axis, int dir) const {
  FaceNeighbors out;
  NodeId cell;
  if (!step_cell(*this, leaf, axis, dir, cell)) return out;  // boundary
  auto it = nodes_.find(cell.packed());
  if (it != nodes_.end() && it->second.children_mask) {
    out.kind = NeighborKind::finer;
    out.ids = face_children(cell, axis, dir);
    out.count = 4;
    return out;
  }
  auto cov = covering_leaf(cell);
  if (!cov) throw AmrError("face_neighbor: topology corrupt");
  out.kind = cov->level == leaf.level ? NeighborKind::same : NeighborKind::coarser;
  out.ids[0] = *cov;
  out.count = 1;
  return out;
}

void Forest::refine(const NodeId& id) {
  {
    auto it = nodes_.find(id.packed());
    if (it == nodes_.end()) throw AmrError("node not in tree");
    if (it->second.children_mask) throw AmrError("refine of a non-leaf");
    if (id.level >= cfg_.max_level) throw AmrError("refine beyond max_level");
  }
  // eager 2:1 balance: coarser face neighbours refine first (octree.cpp:206-223)
  for (int axis = 0; axis < 3; ++axis)
    for (int dir : {-1, +1})
      for (;;) {
        NodeId cell;
        if (!step_cell(*this, id, axis, dir, cell)) break;
        auto cov = covering_leaf(cell);
        if (!cov || cov->level >= id.level) break;
        refine(*cov);
      }
  nodes_[id.packed()].children_mask = 0xFF;
  for (int bk = 0; bk < 2; ++bk)
    for (int bj = 0; bj < 2; ++bj)
      for (int bi = 0; bi < 2; ++bi) nodes_[id.child(bi, bj, bk).packed()] = Node{};
  oplog_.push_back(Op{true, id});
  cache_valid_ = false;
  version_ += 1;
}

void Forest::coarsen(const NodeId& parent) {
  auto it = nodes_.find(parent.packed());
  if (it == nodes_.end()) throw AmrError("node not in tree");
  if (it->second.children_mask != 0xFF) throw AmrError("coarsen of a leaf");
  for (int b = 0; b < 8; ++b) {
    auto c = nodes_.find(parent.child(b & 1, (b >> 1) & 1, (b >> 2) & 1).packed());
    if (c == nodes_.end() || c->second.children_mask)
      throw AmrError("coarsen requires all 8 children to be leaves");
  }
  // balance: a subdivided face neighbour's face children must all be leaves
  for (int axis = 0; axis < 3; ++axis)
    for (int dir : {-1, +1}) {
      NodeId cell;
      if (!step_cell(*this, parent, axis, dir, cell)) continue;
      auto nb = nodes_.find(cell.packed());
      if (nb == nodes_.end() || !nb->second.children_mask) continue;
      for (const NodeId& fc : face_children(cell, axis, dir)) {
        auto f = nodes_.find(fc.packed());
        if (f != nodes_.end() && f->second.children_mask)
          throw AmrError("coarsen would violate 2:1 balance");
      }
    }
  for (int b = 0; b < 8; ++b) nodes_.erase(parent.child(b & 1, (b >> 1) & 1, (b >> 2) & 1).packed());
  nodes_[parent.packed()].children_mask = 0;
  oplog_.push_back(Op{false, parent});
  cache_valid_ = false;
  version_ += 1;
}

bool Forest::is_balanced() const {
  for (const NodeId& leaf : leaves())
    for (int axis = 0; axis < 3; ++axis)
      for (int dir : {-1, +1}) {
        NodeId cell;
        if (!step_cell(*this, leaf, axis, dir, cell)) continue;
        auto it = nodes_.find(cell.packed());
        if (it != nodes_.end() && it->second.children_mask) {
          for (const NodeId& c : face_children(cell, axis, dir))
            if (!is_leaf(c)) return false;
          continue;
        }
        auto cov = covering_leaf(cell);
        if (!cov || leaf.level - cov->level > 1) return false;
      }
  return true;
}

std::vector<Fill> Forest::plan_axis(int axis) const {
  std::vector<Fill> plan;
  const auto& lv = leaves();
  plan.reserve(lv.size() * 2);
  const int t1 = (axis + 1) % 3, t2 = (axis + 2) % 3;
  for (size_t s = 0; s < lv.size(); ++s) {
    const NodeId& leaf = lv[s];
    for (int dir : {-1, +1}) {
      const FaceNeighbors nb = face_neighbor(leaf, axis, dir);
      Fill f{int32_t(s), -1, int8_t(nb.kind), int8_t(axis), int8_t(dir), 0, 0};
      switch (nb.kind) {
        case NeighborKind::boundary:
          plan.push_back(f);
          break;
        case NeighborKind::same:
          f.src = slot_of(nb.ids[0]);
          plan.push_back(f);
          break;
        case NeighborKind::coarser: {
          const uint32_t c[3] = {leaf.ci, leaf.cj, leaf.ck};
          f.src = slot_of(nb.ids[0]);
          f.qt1 = int8_t(c[t1] & 1);
          f.qt2 = int8_t(c[t2] & 1);
          plan.push_back(f);
          break;
        }
        case NeighborKind::finer:
          for (int q = 0; q < 4; ++q) {
            f.src = slot_of(nb.ids[q]);
            f.qt1 = int8_t(q & 1);
            f.qt2 = int8_t(q >> 1);
            plan.push_back(f);
          }
          break;
      }
    }
  }
  return plan;
}

std::vector<int> partition_leaves(const std::vector<uint64_t>& w, int L) {
  if (L < 1) throw AmrError("partition: localities must be >= 1");
  if ((size_t)L > w.size()) throw AmrError("partition: more localities than leaves");
  unsigned __int128 total = 0;
  for (uint64_t x : w) total += x;
  std::vector<int> owner(w.size());
  unsigned __int128 cum = 0;
  int rank = 0;
  const size_t n = w.size();
  for (size_t i = 0; i < n; ++i) {
    owner[i] = rank;
    cum += w[i];
    if (rank + 1 == L) continue;
    const size_t remaining = n - i - 1, needed = size_t(L - rank - 1);
    const bool reach = cum * (unsigned __int128)L >= (unsigned __int128)(rank + 1) * total;
    if (remaining == needed || (reach && remaining >= needed)) ++rank;
  }
  return owner;
}

}  // namespace tmgpu
