// Host-side octree forest: topology, canonical leaf order, face-neighbour
// resolution and the ghost-fill plan. Bit-exact restatement of the reference
// indexing (proj/include/taskmesh/amr/{morton,octree}.hpp,
// src/amr/octree.cpp, src/amr/ghost.cpp:168-210). Grids do not live here:
// the state is a device arena indexed by canonical leaf slot.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace tmgpu {

struct AmrError : std::logic_error {
  using std::logic_error::logic_error;
};

constexpr int kMaxMortonLevel = 20;  // morton.hpp:30

// morton.hpp:32-66
uint64_t morton_encode(int level, uint64_t i, uint64_t j, uint64_t k);
void morton_decode(int level, uint64_t index, uint64_t& i, uint64_t& j, uint64_t& k);
inline uint64_t morton_dfs_rank(int level, uint64_t index) {
  return index << (3 * (kMaxMortonLevel - level));
}

// octree.hpp:23-49
struct NodeId {
  int level = 0;
  uint32_t ci = 0, cj = 0, ck = 0;
  uint64_t packed() const {
    return (uint64_t(level) << 60) | (uint64_t(ci) << 40) | (uint64_t(cj) << 20) | ck;
  }
  static NodeId unpack(uint64_t b) {
    return {int(b >> 60), uint32_t((b >> 40) & 0xFFFFF), uint32_t((b >> 20) & 0xFFFFF),
            uint32_t(b & 0xFFFFF)};
  }
  NodeId child(int bi, int bj, int bk) const {
    return {level + 1, (ci << 1) | uint32_t(bi), (cj << 1) | uint32_t(bj), (ck << 1) | uint32_t(bk)};
  }
  bool operator==(const NodeId& o) const {
    return level == o.level && ci == o.ci && cj == o.cj && ck == o.ck;
  }
};

enum class NeighborKind : uint8_t { same = 0, coarser = 1, finer = 2, boundary = 3 };

struct FaceNeighbors {
  NeighborKind kind = NeighborKind::boundary;
  int count = 0;
  std::array<NodeId, 4> ids{};
};

struct ForestConfig {
  int edge = 8, ghost = 2, vars = 5, max_level = 10;
  std::array<int, 3> root_dims{1, 1, 1};
  std::array<int, 3> bc{0, 0, 0};  // 0 periodic, 1 reflective
};

// One directed ghost fill of one axis pass (ghost.hpp:53-61), by leaf slot.
struct Fill {
  int32_t dst, src;  // src = -1 for boundary fills
  int8_t kind, axis, dir, qt1, qt2;
};

class Forest {
 public:
  explicit Forest(const ForestConfig& cfg);

  const ForestConfig& config() const { return cfg_; }
  double root_extent() const { return root_extent_; }
  double cell_size(int level) const { return root_extent_ / (cfg_.edge * (1 << level)); }
  uint32_t cells_per_axis(int level, int axis) const {
    return uint32_t(cfg_.root_dims[axis]) << level;
  }
  // octree.cpp:42-50, storage coordinates (interior at [ghost, ghost+edge))
  std::array<double, 3> cell_center(const NodeId& id, int i, int j, int k) const;

  bool contains(const NodeId& id) const { return nodes_.count(id.packed()) != 0; }
  bool is_leaf(const NodeId& id) const;

  // octree.cpp:52-77: root raster order, then Morton depth-first order
  const std::vector<NodeId>& leaves() const;
  int slot_of(const NodeId& leaf) const;  // canonical index, -1 if not a leaf
  uint64_t topology_version() const { return version_; }

  void refine(const NodeId& id);  // octree.cpp:200-234 (eager 2:1 cascade)
  void coarsen(const NodeId& parent);  // octree.cpp:236-293 (2:1 check, all children leaves)
  // every split / merge in execution order (cascaded refines included): the
  // sequence the reference's data prolongation/restriction follows (regrid)
  struct Op {
    bool refine;
    NodeId node;
  };
  const std::vector<Op>& oplog() const { return oplog_; }
  void clear_oplog() { oplog_.clear(); }
  std::optional<NodeId> covering_leaf(const NodeId& cell) const;          // octree.cpp:79-90
  FaceNeighbors face_neighbor(const NodeId& leaf, int axis, int dir) const;  // :92-132
  bool is_balanced() const;                                               // :325-361

  // ghost.cpp:168-210 plan_axis_fills, with leaf slots
  std::vector<Fill> plan_axis(int axis) const;

 private:
  struct Node {
    uint8_t children_mask = 0;
  };
  ForestConfig cfg_;
  double root_extent_ = 1.0;
  std::unordered_map<uint64_t, Node> nodes_;
  mutable std::vector<NodeId> leaf_cache_;
  mutable std::unordered_map<uint64_t, int> slot_cache_;
  mutable bool cache_valid_ = false;
  uint64_t version_ = 0;
  std::vector<Op> oplog_;
};

// scenario.cpp: analytic refinement + initial data (kinds: 0 rotating star,
// 1 double white dwarf, 2 Sod, 3 Sedov); state in compact [slot][5][E^3].
void scenario_refine(Forest& f, int kind, int min_level, int max_level, double theta);
void scenario_fill(const Forest& f, int kind, uint64_t seed, double* out);

// octree.cpp:374-399: greedy contiguous partition by weight (uint128 sums).
std::vector<int> partition_leaves(const std::vector<uint64_t>& weights, int localities);

}  // namespace tmgpu
