// Host-side plan of the one-round face exchange for one rank (halo_plan.cpp).
// Pure C++ (no CUDA calls), so the multi-rank bookkeeping is testable on CPU.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "forest.h"
#include "halo.h"

namespace tmgpu {

struct HaloPlan {
  int rank = 0, world = 1, vars = 5;
  std::vector<int> loc2gl;  // local slot -> canonical leaf index
  std::vector<int> gl2loc;  // canonical leaf index -> local slot or -1
  std::vector<PackItem> pack;          // slabs this rank produces each exchange
  std::vector<FaceSrc> faces;          // [local slot][6]
  std::vector<int> face_src;           // [local slot][6] stage-kernel TMA source codes
  std::vector<int> pull_fused;         // pairs (slot, face): faces the fused step pulls
  std::vector<int> pull_all;           // pairs (slot, face): every face
  // multi-GPU overlap: faces needing a received slab vs the rest, and the
  // local leaves with (boundary) / without (interior) such a face
  std::vector<int> pull_fused_local, pull_fused_remote;
  std::vector<int> interior_slots, boundary_slots;
  long long local_doubles = 0;         // slab buffer: [local prolonged | send | recv]
  long long send_base = 0, recv_base = 0, total_doubles = 0;
  std::vector<long long> send_off, send_cnt, recv_off, recv_cnt;  // per peer, relative to base
  // message manifests (tests): per slab, (peer, dst leaf, src leaf, kind, axis, dir)
  std::vector<std::array<int64_t, 6>> send_manifest, recv_manifest;
};

// owner: rank of every canonical leaf (partition_leaves); all zero for one GPU.
HaloPlan build_halo_plan(const Forest& f, const std::vector<int>& owner, int rank, int world);

}  // namespace tmgpu
