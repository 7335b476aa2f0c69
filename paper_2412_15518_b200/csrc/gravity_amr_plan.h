// Host plan of the AMR FMM (gravity_amr.cu): the cell tree of a forest laid
// out as 8^3-cell patches per forest node, and the W/X (M2L) and cross-depth U
// (P2P) pair lists of our adaptive specification (oracle/gravity_amr_oracle.c).
// Pure C++ (no CUDA), testable on CPU.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace tmgpu {

constexpr int kGravMaxLevel = 15;  // cell depth <= 18; 19-bit global coordinates

struct GravLevel {
  int n = 0;                    // forest nodes at this level (Morton order)
  std::vector<int> ijk;         // [n][3] node coordinates
  std::vector<int> nbr;         // [n][27] same-level node, -1 if none ((dz,dy,dx)+1, x fastest)
  std::vector<int> child;       // [n][8] child node at level+1 (octant x fastest), -1 for leaves
  std::vector<int> parent;      // [n] node at level-1 (-1 at level 0)
  std::vector<int> leaf_slot;   // [n] canonical leaf slot or -1
  std::vector<int> internal;    // internal node indices
  // pair lists over the level's cells (flat = node * 512 + (k*8+j)*8+i),
  // CSR offsets [n*512 + 1]; entries (src_level << 40) | src_flat, sorted
  // per target by source (depth, gk, gj, gi)
  std::vector<int64_t> moff, ment;  // W/X: M2L terms into the cell's local expansion
  std::vector<int64_t> poff, pent;  // cross-depth U: P2P terms (leaf cells only)
  std::vector<int> mgeo, pgeo;      // per entry: index into GravPlan::wx_sep / u_sep
};

struct GravPlan {
  int nlevels = 0;  // levels 0..nlevels-1
  std::vector<GravLevel> lv;
  std::vector<int> slot_level, slot_node;  // per canonical leaf slot
  long long m_entries = 0, p_entries = 0;
  // distinct separations R = x_target - x_source of the W/X and cross-depth U
  // entries ([k][3], each computed as centre(t) - centre(s) exactly as the
  // oracle does): the result of that subtraction depends only on the exact
  // separation, so entries share a geometry table bit for bit
  std::vector<double> wx_sep, u_sep;
};

// leaves: [n][4] (level, I, J, K) in canonical order, one root = unit cube.
// Returns false (why set) unless the leaves tile the cube without overlap.
bool build_grav_plan(const int* leaves, long long nleaves, GravPlan& plan, std::string* why);

// Multi-GPU: per level, the nodes (ascending) that are ancestors-or-self of the
// canonical slots [lo, hi) — the patches whose M2L/L2L a rank owning those
// slots must evaluate (their locals flow down to its leaves).
std::vector<std::vector<int>> grav_owned_ancestors(const GravPlan& plan, long long lo, long long hi);

// Multi-GPU locally essential tree (the multipole-moment exchange). A patch is
// owned by rank r when every leaf of its subtree is r's (canonical slots are
// Morton DFS, so a subtree is a contiguous slot range); patches spanning
// ranks form the shared top T. Rank r computes its owned subtrees' moments
// (P2M, M2M), all ranks all-gather the owned subtree roots R (children of T
// or the root), every rank then computes T by M2M, and the owned patches
// other ranks read (V-list neighbourhoods, W/X and cross-depth U sources of
// their targets) are sent point to point. Every moment is computed exactly as
// on one GPU, so the solve stays bitwise.
struct PatchRef {
  int level, node;
};
struct GravLetPlan {
  std::vector<std::vector<int>> owned_internal;  // per level: this rank's owned internal patches
  std::vector<std::vector<int>> top_internal;    // per level: T (shared) patches
  std::vector<std::vector<PatchRef>> roots;      // per rank: its owned subtree roots R_r
  std::vector<std::vector<PatchRef>> send;       // per peer: owned patches the peer reads
  std::vector<std::vector<PatchRef>> recv;       // per peer: the peer's patches this rank reads
  std::vector<int> halo_leaf_slots;              // received leaf patches (their masses are read)
};
GravLetPlan grav_let_plan(const GravPlan& plan, const std::vector<long long>& slot_bounds, int me);

}  // namespace tmgpu
