// Plan of the one-round face exchange (see halo.h / halo_plan.h).
//
// Every fill of the reference plan (plan_axis_fills, ghost.cpp:168-210, all
// three axes, plan order) is classified from this rank's point of view:
//   dst local, src local   same  -> stage kernel reads the neighbour (no work)
//                          finer -> pull computes the 2x2x2 means in place
//                          coarser -> pack a prolonged slab locally, pull it
//   dst local, src remote  -> receive a slab from the source's rank, pull it
//   dst remote, src local  -> pack a slab into the send region for dst's rank
//   boundary               -> pull mirrors the leaf's own interior
// Sender and receiver walk the same global plan order, so the k-th slab
// from rank q to rank r describes the same fill on both sides.
#include "halo_plan.h"

#include <cstring>

namespace tmgpu {

HaloPlan build_halo_plan(const Forest& f, const std::vector<int>& owner, int rank, int world) {
  HaloPlan P;
  P.rank = rank;
  P.world = world;
  P.vars = f.config().vars;
  const int V = P.vars;
  const auto& lv = f.leaves();
  const int ng = (int)lv.size();
  P.gl2loc.assign(ng, -1);
  for (int g = 0; g < ng; ++g)
    if (owner[g] == rank) {
      P.gl2loc[g] = (int)P.loc2gl.size();
      P.loc2gl.push_back(g);
    }
  const int nl = (int)P.loc2gl.size();
  P.faces.assign((size_t)nl * 6, FaceSrc{});
  for (auto& fs : P.faces) {
    std::memset(&fs, 0, sizeof(fs));
    for (int q = 0; q < 4; ++q) fs.src[q] = -1, fs.off[q] = -1;
    fs.kind = 3;
  }
  P.send_cnt.assign(world, 0);
  P.recv_cnt.assign(world, 0);
  std::vector<std::vector<Fill>> plans(3);
  for (int a = 0; a < 3; ++a) plans[a] = f.plan_axis(a);

  // pass 1: sizes (local prolonged, per-peer send / recv)
  for (int a = 0; a < 3; ++a)
    for (const Fill& x : plans[a]) {
      if (x.kind == (int8_t)NeighborKind::boundary) continue;
      const int dst_o = owner[x.dst], src_o = owner[x.src];
      const long long n = slab_doubles(x.kind, V);
      if (dst_o == rank && src_o == rank) {
        if (x.kind == (int8_t)NeighborKind::coarser) P.local_doubles += n;
      } else if (src_o == rank) {
        P.send_cnt[dst_o] += n;
      } else if (dst_o == rank) {
        P.recv_cnt[src_o] += n;
      }
    }
  P.send_off.assign(world, 0);
  P.recv_off.assign(world, 0);
  long long s = 0, r = 0;
  for (int p = 0; p < world; ++p) {
    P.send_off[p] = s;
    P.recv_off[p] = r;
    s += P.send_cnt[p];
    r += P.recv_cnt[p];
  }
  P.send_base = P.local_doubles;
  P.recv_base = P.send_base + s;
  P.total_doubles = P.recv_base + r;

  // pass 2: items and offsets
  long long local_cur = 0;
  std::vector<long long> send_cur(world, 0), recv_cur(world, 0);
  for (int a = 0; a < 3; ++a)
    for (const Fill& x : plans[a]) {
      const int face = 2 * a + (x.dir > 0 ? 1 : 0);
      const int dst_o = owner[x.dst];
      const bool boundary = x.kind == (int8_t)NeighborKind::boundary;
      const int src_o = boundary ? dst_o : owner[x.src];
      const int q = x.kind == (int8_t)NeighborKind::finer ? x.qt2 * 2 + x.qt1 : 0;
      const long long n = slab_doubles(x.kind, V);
      if (dst_o == rank) {
        FaceSrc& fs = P.faces[(size_t)P.gl2loc[x.dst] * 6 + face];
        fs.kind = x.kind;
        if (!boundary) {
          if (src_o == rank && x.kind != (int8_t)NeighborKind::coarser) {
            fs.src[q] = P.gl2loc[x.src];
          } else if (src_o == rank) {  // local prolonged slab
            fs.off[0] = (int32_t)local_cur;
            P.pack.push_back(PackItem{P.gl2loc[x.src], (int32_t)local_cur, x.kind, x.axis, x.dir,
                                      x.qt1, x.qt2, {0, 0, 0}});
            local_cur += n;
          } else {  // received slab
            fs.off[q] = (int32_t)(P.recv_base + P.recv_off[src_o] + recv_cur[src_o]);
            recv_cur[src_o] += n;
            P.recv_manifest.push_back({src_o, (int64_t)lv[x.dst].packed(),
                                       (int64_t)lv[x.src].packed(), x.kind, x.axis, x.dir});
          }
        }
      } else if (!boundary && src_o == rank) {  // slab for another rank
        const long long off = P.send_base + P.send_off[dst_o] + send_cur[dst_o];
        P.pack.push_back(PackItem{P.gl2loc[x.src], (int32_t)off, x.kind, x.axis, x.dir, x.qt1,
                                  x.qt2, {0, 0, 0}});
        send_cur[dst_o] += n;
        P.send_manifest.push_back({dst_o, (int64_t)lv[x.dst].packed(), (int64_t)lv[x.src].packed(),
                                   x.kind, x.axis, x.dir});
      }
    }

  P.face_src.assign((size_t)nl * 6, 0);
  for (int l = 0; l < nl; ++l) {
    bool boundary = false;
    for (int face = 0; face < 6; ++face) {
      const FaceSrc& fs = P.faces[(size_t)l * 6 + face];
      const bool local_same = fs.kind == (int8_t)NeighborKind::same && fs.src[0] >= 0;
      bool remote = false;
      for (int q = 0; q < 4; ++q) remote |= fs.src[q] < 0 && fs.off[q] >= P.recv_base;
      P.face_src[(size_t)l * 6 + face] = local_same ? ((fs.src[0] << 1) | 1) : (l << 1);
      P.pull_all.push_back(l);
      P.pull_all.push_back(face);
      if (!local_same) {
        P.pull_fused.push_back(l);
        P.pull_fused.push_back(face);
        auto& v = remote ? P.pull_fused_remote : P.pull_fused_local;
        v.push_back(l);
        v.push_back(face);
      }
      boundary |= remote;
    }
    (boundary ? P.boundary_slots : P.interior_slots).push_back(l);
  }
  return P;
}

}  // namespace tmgpu
