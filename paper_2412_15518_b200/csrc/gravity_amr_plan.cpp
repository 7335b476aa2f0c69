// AMR FMM plan (see gravity_amr_plan.h). The list definitions are those of
// oracle/gravity_amr_oracle.c (visit(), ent_cmp()); here they are generated
// from node tables instead of dense per-depth arrays, so they scale to the
// 7-level configurations.
#include "gravity_amr_plan.h"

#include <algorithm>
#include <unordered_map>

namespace tmgpu {
namespace {

inline uint64_t key3(uint64_t i, uint64_t j, uint64_t k) { return (i << 42) | (j << 21) | k; }

inline uint64_t morton3(uint64_t i, uint64_t j, uint64_t k, int bits) {
  uint64_t m = 0;
  for (int b = bits - 1; b >= 0; --b)
    m = (m << 3) | (((k >> b) & 1) << 2) | (((j >> b) & 1) << 1) | ((i >> b) & 1);
  return m;
}

struct Pair {
  int64_t tflat;
  int64_t skey;
  int64_t enc;
  int8_t kind, tlevel;
  int8_t sdepth;
  int64_t tg[3], sg[3];  // global cell coordinates of target and source
};

inline double centre(int64_t gi, int d) { return ((double)gi + 0.5) / (double)(1LL << d); }

// exact separation key: depths + 2^(dm+1) (x_t - x_s) as integers, dm the finer depth
struct SepKey {
  int td, sd;
  int64_t i[3];
  bool operator==(const SepKey& o) const {
    return td == o.td && sd == o.sd && i[0] == o.i[0] && i[1] == o.i[1] && i[2] == o.i[2];
  }
};
struct SepHash {
  size_t operator()(const SepKey& k) const {
    uint64_t h = (uint64_t)k.td * 1315423911u + (uint64_t)k.sd * 2654435761u;
    for (int q = 0; q < 3; ++q) h = h * 1000003u ^ (uint64_t)(k.i[q] + (1LL << 40));
    return (size_t)h;
  }
};

struct Builder {
  GravPlan& P;
  std::vector<Pair> pairs;

  bool is_leaf(int level, int node) const { return P.lv[level].leaf_slot[node] >= 0; }

  static bool touches(int da, const int64_t* a, int db, const int64_t* b) {
    const int s = db - da;
    for (int q = 0; q < 3; ++q) {
      const int64_t lo = a[q] << s, hi = (a[q] + 1) << s;
      if (!(b[q] <= hi && b[q] + 1 >= lo)) return false;
    }
    return true;
  }

  static int64_t skey(int depth, const int64_t* g) {
    return ((int64_t)depth << 57) | (g[2] << 38) | (g[1] << 19) | g[0];
  }

  void push(int kind, int tlevel, int64_t tflat, const int64_t* tg, int slevel, int64_t sflat,
            int sdepth, const int64_t* sg) {
    pairs.push_back(Pair{tflat, skey(sdepth, sg), ((int64_t)slevel << 40) | sflat, (int8_t)kind,
                         (int8_t)tlevel, (int8_t)sdepth, {tg[0], tg[1], tg[2]}, {sg[0], sg[1], sg[2]}});
  }

  // b: leaf cell (level lb, flat fb, depth db, global gb); Y: internal cell
  // (level ly, node ny, local yl, global gy)
  void visit(int lb, int64_t fb, const int64_t* gb, int ly, int ny, const int* yl,
             const int64_t* gy) {
    const int db = lb + 3, dc = ly + 4;
    const int cn = P.lv[ly].child[(size_t)ny * 8 + ((yl[2] >> 2) * 2 + (yl[1] >> 2)) * 2 + (yl[0] >> 2)];
    const int lc = ly + 1;
    for (int c = 0; c < 2; ++c)
      for (int bb = 0; bb < 2; ++bb)
        for (int a = 0; a < 2; ++a) {
          const int cl[3] = {((2 * yl[0]) & 7) + a, ((2 * yl[1]) & 7) + bb, ((2 * yl[2]) & 7) + c};
          const int64_t cg[3] = {2 * gy[0] + a, 2 * gy[1] + bb, 2 * gy[2] + c};
          const int64_t cf = (int64_t)cn * 512 + (cl[2] * 8 + cl[1]) * 8 + cl[0];
          if (touches(db, gb, dc, cg)) {
            if (is_leaf(lc, cn)) {
              push(1, lb, fb, gb, lc, cf, dc, cg);
              push(1, lc, cf, cg, lb, fb, db, gb);
            } else {
              visit(lb, fb, gb, lc, cn, cl, cg);
            }
          } else {
            push(0, lb, fb, gb, lc, cf, dc, cg);
            push(0, lc, cf, cg, lb, fb, db, gb);
          }
        }
  }
};

}  // namespace

bool build_grav_plan(const int* leaves, long long nleaves, GravPlan& P, std::string* why) {
  auto fail = [&](const char* m) {
    if (why) *why = m;
    return false;
  };
  P = GravPlan{};
  if (nleaves <= 0) return fail("gravity: no leaves");
  int lmax = 0;
  for (long long s = 0; s < nleaves; ++s) {
    const int l = leaves[4 * s];
    if (l < 0 || l > kGravMaxLevel) return fail("gravity: leaf level out of range");
    for (int q = 1; q < 4; ++q)
      if (leaves[4 * s + q] < 0 || leaves[4 * s + q] >= (1 << l))
        return fail("gravity: leaf outside the unit root");
    lmax = std::max(lmax, l);
  }
  P.nlevels = lmax + 1;
  P.lv.resize(P.nlevels);
  // node sets: value = 1 internal, 2 + slot for leaves
  std::vector<std::unordered_map<uint64_t, long long>> set(P.nlevels);
  uint64_t vol = 0;
  const uint64_t full = 1ULL << (3 * lmax);
  for (long long s = 0; s < nleaves; ++s) {
    const int l = leaves[4 * s];
    uint64_t I = leaves[4 * s + 1], J = leaves[4 * s + 2], K = leaves[4 * s + 3];
    if (!set[l].emplace(key3(I, J, K), 2 + s).second) return fail("gravity: overlapping leaves");
    vol += 1ULL << (3 * (lmax - l));
    for (int a = l - 1; a >= 0; --a) {
      I >>= 1, J >>= 1, K >>= 1;
      auto it = set[a].find(key3(I, J, K));
      if (it != set[a].end()) {
        if (it->second != 1) return fail("gravity: overlapping leaves");
        break;
      }
      set[a].emplace(key3(I, J, K), 1);
    }
  }
  if (vol != full) return fail("gravity: leaves do not tile the unit root");
  // per-level node order (Morton) and tables
  std::vector<std::unordered_map<uint64_t, int>> index(P.nlevels);
  for (int l = 0; l < P.nlevels; ++l) {
    std::vector<std::pair<uint64_t, uint64_t>> keys;  // morton, key
    keys.reserve(set[l].size());
    for (auto& kv : set[l]) {
      const uint64_t k = kv.first;
      keys.emplace_back(morton3(k >> 42, (k >> 21) & 0x1FFFFF, k & 0x1FFFFF, l), k);
    }
    std::sort(keys.begin(), keys.end());
    GravLevel& L = P.lv[l];
    L.n = (int)keys.size();
    L.ijk.resize((size_t)L.n * 3);
    L.leaf_slot.assign(L.n, -1);
    for (int n = 0; n < L.n; ++n) {
      const uint64_t k = keys[n].second;
      L.ijk[3 * n] = (int)(k >> 42);
      L.ijk[3 * n + 1] = (int)((k >> 21) & 0x1FFFFF);
      L.ijk[3 * n + 2] = (int)(k & 0x1FFFFF);
      index[l][k] = n;
      const long long v = set[l][k];
      if (v >= 2) L.leaf_slot[n] = (int)(v - 2);
      else L.internal.push_back(n);
    }
  }
  P.slot_level.assign(nleaves, 0);
  P.slot_node.assign(nleaves, 0);
  for (int l = 0; l < P.nlevels; ++l) {
    GravLevel& L = P.lv[l];
    const int m = 1 << l;
    L.nbr.assign((size_t)L.n * 27, -1);
    L.child.assign((size_t)L.n * 8, -1);
    L.parent.assign(L.n, -1);
    for (int n = 0; n < L.n; ++n) {
      const int I = L.ijk[3 * n], J = L.ijk[3 * n + 1], K = L.ijk[3 * n + 2];
      if (L.leaf_slot[n] >= 0) {
        P.slot_level[L.leaf_slot[n]] = l;
        P.slot_node[L.leaf_slot[n]] = n;
      }
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int a = I + dx, b = J + dy, c = K + dz;
            if (a < 0 || b < 0 || c < 0 || a >= m || b >= m || c >= m) continue;
            auto it = index[l].find(key3(a, b, c));
            if (it != index[l].end()) L.nbr[(size_t)n * 27 + ((dz + 1) * 3 + (dy + 1)) * 3 + dx + 1] = it->second;
          }
      if (l > 0) L.parent[n] = index[l - 1].at(key3(I >> 1, J >> 1, K >> 1));
      if (L.leaf_slot[n] < 0)
        for (int o = 0; o < 8; ++o)
          L.child[(size_t)n * 8 + o] =
              index[l + 1].at(key3(2 * I + (o & 1), 2 * J + ((o >> 1) & 1), 2 * K + (o >> 2)));
    }
  }
  // W / X / cross-depth U pairs (oracle visit(): leaf cells in canonical order)
  Builder B{P, {}};
  for (long long s = 0; s < nleaves; ++s) {
    const int l = P.slot_level[s], n = P.slot_node[s];
    const GravLevel& L = P.lv[l];
    bool any = false;
    for (int o = 0; o < 27 && !any; ++o) {
      const int nb = L.nbr[(size_t)n * 27 + o];
      any = nb >= 0 && L.leaf_slot[nb] < 0;
    }
    if (!any) continue;
    for (int c = 0; c < 512; ++c) {
      const int bl[3] = {c & 7, (c >> 3) & 7, c >> 6};
      const int64_t gb[3] = {8LL * L.ijk[3 * n] + bl[0], 8LL * L.ijk[3 * n + 1] + bl[1],
                             8LL * L.ijk[3 * n + 2] + bl[2]};
      const int64_t fb = (int64_t)n * 512 + c;
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            if (!dx && !dy && !dz) continue;
            int yl[3] = {bl[0] + dx, bl[1] + dy, bl[2] + dz};
            int off[3];
            for (int q = 0; q < 3; ++q) {
              off[q] = yl[q] < 0 ? -1 : (yl[q] > 7 ? 1 : 0);
              yl[q] -= 8 * off[q];
            }
            if (!off[0] && !off[1] && !off[2]) continue;  // own (leaf) node
            const int ny = L.nbr[(size_t)n * 27 + ((off[2] + 1) * 3 + (off[1] + 1)) * 3 + off[0] + 1];
            if (ny < 0 || L.leaf_slot[ny] >= 0) continue;
            const int64_t gy[3] = {gb[0] + dx, gb[1] + dy, gb[2] + dz};
            B.visit(l, fb, gb, l, ny, yl, gy);
          }
    }
  }
  std::sort(B.pairs.begin(), B.pairs.end(), [](const Pair& a, const Pair& b) {
    if (a.kind != b.kind) return a.kind < b.kind;
    if (a.tlevel != b.tlevel) return a.tlevel < b.tlevel;
    if (a.tflat != b.tflat) return a.tflat < b.tflat;
    return a.skey < b.skey;
  });
  for (int l = 0; l < P.nlevels; ++l) {
    GravLevel& L = P.lv[l];
    L.moff.assign((size_t)L.n * 512 + 1, 0);
    L.poff.assign((size_t)L.n * 512 + 1, 0);
  }
  std::unordered_map<SepKey, int, SepHash> sep[2];
  for (const Pair& x : B.pairs) {
    GravLevel& L = P.lv[x.tlevel];
    (x.kind == 0 ? L.moff : L.poff)[x.tflat + 1] += 1;
    (x.kind == 0 ? L.ment : L.pent).push_back(x.enc);
    (x.kind == 0 ? P.m_entries : P.p_entries) += 1;
    const int td = x.tlevel + 3, sd = x.sdepth, dm = std::max(td, sd);
    SepKey k{td, sd, {0, 0, 0}};
    for (int q = 0; q < 3; ++q)
      k.i[q] = (2 * x.tg[q] + 1) * (1LL << (dm - td)) - (2 * x.sg[q] + 1) * (1LL << (dm - sd));
    std::vector<double>& tab = x.kind == 0 ? P.wx_sep : P.u_sep;
    auto it = sep[x.kind].find(k);
    int gi;
    if (it == sep[x.kind].end()) {
      gi = (int)(tab.size() / 3);
      sep[x.kind].emplace(k, gi);
      for (int q = 0; q < 3; ++q) tab.push_back(centre(x.tg[q], td) - centre(x.sg[q], sd));
    } else {
      gi = it->second;
    }
    (x.kind == 0 ? L.mgeo : L.pgeo).push_back(gi);
  }
  for (int l = 0; l < P.nlevels; ++l) {
    GravLevel& L = P.lv[l];
    for (size_t t = 1; t < L.moff.size(); ++t) L.moff[t] += L.moff[t - 1];
    for (size_t t = 1; t < L.poff.size(); ++t) L.poff[t] += L.poff[t - 1];
  }
  return true;
}

std::vector<std::vector<int>> grav_owned_ancestors(const GravPlan& P, long long lo, long long hi) {
  std::vector<std::vector<char>> mark(P.nlevels);
  for (int l = 0; l < P.nlevels; ++l) mark[l].assign(P.lv[l].n, 0);
  for (long long s = lo; s < hi; ++s) {
    int l = P.slot_level[s], n = P.slot_node[s];
    while (l >= 0 && n >= 0 && !mark[l][n]) {
      mark[l][n] = 1;
      n = P.lv[l].parent[n];
      --l;
    }
  }
  std::vector<std::vector<int>> out(P.nlevels);
  for (int l = 0; l < P.nlevels; ++l)
    for (int n = 0; n < P.lv[l].n; ++n)
      if (mark[l][n]) out[l].push_back(n);
  return out;
}

// patches whose moments a rank owning slots [lo, hi) reads: the 27-patch
// neighbourhoods of its M2L patches, their W/X sources, the cross-depth U
// sources of its leaf cells (mark[l][n] = 1)
static std::vector<std::vector<char>> moment_reads(const GravPlan& P, long long lo, long long hi) {
  const auto need = grav_owned_ancestors(P, lo, hi);
  std::vector<std::vector<char>> mark(P.nlevels);
  for (int l = 0; l < P.nlevels; ++l) mark[l].assign(P.lv[l].n, 0);
  auto add_src = [&](int64_t enc) { mark[(int)(enc >> 40)][(int)((enc & ((1LL << 40) - 1)) >> 9)] = 1; };
  for (int l = 0; l < P.nlevels; ++l) {
    const GravLevel& L = P.lv[l];
    for (int n : need[l]) {
      for (int o = 0; o < 27; ++o) {
        const int nb = L.nbr[(size_t)n * 27 + o];
        if (nb >= 0) mark[l][nb] = 1;
      }
      for (int64_t e = L.moff[(size_t)n * 512]; e < L.moff[(size_t)(n + 1) * 512]; ++e) add_src(L.ment[e]);
    }
  }
  for (long long s = lo; s < hi; ++s) {
    const GravLevel& L = P.lv[P.slot_level[s]];
    const int n = P.slot_node[s];
    for (int64_t e = L.poff[(size_t)n * 512]; e < L.poff[(size_t)(n + 1) * 512]; ++e) add_src(L.pent[e]);
  }
  return mark;
}

GravLetPlan grav_let_plan(const GravPlan& P, const std::vector<long long>& bounds, int me) {
  const int R = (int)bounds.size() - 1;
  auto rank_of = [&](long long slot) {
    return (int)(std::upper_bound(bounds.begin(), bounds.end(), slot) - bounds.begin()) - 1;
  };
  // owner per patch (-1: spans ranks), bottom-up from the leaf slots
  std::vector<std::vector<int>> own(P.nlevels);
  for (int l = P.nlevels - 1; l >= 0; --l) {
    const GravLevel& L = P.lv[l];
    own[l].assign(L.n, -1);
    for (int n = 0; n < L.n; ++n) {
      if (L.leaf_slot[n] >= 0) {
        own[l][n] = rank_of(L.leaf_slot[n]);
        continue;
      }
      int o = own[l + 1][L.child[(size_t)n * 8]];
      for (int c = 1; c < 8 && o >= 0; ++c)
        if (own[l + 1][L.child[(size_t)n * 8 + c]] != o) o = -1;
      own[l][n] = o;
    }
  }
  GravLetPlan G;
  G.owned_internal.resize(P.nlevels);
  G.top_internal.resize(P.nlevels);
  G.roots.resize(R);
  G.send.resize(R);
  G.recv.resize(R);
  std::vector<std::vector<char>> avail(P.nlevels);  // computed or all-gathered on every rank
  for (int l = 0; l < P.nlevels; ++l) {
    const GravLevel& L = P.lv[l];
    avail[l].assign(L.n, 0);
    for (int n = 0; n < L.n; ++n) {
      const int o = own[l][n];
      const bool leaf = L.leaf_slot[n] >= 0;
      if (o < 0) {
        if (!leaf) G.top_internal[l].push_back(n);
        avail[l][n] = 1;
        continue;
      }
      if (o == me && !leaf) G.owned_internal[l].push_back(n);
      if (l == 0 || own[l - 1][L.parent[n]] < 0) {
        G.roots[o].push_back(PatchRef{l, n});
        avail[l][n] = 1;
      }
    }
  }
  // point-to-point halo: what rank q reads of rank r's owned, non-root patches
  for (int q = 0; q < R; ++q) {
    if (q == me && R == 1) break;
    const auto reads = moment_reads(P, bounds[q], bounds[q + 1]);
    for (int l = 0; l < P.nlevels; ++l)
      for (int n = 0; n < P.lv[l].n; ++n) {
        if (!reads[l][n]) continue;
        const int o = own[l][n];
        if (o == q) continue;
        // other ranks' leaf patches this rank reads: their masses feed its P2P
        if (q == me && o >= 0 && P.lv[l].leaf_slot[n] >= 0) G.halo_leaf_slots.push_back(P.lv[l].leaf_slot[n]);
        if (avail[l][n]) continue;
        if (q == me)
          G.recv[o].push_back(PatchRef{l, n});
        else if (o == me)
          G.send[q].push_back(PatchRef{l, n});
      }
  }
  return G;
}

}  // namespace tmgpu
