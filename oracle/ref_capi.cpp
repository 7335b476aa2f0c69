// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference mini-app ("taskmesh",
// /root/reference/proj), compiled together with the reference's own sources
// where they lie by oracle/Makefile into oracle/_ref/libtmref.so. Python
// tests and bench.py's reference / cpu_baseline legs reach the reference
// through these entry points (ctypes), so every comparison is against the
// reference's real code path:
//   stage kernel        proj/src/hydro/stage.cpp:222-246 (stage_subgrid, make_stage_kernel)
//   max_wavespeed       proj/src/hydro/stage.cpp:248-272
//   rk3_combine         proj/include/taskmesh/hydro/rk3.hpp:18-27
//   morton / NodeId     proj/include/taskmesh/amr/morton.hpp:32-66, octree.hpp:29-41
//   Tree                proj/src/amr/octree.cpp (leaves, face_neighbor, refine, flag)
//   ghost exchange      proj/src/amr/ghost.cpp:168-296 (plan_axis_fills, fill_ghosts_sync)
//   partition_leaves    proj/src/amr/octree.cpp:374-399
//   aggregation         proj/src/aggregator.cpp (AggregationRegion over task::Scheduler)
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "taskmesh/aggregator.hpp"
#include "taskmesh/amr/ghost.hpp"
#include "taskmesh/amr/morton.hpp"
#include "taskmesh/amr/octree.hpp"
#include "taskmesh/bufferpool.hpp"
#include "taskmesh/hydro/euler.hpp"
#include "taskmesh/hydro/limiter.hpp"
#include "taskmesh/hydro/rk3.hpp"
#include "taskmesh/hydro/stage.hpp"
#include "taskmesh/taskgraph.hpp"

using namespace taskmesh;

namespace {

void put_err(char* err, std::size_t errlen, const char* msg) {
  if (!err || errlen == 0) return;
  std::snprintf(err, errlen, "%s", msg);
}

hydro::StageGeom geom_of(int edge, int ghost, int vars) {
  hydro::StageGeom g;
  g.edge = edge;
  g.ghost = ghost;
  g.vars = vars;
  return g;
}

struct TreeHandle {
  std::unique_ptr<amr::Tree> tree;
};

amr::Tree& T(void* h) { return *static_cast<TreeHandle*>(h)->tree; }

}  // namespace

extern "C" {

// ---------------------------------------------------------------- hydro
// Error codes: 0 ok, 1 SolverError (message in err), 2 other exception.
int tmref_stage_fused(const double* in, double* out, std::size_t in_slice,
                      std::size_t out_slice, std::size_t count, int edge,
                      int ghost, int vars, unsigned lane_width, char* err,
                      std::size_t errlen) {
  try {
    auto spec = hydro::make_stage_kernel(geom_of(edge, ghost, vars), lane_width, 1);
    spec.fn(in, out, in_slice, out_slice, count);
    return 0;
  } catch (const hydro::SolverError& e) {
    put_err(err, errlen, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 2;
  }
}

std::size_t tmref_in_slice(int edge, int ghost, int vars) {
  return geom_of(edge, ghost, vars).in_slice();
}
std::size_t tmref_out_slice(int edge, int ghost, int vars) {
  return geom_of(edge, ghost, vars).out_slice();
}

void tmref_encode_header(int mode, double dx, double dt, double gamma, double ax,
                         double ay, double az, double* out8) {
  hydro::StageParams p;
  p.mode = mode == 0 ? hydro::Mode::scalar : hydro::Mode::euler;
  p.dx = dx;
  p.dt = dt;
  p.gamma = gamma;
  p.advect = {ax, ay, az};
  hydro::encode_header(p, {out8, hydro::kHeaderDoubles});
}

double tmref_max_wavespeed(const double* header8, int edge, int ghost, int vars,
                           const double* ghosted) {
  auto p = hydro::decode_header({header8, hydro::kHeaderDoubles});
  return hydro::max_wavespeed(p, geom_of(edge, ghost, vars), ghosted);
}

double tmref_rk3_combine(int stage, double u0, double v) {
  return hydro::rk3_combine(stage, u0, v);
}

double tmref_minmod_scalar(double a, double b) { return hydro::minmod(a, b); }

double tmref_minmod_lane(double a, double b) {
  using P = lanes::LanePack<1>;
  return hydro::minmod(P(a), P(b)).v[0];
}

void tmref_reconstruct_face(double um1, double u0, double up1, double up2,
                            double* lr) {
  auto f = hydro::reconstruct_face_scalar(um1, u0, up1, up2);
  lr[0] = f.left.v[0];
  lr[1] = f.right.v[0];
}

void tmref_rusanov_euler(const double* ql, const double* qr, double gamma,
                         int axis, double* f5) {
  using P = lanes::LanePack<1>;
  hydro::Prim<P> l{P(ql[0]), P(ql[1]), P(ql[2]), P(ql[3]), P(ql[4])};
  hydro::Prim<P> r{P(qr[0]), P(qr[1]), P(qr[2]), P(qr[3]), P(qr[4])};
  auto f = hydro::rusanov_euler(l, r, P(gamma), axis);
  f5[0] = f.rho.v[0];
  f5[1] = f.mx.v[0];
  f5[2] = f.my.v[0];
  f5[3] = f.mz.v[0];
  f5[4] = f.e.v[0];
}

double tmref_rusanov_scalar(double a, double l, double r) {
  using P = lanes::LanePack<1>;
  return hydro::rusanov_scalar(P(a), P(l), P(r)).v[0];
}

// ---------------------------------------------------------------- indexing
int tmref_morton_encode(int level, std::uint64_t i, std::uint64_t j,
                        std::uint64_t k, std::uint64_t* index) {
  try {
    *index = amr::morton_encode(level, i, j, k).index;
    return 0;
  } catch (const amr::AmrError&) {
    return 1;
  }
}

int tmref_morton_decode(int level, std::uint64_t index, std::uint64_t* ijk) {
  try {
    auto c = amr::morton_decode(amr::MortonKey{level, index});
    ijk[0] = c.i;
    ijk[1] = c.j;
    ijk[2] = c.k;
    return 0;
  } catch (const amr::AmrError&) {
    return 1;
  }
}

std::uint64_t tmref_morton_dfs_rank(int level, std::uint64_t index) {
  return amr::morton_dfs_rank(amr::MortonKey{level, index});
}

int tmref_partition_leaves(const std::uint64_t* weights, std::size_t n,
                           int localities, int* owner) {
  try {
    auto o = amr::partition_leaves(std::vector<std::uint64_t>(weights, weights + n),
                                   localities);
    std::copy(o.begin(), o.end(), owner);
    return 0;
  } catch (const amr::AmrError&) {
    return 1;
  }
}

void tmref_prolong_cell(double c, double xm, double xp, double ym, double yp,
                        double zm, double zp, double* out8) {
  auto f = amr::prolong_cell(c, xm, xp, ym, yp, zm, zp);
  std::copy(f.begin(), f.end(), out8);
}

// ---------------------------------------------------------------- tree
// bc[a]: 0 periodic, 1 reflective.
void* tmref_tree_create(int edge, int ghost, int vars, int max_level,
                        const int* root_dims, const int* bc) {
  amr::TreeConfig cfg;
  cfg.edge = edge;
  cfg.ghost = ghost;
  cfg.vars = vars;
  cfg.max_level = max_level;
  for (int a = 0; a < 3; ++a) {
    cfg.root_dims[a] = root_dims[a];
    cfg.bc[a] = bc[a] ? amr::Boundary::reflective : amr::Boundary::periodic;
  }
  auto* h = new TreeHandle;
  h->tree = std::make_unique<amr::Tree>(cfg);
  return h;
}

void tmref_tree_destroy(void* h) { delete static_cast<TreeHandle*>(h); }

int tmref_tree_refine(void* h, std::uint64_t packed) {
  try {
    T(h).refine(amr::NodeId::unpack(packed));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

int tmref_tree_coarsen(void* h, std::uint64_t packed) {
  try {
    T(h).coarsen(amr::NodeId::unpack(packed));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

std::size_t tmref_tree_leaves(void* h, std::uint64_t* out, std::size_t cap) {
  const auto& lv = T(h).leaves();
  for (std::size_t i = 0; i < lv.size() && i < cap; ++i) out[i] = lv[i].packed();
  return lv.size();
}

double* tmref_tree_grid(void* h, std::uint64_t packed) {
  auto& n = T(h).at(amr::NodeId::unpack(packed));
  return n.grid ? n.grid->raw().data() : nullptr;
}

void tmref_tree_fill_ghosts(void* h) { amr::ghost::fill_ghosts_sync(T(h)); }

int tmref_tree_flag(void* h, std::uint64_t packed, double theta) {
  return T(h).flag_refinement(amr::NodeId::unpack(packed), theta) ? 1 : 0;
}

int tmref_tree_balanced(void* h) { return T(h).is_balanced() ? 1 : 0; }

double tmref_tree_cell_size(void* h, int level) { return T(h).cell_size(level); }

void tmref_tree_cell_center(void* h, std::uint64_t packed, int i, int j, int k,
                            double* xyz) {
  auto c = T(h).cell_center(amr::NodeId::unpack(packed), i, j, k);
  xyz[0] = c[0];
  xyz[1] = c[1];
  xyz[2] = c[2];
}

// kind: 0 same, 1 coarser, 2 finer, 3 boundary (NeighborKind order).
int tmref_tree_face_neighbor(void* h, std::uint64_t packed, int axis, int dir,
                             std::uint64_t* ids4, int* count) {
  auto nb = T(h).face_neighbor(amr::NodeId::unpack(packed), axis, dir);
  *count = nb.count;
  for (int q = 0; q < nb.count; ++q) ids4[q] = nb.ids[q].packed();
  return static_cast<int>(nb.kind);
}

// One row per FillEntry: dst, src, kind, axis, dir, qt1, qt2 (7 x int64).
std::size_t tmref_tree_plan(void* h, int axis, std::int64_t* rows,
                            std::size_t cap) {
  auto plan = amr::ghost::plan_axis_fills(T(h), axis);
  for (std::size_t r = 0; r < plan.size() && r < cap; ++r) {
    const auto& f = plan[r];
    std::int64_t* o = rows + 7 * r;
    o[0] = static_cast<std::int64_t>(f.dst.packed());
    o[1] = f.kind == amr::NeighborKind::boundary
               ? -1
               : static_cast<std::int64_t>(f.src.packed());
    o[2] = static_cast<int>(f.kind);
    o[3] = f.axis;
    o[4] = f.dir;
    o[5] = f.qt1;
    o[6] = f.qt2;
  }
  return plan.size();
}

// ------------------------------------------------- composed hydro step (bench)
// The reference ships no driver (proj/tools/taskmesh_cli.cpp:1); this composes
// the specified SSP-RK3 step from the reference's own calls:
// per stage fill_ghosts_sync -> AggregationRegion(make_stage_kernel) over a
// task::Scheduler -> rk3_combine per interior value. Euler mode, one dt for
// all leaves, dx per leaf level. Returns 0 ok, 1 solver error, 2 other.
int tmref_hydro_step(void* h, double dt, double gamma, unsigned workers,
                     unsigned lane_width, std::size_t max_slices,
                     double* seconds_exchange, double* seconds_stage,
                     char* err, std::size_t errlen) {
  using clock = std::chrono::steady_clock;
  try {
    amr::Tree& tree = T(h);
    const auto& cfg = tree.config();
    const hydro::StageGeom g = geom_of(cfg.edge, cfg.ghost, cfg.vars);
    const std::vector<amr::NodeId> leaves = tree.leaves();
    const std::size_t n = leaves.size();
    const std::size_t ni = g.interior_elems();
    const int E = cfg.edge, G = cfg.ghost;

    std::vector<double> u0(n * ni);
    for (std::size_t l = 0; l < n; ++l) {
      const amr::SubGrid& sg = *tree.at(leaves[l]).grid;
      for (int var = 0; var < cfg.vars; ++var)
        sg.copy_interior_out(var, {u0.data() + l * ni + var * E * E * E,
                                   static_cast<std::size_t>(E) * E * E});
    }

    task::Scheduler sched(workers);
    agg::ExecutorPool execs(std::max(1u, workers));
    mem::BufferPool pool;
    auto spec = hydro::make_stage_kernel(g, lane_width, 1);
    double t_ex = 0.0, t_st = 0.0;
    std::vector<double> slice(spec.in_slice);
    for (int stage = 1; stage <= 3; ++stage) {
      auto t0 = clock::now();
      amr::ghost::fill_ghosts_sync(tree);
      auto t1 = clock::now();
      agg::AggregationRegion region(sched, execs, pool, spec, max_slices, n);
      std::vector<task::Future<agg::SliceOutput>> futs;
      futs.reserve(n);
      for (std::size_t l = 0; l < n; ++l) {
        hydro::StageParams p;
        p.mode = hydro::Mode::euler;
        p.dx = tree.cell_size(leaves[l].level);
        p.dt = dt;
        p.gamma = gamma;
        hydro::encode_header(p, {slice.data(), hydro::kHeaderDoubles});
        auto raw = tree.at(leaves[l]).grid->raw();
        std::memcpy(slice.data() + hydro::kHeaderDoubles, raw.data(),
                    raw.size() * sizeof(double));
        futs.push_back(region.submit_slice(slice));
      }
      region.flush();
      auto outs = sched.run_until(task::when_all(sched, std::move(futs)));
      for (std::size_t l = 0; l < n; ++l) {
        auto v = outs[l].values();
        amr::SubGrid& sg = *tree.at(leaves[l]).grid;
        std::size_t q = 0;
        for (int var = 0; var < cfg.vars; ++var)
          for (int k = G; k < G + E; ++k)
            for (int j = G; j < G + E; ++j)
              for (int i = G; i < G + E; ++i, ++q)
                sg.at(var, i, j, k) =
                    hydro::rk3_combine(stage, u0[l * ni + q], v[q]);
      }
      auto t2 = clock::now();
      t_ex += std::chrono::duration<double>(t1 - t0).count();
      t_st += std::chrono::duration<double>(t2 - t1).count();
    }
    if (seconds_exchange) *seconds_exchange = t_ex;
    if (seconds_stage) *seconds_stage = t_st;
    return 0;
  } catch (const hydro::SolverError& e) {
    put_err(err, errlen, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 2;
  }
}

// Aggregated stage only, over caller-packed slices (bench: kernel throughput of
// the reference with all host threads). Returns seconds, or -1 on error.
double tmref_stage_aggregated(const double* packed_in, std::size_t count,
                              int edge, int ghost, int vars, unsigned workers,
                              unsigned lane_width, std::size_t max_slices,
                              double* packed_out) {
  using clock = std::chrono::steady_clock;
  try {
    const hydro::StageGeom g = geom_of(edge, ghost, vars);
    task::Scheduler sched(workers);
    agg::ExecutorPool execs(std::max(1u, workers));
    mem::BufferPool pool;
    auto spec = hydro::make_stage_kernel(g, lane_width, 1);
    auto t0 = clock::now();
    agg::AggregationRegion region(sched, execs, pool, spec, max_slices, count);
    std::vector<task::Future<agg::SliceOutput>> futs;
    futs.reserve(count);
    for (std::size_t s = 0; s < count; ++s)
      futs.push_back(region.submit_slice(
          {packed_in + s * spec.in_slice, spec.in_slice}));
    region.flush();
    auto outs = sched.run_until(task::when_all(sched, std::move(futs)));
    auto t1 = clock::now();
    if (packed_out)
      for (std::size_t s = 0; s < count; ++s) {
        auto v = outs[s].values();
        std::memcpy(packed_out + s * spec.out_slice, v.data(),
                    v.size() * sizeof(double));
      }
    return std::chrono::duration<double>(t1 - t0).count();
  } catch (const std::exception&) {
    return -1.0;
  }
}

}  // extern "C"
