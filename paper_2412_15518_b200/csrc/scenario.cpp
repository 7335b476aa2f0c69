// Synthetic scenarios (the configs of BASELINE.json): analytic initial data
// and analytic refinement rules. Host C++; the reference ships no scenario
// code (its CLI is a stub, proj/tools/taskmesh_cli.cpp:1), so these follow
// SURVEY.md §8(d) and SPEC.md:620-631.
//
//  kind 0  rotating star     rho = max(1-r^2/R^2,0)^1.5 + 1e-3, R = 0.3 about the box
//                            centre; p = 0.5 rho^(5/3); rigid rotation about z
//                            (u,v,w) = (-(y-1/2), x-1/2, 0); then rho *= 1 + 1e-3 U(-1,1)
//                            from std::mt19937_64(seed), drawn in canonical leaf order,
//                            (k,j,i) cell order. Refinement: |grad rho0| dx / rho0 > theta
//                            (analytic gradient) at any cell centre of the leaf.
//  kind 1  double white dwarf two such polytropes at (0.35,.5,.5) R=0.12 and
//                            (0.65,.5,.5) R=0.09 (amplitude 0.6), same rotation; refine
//                            every leaf intersecting |x - c| < 0.28 (geometric).
//  kind 2  Sod               (rho,p) = (1,1) for x < 1/2 else (0.125,0.1), u = 0;
//                            refine leaves touching the x = 1/2 plane.
//  kind 3  Sedov             rho = 1, p = 1e-5, E0 = 1 deposited in the 2^3 cells
//                            nearest the centre at the finest level; refine |x-c| < 0.15.
#include <algorithm>
#include <cmath>
#include <random>

#include "forest.h"

namespace tmgpu {

namespace {

constexpr double kGamma = 1.4;

struct Prim5 {
  double rho, u, v, w, p;
};

double star_rho0(double x, double y, double z, double cx, double R, double amp) {
  const double r2 = (x - cx) * (x - cx) + (y - 0.5) * (y - 0.5) + (z - 0.5) * (z - 0.5);
  const double q = 1.0 - r2 / (R * R);
  return amp * (q > 0.0 ? std::pow(q, 1.5) : 0.0);
}

// |grad rho0| for one polytrope
double star_grad(double x, double y, double z, double cx, double R, double amp) {
  const double r2 = (x - cx) * (x - cx) + (y - 0.5) * (y - 0.5) + (z - 0.5) * (z - 0.5);
  const double q = 1.0 - r2 / (R * R);
  if (q <= 0.0) return 0.0;
  return amp * 1.5 * std::sqrt(q) * 2.0 * std::sqrt(r2) / (R * R);
}

Prim5 prim_at(int kind, double x, double y, double z) {
  switch (kind) {
    case 0: {
      const double rho = star_rho0(x, y, z, 0.5, 0.3, 1.0) + 1e-3;
      return {rho, -(y - 0.5), x - 0.5, 0.0, 0.5 * std::pow(rho, 5.0 / 3.0)};
    }
    case 1: {
      const double rho =
          star_rho0(x, y, z, 0.35, 0.12, 1.0) + star_rho0(x, y, z, 0.65, 0.09, 0.6) + 1e-3;
      return {rho, -(y - 0.5), x - 0.5, 0.0, 0.5 * std::pow(rho, 5.0 / 3.0)};
    }
    case 2:
      return x < 0.5 ? Prim5{1.0, 0, 0, 0, 1.0} : Prim5{0.125, 0, 0, 0, 0.1};
    default:
      return {1.0, 0, 0, 0, 1e-5};
  }
}

// Leaf box [lo, hi) in physical coordinates.
void leaf_box(const Forest& f, const NodeId& id, double lo[3], double hi[3]) {
  const double ext = f.root_extent() / double(1u << id.level);
  const uint32_t c[3] = {id.ci, id.cj, id.ck};
  for (int a = 0; a < 3; ++a) {
    lo[a] = c[a] * ext;
    hi[a] = (c[a] + 1) * ext;
  }
}

double box_dist(const double lo[3], const double hi[3], const double c[3]) {
  double d2 = 0;
  for (int a = 0; a < 3; ++a) {
    const double t = c[a] < lo[a] ? lo[a] - c[a] : c[a] > hi[a] ? c[a] - hi[a] : 0.0;
    d2 += t * t;
  }
  return std::sqrt(d2);
}

bool wants_refine(const Forest& f, int kind, const NodeId& id, double theta) {
  double lo[3], hi[3];
  leaf_box(f, id, lo, hi);
  const double ctr[3] = {0.5, 0.5, 0.5};
  switch (kind) {
    case 0: {
      const int E = f.config().edge, G = f.config().ghost;
      const double dx = f.cell_size(id.level);
      for (int k = G; k < G + E; ++k)
        for (int j = G; j < G + E; ++j)
          for (int i = G; i < G + E; ++i) {
            auto c = f.cell_center(id, i, j, k);
            const double rho = star_rho0(c[0], c[1], c[2], 0.5, 0.3, 1.0) + 1e-3;
            if (star_grad(c[0], c[1], c[2], 0.5, 0.3, 1.0) * dx / rho > theta) return true;
          }
      return false;
    }
    case 1:
      return box_dist(lo, hi, ctr) < 0.28;
    case 2:
      return lo[0] <= 0.5 && 0.5 <= hi[0];
    default:
      return box_dist(lo, hi, ctr) < 0.15;
  }
}

}  // namespace

// Uniform refinement to `min_level`, then repeated sweeps refining every leaf
// the rule selects (in canonical order, 2:1 cascades included) up to max_level.
void scenario_refine(Forest& f, int kind, int min_level, int max_level, double theta) {
  for (int l = 0; l < min_level; ++l) {
    const std::vector<NodeId> lv = f.leaves();
    for (const NodeId& id : lv)
      if (id.level == l && f.is_leaf(id)) f.refine(id);
  }
  for (int l = min_level; l < max_level; ++l) {
    const std::vector<NodeId> lv = f.leaves();
    for (const NodeId& id : lv)
      if (id.level == l && f.is_leaf(id) && wants_refine(f, kind, id, theta)) f.refine(id);
  }
}

// Interior conserved state in compact [slot][5][E^3] (k,j,i) order.
void scenario_fill(const Forest& f, int kind, uint64_t seed, double* out) {
  const int E = f.config().edge, G = f.config().ghost;
  const size_t e3 = size_t(E) * E * E;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(-1.0, 1.0);
  const auto& lv = f.leaves();
  int finest = 0;
  for (const NodeId& id : lv) finest = std::max(finest, id.level);
  const double hf = f.cell_size(finest);
  for (size_t s = 0; s < lv.size(); ++s) {
    double* o = out + s * 5 * e3;
    size_t n = 0;
    for (int k = G; k < G + E; ++k)
      for (int j = G; j < G + E; ++j)
        for (int i = G; i < G + E; ++i, ++n) {
          auto c = f.cell_center(lv[s], i, j, k);
          Prim5 q = prim_at(kind, c[0], c[1], c[2]);
          if (kind <= 1) q.rho *= 1.0 + 1e-3 * unif(rng);
          double e = q.p / (kGamma - 1.0) + 0.5 * q.rho * (q.u * q.u + q.v * q.v + q.w * q.w);
          if (kind == 3 && lv[s].level == finest && std::fabs(c[0] - 0.5) < hf &&
              std::fabs(c[1] - 0.5) < hf && std::fabs(c[2] - 0.5) < hf)
            e += 1.0 / (8.0 * hf * hf * hf);  // E0 = 1 over the 8 central cells
          o[n] = q.rho;
          o[e3 + n] = q.rho * q.u;
          o[2 * e3 + n] = q.rho * q.v;
          o[3 * e3 + n] = q.rho * q.w;
          o[4 * e3 + n] = e;
        }
  }
}

}  // namespace tmgpu
