/* TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * Plain-C restatement of the reference per-subgrid hot path. Citations are
 * into /root/reference/proj. Parity is pinned (see tm_oracle.h): this file is
 * compared bitwise against the unmodified reference (oracle/_ref/libtmref.so)
 * by tests/test_oracle_pin.py. Build: oracle/Makefile, -O2 -ffp-contract=off
 * like the reference (CMakeLists.txt:12-14), so every + - * / and sqrt is one
 * IEEE round-to-nearest operation in the reference's association order.
 */
#include "tm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define RHO_FLOOR 1e-10      /* euler.hpp:15 */
#define P_FLOOR 1e-12        /* euler.hpp:16 */

/* ------------------------------------------------------------ limiter */
/* limiter.hpp:13-16 (scalar form, used by ghost prolongation) */
double tmo_minmod_scalar(double a, double b) {
  if (a * b <= 0.0) return 0.0;
  return fabs(a) < fabs(b) ? a : b;
}

/* limiter.hpp:18-26 (lane form, used by the stage): select(a*b > 0,
 * select(|a|<|b|, a, b), 0) */
double tmo_minmod_lane(double a, double b) {
  int same = (a * b) > 0.0;
  double smaller = fabs(a) < fabs(b) ? a : b;
  return same ? smaller : 0.0;
}

/* lanes.hpp:109-113 vmax: x > f ? x : f */
static inline double vmax_(double a, double b) { return a > b ? a : b; }
/* std::max(a, b) == (a < b) ? b : a */
static inline double stdmax_(double a, double b) { return (a < b) ? b : a; }

/* euler.hpp:27-35 */
void tmo_reconstruct_face(double um1, double u0, double up1, double up2, double* lr) {
  lr[0] = u0 + 0.5 * tmo_minmod_lane(u0 - um1, up1 - u0);
  lr[1] = up1 - 0.5 * tmo_minmod_lane(up1 - u0, up2 - up1);
}

/* euler.hpp:45-50 */
double tmo_rusanov_scalar(double a, double l, double r) {
  return 0.5 * (a * l + a * r) - 0.5 * fabs(a) * (r - l);
}

/* euler.hpp:78-89 prim_to_cons */
static void prim_to_cons(const double* q, double gamma, double* c) {
  c[0] = q[0];
  c[1] = q[0] * q[1];
  c[2] = q[0] * q[2];
  c[3] = q[0] * q[3];
  c[4] = q[4] / (gamma - 1.0) + 0.5 * q[0] * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
}

/* euler.hpp:96-114 euler_flux */
static void euler_flux(const double* q, double gamma, int axis, double* f) {
  double un = q[1 + axis];
  double c[5];
  prim_to_cons(q, gamma, c);
  f[0] = c[0] * un;
  f[1] = c[1] * un;
  f[2] = c[2] * un;
  f[3] = c[3] * un;
  f[1 + axis] = f[1 + axis] + q[4];
  f[4] = (c[4] + q[4]) * un;
}

/* euler.hpp:91-94 sound_speed */
static double sound_speed(const double* q, double gamma) { return sqrt(gamma * q[4] / q[0]); }

/* euler.hpp:116-137 rusanov_euler; q = (rho,u,v,w,p) */
void tmo_rusanov_euler(const double* ql, const double* qr, double gamma, int axis, double* f) {
  double smax = vmax_(fabs(ql[1 + axis]) + sound_speed(ql, gamma),
                      fabs(qr[1 + axis]) + sound_speed(qr, gamma));
  double fl[5], fr[5], ul[5], ur[5];
  euler_flux(ql, gamma, axis, fl);
  euler_flux(qr, gamma, axis, fr);
  prim_to_cons(ql, gamma, ul);
  prim_to_cons(qr, gamma, ur);
  for (int v = 0; v < 5; ++v) f[v] = 0.5 * (fl[v] + fr[v]) - 0.5 * smax * (ur[v] - ul[v]);
}

/* ------------------------------------------------------------ stage */
/* stage.cpp:93-218 at lane width 1 (output is W-invariant, stage.hpp:69).
 * grav (OUR extension, not in the reference): optional [3][E^3]
 * gravitational acceleration; after the z update and before the floors,
 * m_q += dt*(rho*g_q) and E += dt*(rho*((u*gx + v*gy) + w*gz)) with the stage
 * input's primitives (density floored as in cons -> prim). */
static int stage_impl(const double* h, int E, int G, int V, const double* in, const double* grav,
                      double* out, int* bad_cell) {
  const int S = E + 2 * G;
  const size_t s2 = (size_t)S * S, s3 = s2 * S;
  const size_t e2 = (size_t)E * E, e3 = e2 * E;
  const int euler = h[0] != 0.0;          /* decode_header stage.cpp:21-29 */
  const double dx = h[1], dt = h[2], gamma = h[3];
  const double advect[3] = {h[4], h[5], h[6]};
  const double cdt = dt / dx;
  const size_t face_elems = (size_t)V * e2, interior = (size_t)V * e3;
  size_t n = 0;
  /* stage.cpp:102-110: out interior starts as a copy */
  for (int var = 0; var < V; ++var)
    for (int k = G; k < G + E; ++k)
      for (int j = G; j < G + E; ++j)
        for (int i = G; i < G + E; ++i) out[n++] = in[var * s3 + k * s2 + j * S + i];

  double* cons = (double*)malloc(sizeof(double) * (size_t)V * S);
  double* prim = (double*)malloc(sizeof(double) * 5 * (size_t)S);
  /* stage.cpp:114: flux scratch zeroed once per call (scalar mode never
   * writes vars > 0, which therefore stay zero) */
  double* flux = (double*)calloc((size_t)V * (E + 1), sizeof(double));
  for (int axis = 0; axis < 3; ++axis) {
    const size_t sa = axis == 0 ? 1 : axis == 1 ? (size_t)S : s2;
    const int t1 = (axis + 1) % 3, t2 = (axis + 2) % 3;
    const size_t st1 = t1 == 0 ? 1 : t1 == 1 ? (size_t)S : s2;
    const size_t st2 = t2 == 0 ? 1 : t2 == 1 ? (size_t)S : s2;
    for (int c2 = 0; c2 < E; ++c2)
      for (int c1 = 0; c1 < E; ++c1) {
        const size_t pb = (size_t)(G + c1) * st1 + (size_t)(G + c2) * st2;
        for (int var = 0; var < V; ++var)
          for (int sx = 0; sx < S; ++sx) cons[var * S + sx] = in[var * s3 + pb + sx * sa];
        if (euler) {
          /* stage.cpp:141-153 cons -> prim (true divisions, std::max floors) */
          for (int q = 0; q < S; ++q) {
            double rho = stdmax_(cons[q], RHO_FLOOR);
            double iu = cons[S + q] / rho, iv = cons[2 * S + q] / rho, iw = cons[3 * S + q] / rho;
            double ke = 0.5 * rho * (iu * iu + iv * iv + iw * iw);
            prim[0 * S + q] = rho;
            prim[1 * S + q] = iu;
            prim[2 * S + q] = iv;
            prim[3 * S + q] = iw;
            prim[4 * S + q] = stdmax_((gamma - 1.0) * (cons[4 * S + q] - ke), P_FLOOR);
          }
          /* stage.cpp:57-91 faces_euler */
          for (int f = 0; f <= E; ++f) {
            double ql[5], qr[5], lr[2], fx[5];
            for (int v = 0; v < 5; ++v) {
              const double* p = prim + v * S + G + f;
              tmo_reconstruct_face(p[-2], p[-1], p[0], p[1], lr);
              ql[v] = lr[0];
              qr[v] = lr[1];
            }
            ql[0] = vmax_(ql[0], RHO_FLOOR);
            qr[0] = vmax_(qr[0], RHO_FLOOR);
            ql[4] = vmax_(ql[4], P_FLOOR);
            qr[4] = vmax_(qr[4], P_FLOOR);
            tmo_rusanov_euler(ql, qr, gamma, axis, fx);
            for (int v = 0; v < 5; ++v) flux[v * (E + 1) + f] = fx[v];
          }
        } else {
          /* stage.cpp:44-55 faces_scalar on var 0 */
          for (int f = 0; f <= E; ++f) {
            double lr[2];
            const double* p = cons + G + f;
            tmo_reconstruct_face(p[-2], p[-1], p[0], p[1], lr);
            flux[f] = tmo_rusanov_scalar(advect[axis], lr[0], lr[1]);
          }
        }
        /* stage.cpp:166-183 divergence update + boundary-face record */
        for (int var = 0; var < V; ++var) {
          const double* fx = flux + var * (E + 1);
          for (int c0 = 0; c0 < E; ++c0) {
            int cc[3];
            cc[axis] = c0;
            cc[t1] = c1;
            cc[t2] = c2;
            size_t oi = (((size_t)var * E + cc[2]) * E + cc[1]) * E + cc[0];
            out[oi] -= cdt * (fx[c0 + 1] - fx[c0]);
          }
          size_t fo = (size_t)var * e2 + (size_t)c2 * E + c1;
          out[interior + (size_t)(2 * axis + 0) * face_elems + fo] = fx[0];
          out[interior + (size_t)(2 * axis + 1) * face_elems + fo] = fx[E];
        }
      }
  }
  free(cons);
  free(prim);
  free(flux);
  if (grav && euler && V == 5) {
    for (int k = 0; k < E; ++k)
      for (int j = 0; j < E; ++j)
        for (int i = 0; i < E; ++i) {
          const size_t c = ((size_t)k * E + j) * E + i;
          const size_t q = (size_t)(k + G) * s2 + (size_t)(j + G) * S + (i + G);
          const double rho = stdmax_(in[q], RHO_FLOOR);
          const double iu = in[s3 + q] / rho, iv = in[2 * s3 + q] / rho, iw = in[3 * s3 + q] / rho;
          const double gx = grav[c], gy = grav[e3 + c], gz = grav[2 * e3 + c];
          out[e3 + c] = out[e3 + c] + dt * (rho * gx);
          out[2 * e3 + c] = out[2 * e3 + c] + dt * (rho * gy);
          out[3 * e3 + c] = out[3 * e3 + c] + dt * (rho * gz);
          out[4 * e3 + c] = out[4 * e3 + c] + dt * (rho * ((iu * gx + iv * gy) + iw * gz));
        }
  }
  /* stage.cpp:187-208 floors */
  double floor_hits = 0.0;
  if (euler) {
    for (size_t c = 0; c < e3; ++c) {
      double* rho = out + c;
      double mx = out[e3 + c], my = out[2 * e3 + c], mz = out[3 * e3 + c];
      double* et = out + 4 * e3 + c;
      if (*rho < RHO_FLOOR) {
        *rho = RHO_FLOOR;
        floor_hits += 1.0;
      }
      double ke = 0.5 * (mx * mx + my * my + mz * mz) / *rho;
      double p = (gamma - 1.0) * (*et - ke);
      if (p < P_FLOOR) {
        *et = P_FLOOR / (gamma - 1.0) + ke;
        floor_hits += 1.0;
      }
    }
  }
  /* stage.cpp:209-216 non-finite check, first in var-major order */
  for (size_t c = 0; c < interior; ++c)
    if (!isfinite(out[c])) {
      size_t cell = c % e3;
      if (bad_cell) {
        bad_cell[0] = (int)(cell % E);
        bad_cell[1] = (int)(cell / E % E);
        bad_cell[2] = (int)(cell / e2);
      }
      return 1;
    }
  out[interior + 6 * face_elems] = floor_hits;
  return 0;
}

int tmo_stage_subgrid(const double* h, int E, int G, int V, const double* in, double* out,
                      int* bad_cell) {
  return stage_impl(h, E, G, V, in, NULL, out, bad_cell);
}

int tmo_stage_subgrid_grav(const double* h, int E, int G, int V, const double* in,
                           const double* grav, double* out, int* bad_cell) {
  return stage_impl(h, E, G, V, in, grav, out, bad_cell);
}

/* stage.cpp:229-246 make_stage_kernel's fused body */
int tmo_stage_fused(const double* in, double* out, size_t in_slice, size_t out_slice,
                    size_t count, int E, int G, int V, size_t* bad_slice, int* bad_cell) {
  for (size_t s = 0; s < count; ++s) {
    const double* slice = in + s * in_slice;
    if (tmo_stage_subgrid(slice, E, G, V, slice + 8, out + s * out_slice, bad_cell)) {
      if (bad_slice) *bad_slice = s;
      return 1;
    }
  }
  return 0;
}

/* stage.cpp:248-272 */
double tmo_max_wavespeed(const double* h, int E, int G, int V, const double* g) {
  (void)V;
  const double gamma = h[3];
  if (h[0] == 0.0) return sqrt(h[4] * h[4] + h[5] * h[5] + h[6] * h[6]);
  const int S = E + 2 * G;
  const size_t s2 = (size_t)S * S, s3 = s2 * S;
  double smax = 0.0;
  for (int k = G; k < G + E; ++k)
    for (int j = G; j < G + E; ++j)
      for (int i = G; i < G + E; ++i) {
        size_t c = k * s2 + j * S + i;
        double rho = stdmax_(g[c], RHO_FLOOR);
        double iu = g[s3 + c] / rho, iv = g[2 * s3 + c] / rho, iw = g[3 * s3 + c] / rho;
        double ke = 0.5 * rho * (iu * iu + iv * iv + iw * iw);
        double pr = stdmax_((gamma - 1.0) * (g[4 * s3 + c] - ke), P_FLOOR);
        double s = sqrt(iu * iu + iv * iv + iw * iw) + sqrt(gamma * pr / rho);
        smax = stdmax_(smax, s);
      }
  return smax;
}

/* rk3.hpp:18-27 */
double tmo_rk3_combine(int stage, double u0, double v) {
  switch (stage) {
    case 1:
      return v;
    case 2:
      return u0 + 0.25 * (v - u0);
    default:
      return u0 + (2.0 / 3.0) * (v - u0);
  }
}

/* ------------------------------------------------------------ indexing */
/* morton.hpp:32-46 */
int tmo_morton_encode(int level, uint64_t i, uint64_t j, uint64_t k, uint64_t* index) {
  if (level < 0 || level > 20) return 1;
  const uint64_t limit = 1ull << level;
  if (i >= limit || j >= limit || k >= limit) return 1;
  uint64_t idx = 0;
  for (int b = 0; b < level; ++b) {
    idx |= ((i >> b) & 1ull) << (3 * b);
    idx |= ((j >> b) & 1ull) << (3 * b + 1);
    idx |= ((k >> b) & 1ull) << (3 * b + 2);
  }
  *index = idx;
  return 0;
}

/* morton.hpp:48-60 */
int tmo_morton_decode(int level, uint64_t index, uint64_t* ijk) {
  if (level < 0 || level > 20) return 1;
  if (index >> (3 * level) != 0) return 1;
  ijk[0] = ijk[1] = ijk[2] = 0;
  for (int b = 0; b < level; ++b) {
    ijk[0] |= ((index >> (3 * b)) & 1ull) << b;
    ijk[1] |= ((index >> (3 * b + 1)) & 1ull) << b;
    ijk[2] |= ((index >> (3 * b + 2)) & 1ull) << b;
  }
  return 0;
}

/* morton.hpp:64-66 */
uint64_t tmo_morton_dfs_rank(int level, uint64_t index) { return index << (3 * (20 - level)); }

/* octree.cpp:374-399 */
int tmo_partition_leaves(const uint64_t* w, size_t n, int L, int* owner) {
  if (L < 1 || (size_t)L > n) return 1;
  unsigned __int128 total = 0, cum = 0;
  for (size_t i = 0; i < n; ++i) total += w[i];
  int rank = 0;
  for (size_t i = 0; i < n; ++i) {
    owner[i] = rank;
    cum += w[i];
    if (rank + 1 == L) continue;
    size_t remaining = n - i - 1;
    size_t needed = (size_t)(L - rank - 1);
    int must = remaining == needed;
    int want = cum * (unsigned __int128)L >= (unsigned __int128)(rank + 1) * total;
    if (must || (want && remaining >= needed)) rank += 1;
  }
  return 0;
}

/* ------------------------------------------------------------ tree */
/* NodeId packing, octree.hpp:29-41 */
#define PK(l, i, j, k) (((uint64_t)(l) << 60) | ((uint64_t)(i) << 40) | ((uint64_t)(j) << 20) | (uint64_t)(k))
#define LV(p) ((int)((p) >> 60))
#define CI(p) ((uint32_t)(((p) >> 40) & 0xFFFFF))
#define CJ(p) ((uint32_t)(((p) >> 20) & 0xFFFFF))
#define CK(p) ((uint32_t)((p)&0xFFFFF))

struct tmo_tree {
  int E, G, V;
  int root[3];
  int bc[3];
  uint64_t* nodes; /* sorted packed ids, all nodes */
  unsigned char* leaf;
  size_t nnodes;
  uint64_t* leaves; /* canonical order */
  size_t nleaves;
};

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

static long find_node(const tmo_tree* t, uint64_t p) {
  size_t lo = 0, hi = t->nnodes;
  while (lo < hi) {
    size_t mid = (lo + hi) / 2;
    if (t->nodes[mid] < p) lo = mid + 1;
    else hi = mid;
  }
  return (lo < t->nnodes && t->nodes[lo] == p) ? (long)lo : -1;
}

/* octree.cpp:52-77 rank: (root raster index, morton dfs rank) */
static const tmo_tree* g_sort_tree;
static void leaf_rank(const tmo_tree* t, uint64_t p, uint64_t* r0, uint64_t* r1) {
  int l = LV(p);
  uint32_t ri = CI(p) >> l, rj = CJ(p) >> l, rk = CK(p) >> l;
  *r0 = ((uint64_t)rk * t->root[1] + rj) * t->root[0] + ri;
  uint64_t mask = (1u << l) - 1, idx = 0;
  tmo_morton_encode(l, CI(p) & mask, CJ(p) & mask, CK(p) & mask, &idx);
  *r1 = tmo_morton_dfs_rank(l, idx);
}
static int cmp_leaf(const void* a, const void* b) {
  uint64_t a0, a1, b0, b1;
  leaf_rank(g_sort_tree, *(const uint64_t*)a, &a0, &a1);
  leaf_rank(g_sort_tree, *(const uint64_t*)b, &b0, &b1);
  if (a0 != b0) return a0 < b0 ? -1 : 1;
  if (a1 != b1) return a1 < b1 ? -1 : 1;
  return 0;
}

tmo_tree* tmo_tree_create(int E, int G, int V, const int* root_dims, const int* bc,
                          const uint64_t* leaves, size_t n) {
  tmo_tree* t = (tmo_tree*)calloc(1, sizeof(tmo_tree));
  t->E = E;
  t->G = G;
  t->V = V;
  for (int a = 0; a < 3; ++a) {
    t->root[a] = root_dims[a];
    t->bc[a] = bc[a];
  }
  size_t cap = 0;
  for (size_t i = 0; i < n; ++i) cap += (size_t)LV(leaves[i]) + 1;
  uint64_t* all = (uint64_t*)malloc(sizeof(uint64_t) * (cap ? cap : 1));
  size_t m = 0;
  for (size_t i = 0; i < n; ++i) {
    uint64_t p = leaves[i];
    for (int l = LV(p); l >= 0; --l) {
      int s = LV(p) - l;
      all[m++] = PK(l, CI(p) >> s, CJ(p) >> s, CK(p) >> s);
    }
  }
  qsort(all, m, sizeof(uint64_t), cmp_u64);
  size_t u = 0;
  for (size_t i = 0; i < m; ++i)
    if (u == 0 || all[u - 1] != all[i]) all[u++] = all[i];
  t->nodes = all;
  t->nnodes = u;
  t->leaf = (unsigned char*)calloc(u ? u : 1, 1);
  for (size_t i = 0; i < n; ++i) t->leaf[find_node(t, leaves[i])] = 1;
  t->leaves = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  memcpy(t->leaves, leaves, sizeof(uint64_t) * n);
  t->nleaves = n;
  g_sort_tree = t;
  qsort(t->leaves, n, sizeof(uint64_t), cmp_leaf);
  return t;
}

void tmo_tree_destroy(tmo_tree* t) {
  if (!t) return;
  free(t->nodes);
  free(t->leaf);
  free(t->leaves);
  free(t);
}

size_t tmo_tree_leaves(const tmo_tree* t, uint64_t* out, size_t cap) {
  for (size_t i = 0; i < t->nleaves && i < cap; ++i) out[i] = t->leaves[i];
  return t->nleaves;
}

/* octree.cpp:79-90 covering_leaf; returns 1 and the leaf, or 0 */
static int covering_leaf(const tmo_tree* t, uint64_t cell, uint64_t* out) {
  int L = LV(cell);
  for (int l = L; l >= 0; --l) {
    int s = L - l;
    uint64_t probe = PK(l, CI(cell) >> s, CJ(cell) >> s, CK(cell) >> s);
    long at = find_node(t, probe);
    if (at >= 0) {
      if (t->leaf[at]) {
        *out = probe;
        return 1;
      }
      return 0;
    }
  }
  return 0;
}

/* octree.cpp:92-132 face_neighbor; kind 0 same, 1 coarser, 2 finer, 3 boundary,
 * -1 topology corrupt */
int tmo_tree_face_neighbor(const tmo_tree* t, uint64_t leaf, int axis, int dir,
                           uint64_t* ids, int* count) {
  int l = LV(leaf);
  int64_t c[3] = {CI(leaf), CJ(leaf), CK(leaf)};
  c[axis] += dir > 0 ? 1 : -1;
  int64_t extent = (int64_t)((uint32_t)t->root[axis] << l);
  *count = 0;
  if (c[axis] < 0 || c[axis] >= extent) {
    if (t->bc[axis]) return 3;
    c[axis] = (c[axis] + extent) % extent;
  }
  uint64_t cell = PK(l, c[0], c[1], c[2]);
  long at = find_node(t, cell);
  if (at >= 0 && !t->leaf[at]) {
    int face_bit = dir > 0 ? 0 : 1;
    int t1 = (axis + 1) % 3, t2 = (axis + 2) % 3;
    for (int b2 = 0; b2 < 2; ++b2)
      for (int b1 = 0; b1 < 2; ++b1) {
        int bits[3];
        bits[axis] = face_bit;
        bits[t1] = b1;
        bits[t2] = b2;
        ids[(*count)++] = PK(l + 1, ((uint32_t)c[0] << 1) | (uint32_t)bits[0],
                             ((uint32_t)c[1] << 1) | (uint32_t)bits[1],
                             ((uint32_t)c[2] << 1) | (uint32_t)bits[2]);
      }
    return 2;
  }
  uint64_t cov;
  if (!covering_leaf(t, cell, &cov)) return -1;
  ids[0] = cov;
  *count = 1;
  return LV(cov) == l ? 0 : 1;
}

/* ghost.cpp:168-210 plan_axis_fills */
size_t tmo_tree_plan(const tmo_tree* t, int axis, int64_t* rows, size_t cap) {
  size_t r = 0;
  for (size_t li = 0; li < t->nleaves; ++li) {
    uint64_t leaf = t->leaves[li];
    for (int d = 0; d < 2; ++d) {
      int dir = d == 0 ? -1 : 1;
      uint64_t ids[4];
      int cnt;
      int kind = tmo_tree_face_neighbor(t, leaf, axis, dir, ids, &cnt);
      int nent = kind == 2 ? 4 : 1;
      for (int q = 0; q < nent; ++q, ++r) {
        if (r >= cap) continue;
        int64_t* o = rows + 7 * r;
        o[0] = (int64_t)leaf;
        o[1] = kind == 3 ? -1 : (int64_t)ids[q];
        o[2] = kind;
        o[3] = axis;
        o[4] = dir;
        if (kind == 1) {
          uint32_t c[3] = {CI(leaf), CJ(leaf), CK(leaf)};
          o[5] = c[(axis + 1) % 3] & 1;
          o[6] = c[(axis + 2) % 3] & 1;
        } else if (kind == 2) {
          o[5] = q & 1; /* qt1 inner loop */
          o[6] = q >> 1;
        } else {
          o[5] = o[6] = 0;
        }
      }
    }
  }
  return r;
}

/* ghost.cpp:26-38 axis_coords */
static inline void axc(int axis, int na, int v1, int v2, int* i, int* j, int* k) {
  int c[3];
  c[axis] = na;
  c[(axis + 1) % 3] = v1;
  c[(axis + 2) % 3] = v2;
  *i = c[0];
  *j = c[1];
  *k = c[2];
}

typedef struct {
  int E, G, V, E2S;
} geo;

static double* gat(double* g, const geo* t, int var, int i, int j, int k) {
  size_t S = (size_t)t->E2S;
  return g + ((size_t)var * S + k) * S * S + (size_t)j * S + i;
}

/* ghost.cpp:40-49 / 55-68 */
static void same_slab(const geo* t, double* src, double* dst, int axis, int dir) {
  const int G = t->G, E = t->E, S = t->E2S;
  int i, j, k;
  for (int var = 0; var < t->V; ++var)
    for (int v2 = 0; v2 < S; ++v2)
      for (int v1 = 0; v1 < S; ++v1)
        for (int q = 0; q < G; ++q) {
          int ns = dir > 0 ? G + q : E + q;
          int nd = dir > 0 ? G + E + q : q;
          axc(axis, ns, v1, v2, &i, &j, &k);
          double v = *gat(src, t, var, i, j, k);
          axc(axis, nd, v1, v2, &i, &j, &k);
          *gat(dst, t, var, i, j, k) = v;
        }
}

/* ghost.cpp:70-96 extract_prolonged_slab (into slab, ghost.cpp order) */
static void extract_prolonged(const geo* t, double* src, int axis, int dir, int qt1, int qt2,
                              double* out) {
  const int G = t->G, E = t->E;
  size_t n = 0;
  int i, j, k, im, jm, km, ip, jp, kp;
  for (int var = 0; var < t->V; ++var)
    for (int f2 = 0; f2 < E; ++f2)
      for (int f1 = 0; f1 < E; ++f1)
        for (int dd = 0; dd < G; ++dd) {
          int cd = dd / 2;
          int sub = dd - 2 * cd;
          int na = dir > 0 ? G + cd : G + E - 1 - cd;
          int ct1 = G + qt1 * (E / 2) + f1 / 2;
          int ct2 = G + qt2 * (E / 2) + f2 / 2;
          axc(axis, na, ct1, ct2, &i, &j, &k);
          axc(axis, na - 1, ct1, ct2, &im, &jm, &km);
          axc(axis, na + 1, ct1, ct2, &ip, &jp, &kp);
          double c = *gat(src, t, var, i, j, k);
          double s = tmo_minmod_scalar(*gat(src, t, var, ip, jp, kp) - c,
                                       c - *gat(src, t, var, im, jm, km));
          double off = 0.25 * s;
          int sign = dir > 0 ? (sub == 0 ? -1 : +1) : (sub == 0 ? +1 : -1);
          out[n++] = sign > 0 ? c + off : c - off;
        }
}

/* ghost.cpp:98-111 */
static void apply_prolonged(const geo* t, double* dst, int axis, int dir, const double* in) {
  const int G = t->G, E = t->E;
  size_t n = 0;
  int i, j, k;
  for (int var = 0; var < t->V; ++var)
    for (int f2 = 0; f2 < E; ++f2)
      for (int f1 = 0; f1 < E; ++f1)
        for (int dd = 0; dd < G; ++dd) {
          int na = dir > 0 ? G + E + dd : G - 1 - dd;
          axc(axis, na, G + f1, G + f2, &i, &j, &k);
          *gat(dst, t, var, i, j, k) = in[n++];
        }
}

/* ghost.cpp:113-149 restricted extract + apply */
static void restricted_slab(const geo* t, double* src, double* dst, int axis, int dir,
                            int qt1, int qt2) {
  const int G = t->G, E = t->E;
  int i, j, k;
  for (int var = 0; var < t->V; ++var)
    for (int c2 = 0; c2 < E / 2; ++c2)
      for (int c1 = 0; c1 < E / 2; ++c1)
        for (int dd = 0; dd < G; ++dd) {
          double acc = 0.0;
          for (int dn = 0; dn < 2; ++dn)
            for (int d1 = 0; d1 < 2; ++d1)
              for (int d2 = 0; d2 < 2; ++d2) {
                int fn = dir > 0 ? G + 2 * dd + dn : G + E - 1 - (2 * dd + dn);
                axc(axis, fn, G + 2 * c1 + d1, G + 2 * c2 + d2, &i, &j, &k);
                acc += *gat(src, t, var, i, j, k);
              }
          double v = acc * 0.125;
          int na = dir > 0 ? G + E + dd : G - 1 - dd;
          axc(axis, na, G + qt1 * (E / 2) + c1, G + qt2 * (E / 2) + c2, &i, &j, &k);
          *gat(dst, t, var, i, j, k) = v;
        }
}

/* ghost.cpp:151-166 */
static void reflective(const geo* t, double* g, int axis, int dir, int nmv) {
  const int G = t->G, E = t->E, S = t->E2S;
  int gi, gj, gk, ii, ij, ik;
  for (int var = 0; var < t->V; ++var) {
    double sign = var == nmv ? -1.0 : 1.0;
    for (int v2 = 0; v2 < S; ++v2)
      for (int v1 = 0; v1 < S; ++v1)
        for (int dd = 0; dd < G; ++dd) {
          int ng = dir > 0 ? G + E + dd : G - 1 - dd;
          int ni = dir > 0 ? G + E - 1 - dd : G + dd;
          axc(axis, ng, v1, v2, &gi, &gj, &gk);
          axc(axis, ni, v1, v2, &ii, &ij, &ik);
          *gat(g, t, var, gi, gj, gk) = sign * *gat(g, t, var, ii, ij, ik);
        }
  }
}

static long leaf_index(const tmo_tree* t, uint64_t p) {
  for (size_t i = 0; i < t->nleaves; ++i)
    if (t->leaves[i] == p) return (long)i;
  return -1;
}

/* ghost.cpp:282-296 fill_ghosts_sync: per axis, stage every prolonged slab,
 * then apply all fills in plan order. */
int tmo_fill_ghosts_sync(const tmo_tree* t, double** grids) {
  geo g = {t->E, t->G, t->V, t->E + 2 * t->G};
  size_t cap = 16 * t->nleaves + 16;
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * 7 * cap);
  long* dsti = (long*)malloc(sizeof(long) * cap);
  long* srci = (long*)malloc(sizeof(long) * cap);
  size_t pslab = (size_t)t->V * t->G * t->E * t->E;
  for (int axis = 0; axis < 3; ++axis) {
    size_t n = tmo_tree_plan(t, axis, rows, cap);
    double* staged = (double*)malloc(sizeof(double) * pslab * (n ? n : 1));
    for (size_t r = 0; r < n; ++r) {
      const int64_t* o = rows + 7 * r;
      dsti[r] = leaf_index(t, (uint64_t)o[0]);
      srci[r] = o[1] >= 0 ? leaf_index(t, (uint64_t)o[1]) : -1;
      if (o[2] == 1)
        extract_prolonged(&g, grids[srci[r]], axis, (int)o[4], (int)o[5], (int)o[6],
                          staged + r * pslab);
    }
    for (size_t r = 0; r < n; ++r) {
      const int64_t* o = rows + 7 * r;
      double* dst = grids[dsti[r]];
      int dir = (int)o[4];
      switch (o[2]) {
        case 3:
          reflective(&g, dst, axis, dir, t->V == 5 ? 1 + axis : -1);
          break;
        case 1:
          apply_prolonged(&g, dst, axis, dir, staged + r * pslab);
          break;
        case 0:
          same_slab(&g, grids[srci[r]], dst, axis, dir);
          break;
        case 2:
          restricted_slab(&g, grids[srci[r]], dst, axis, dir, (int)o[5], (int)o[6]);
          break;
        default:
          free(staged);
          free(rows);
          free(dsti);
          free(srci);
          return 1;
      }
    }
    free(staged);
  }
  free(rows);
  free(dsti);
  free(srci);
  return 0;
}

/* octree.cpp:306-323 flag_refinement (density = var 0) */
int tmo_flag_refinement(const tmo_tree* t, const double* grid, double theta, double rho_floor) {
  geo g = {t->E, t->G, t->V, t->E + 2 * t->G};
  double* gg = (double*)grid;
  const int G = t->G, E = t->E;
  for (int k = G; k < G + E; ++k)
    for (int j = G; j < G + E; ++j)
      for (int i = G; i < G + E; ++i) {
        double gx = 0.5 * (*gat(gg, &g, 0, i + 1, j, k) - *gat(gg, &g, 0, i - 1, j, k));
        double gy = 0.5 * (*gat(gg, &g, 0, i, j + 1, k) - *gat(gg, &g, 0, i, j - 1, k));
        double gz = 0.5 * (*gat(gg, &g, 0, i, j, k + 1) - *gat(gg, &g, 0, i, j, k - 1));
        double mag = sqrt(gx * gx + gy * gy + gz * gz);
        double rho = stdmax_(*gat(gg, &g, 0, i, j, k), rho_floor);
        if (mag / rho > theta) return 1;
      }
  return 0;
}

/* Reflux at refinement jumps — our restatement (parity unpinned): the
 * reference declares FluxRegister (proj/include/taskmesh/amr/flux_register.hpp:
 * 21-63) without a definition; SPEC.md:383-391 gives the correction
 * (sum fine_flux*fine_area - coarse_flux*coarse_area)*dt/volume, the header
 * the sign -dir, the weight w = stage coefficient * dt, the 2x2 arithmetic
 * mean (restrict_face) and the sorted (leaf, axis, dir) application order.
 * faces[l]: leaf l's stage face-flux blocks [6][V][E^2] (stage.hpp:8-12,
 * block 2*axis+side, entry var*E^2 + c2*E + c1); dx[l] its cell size.
 * grids: ghosted leaf states after the stage (and its RK combine). */
int tmo_reflux_apply(const tmo_tree* t, double** grids, double* const* faces, int E, int G, int V,
                     const double* dx, double dt, double coef) {
  const int S = E + 2 * G, E2 = E * E, H = E / 2;
  const double w = coef * dt;
  for (size_t li = 0; li < t->nleaves; ++li) {
    const double cw = w / dx[li];
    for (int axis = 0; axis < 3; ++axis)
      for (int d = 0; d < 2; ++d) {
        const int dir = d == 0 ? -1 : 1;
        uint64_t ids[4];
        int cnt;
        if (tmo_tree_face_neighbor(t, t->leaves[li], axis, dir, ids, &cnt) != 2) continue;
        long fl[4];
        for (int q = 0; q < 4; ++q) {
          fl[q] = leaf_index(t, ids[q]);
          if (fl[q] < 0) return -1;
        }
        const int side_c = dir > 0 ? 1 : 0, side_f = 1 - side_c;
        for (int v = 0; v < V; ++v)
          for (int c2 = 0; c2 < E; ++c2)
            for (int c1 = 0; c1 < E; ++c1) {
              const double* Ff = faces[fl[(c2 / H) * 2 + c1 / H]] + (size_t)((2 * axis + side_f) * V + v) * E2;
              const int f1 = 2 * (c1 % H), f2 = 2 * (c2 % H);
              const double mean = (((Ff[f2 * E + f1] + Ff[f2 * E + f1 + 1]) + Ff[(f2 + 1) * E + f1]) +
                                   Ff[(f2 + 1) * E + f1 + 1]) * 0.25;
              const double coarse = faces[li][(size_t)((2 * axis + side_c) * V + v) * E2 + c2 * E + c1];
              const double delta = mean - coarse;
              int x[3];
              x[axis] = side_c ? E - 1 : 0;
              x[(axis + 1) % 3] = c1;
              x[(axis + 2) % 3] = c2;
              double* u = grids[li] + (((size_t)v * S + x[2] + G) * S + x[1] + G) * S + x[0] + G;
              *u = dir > 0 ? *u - cw * delta : *u + cw * delta;
            }
      }
  }
  return 0;
}
