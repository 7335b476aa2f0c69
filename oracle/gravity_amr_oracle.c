/* TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * Plain-C restatement of OUR adaptive (AMR) extension of the cell-level FMM
 * gravity specification. PARITY UNPINNED w.r.t. the reference:
 * the reference has no gravity code (prose only, PAPER.md:120,233,
 * 238,241,347). csrc/gravity_amr.cu must equal this file bitwise
 * (-ffp-contract=off / -fmad=false); the file itself is checked against direct
 * O(N^2) summation, momentum conservation, and (on a uniform forest) against
 * the uniform specification tmo_grav_solve, bit for bit.
 *
 * Geometry: one root = the unit cube, isolated boundaries, G = 1. A forest
 * leaf at level l with node coordinates (I,J,K) holds 8^3 cells at cell depth
 * d = l + 3, cell (i,j,k) at global coordinates (8I+i, 8J+j, 8K+k) with centre
 * ((gi + 0.5) h_d, ...), h_d = 2^-d. The cell tree over depths 0..Dmax has a
 * cell of depth d "internal" when finer leaves cover it, "leaf" when it is a
 * cell of a forest leaf, missing otherwise (covered by a coarser leaf cell).
 *
 * The algorithm is the classic adaptive FMM (U, V, W, X lists) over that cell
 * tree with the uniform specification's operators (order-2 Cartesian moments,
 * Dehnen-truncated M2L, L2L, monopole P2P):
 *   P2M   leaf cells: (m, 0, 0)
 *   M2M   internal cells from their 8 children, (c, b, a) loop order
 *   V     every existing cell at depth >= 2: the 189-cell stencil of the
 *         uniform spec (two partial sums over the lower / upper three source
 *         planes, dz, dy ascending, per row even source x then odd, then
 *         added), skipping missing/outside cells
 *   W, X  for every leaf cell b (canonical leaf order, cells (k,j,i)), every
 *         internal colleague Y (same depth, max|offset| = 1, dz,dy,dx
 *         ascending) is visited: each child y (z,y,x order) adjacent to b
 *         (closed boxes touch) is a leaf -> U pair (b, y), or internal ->
 *         visited in turn; a child not adjacent to b -> W(b) += y and
 *         X(y) += b. W and X entries are M2L terms (R = x_target - x_source).
 *   order L(t) = V-sum, then + each W/X entry of t sorted by source
 *         (depth, gk, gj, gi) ascending, then L = shift(L(parent)) + L
 *   L2P   leaf cells: phi = L0, g = -L_i; then P2P with the 26 same-depth
 *         leaf neighbours (dz, dy, dx ascending), then the cross-depth U
 *         pairs of the cell sorted by source (depth, gk, gj, gi)
 *   AM    optional (flag 1): angular-momentum correction, see
 *         tmo_grav_am_correct below.
 * On a uniform forest no W/X/U-cross pairs exist and every step is the
 * uniform specification's, so both solvers agree bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "tm_oracle.h"

static inline long cix(long n, long i, long j, long k) { return (k * n + j) * n + i; }

typedef struct {
  long n;         /* cells per axis = 2^d */
  uint8_t* type;  /* 0 missing, 1 internal, 2 leaf */
  double* mom;    /* [n^3][10] */
  double* loc;    /* [n^3][10] */
  long* out;      /* leaf cell -> output index (slot*512 + c), else -1 */
} GDepth;

typedef struct {
  int kind; /* 0 = M2L (W/X), 1 = P2P (U cross-depth) */
  int td;
  long tidx;
  int sd;
  long si, sj, sk;
} GEnt;

typedef struct {
  GEnt* e;
  size_t n, cap;
  int err;
} GList;

static void push(GList* L, int kind, int td, long tidx, int sd, long si, long sj, long sk) {
  if (L->n == L->cap) {
    size_t nc = L->cap ? 2 * L->cap : 1024;
    GEnt* p = (GEnt*)realloc(L->e, nc * sizeof(GEnt));
    if (!p) {
      L->err = 1;
      return;
    }
    L->e = p;
    L->cap = nc;
  }
  GEnt* x = &L->e[L->n++];
  x->kind = kind;
  x->td = td;
  x->tidx = tidx;
  x->sd = sd;
  x->si = si;
  x->sj = sj;
  x->sk = sk;
}

static int ent_cmp(const void* pa, const void* pb) {
  const GEnt* a = (const GEnt*)pa;
  const GEnt* b = (const GEnt*)pb;
#define CMP(f) \
  if (a->f != b->f) return a->f < b->f ? -1 : 1;
  CMP(kind) CMP(td) CMP(tidx) CMP(sd) CMP(sk) CMP(sj) CMP(si)
#undef CMP
  return 0;
}

/* closed boxes of cell A (depth da, coords a) and cell B (depth db >= da) touch */
static int touches(int da, const long* a, int db, const long* b) {
  const int s = db - da;
  for (int q = 0; q < 3; ++q) {
    const long lo = a[q] << s, hi = (a[q] + 1) << s;
    if (!(b[q] <= hi && b[q] + 1 >= lo)) return 0;
  }
  return 1;
}

static void visit(GDepth* dep, GList* L, int db, const long* b, long bidx, int dy, const long* Y) {
  const long n = dep[dy + 1].n;
  for (int c = 0; c < 2; ++c)
    for (int bb = 0; bb < 2; ++bb)
      for (int a = 0; a < 2; ++a) {
        const long y[3] = {2 * Y[0] + a, 2 * Y[1] + bb, 2 * Y[2] + c};
        const long yidx = cix(n, y[0], y[1], y[2]);
        const uint8_t t = dep[dy + 1].type[yidx];
        if (touches(db, b, dy + 1, y)) {
          if (t == 2) {
            push(L, 1, db, bidx, dy + 1, y[0], y[1], y[2]);
            push(L, 1, dy + 1, yidx, db, b[0], b[1], b[2]);
          } else if (t == 1) {
            visit(dep, L, db, b, bidx, dy + 1, y);
          } else {
            L->err = 2;
          }
        } else {
          push(L, 0, db, bidx, dy + 1, y[0], y[1], y[2]);
          push(L, 0, dy + 1, yidx, db, b[0], b[1], b[2]);
        }
      }
}

/* flags & 2 (tests): "count mode" — every M2L adds the source's mass to L0
 * and every P2P adds 1 to phi, so with unit masses phi counts the leaf cells
 * each leaf cell interacted with: exactly n - 1 iff every pair is covered once. */
static void m2l_k(const double* mom, const double* R, double* out, int cnt) {
  if (cnt)
    out[0] += mom[0];
  else
    tmo_grav_m2l(mom, R, out);
}

static inline double centre(long gi, int d) { return ((double)gi + 0.5) / (double)(1L << d); }

/* Angular-momentum correction (our specification of PAPER.md:233's "special
 * technique"; the paper does not define it): the truncated M2L forces are
 * exactly opposite but not central, so the total torque sum r x m g is not
 * zero. The correction adds the rigid-rotation field w x (x - R) about the
 * centre of mass R with J w = -tau (J the inertia tensor of the leaf-cell
 * point masses about R, tau the torque about R): afterwards the total torque
 * is zero and the total force is unchanged (sum m (x - R) = 0) to round-off.
 * Sums: 16 per-cell values, reduced by an adjacent-pair binary tree over the
 * cells in output order (slot-major, 512 per slot), the slot count padded with
 * zeros to a power of two. nslots leaves; x, y, z: cell centres. */
static void am_values(double m, double x, double y, double z, double gx, double gy, double gz,
                      double* v) {
  v[0] = m;
  v[1] = m * x;
  v[2] = m * y;
  v[3] = m * z;
  v[4] = m * gx;
  v[5] = m * gy;
  v[6] = m * gz;
  v[7] = m * (y * gz - z * gy);
  v[8] = m * (z * gx - x * gz);
  v[9] = m * (x * gy - y * gx);
  v[10] = v[1] * x;
  v[11] = v[1] * y;
  v[12] = v[1] * z;
  v[13] = v[2] * y;
  v[14] = v[2] * z;
  v[15] = v[3] * z;
}

/* S[16] sums -> R[3], w[3] */
void tmo_grav_am_solve(const double* S, double* R, double* w) {
  const double M = S[0];
  R[0] = S[1] / M;
  R[1] = S[2] / M;
  R[2] = S[3] / M;
  const double F[3] = {S[4], S[5], S[6]};
  const double tau[3] = {S[7] - (R[1] * F[2] - R[2] * F[1]), S[8] - (R[2] * F[0] - R[0] * F[2]),
                         S[9] - (R[0] * F[1] - R[1] * F[0])};
  const double cxx = S[10] - (M * R[0]) * R[0], cxy = S[11] - (M * R[0]) * R[1],
               cxz = S[12] - (M * R[0]) * R[2], cyy = S[13] - (M * R[1]) * R[1],
               cyz = S[14] - (M * R[1]) * R[2], czz = S[15] - (M * R[2]) * R[2];
  const double tr = (cxx + cyy) + czz;
  const double j00 = tr - cxx, j11 = tr - cyy, j22 = tr - czz, j01 = -cxy, j02 = -cxz, j12 = -cyz;
  const double a00 = j11 * j22 - j12 * j12, a01 = j02 * j12 - j01 * j22, a02 = j01 * j12 - j02 * j11,
               a11 = j00 * j22 - j02 * j02, a12 = j01 * j02 - j00 * j12, a22 = j00 * j11 - j01 * j01;
  const double det = (j00 * a00 + j01 * a01) + j02 * a02;
  if (!(det > 0.0)) {
    w[0] = w[1] = w[2] = 0.0;
    return;
  }
  const double b0 = -tau[0], b1 = -tau[1], b2 = -tau[2];
  w[0] = ((a00 * b0 + a01 * b1) + a02 * b2) / det;
  w[1] = ((a01 * b0 + a11 * b1) + a12 * b2) / det;
  w[2] = ((a02 * b0 + a12 * b1) + a22 * b2) / det;
}

/* adjacent-pair tree reduction of v[n][16] (n a power of two) into S[16] */
static void pair_tree(double* v, long n, double* S) {
  for (long s = 1; s < n; s <<= 1)
    for (long c = 0; c + s < n; c += 2 * s)
      for (int q = 0; q < 16; ++q) v[c * 16 + q] = v[c * 16 + q] + v[(c + s) * 16 + q];
  for (int q = 0; q < 16; ++q) S[q] = v[q];
}

/* leaves: [n][4] = (level, I, J, K); mass [n][512]; pos [n*512][3] centres.
 * Applies the correction to g ([3][n*512]). Returns the sums in S (optional). */
int tmo_grav_am_correct(long nleaves, const double* mass, const double* pos, double* g,
                        double* S_out, double* w_out) {
  long P = 1;
  while (P < nleaves) P <<= 1;
  const long ncell = nleaves * 512, npad = P * 512;
  double* v = (double*)calloc((size_t)npad * 16, sizeof(double));
  if (!v) return -1;
  for (long c = 0; c < ncell; ++c)
    am_values(mass[c], pos[3 * c], pos[3 * c + 1], pos[3 * c + 2], g[c], g[ncell + c],
              g[2 * ncell + c], v + c * 16);
  double S[16], R[3], w[3];
  pair_tree(v, npad, S);
  free(v);
  tmo_grav_am_solve(S, R, w);
  for (long c = 0; c < ncell; ++c) {
    const double dx = pos[3 * c] - R[0], dy = pos[3 * c + 1] - R[1], dz = pos[3 * c + 2] - R[2];
    g[c] = g[c] + (w[1] * dz - w[2] * dy);
    g[ncell + c] = g[ncell + c] + (w[2] * dx - w[0] * dz);
    g[2 * ncell + c] = g[2 * ncell + c] + (w[0] * dy - w[1] * dx);
  }
  if (S_out) memcpy(S_out, S, sizeof(S));
  if (w_out) memcpy(w_out, w, sizeof(w));
  return 0;
}

static void free_depths(GDepth* dep, int Dmax) {
  for (int d = 0; d <= Dmax; ++d) {
    free(dep[d].type);
    free(dep[d].mom);
    free(dep[d].loc);
    free(dep[d].out);
  }
}

/* Returns 0; -1 out of memory / too deep; -2 leaves do not tile the cube.
 * counts (optional): [0] W/X entries, [1] U-cross entries (both directions). */
int tmo_grav_amr_solve_ex(long nleaves, const int* leaves, const double* mass, int flags,
                          double* phi, double* g, long* counts) {
  const int cnt = (flags & 2) != 0;
  int Dmax = 0;
  for (long s = 0; s < nleaves; ++s)
    if (leaves[4 * s] + 3 > Dmax) Dmax = leaves[4 * s] + 3;
  if (Dmax > 8) return -1;
  GDepth dep[9];
  memset(dep, 0, sizeof(dep));
  for (int d = 0; d <= Dmax; ++d) {
    const long n = 1L << d, n3 = n * n * n;
    dep[d].n = n;
    dep[d].type = (uint8_t*)calloc((size_t)n3, 1);
    dep[d].mom = (double*)calloc((size_t)n3 * 10, sizeof(double));
    dep[d].loc = (double*)calloc((size_t)n3 * 10, sizeof(double));
    dep[d].out = (long*)malloc((size_t)n3 * sizeof(long));
    if (!dep[d].type || !dep[d].mom || !dep[d].loc || !dep[d].out) {
      free_depths(dep, Dmax);
      return -1;
    }
    for (long c = 0; c < n3; ++c) dep[d].out[c] = -1;
  }
  /* P2M + cell types */
  for (long s = 0; s < nleaves; ++s) {
    const int d = leaves[4 * s] + 3;
    const long n = dep[d].n;
    for (int c = 0; c < 512; ++c) {
      const long gi = 8L * leaves[4 * s + 1] + (c & 7), gj = 8L * leaves[4 * s + 2] + ((c >> 3) & 7),
                 gk = 8L * leaves[4 * s + 3] + (c >> 6);
      if (gi >= n || gj >= n || gk >= n) {
        free_depths(dep, Dmax);
        return -2;
      }
      const long idx = cix(n, gi, gj, gk);
      if (dep[d].type[idx]) {
        free_depths(dep, Dmax);
        return -2;
      }
      dep[d].type[idx] = 2;
      dep[d].out[idx] = s * 512 + c;
      dep[d].mom[idx * 10] = cnt ? 1.0 : mass[s * 512 + c];
      for (int dd = d - 1; dd >= 0; --dd) {
        const int sh = d - dd;
        uint8_t* t = &dep[dd].type[cix(dep[dd].n, gi >> sh, gj >> sh, gk >> sh)];
        if (*t == 2) {
          free_depths(dep, Dmax);
          return -2;
        }
        *t = 1;
      }
    }
  }
  for (int d = 0; d < Dmax; ++d) { /* every internal cell has 8 existing children */
    const long n = dep[d].n;
    for (long k = 0; k < n; ++k)
      for (long j = 0; j < n; ++j)
        for (long i = 0; i < n; ++i) {
          if (dep[d].type[cix(n, i, j, k)] != 1) continue;
          for (int q = 0; q < 8; ++q)
            if (!dep[d + 1].type[cix(2 * n, 2 * i + (q & 1), 2 * j + ((q >> 1) & 1), 2 * k + (q >> 2))]) {
              free_depths(dep, Dmax);
              return -2;
            }
        }
  }
  if (!dep[0].type[0]) {
    free_depths(dep, Dmax);
    return -2;
  }
  /* M2M */
  for (int d = Dmax - 1; d >= 0; --d) {
    const long n = dep[d].n;
    const double hc = 1.0 / (double)dep[d + 1].n;
#pragma omp parallel for schedule(dynamic, 1)
    for (long K = 0; K < n; ++K)
      for (long J = 0; J < n; ++J)
        for (long I = 0; I < n; ++I) {
          if (dep[d].type[cix(n, I, J, K)] != 1) continue;
          double* out = dep[d].mom + cix(n, I, J, K) * 10;
          for (int c = 0; c < 2; ++c)
            for (int b = 0; b < 2; ++b)
              for (int a = 0; a < 2; ++a) {
                const double s[3] = {(a - 0.5) * hc, (b - 0.5) * hc, (c - 0.5) * hc};
                tmo_grav_m2m(dep[d + 1].mom + cix(2 * n, 2 * I + a, 2 * J + b, 2 * K + c) * 10, s, out);
              }
        }
  }
  /* V lists */
  for (int d = 2; d <= Dmax; ++d) {
    const long m = dep[d].n;
    const double h = 1.0 / (double)m;
#pragma omp parallel for schedule(dynamic, 1)
    for (long k = 0; k < m; ++k)
      for (long j = 0; j < m; ++j)
        for (long i = 0; i < m; ++i) {
          if (!dep[d].type[cix(m, i, j, k)]) continue;
          double* out = dep[d].loc + cix(m, i, j, k) * 10;
          double part[2][10] = {{0}};  /* lower / upper three source planes */
          for (long dz = -2 - (k & 1); dz <= 3 - (k & 1); ++dz)
            for (long dy = -2 - (j & 1); dy <= 3 - (j & 1); ++dy)
              for (int pe = 0; pe < 2; ++pe)  /* even source x, then odd */
              for (long dx = -2 - (i & 1) + pe; dx <= 3 - (i & 1); dx += 2) {
                if (labs(dx) <= 1 && labs(dy) <= 1 && labs(dz) <= 1) continue;
                const long si = i + dx, sj = j + dy, sk = k + dz;
                if (si < 0 || sj < 0 || sk < 0 || si >= m || sj >= m || sk >= m) continue;
                if (!dep[d].type[cix(m, si, sj, sk)]) continue;
                const double R[3] = {-(double)dx * h, -(double)dy * h, -(double)dz * h};
                m2l_k(dep[d].mom + cix(m, si, sj, sk) * 10, R, part[dz + (k & 1) >= 1], cnt);
              }
          for (int q = 0; q < 10; ++q) out[q] = part[0][q] + part[1][q];
        }
  }
  /* W / X / U-cross lists */
  GList L = {0, 0, 0, 0};
  for (long s = 0; s < nleaves; ++s) {
    const int d = leaves[4 * s] + 3;
    const long n = dep[d].n;
    for (int c = 0; c < 512; ++c) {
      const long b[3] = {8L * leaves[4 * s + 1] + (c & 7), 8L * leaves[4 * s + 2] + ((c >> 3) & 7),
                         8L * leaves[4 * s + 3] + (c >> 6)};
      const long bidx = cix(n, b[0], b[1], b[2]);
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            if (!dx && !dy && !dz) continue;
            const long Y[3] = {b[0] + dx, b[1] + dy, b[2] + dz};
            if (Y[0] < 0 || Y[1] < 0 || Y[2] < 0 || Y[0] >= n || Y[1] >= n || Y[2] >= n) continue;
            if (dep[d].type[cix(n, Y[0], Y[1], Y[2])] == 1) visit(dep, &L, d, b, bidx, d, Y);
          }
    }
  }
  if (L.err) {
    free(L.e);
    free_depths(dep, Dmax);
    return L.err == 1 ? -1 : -2;
  }
  qsort(L.e, L.n, sizeof(GEnt), ent_cmp);
  if (counts) {
    counts[0] = counts[1] = 0;
    for (size_t q = 0; q < L.n; ++q) ++counts[L.e[q].kind];
  }
  for (size_t q = 0; q < L.n; ++q) { /* M2L entries (sorted, kind 0 first) */
    const GEnt* x = &L.e[q];
    if (x->kind != 0) break;
    const long tn = dep[x->td].n;
    const long ti = x->tidx % tn, tj = (x->tidx / tn) % tn, tk = x->tidx / (tn * tn);
    const double R[3] = {centre(ti, x->td) - centre(x->si, x->sd), centre(tj, x->td) - centre(x->sj, x->sd),
                         centre(tk, x->td) - centre(x->sk, x->sd)};
    m2l_k(dep[x->sd].mom + cix(dep[x->sd].n, x->si, x->sj, x->sk) * 10, R,
          dep[x->td].loc + x->tidx * 10, cnt);
  }
  /* L2L */
  for (int d = 3; d <= Dmax; ++d) {
    const long m = dep[d].n;
    const double h = 1.0 / (double)m;
#pragma omp parallel for schedule(dynamic, 1)
    for (long k = 0; k < m; ++k)
      for (long j = 0; j < m; ++j)
        for (long i = 0; i < m; ++i) {
          if (!dep[d].type[cix(m, i, j, k)]) continue;
          const double s[3] = {((i & 1) - 0.5) * h, ((j & 1) - 0.5) * h, ((k & 1) - 0.5) * h};
          double sh[10];
          tmo_grav_l2l(dep[d - 1].loc + cix(dep[d - 1].n, i >> 1, j >> 1, k >> 1) * 10, s, sh);
          double* out = dep[d].loc + cix(m, i, j, k) * 10;
          for (int q = 0; q < 10; ++q) out[q] = sh[q] + out[q];
        }
  }
  /* L2P + same-depth P2P */
  const long ncell = nleaves * 512;
#pragma omp parallel for schedule(dynamic, 4)
  for (long s = 0; s < nleaves; ++s) {
    const int d = leaves[4 * s] + 3;
    const long N = dep[d].n;
    const double h = 1.0 / (double)N;
    for (int c = 0; c < 512; ++c) {
      const long i = 8L * leaves[4 * s + 1] + (c & 7), j = 8L * leaves[4 * s + 2] + ((c >> 3) & 7),
                 k = 8L * leaves[4 * s + 3] + (c >> 6);
      const double* Lc = dep[d].loc + cix(N, i, j, k) * 10;
      double p = Lc[0], gx = -Lc[1], gy = -Lc[2], gz = -Lc[3];
      for (long dz = -1; dz <= 1; ++dz)
        for (long dy = -1; dy <= 1; ++dy)
          for (long dx = -1; dx <= 1; ++dx) {
            if (!dx && !dy && !dz) continue;
            const long si = i + dx, sj = j + dy, sk = k + dz;
            if (si < 0 || sj < 0 || sk < 0 || si >= N || sj >= N || sk >= N) continue;
            if (dep[d].type[cix(N, si, sj, sk)] != 2) continue;
            if (cnt) {
              p += 1.0;
              continue;
            }
            const double nm = -dep[d].mom[cix(N, si, sj, sk) * 10];
            double w[4];
            tmo_grav_p2p_geom(-(double)dx * h, -(double)dy * h, -(double)dz * h, w);
            p = fma(nm, w[0], p);
            gx = fma(nm, w[1], gx);
            gy = fma(nm, w[2], gy);
            gz = fma(nm, w[3], gz);
          }
      const long o = s * 512 + c;
      phi[o] = p;
      g[o] = gx;
      g[ncell + o] = gy;
      g[2 * ncell + o] = gz;
    }
  }
  /* cross-depth U pairs */
  for (size_t q = 0; q < L.n; ++q) {
    const GEnt* x = &L.e[q];
    if (x->kind != 1) continue;
    const long tn = dep[x->td].n;
    const long ti = x->tidx % tn, tj = (x->tidx / tn) % tn, tk = x->tidx / (tn * tn);
    const long o = dep[x->td].out[x->tidx];
    if (cnt) {
      phi[o] += 1.0;
      continue;
    }
    const double nm = -dep[x->sd].mom[cix(dep[x->sd].n, x->si, x->sj, x->sk) * 10];
    double w[4];
    tmo_grav_p2p_geom(centre(ti, x->td) - centre(x->si, x->sd), centre(tj, x->td) - centre(x->sj, x->sd),
                      centre(tk, x->td) - centre(x->sk, x->sd), w);
    phi[o] = fma(nm, w[0], phi[o]);
    g[o] = fma(nm, w[1], g[o]);
    g[ncell + o] = fma(nm, w[2], g[ncell + o]);
    g[2 * ncell + o] = fma(nm, w[3], g[2 * ncell + o]);
  }
  free(L.e);
  free_depths(dep, Dmax);
  if (flags & 1) {
    double* pos = (double*)malloc((size_t)ncell * 3 * sizeof(double));
    if (!pos) return -1;
    for (long s = 0; s < nleaves; ++s) {
      const int d = leaves[4 * s] + 3;
      for (int c = 0; c < 512; ++c) {
        double* x = pos + (s * 512 + c) * 3;
        x[0] = centre(8L * leaves[4 * s + 1] + (c & 7), d);
        x[1] = centre(8L * leaves[4 * s + 2] + ((c >> 3) & 7), d);
        x[2] = centre(8L * leaves[4 * s + 3] + (c >> 6), d);
      }
    }
    const int r = tmo_grav_am_correct(nleaves, mass, pos, g, NULL, NULL);
    free(pos);
    if (r) return r;
  }
  return 0;
}

int tmo_grav_amr_solve(long nleaves, const int* leaves, const double* mass, int flags, double* phi,
                       double* g) {
  return tmo_grav_amr_solve_ex(nleaves, leaves, mass, flags, phi, g, NULL);
}

/* Direct summation over all leaf-cell pairs (accuracy reference). */
int tmo_grav_amr_direct(long nleaves, const int* leaves, const double* mass, double* phi, double* g) {
  const long n = nleaves * 512;
  double* pos = (double*)malloc((size_t)n * 3 * sizeof(double));
  if (!pos) return -1;
  for (long s = 0; s < nleaves; ++s) {
    const int d = leaves[4 * s] + 3;
    for (int c = 0; c < 512; ++c) {
      double* x = pos + (s * 512 + c) * 3;
      x[0] = centre(8L * leaves[4 * s + 1] + (c & 7), d);
      x[1] = centre(8L * leaves[4 * s + 2] + ((c >> 3) & 7), d);
      x[2] = centre(8L * leaves[4 * s + 3] + (c >> 6), d);
    }
  }
  for (long t = 0; t < n; ++t) {
    double p = 0, gx = 0, gy = 0, gz = 0;
    for (long s = 0; s < n; ++s) {
      if (s == t) continue;
      const double Rx = pos[3 * t] - pos[3 * s], Ry = pos[3 * t + 1] - pos[3 * s + 1],
                   Rz = pos[3 * t + 2] - pos[3 * s + 2];
      const double ir = 1.0 / sqrt(Rx * Rx + Ry * Ry + Rz * Rz);
      const double ir3 = ir * ir * ir;
      p -= mass[s] * ir;
      gx -= mass[s] * Rx * ir3;
      gy -= mass[s] * Ry * ir3;
      gz -= mass[s] * Rz * ir3;
    }
    phi[t] = p;
    g[t] = gx;
    g[n + t] = gy;
    g[2 * n + t] = gz;
  }
  free(pos);
  return 0;
}
