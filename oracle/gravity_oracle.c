/* TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * Plain-C restatement of OUR cell-level FMM gravity specification (DESIGN.md
 * §7). PARITY UNPINNED w.r.t. the reference: the reference mini-app has no
 * gravity code at all (SPEC.md:8 puts "the FMM gravity solver and its
 * angular-momentum-conserving modification" out of scope; only prose exists:
 * PAPER.md:120,233,238,241,347). This file is the specification the GPU
 * kernels must match bitwise (same operation order, -ffp-contract=off); it is
 * itself checked against direct O(N^2) summation (tmo_grav_direct) for
 * accuracy and against momentum conservation by tests/test_gravity.py.
 *
 * Specification (uniform cell level D, N = 2^D cells per axis, unit box,
 * isolated boundaries, G = 1, cell (i,j,k) centre ((i+.5)h, (j+.5)h, (k+.5)h)):
 *   masses   m = rho * h^3 at the finest level (monopoles at cell centres)
 *   M2M      parent moments (M, D_i, Q_ij about the parent centre) from its 8
 *            children in (c, b, a) = (z, y, x) loop order, x fastest
 *   M2L      at every level l >= 2, target cell c sums over the cells c' whose
 *            parent is one of the 27 neighbours of parent(c) but with
 *            max|c - c'| >= 2 (the 189-cell interaction list), loops dz, dy
 *            ascending and in each row the sources with even x first, then odd
 *            (dx ascending within each), as two partial sums — sources in the lower three planes
 *            (z' < 2 (z >> 1) + 1) and in the upper three — added at the end
 *            (the GPU gives each half its own thread); R = x_c - x_c';
 *            order-2 Cartesian multipoles -> local
 *            Taylor coefficients truncated at |alpha| + |beta| <= 2 (Dehnen):
 *              L0   = -(M/r - D_i D1_i + Q_ij D2_ij / 2)
 *              L_i  = -(M D1_i - D_j D2_ij)
 *              L_ij = -(M D2_ij)
 *            With this truncation the mutual M2L forces of every pair are
 *            exactly opposite, so the FMM conserves linear momentum
 *             to round-off. Arithmetic: geometry per separation
 *            (tmo_grav_geom), then a fixed sequence of 27 fused multiply-adds,
 *            one product and one add (tmo_grav_m2l_geom) — C fma() and the GPU's DFMA are the same
 *            correctly rounded operation, so the kernels match bit for bit
 *   L2L      L(c) = shift(L(parent(c))) + M2L-sum(c) (levels 3..D)
 *   L2P+P2P  at the finest level (expansion centre = cell centre, so L2P is
 *            phi = L0, g = -L_i) plus direct monopole sums over the 26
 *            neighbours (dz, dy, dx ascending): phi += -m'/r, g += -m' R/r^3
 *            as fused multiply-adds with the geometry of tmo_grav_p2p_geom
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "tm_oracle.h"

/* symmetric 3x3 index map for the 6 unique components: xx xy xz yy yz zz */
static const int S2[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};

/* Moments: [0] M, [1..3] D, [4..9] Q (xx xy xz yy yz zz). Locals: [0] L0,
 * [1..3] L_i, [4..9] L_ij. */

/* M2L geometry of the separation R = x_target - x_source: e[13] =
 * [ir, D1 x y z, D2 xx xy xz yy yz zz, D2/2 xx yy zz] with D1_i = -R_i/r^3,
 * D2_ij = 3 R_i R_j / r^5 - delta_ij / r^3 (the halving is exact). */
void tmo_grav_geom(const double* R, double* e) {
  const double x = R[0], y = R[1], z = R[2];
  const double r2 = x * x + y * y + z * z;
  const double r = sqrt(r2);
  const double ir = 1.0 / r;
  const double ir2 = ir * ir;
  const double ir3 = ir * ir2, ir5 = ir3 * ir2;
  e[0] = ir;
  for (int i = 0; i < 3; ++i) e[1 + i] = -R[i] * ir3;
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j) e[4 + S2[i][j]] = 3.0 * R[i] * R[j] * ir5 - (i == j ? ir3 : 0.0);
  e[10] = 0.5 * e[4];
  e[11] = 0.5 * e[7];
  e[12] = 0.5 * e[9];
}

/* One M2L term with known geometry, accumulated into out (10 locals):
 *   L0   += t,  t = -M ir + D_i D1_i - (1/2) Q_ij D2_ij, formed on its own
 *          (one product, then a chain of 9 fused multiply-adds) and then added,
 *          so the long L0 chain does not serialise successive terms
 *   L_i  += -M D1_i + D_j D2_ij   (4 fused multiply-adds into L_i)
 *   L_ij += -M D2_ij              (1 fused multiply-add)
 * (Q symmetric: (1/2) Q_ij D2_ij = sum_i Q_ii (D2_ii/2) + sum_{i<j} Q_ij D2_ij). */
void tmo_grav_m2l_geom(const double* mom, const double* e, double* out) {
  const double nM = -mom[0];
  double o = nM * e[0];
  o = fma(mom[1], e[1], o);
  o = fma(mom[2], e[2], o);
  o = fma(mom[3], e[3], o);
  o = fma(-mom[4], e[10], o);
  o = fma(-mom[5], e[5], o);
  o = fma(-mom[6], e[6], o);
  o = fma(-mom[7], e[11], o);
  o = fma(-mom[8], e[8], o);
  o = fma(-mom[9], e[12], o);
  out[0] = out[0] + o;
  for (int i = 0; i < 3; ++i) {
    double t = out[1 + i];
    t = fma(nM, e[1 + i], t);
    for (int j = 0; j < 3; ++j) t = fma(mom[1 + j], e[4 + S2[i][j]], t);
    out[1 + i] = t;
  }
  for (int q = 0; q < 6; ++q) out[4 + q] = fma(nM, e[4 + q], out[4 + q]);
}

void tmo_grav_m2l(const double* mom, const double* R, double* out /* 10, accumulated */) {
  double e[13];
  tmo_grav_geom(R, e);
  tmo_grav_m2l_geom(mom, e, out);
}

/* P2P geometry of R: w[4] = [1/r, R_x/r^3, R_y/r^3, R_z/r^3]; the monopole
 * term is then phi += -m w0, g_i += -m w_i (fused multiply-adds). */
void tmo_grav_p2p_geom(double Rx, double Ry, double Rz, double* w) {
  const double r2 = Rx * Rx + Ry * Ry + Rz * Rz;
  const double ir = 1.0 / sqrt(r2);
  const double ir3 = ir * ir * ir;
  w[0] = ir;
  w[1] = Rx * ir3;
  w[2] = Ry * ir3;
  w[3] = Rz * ir3;
}

/* child moments shifted by s (child centre - parent centre), accumulated */
void tmo_grav_m2m(const double* ch, const double* s, double* out) {
  const double M = ch[0];
  out[0] += M;
  for (int i = 0; i < 3; ++i) out[1 + i] += ch[1 + i] + M * s[i];
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j)
      out[4 + S2[i][j]] += ch[4 + S2[i][j]] + ch[1 + i] * s[j] + s[i] * ch[1 + j] + M * s[i] * s[j];
}

/* parent local shifted to a child centre (s = child - parent) */
void tmo_grav_l2l(const double* L, const double* s, double* out) {
  double Lm[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Lm[i][j] = L[4 + S2[i][j]];
  double t1 = 0.0, t2 = 0.0;
  for (int i = 0; i < 3; ++i) t1 += L[1 + i] * s[i];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t2 += Lm[i][j] * s[i] * s[j];
  out[0] = L[0] + t1 + 0.5 * t2;
  for (int i = 0; i < 3; ++i) {
    double t = 0.0;
    for (int j = 0; j < 3; ++j) t += Lm[i][j] * s[j];
    out[1 + i] = L[1 + i] + t;
  }
  for (int k = 0; k < 6; ++k) out[4 + k] = L[4 + k];
}

static inline long cidx(long n, long i, long j, long k) { return (k * n + j) * n + i; }

/* Full solve. mass: N^3 finest-level masses ((k,j,i) order, x fastest),
 * N = 2^D. Outputs phi[N^3], g[3][N^3]. Returns 0. */
int tmo_grav_solve(int D, const double* mass, double* phi, double* g) {
  long n[32] = {0};
  double* mom[32];
  double* loc[32];
  for (int l = 0; l <= D; ++l) {
    n[l] = 1L << l;
    mom[l] = (double*)calloc((size_t)(n[l] * n[l] * n[l]) * 10, sizeof(double));
    loc[l] = (double*)calloc((size_t)(n[l] * n[l] * n[l]) * 10, sizeof(double));
  }
  const long N = n[D];
  for (long c = 0; c < N * N * N; ++c) mom[D][c * 10] = mass[c];
  /* M2M, levels D-1 .. 0 */
  for (int l = D - 1; l >= 0; --l) {
    const double hc = 1.0 / (double)n[l + 1];
    for (long K = 0; K < n[l]; ++K)
      for (long J = 0; J < n[l]; ++J)
        for (long I = 0; I < n[l]; ++I) {
          double* out = mom[l] + cidx(n[l], I, J, K) * 10;
          for (int c = 0; c < 2; ++c)
            for (int b = 0; b < 2; ++b)
              for (int a = 0; a < 2; ++a) {
                const double s[3] = {(a - 0.5) * hc, (b - 0.5) * hc, (c - 0.5) * hc};
                tmo_grav_m2m(mom[l + 1] + cidx(n[l + 1], 2 * I + a, 2 * J + b, 2 * K + c) * 10, s,
                             out);
              }
        }
  }
  /* M2L (into loc as the per-level M2L sums), levels 2..D */
  for (int l = 2; l <= D; ++l) {
    const long m = n[l];
    const double h = 1.0 / (double)m;
    for (long k = 0; k < m; ++k)
      for (long j = 0; j < m; ++j)
        for (long i = 0; i < m; ++i) {
          double* out = loc[l] + cidx(m, i, j, k) * 10;
          double part[2][10] = {{0}};
          for (long dz = -2 - (k & 1); dz <= 3 - (k & 1); ++dz)
            for (long dy = -2 - (j & 1); dy <= 3 - (j & 1); ++dy)
              for (int pe = 0; pe < 2; ++pe)  /* even source x, then odd */
              for (long dx = -2 - (i & 1) + pe; dx <= 3 - (i & 1); dx += 2) {
                if (labs(dx) <= 1 && labs(dy) <= 1 && labs(dz) <= 1) continue;
                const long si = i + dx, sj = j + dy, sk = k + dz;
                if (si < 0 || sj < 0 || sk < 0 || si >= m || sj >= m || sk >= m) continue;
                const double R[3] = {-(double)dx * h, -(double)dy * h, -(double)dz * h};
                tmo_grav_m2l(mom[l] + cidx(m, si, sj, sk) * 10, R, part[dz + (k & 1) >= 1]);
              }
          for (int q = 0; q < 10; ++q) out[q] = part[0][q] + part[1][q];
        }
  }
  /* L2L, levels 3..D: loc = shift(parent) + own M2L sum */
  for (int l = 3; l <= D; ++l) {
    const long m = n[l];
    const double h = 1.0 / (double)m;
    for (long k = 0; k < m; ++k)
      for (long j = 0; j < m; ++j)
        for (long i = 0; i < m; ++i) {
          const double s[3] = {((i & 1) - 0.5) * h, ((j & 1) - 0.5) * h, ((k & 1) - 0.5) * h};
          double sh[10];
          tmo_grav_l2l(loc[l - 1] + cidx(n[l - 1], i >> 1, j >> 1, k >> 1) * 10, s, sh);
          double* out = loc[l] + cidx(m, i, j, k) * 10;
          for (int q = 0; q < 10; ++q) out[q] = sh[q] + out[q];
        }
  }
  /* L2P + P2P at the finest level */
  const double h = 1.0 / (double)N;
  for (long k = 0; k < N; ++k)
    for (long j = 0; j < N; ++j)
      for (long i = 0; i < N; ++i) {
        const long c = cidx(N, i, j, k);
        const double* L = loc[D] + c * 10;
        double p = L[0], gx = -L[1], gy = -L[2], gz = -L[3];
        for (long dz = -1; dz <= 1; ++dz)
          for (long dy = -1; dy <= 1; ++dy)
            for (long dx = -1; dx <= 1; ++dx) {
              if (!dx && !dy && !dz) continue;
              const long si = i + dx, sj = j + dy, sk = k + dz;
              if (si < 0 || sj < 0 || sk < 0 || si >= N || sj >= N || sk >= N) continue;
              const double nm = -mass[cidx(N, si, sj, sk)];
              double w[4];
              tmo_grav_p2p_geom(-(double)dx * h, -(double)dy * h, -(double)dz * h, w);
              p = fma(nm, w[0], p);
              gx = fma(nm, w[1], gx);
              gy = fma(nm, w[2], gy);
              gz = fma(nm, w[3], gz);
            }
        phi[c] = p;
        g[c] = gx;
        g[N * N * N + c] = gy;
        g[2 * N * N * N + c] = gz;
      }
  for (int l = 0; l <= D; ++l) {
    free(mom[l]);
    free(loc[l]);
  }
  return 0;
}

/* Direct O(N^2) summation over all cell pairs (accuracy reference). */
int tmo_grav_direct(int D, const double* mass, double* phi, double* g) {
  const long N = 1L << D, n3 = N * N * N;
  const double h = 1.0 / (double)N;
  for (long c = 0; c < n3; ++c) {
    const long i = c % N, j = (c / N) % N, k = c / (N * N);
    double p = 0, gx = 0, gy = 0, gz = 0;
    for (long s = 0; s < n3; ++s) {
      if (s == c) continue;
      const long si = s % N, sj = (s / N) % N, sk = s / (N * N);
      const double Rx = (double)(i - si) * h, Ry = (double)(j - sj) * h, Rz = (double)(k - sk) * h;
      const double r2 = Rx * Rx + Ry * Ry + Rz * Rz;
      const double ir = 1.0 / sqrt(r2);
      const double ir3 = ir * ir * ir;
      p -= mass[s] * ir;
      gx -= mass[s] * Rx * ir3;
      gy -= mass[s] * Ry * ir3;
      gz -= mass[s] * Rz * ir3;
    }
    phi[c] = p;
    g[c] = gx;
    g[n3 + c] = gy;
    g[2 * n3 + c] = gz;
  }
  return 0;
}
