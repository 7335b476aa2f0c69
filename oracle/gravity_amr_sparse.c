/* TEST INFRASTRUCTURE ONLY — the checker and the CPU baseline, never the product.
 *
 * Patch-sparse restatement of the adaptive FMM specification of
 * gravity_amr_oracle.c (PARITY UNPINNED w.r.t. the reference,
 * which has no gravity code). Same operators, same lists, same
 * per-target operation order, so the results are bit for bit those of
 * tmo_grav_amr_solve_ex (tests/test_gravity_amr.py compares the two on random
 * forests) — but stored the way the forest is:
 *
 *   * cells of depth d >= 3 live in the 8^3 patch of their forest node
 *     (level d - 3), found through a per-level hash of node coordinates; the
 *     depths 0..2 above the root patch are three tiny dense arrays. Memory is
 *     O(cells), so deep forests (configs[4], leaf level 7) fit, where the dense
 *     restatement's 2^(3d) arrays stop at leaf level 5;
 *   * the M2L geometry of the 343 same-depth offsets and the P2P geometry of
 *     the 27 neighbour offsets are tabulated per depth (the separation R =
 *     -(dx h, dy h, dz h) is the same double for every target, so the table
 *     entry is the bits the per-pair computation gives);
 *   * leaf cells evaluate only L0 and L_i (their L_ij are never read: L2P
 *     takes phi = L0, g = -L_i, and a leaf cell has no children);
 *   * the W/X/U lists are built in parallel over leaves and bucketed per
 *     target (CSR), each target's entries sorted by source (depth, k, j, i) —
 *     the dense restatement's global qsort order restricted to one target;
 *   * every phase runs OpenMP over independent targets (each target's own
 *     operation sequence is unchanged, so the thread count cannot change a bit).
 *
 * This is the CPU baseline of the gravity half of bench.py (cpu_baseline,
 * --impl reference) and the oracle for forests deeper than leaf level 5. */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "tm_oracle.h"

#define MAXL 18 /* forest levels 0..17 (cell depth <= 20: 20-bit coordinates in keys) */

typedef struct {
  long n, cap;
  uint64_t* hkey; /* open addressing: key + 1 (0 = empty) */
  int* hval;
  int *I, *J, *K;
  int* leaf; /* leaf slot or -1 (internal) */
  int* nb;   /* [n][27] same-level neighbour node or -1 */
  int* ch;   /* [n][8] child nodes (internal) */
  double* mom; /* [n][512][10] */
  double* loc; /* [n][512][10] */
} SLevel;

typedef struct {
  int nl;
  SLevel lv[MAXL];
  double* dmom[3];
  double* dloc[3];
  long base[MAXL + 1]; /* flat target ids: (base[l] + node) * 512 + c */
} SForest;

static inline uint64_t hkey(long I, long J, long K) {
  return (uint64_t)I | ((uint64_t)J << 21) | ((uint64_t)K << 42);
}
static inline uint64_t hmix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  return x;
}

static int find(const SLevel* L, long I, long J, long K) {
  if (!L->cap) return -1;
  const uint64_t k = hkey(I, J, K) + 1;
  for (uint64_t h = hmix(k) & (L->cap - 1);; h = (h + 1) & (L->cap - 1)) {
    if (L->hkey[h] == k) return L->hval[h];
    if (!L->hkey[h]) return -1;
  }
}

/* insert (returns node index; *fresh = 1 when new); -1 on allocation failure */
static int insert(SLevel* L, long I, long J, long K, int leaf, int* fresh) {
  const uint64_t k = hkey(I, J, K) + 1;
  uint64_t h = hmix(k) & (L->cap - 1);
  for (;; h = (h + 1) & (L->cap - 1)) {
    if (L->hkey[h] == k) {
      *fresh = 0;
      return L->hval[h];
    }
    if (!L->hkey[h]) break;
  }
  const int n = (int)L->n++;
  L->hkey[h] = k;
  L->hval[h] = n;
  L->I[n] = (int)I;
  L->J[n] = (int)J;
  L->K[n] = (int)K;
  L->leaf[n] = leaf;
  *fresh = 1;
  return n;
}

static void sforest_free(SForest* F) {
  for (int l = 0; l < MAXL; ++l) {
    SLevel* L = &F->lv[l];
    free(L->hkey), free(L->hval), free(L->I), free(L->J), free(L->K), free(L->leaf), free(L->nb), free(L->ch);
    free(L->mom), free(L->loc);
  }
  for (int d = 0; d < 3; ++d) free(F->dmom[d]), free(F->dloc[d]);
}

/* 0 ok, -1 memory / too deep, -2 leaves do not tile the unit cube */
static int sforest_build(SForest* F, long nleaves, const int* leaves) {
  memset(F, 0, sizeof(*F));
  long cnt[MAXL] = {0};
  for (long s = 0; s < nleaves; ++s) {
    const int l = leaves[4 * s];
    if (l < 0 || l >= MAXL) return -1;
    if (l + 1 > F->nl) F->nl = l + 1;
    for (int a = 0; a <= l; ++a) ++cnt[a];
  }
  if (!F->nl) return -2;
  for (int l = 0; l < F->nl; ++l) {
    SLevel* L = &F->lv[l];
    long cap = 16;
    while (cap < 2 * cnt[l]) cap <<= 1;
    L->cap = cap;
    L->hkey = (uint64_t*)calloc((size_t)cap, sizeof(uint64_t));
    L->hval = (int*)malloc((size_t)cap * sizeof(int));
    L->I = (int*)malloc((size_t)cnt[l] * sizeof(int) + 4);
    L->J = (int*)malloc((size_t)cnt[l] * sizeof(int) + 4);
    L->K = (int*)malloc((size_t)cnt[l] * sizeof(int) + 4);
    L->leaf = (int*)malloc((size_t)cnt[l] * sizeof(int) + 4);
    if (!L->hkey || !L->hval || !L->I || !L->J || !L->K || !L->leaf) return -1;
  }
  for (long s = 0; s < nleaves; ++s) {
    const int l = leaves[4 * s];
    const long I = leaves[4 * s + 1], J = leaves[4 * s + 2], K = leaves[4 * s + 3];
    const long n = 1L << l;
    if (I < 0 || J < 0 || K < 0 || I >= n || J >= n || K >= n) return -2;
    int fresh;
    const int nd = insert(&F->lv[l], I, J, K, (int)s, &fresh);
    if (!fresh) return -2; /* duplicate leaf, or a leaf that is another leaf's ancestor */
    (void)nd;
    for (int a = l - 1; a >= 0; --a) {
      const int sh = l - a;
      const int q = insert(&F->lv[a], I >> sh, J >> sh, K >> sh, -1, &fresh);
      if (F->lv[a].leaf[q] >= 0) return -2; /* covered by a coarser leaf */
      if (!fresh) break;                     /* its ancestors exist already */
    }
  }
  if (find(&F->lv[0], 0, 0, 0) < 0) return -2;
  long acc = 0;
  for (int l = 0; l < F->nl; ++l) {
    SLevel* L = &F->lv[l];
    F->base[l] = acc;
    acc += L->n;
    L->nb = (int*)malloc((size_t)L->n * 27 * sizeof(int) + 4);
    L->ch = (int*)malloc((size_t)L->n * 8 * sizeof(int) + 4);
    L->mom = (double*)calloc((size_t)L->n * 5120, sizeof(double));
    L->loc = (double*)calloc((size_t)L->n * 5120, sizeof(double));
    if (!L->nb || !L->ch || !L->mom || !L->loc) return -1;
  }
  F->base[F->nl] = acc;
  int bad = 0;
  for (int l = 0; l < F->nl; ++l) {
    SLevel* L = &F->lv[l];
    const long n = 1L << l;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (long q = 0; q < L->n; ++q) {
      const long I = L->I[q], J = L->J[q], K = L->K[q];
      for (int o = 0; o < 27; ++o) {
        const long a = I + o % 3 - 1, b = J + (o / 3) % 3 - 1, c = K + o / 9 - 1;
        L->nb[q * 27 + o] = (a < 0 || b < 0 || c < 0 || a >= n || b >= n || c >= n) ? -1 : find(L, a, b, c);
      }
      for (int o = 0; o < 8; ++o) {
        const int x = L->leaf[q] >= 0 || l + 1 >= F->nl
                          ? -1
                          : find(&F->lv[l + 1], 2 * I + (o & 1), 2 * J + ((o >> 1) & 1), 2 * K + (o >> 2));
        L->ch[q * 8 + o] = x;
        if (L->leaf[q] < 0 && x < 0) bad = 1; /* an internal node without all 8 children */
      }
    }
  }
  if (bad) return -2;
  for (int d = 0; d < 3; ++d) {
    const size_t n3 = (size_t)1 << (3 * d);
    F->dmom[d] = (double*)calloc(n3 * 10, sizeof(double));
    F->dloc[d] = (double*)calloc(n3 * 10, sizeof(double));
    if (!F->dmom[d] || !F->dloc[d]) return -1;
  }
  return 0;
}

static inline long cix(long n, long i, long j, long k) { return (k * n + j) * n + i; }
static inline int lcell(long gi, long gj, long gk) { return (int)(((gk & 7) * 8 + (gj & 7)) * 8 + (gi & 7)); }
static inline double centre(long gi, int d) { return ((double)gi + 0.5) / (double)(1L << d); }

/* cell type at depth d: 0 missing / outside, 1 internal, 2 leaf; node index in *nd (d >= 3) */
static inline int ctype(const SForest* F, int d, long gi, long gj, long gk, int* nd) {
  const long n = 1L << d;
  if (gi < 0 || gj < 0 || gk < 0 || gi >= n || gj >= n || gk >= n) return 0;
  if (d < 3) return 1;
  if (d - 3 >= F->nl) return 0;
  const SLevel* L = &F->lv[d - 3];
  const int q = find(L, gi >> 3, gj >> 3, gk >> 3);
  if (nd) *nd = q;
  if (q < 0) return 0;
  return L->leaf[q] >= 0 ? 2 : 1;
}

static inline double* momp(const SForest* F, int d, long gi, long gj, long gk) {
  if (d < 3) return F->dmom[d] + cix(1L << d, gi, gj, gk) * 10;
  const SLevel* L = &F->lv[d - 3];
  return L->mom + ((long)find(L, gi >> 3, gj >> 3, gk >> 3) * 512 + lcell(gi, gj, gk)) * 10;
}

/* tmo_grav_m2l_geom restricted to L0, L_i (the same operations for those) */
static void m2l_geom4(const double* mom, const double* e, double* out) {
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
  static const int S2[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
  for (int i = 0; i < 3; ++i) {
    double t = out[1 + i];
    t = fma(nM, e[1 + i], t);
    for (int j = 0; j < 3; ++j) t = fma(mom[1 + j], e[4 + S2[i][j]], t);
    out[1 + i] = t;
  }
}

static inline void m2l_any(const double* mom, const double* e, double* out, int full, int cnt) {
  if (cnt)
    out[0] += mom[0];
  else if (full)
    tmo_grav_m2l_geom(mom, e, out);
  else
    m2l_geom4(mom, e, out);
}

/* V list of one target cell (global coords at depth d): the specification's
 * two partial sums over the 189-cell stencil; sources resolve through the
 * target node's 27 neighbours (depth >= 3) or the dense depth-2 array */
static void vlist_cell(const SForest* F, int d, const double* tab, long gi, long gj, long gk, const int* nb27,
                       const double* lvmom, double* out, int full, int cnt) {
  const long m = 1L << d;
  double part[2][10];
  memset(part, 0, sizeof(part));
  const long I0 = (gi >> 3) - 1, J0 = (gj >> 3) - 1, K0 = (gk >> 3) - 1;
  for (long dz = -2 - (gk & 1); dz <= 3 - (gk & 1); ++dz)
    for (long dy = -2 - (gj & 1); dy <= 3 - (gj & 1); ++dy)
      for (int pe = 0; pe < 2; ++pe)
        for (long dx = -2 - (gi & 1) + pe; dx <= 3 - (gi & 1); dx += 2) {
          if (labs(dx) <= 1 && labs(dy) <= 1 && labs(dz) <= 1) continue;
          const long si = gi + dx, sj = gj + dy, sk = gk + dz;
          if (si < 0 || sj < 0 || sk < 0 || si >= m || sj >= m || sk >= m) continue;
          const double* src;
          if (d < 3) {
            src = F->dmom[d] + cix(m, si, sj, sk) * 10;
          } else {
            const int o = (int)(((sk >> 3) - K0) * 9 + ((sj >> 3) - J0) * 3 + ((si >> 3) - I0));
            const int q = nb27[o];
            if (q < 0) continue; /* missing cell */
            src = lvmom + ((long)q * 512 + lcell(si, sj, sk)) * 10;
          }
          m2l_any(src, tab + (((dz + 3) * 7 + (dy + 3)) * 7 + (dx + 3)) * 13, part[dz + (gk & 1) >= 1], full, cnt);
        }
  const int nq = full ? 10 : 4;
  for (int q = 0; q < nq; ++q) out[q] = part[0][q] + part[1][q];
}


/* ---- V lists of one node patch, four same-x-parity targets per vector ------
 * The 12^3 source window of the patch (its 27-node neighbourhood; missing or
 * outside cells are zero moments: adding a zero-moment term is an exact no-op,
 * because every accumulator starts at +0 and a sum started at +0 never becomes
 * -0) is stored per component with x split by parity, so the sources of the
 * four targets x = a, a+2, a+4, a+6 under one offset are four consecutive
 * doubles. Every lane runs the scalar operation sequence of tmo_grav_m2l_geom
 * (vector FMA = four correctly rounded fma(); negation = sign flip). */
#if defined(__AVX2__) && defined(__FMA__)
#include <immintrin.h>
typedef __m256d V4;
static inline V4 vld(const double* p) { return _mm256_loadu_pd(p); }
static inline V4 vset(double x) { return _mm256_set1_pd(x); }
static inline V4 vfma(V4 a, V4 b, V4 c) { return _mm256_fmadd_pd(a, b, c); }
static inline V4 vmul(V4 a, V4 b) { return _mm256_mul_pd(a, b); }
static inline V4 vadd(V4 a, V4 b) { return _mm256_add_pd(a, b); }
static inline V4 vneg(V4 a) { return _mm256_xor_pd(a, _mm256_set1_pd(-0.0)); }
static inline void vst(double* p, V4 a) { _mm256_storeu_pd(p, a); }
#else
typedef struct {
  double x[4];
} V4;
static inline V4 vld(const double* p) {
  V4 r;
  for (int i = 0; i < 4; ++i) r.x[i] = p[i];
  return r;
}
static inline V4 vset(double v) {
  V4 r;
  for (int i = 0; i < 4; ++i) r.x[i] = v;
  return r;
}
static inline V4 vfma(V4 a, V4 b, V4 c) {
  V4 r;
  for (int i = 0; i < 4; ++i) r.x[i] = fma(a.x[i], b.x[i], c.x[i]);
  return r;
}
static inline V4 vmul(V4 a, V4 b) {
  V4 r;
  for (int i = 0; i < 4; ++i) r.x[i] = a.x[i] * b.x[i];
  return r;
}
static inline V4 vadd(V4 a, V4 b) {
  V4 r;
  for (int i = 0; i < 4; ++i) r.x[i] = a.x[i] + b.x[i];
  return r;
}
static inline V4 vneg(V4 a) {
  for (int i = 0; i < 4; ++i) a.x[i] = -a.x[i];
  return a;
}
static inline void vst(double* p, V4 a) {
  for (int i = 0; i < 4; ++i) p[i] = a.x[i];
}
#endif

#define WIN_Q 1728 /* doubles per component: [wz 12][wy 12][parity 2][half-x 6] */

static void vlist_node(const int* nb27, const double* lvmom, const double* tab, double* loc, int full,
                       double* win) {
  for (int wz = 0; wz < 12; ++wz)
    for (int wy = 0; wy < 12; ++wy)
      for (int wx = 0; wx < 12; ++wx) {
        const int oz = wz < 2 ? -1 : (wz > 9 ? 1 : 0), oy = wy < 2 ? -1 : (wy > 9 ? 1 : 0),
                  ox = wx < 2 ? -1 : (wx > 9 ? 1 : 0);
        const int q = nb27[((oz + 1) * 3 + (oy + 1)) * 3 + ox + 1];
        const int at = (wz * 12 + wy) * 12 + (wx & 1) * 6 + (wx >> 1);
        if (q < 0) {
          for (int c = 0; c < 10; ++c) win[c * WIN_Q + at] = 0.0;
          continue;
        }
        const int lx = wx - 2 - 8 * ox, ly = wy - 2 - 8 * oy, lz = wz - 2 - 8 * oz;
        const double* m = lvmom + ((long)q * 512 + (lz * 8 + ly) * 8 + lx) * 10;
        for (int c = 0; c < 10; ++c) win[c * WIN_Q + at] = m[c];
      }
  const int nq = full ? 10 : 4;
  for (int k = 0; k < 8; ++k)
    for (int j = 0; j < 8; ++j)
      for (int a = 0; a < 2; ++a) {
        V4 part[2][10];
        for (int h = 0; h < 2; ++h)
          for (int c = 0; c < 10; ++c) part[h][c] = vset(0.0);
        for (int dz = -2 - (k & 1); dz <= 3 - (k & 1); ++dz)
          for (int dy = -2 - (j & 1); dy <= 3 - (j & 1); ++dy)
            for (int pe = 0; pe < 2; ++pe)
              for (int dx = -2 - a + pe; dx <= 3 - a; dx += 2) {
                if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1) continue;
                const double* e = tab + (((dz + 3) * 7 + (dy + 3)) * 7 + (dx + 3)) * 13;
                const int sx = a + dx + 2;
                const double* src = win + ((k + dz + 2) * 12 + (j + dy + 2)) * 12 + (sx & 1) * 6 + (sx >> 1);
                V4* o = part[dz + (k & 1) >= 1];
                const V4 m0 = vld(src), nM = vneg(m0);
                const V4 m1 = vld(src + WIN_Q), m2 = vld(src + 2 * WIN_Q), m3 = vld(src + 3 * WIN_Q);
                V4 t = vmul(nM, vset(e[0]));
                t = vfma(m1, vset(e[1]), t);
                t = vfma(m2, vset(e[2]), t);
                t = vfma(m3, vset(e[3]), t);
                t = vfma(vneg(vld(src + 4 * WIN_Q)), vset(e[10]), t);
                t = vfma(vneg(vld(src + 5 * WIN_Q)), vset(e[5]), t);
                t = vfma(vneg(vld(src + 6 * WIN_Q)), vset(e[6]), t);
                t = vfma(vneg(vld(src + 7 * WIN_Q)), vset(e[11]), t);
                t = vfma(vneg(vld(src + 8 * WIN_Q)), vset(e[8]), t);
                t = vfma(vneg(vld(src + 9 * WIN_Q)), vset(e[12]), t);
                o[0] = vadd(o[0], t);
                /* L_i: fma(nM, D1_i), then D_j D2_ij (S2 = xx xy xz / xy yy yz / xz yz zz) */
                o[1] = vfma(m3, vset(e[6]), vfma(m2, vset(e[5]), vfma(m1, vset(e[4]), vfma(nM, vset(e[1]), o[1]))));
                o[2] = vfma(m3, vset(e[8]), vfma(m2, vset(e[7]), vfma(m1, vset(e[5]), vfma(nM, vset(e[2]), o[2]))));
                o[3] = vfma(m3, vset(e[9]), vfma(m2, vset(e[8]), vfma(m1, vset(e[6]), vfma(nM, vset(e[3]), o[3]))));
                if (full)
                  for (int c = 0; c < 6; ++c) o[4 + c] = vfma(nM, vset(e[4 + c]), o[4 + c]);
              }
        for (int c = 0; c < nq; ++c) {
          double v[4];
          vst(v, vadd(part[0][c], part[1][c]));
          for (int x = 0; x < 4; ++x) loc[((k * 8 + j) * 8 + a + 2 * x) * 10 + c] = v[x];
        }
      }
}

typedef struct {
  int64_t t;   /* flat target id */
  uint64_t s;  /* source key: depth << 60 | k << 40 | j << 20 | i */
} SEnt;

typedef struct {
  SEnt* e;
  size_t n, cap;
  int err;
} SBuf;

static void spush(SBuf* B, int64_t t, int sd, long si, long sj, long sk) {
  if (B->n == B->cap) {
    size_t nc = B->cap ? 2 * B->cap : 4096;
    SEnt* p = (SEnt*)realloc(B->e, nc * sizeof(SEnt));
    if (!p) {
      B->err = 1;
      return;
    }
    B->e = p;
    B->cap = nc;
  }
  SEnt* x = &B->e[B->n++];
  x->t = t;
  x->s = ((uint64_t)sd << 60) | ((uint64_t)sk << 40) | ((uint64_t)sj << 20) | (uint64_t)si;
}

static inline int64_t flat(const SForest* F, int d, int nd, long gi, long gj, long gk) {
  return (F->base[d - 3] + nd) * 512 + lcell(gi, gj, gk);
}

/* closed boxes of cell A (depth da) and cell B (depth db >= da) touch */
static int touches(int da, const long* a, int db, const long* b) {
  const int s = db - da;
  for (int q = 0; q < 3; ++q) {
    const long lo = a[q] << s, hi = (a[q] + 1) << s;
    if (!(b[q] <= hi && b[q] + 1 >= lo)) return 0;
  }
  return 1;
}

/* gravity_amr_oracle.c visit(): bufs[0] M2L (W/X), bufs[1] U cross-depth */
static void svisit(const SForest* F, SBuf* bufs, int db, const long* b, int64_t bflat, int dy, const long* Y) {
  for (int c = 0; c < 2; ++c)
    for (int bb = 0; bb < 2; ++bb)
      for (int a = 0; a < 2; ++a) {
        const long y[3] = {2 * Y[0] + a, 2 * Y[1] + bb, 2 * Y[2] + c};
        int nd = -1;
        const int t = ctype(F, dy + 1, y[0], y[1], y[2], &nd);
        if (t == 0) {
          bufs[0].err = 2;
          return;
        }
        const int64_t yflat = flat(F, dy + 1, nd, y[0], y[1], y[2]);
        if (touches(db, b, dy + 1, y)) {
          if (t == 2) {
            spush(&bufs[1], bflat, dy + 1, y[0], y[1], y[2]);
            spush(&bufs[1], yflat, db, b[0], b[1], b[2]);
          } else {
            svisit(F, bufs, db, b, bflat, dy + 1, y);
          }
        } else {
          spush(&bufs[0], bflat, dy + 1, y[0], y[1], y[2]);
          spush(&bufs[0], yflat, db, b[0], b[1], b[2]);
        }
      }
}

static int cmp_src(const void* pa, const void* pb) {
  const uint64_t a = ((const SEnt*)pa)->s, b = ((const SEnt*)pb)->s;
  return a < b ? -1 : (a > b ? 1 : 0);
}

/* per-thread buffers -> CSR over targets, each target's entries sorted by source */
static int to_csr(SBuf* tb, int nth, long ntarget, long** off_out, SEnt** ent_out, long* total) {
  long* off = (long*)calloc((size_t)ntarget + 1, sizeof(long));
  if (!off) return -1;
  long tot = 0;
  for (int t = 0; t < nth; ++t) {
    tot += (long)tb[t].n;
    for (size_t q = 0; q < tb[t].n; ++q) ++off[tb[t].e[q].t + 1];
  }
  for (long i = 0; i < ntarget; ++i) off[i + 1] += off[i];
  SEnt* ent = (SEnt*)malloc((size_t)(tot ? tot : 1) * sizeof(SEnt));
  long* fill = (long*)malloc((size_t)(ntarget ? ntarget : 1) * sizeof(long));
  if (!ent || !fill) {
    free(off), free(ent), free(fill);
    return -1;
  }
  memcpy(fill, off, (size_t)ntarget * sizeof(long));
  for (int t = 0; t < nth; ++t)
    for (size_t q = 0; q < tb[t].n; ++q) ent[fill[tb[t].e[q].t]++] = tb[t].e[q];
  free(fill);
#pragma omp parallel for schedule(dynamic, 1024)
  for (long i = 0; i < ntarget; ++i)
    if (off[i + 1] - off[i] > 1) qsort(ent + off[i], (size_t)(off[i + 1] - off[i]), sizeof(SEnt), cmp_src);
  *off_out = off;
  *ent_out = ent;
  *total = tot;
  return 0;
}

static inline void skey_decode(uint64_t s, int* d, long* i, long* j, long* k) {
  *d = (int)(s >> 60);
  *k = (long)((s >> 40) & 0xfffff);
  *j = (long)((s >> 20) & 0xfffff);
  *i = (long)(s & 0xfffff);
}

/* flat target id -> (level, node, cell) */
static inline void flat_decode(const SForest* F, int64_t t, int* l, int* nd, int* c) {
  const long node = t >> 9;
  int a = 0;
  while (a + 1 < F->nl && F->base[a + 1] <= node) ++a;
  *l = a;
  *nd = (int)(node - F->base[a]);
  *c = (int)(t & 511);
}

#include <stdio.h>
#include <time.h>
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
/* TMO_TIMING=1: per-phase wall times on stderr (CPU baseline breakdown) */
#define PHASE(name)                                                   \
  do {                                                                \
    if (timing) {                                                     \
      const double t_ = now_s();                                      \
      fprintf(stderr, "tmo_grav_amr_sparse %-10s %.3f s\n", name, t_ - t_prev); \
      t_prev = t_;                                                    \
    }                                                                 \
  } while (0)

struct tmo_grav_plan;
typedef struct tmo_grav_plan tmo_grav_plan;
struct tmo_grav_plan {
  SForest F;
  long nleaves;
  int* leaves;
  double *tab, *ptab;
  long *moff, *poff;
  SEnt *ment, *pent;
  long nm, np;
};

static int plan_tables(tmo_grav_plan* P) {
  const int nl = P->F.nl, Dmax = nl - 1 + 3;
  /* geometry tables: M2L [depth][7^3][13], P2P [depth][27][4] */
  double* tab = (double*)malloc((size_t)(Dmax + 1) * 343 * 13 * sizeof(double));
  double* ptab = (double*)malloc((size_t)(Dmax + 1) * 27 * 4 * sizeof(double));
  P->tab = tab;
  P->ptab = ptab;
  if (!tab || !ptab) return -1;
  for (int d = 0; d <= Dmax; ++d) {
    const double h = 1.0 / (double)(1L << d);
    for (int o = 0; o < 343; ++o) {
      const long dx = o % 7 - 3, dy = (o / 7) % 7 - 3, dz = o / 49 - 3;
      const double R[3] = {-(double)dx * h, -(double)dy * h, -(double)dz * h};
      if (dx || dy || dz) tmo_grav_geom(R, tab + ((size_t)d * 343 + o) * 13);
    }
    for (int o = 0; o < 27; ++o) {
      const long dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
      if (dx || dy || dz)
        tmo_grav_p2p_geom(-(double)dx * h, -(double)dy * h, -(double)dz * h, ptab + ((size_t)d * 27 + o) * 4);
    }
  }
  return 0;
}

static int plan_lists(tmo_grav_plan* P, const int* leaves) {
  const long nleaves = P->nleaves;
  const int nl = P->F.nl;
  /* W / X / U-cross lists, parallel over leaves */
  int nth = 1;
#ifdef _OPENMP
  nth = omp_get_max_threads();
#endif
  SBuf* tb = (SBuf*)calloc((size_t)nth * 2, sizeof(SBuf));
  if (!tb) return -1;
#pragma omp parallel for schedule(dynamic, 8)
  for (long s = 0; s < nleaves; ++s) {
    int me = 0;
#ifdef _OPENMP
    me = omp_get_thread_num();
#endif
    SBuf* bufs = tb + 2 * me;
    const int l = leaves[4 * s], d = l + 3;
    const int nd = find(&P->F.lv[l], leaves[4 * s + 1], leaves[4 * s + 2], leaves[4 * s + 3]);
    for (int c = 0; c < 512; ++c) {
      const long b[3] = {8L * leaves[4 * s + 1] + (c & 7), 8L * leaves[4 * s + 2] + ((c >> 3) & 7),
                         8L * leaves[4 * s + 3] + (c >> 6)};
      const int64_t bflat = flat(&P->F, d, nd, b[0], b[1], b[2]);
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            if (!dx && !dy && !dz) continue;
            const long Y[3] = {b[0] + dx, b[1] + dy, b[2] + dz};
            if (ctype(&P->F, d, Y[0], Y[1], Y[2], NULL) == 1) svisit(&P->F, bufs, d, b, bflat, d, Y);
          }
    }
  }
  int lerr = 0;
  for (int t = 0; t < 2 * nth; ++t) lerr |= tb[t].err;
  long *moff = NULL, *poff = NULL;
  SEnt *ment = NULL, *pent = NULL;
  long nm = 0, np = 0;
  const long ntarget = P->F.base[nl] * 512;
  if (!lerr) {
    SBuf* m0 = (SBuf*)malloc((size_t)nth * sizeof(SBuf));
    SBuf* p0 = (SBuf*)malloc((size_t)nth * sizeof(SBuf));
    if (!m0 || !p0) lerr = 1;
    for (int t = 0; t < nth && !lerr; ++t) m0[t] = tb[2 * t], p0[t] = tb[2 * t + 1];
    if (!lerr && to_csr(m0, nth, ntarget, &moff, &ment, &nm)) lerr = 1;
    if (!lerr && to_csr(p0, nth, ntarget, &poff, &pent, &np)) lerr = 1;
    free(m0), free(p0);
  }
  for (int t = 0; t < 2 * nth; ++t) free(tb[t].e);
  free(tb);
  P->moff = moff, P->ment = ment, P->poff = poff, P->pent = pent, P->nm = nm, P->np = np;
  if (lerr) return lerr == 2 ? -2 : -1;
  return 0;
}

void tmo_grav_plan_destroy(tmo_grav_plan* P) {
  if (!P) return;
  sforest_free(&P->F);
  free(P->leaves), free(P->tab), free(P->ptab), free(P->moff), free(P->poff), free(P->ment), free(P->pent);
  free(P);
}

/* The topology-only part, done once per forest like the GPU plan: node
 * patches, geometry tables, W/X/U lists. rc: 0, -1 memory, -2 bad tiling. */
tmo_grav_plan* tmo_grav_plan_create(long nleaves, const int* leaves, int* rc_out) {
  tmo_grav_plan* P = (tmo_grav_plan*)calloc(1, sizeof(tmo_grav_plan));
  int rc = P ? 0 : -1;
  if (!rc) {
    P->nleaves = nleaves;
    P->leaves = (int*)malloc((size_t)(nleaves ? nleaves : 1) * 4 * sizeof(int));
    rc = P->leaves ? sforest_build(&P->F, nleaves, leaves) : -1;
    if (P->leaves) memcpy(P->leaves, leaves, (size_t)nleaves * 4 * sizeof(int));
  }
  if (!rc) rc = plan_tables(P);
  if (!rc) rc = plan_lists(P, leaves);
  if (rc_out) *rc_out = rc;
  if (rc) {
    tmo_grav_plan_destroy(P);
    return NULL;
  }
  return P;
}

int tmo_grav_plan_solve(tmo_grav_plan* P, const double* mass, int flags, double* phi, double* g,
                        long* counts) {
  const int cnt = (flags & 2) != 0;
  const int timing = getenv("TMO_TIMING") != NULL;
  double t_prev = timing ? now_s() : 0.0;
  SForest F = P->F; /* shallow: the arrays are the plan's */
  const long nleaves = P->nleaves;
  const int* leaves = P->leaves;
  const int nl = F.nl;
  const double *tab = P->tab, *ptab = P->ptab;
  const long *moff = P->moff, *poff = P->poff;
  const SEnt *ment = P->ment, *pent = P->pent;
  const long ntarget = F.base[nl] * 512;
  if (counts) counts[0] = P->nm, counts[1] = P->np;
  /* internal moments accumulate (M2M): zero them */
  for (int l = 0; l < nl; ++l) {
    SLevel* L = &F.lv[l];
#pragma omp parallel for schedule(static)
    for (long q = 0; q < L->n; ++q)
      if (L->leaf[q] < 0) memset(L->mom + q * 5120, 0, 5120 * sizeof(double));
  }
  for (int d = 0; d < 3; ++d) memset(F.dmom[d], 0, ((size_t)1 << (3 * d)) * 10 * sizeof(double));
  /* P2M */
  for (int l = 0; l < nl; ++l) {
    SLevel* L = &F.lv[l];
#pragma omp parallel for schedule(static)
    for (long q = 0; q < L->n; ++q) {
      const int s = L->leaf[q];
      if (s < 0) continue;
      for (int c = 0; c < 512; ++c) L->mom[((long)q * 512 + c) * 10] = cnt ? 1.0 : mass[(long)s * 512 + c];
    }
  }
  /* M2M: patches bottom-up, then the dense depths 2, 1, 0 */
  for (int l = nl - 2; l >= 0; --l) {
    SLevel* L = &F.lv[l];
    const SLevel* C = &F.lv[l + 1];
    const double hc = 1.0 / (double)(1L << (l + 4));
#pragma omp parallel for schedule(dynamic, 4)
    for (long q = 0; q < L->n; ++q) {
      if (L->leaf[q] >= 0) continue;
      for (int c = 0; c < 512; ++c) {
        const int i = c & 7, j = (c >> 3) & 7, k = c >> 6;
        const int cn = L->ch[q * 8 + ((k >> 2) * 2 + (j >> 2)) * 2 + (i >> 2)];
        double* out = L->mom + ((long)q * 512 + c) * 10;
        for (int cc = 0; cc < 2; ++cc)
          for (int b = 0; b < 2; ++b)
            for (int a = 0; a < 2; ++a) {
              const double s[3] = {(a - 0.5) * hc, (b - 0.5) * hc, (cc - 0.5) * hc};
              const int ci = ((2 * i) & 7) + a, cj = ((2 * j) & 7) + b, ck = ((2 * k) & 7) + cc;
              tmo_grav_m2m(C->mom + ((long)cn * 512 + (ck * 8 + cj) * 8 + ci) * 10, s, out);
            }
      }
    }
  }
  for (int d = 2; d >= 0; --d) {
    const long n = 1L << d;
    const double hc = 1.0 / (double)(2 * n);
    for (long K = 0; K < n; ++K)
      for (long J = 0; J < n; ++J)
        for (long I = 0; I < n; ++I) {
          double* out = F.dmom[d] + cix(n, I, J, K) * 10;
          for (int c = 0; c < 2; ++c)
            for (int b = 0; b < 2; ++b)
              for (int a = 0; a < 2; ++a) {
                const double s[3] = {(a - 0.5) * hc, (b - 0.5) * hc, (c - 0.5) * hc};
                tmo_grav_m2m(momp(&F, d + 1, 2 * I + a, 2 * J + b, 2 * K + c), s, out);
              }
        }
  }
  PHASE("p2m+m2m");
  /* V lists: dense depth 2, then every patch */
  for (long t = 0; t < 64; ++t)
    vlist_cell(&F, 2, tab + 2 * 343 * 13, t & 3, (t >> 2) & 3, t >> 4, NULL, NULL, F.dloc[2] + t * 10, 1, cnt);
  {
    const long nodes = F.base[nl];
#pragma omp parallel
    {
      double* win = cnt ? NULL : (double*)malloc(10 * WIN_Q * sizeof(double));
#pragma omp for schedule(dynamic, 1)
      for (long f = 0; f < nodes; ++f) {
        int l = 0;
        while (l + 1 < nl && F.base[l + 1] <= f) ++l;
        SLevel* L = &F.lv[l];
        const long q = f - F.base[l];
        const int d = l + 3;
        const double* tb = tab + (size_t)d * 343 * 13;
        const int full = L->leaf[q] < 0 || l == 0; /* a leaf root keeps all ten */
        if (win) {
          vlist_node(L->nb + q * 27, L->mom, tb, L->loc + (long)q * 5120, full, win);
          continue;
        }
        const long I = L->I[q], J = L->J[q], K = L->K[q];
        for (int c = 0; c < 512; ++c)
          vlist_cell(&F, d, tb, 8 * I + (c & 7), 8 * J + ((c >> 3) & 7), 8 * K + (c >> 6), L->nb + q * 27,
                     L->mom, L->loc + ((long)q * 512 + c) * 10, full, cnt);
      }
      free(win);
    }
  }
  PHASE("v-list");
  /* W / X M2L per target, in source order, after the V sum */
#pragma omp parallel for schedule(dynamic, 4096)
  for (long t = 0; t < ntarget; ++t) {
    if (moff[t + 1] == moff[t]) continue;
    int l, nd, c;
    flat_decode(&F, t, &l, &nd, &c);
    const SLevel* L = &F.lv[l];
    const int td = l + 3;
    const long ti = 8L * L->I[nd] + (c & 7), tj = 8L * L->J[nd] + ((c >> 3) & 7), tk = 8L * L->K[nd] + (c >> 6);
    double* out = L->loc + ((long)nd * 512 + c) * 10;
    const int full = L->leaf[nd] < 0 || l == 0;
    for (long e = moff[t]; e < moff[t + 1]; ++e) {
      int sd;
      long si, sj, sk;
      skey_decode(ment[e].s, &sd, &si, &sj, &sk);
      const double R[3] = {centre(ti, td) - centre(si, sd), centre(tj, td) - centre(sj, sd),
                           centre(tk, td) - centre(sk, sd)};
      double ge[13];
      if (!cnt) tmo_grav_geom(R, ge);
      m2l_any(momp(&F, sd, si, sj, sk), ge, out, full, cnt);
    }
  }
  PHASE("w/x m2l");
  /* L2L: depth 3 from the dense depth 2, then patch levels top-down */
  for (int l = 0; l < nl; ++l) {
    SLevel* L = &F.lv[l];
    const int d = l + 3;
    const double h = 1.0 / (double)(1L << d);
#pragma omp parallel for schedule(dynamic, 4)
    for (long q = 0; q < L->n; ++q) {
      const long I = L->I[q], J = L->J[q], K = L->K[q];
      for (int c = 0; c < 512; ++c) {
        const long i = 8 * I + (c & 7), j = 8 * J + ((c >> 3) & 7), k = 8 * K + (c >> 6);
        const double s[3] = {((i & 1) - 0.5) * h, ((j & 1) - 0.5) * h, ((k & 1) - 0.5) * h};
        const double* par;
        if (l == 0) {
          par = F.dloc[2] + cix(4, i >> 1, j >> 1, k >> 1) * 10;
        } else {
          const SLevel* P = &F.lv[l - 1];
          const int pn = find(P, (i >> 1) >> 3, (j >> 1) >> 3, (k >> 1) >> 3);
          par = P->loc + ((long)pn * 512 + lcell(i >> 1, j >> 1, k >> 1)) * 10;
        }
        double sh[10];
        tmo_grav_l2l(par, s, sh);
        double* out = L->loc + ((long)q * 512 + c) * 10;
        const int nq = (L->leaf[q] < 0 || l == 0) ? 10 : 4;
        for (int x = 0; x < nq; ++x) out[x] = sh[x] + out[x];
      }
    }
  }
  PHASE("l2l");
  /* L2P + same-depth P2P, then the cross-depth U pairs in source order */
  const long ncell = nleaves * 512;
#pragma omp parallel for schedule(dynamic, 4)
  for (long s = 0; s < nleaves; ++s) {
    const int l = leaves[4 * s], d = l + 3;
    const SLevel* L = &F.lv[l];
    const int nd = find(L, leaves[4 * s + 1], leaves[4 * s + 2], leaves[4 * s + 3]);
    const long N = 1L << d;
    const long I0 = leaves[4 * s + 1] - 1, J0 = leaves[4 * s + 2] - 1, K0 = leaves[4 * s + 3] - 1;
    const double* pt = ptab + (size_t)d * 27 * 4;
    for (int c = 0; c < 512; ++c) {
      const long i = 8L * leaves[4 * s + 1] + (c & 7), j = 8L * leaves[4 * s + 2] + ((c >> 3) & 7),
                 k = 8L * leaves[4 * s + 3] + (c >> 6);
      const double* Lc = L->loc + ((long)nd * 512 + c) * 10;
      double p = Lc[0], gx = -Lc[1], gy = -Lc[2], gz = -Lc[3];
      for (long dz = -1; dz <= 1; ++dz)
        for (long dy = -1; dy <= 1; ++dy)
          for (long dx = -1; dx <= 1; ++dx) {
            if (!dx && !dy && !dz) continue;
            const long si = i + dx, sj = j + dy, sk = k + dz;
            if (si < 0 || sj < 0 || sk < 0 || si >= N || sj >= N || sk >= N) continue;
            const int q = L->nb[(long)nd * 27 + ((sk >> 3) - K0) * 9 + ((sj >> 3) - J0) * 3 + ((si >> 3) - I0)];
            if (q < 0 || L->leaf[q] < 0) continue; /* same-depth leaf cells only */
            if (cnt) {
              p += 1.0;
              continue;
            }
            const double nm = -L->mom[((long)q * 512 + lcell(si, sj, sk)) * 10];
            const double* w = pt + ((dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)) * 4;
            p = fma(nm, w[0], p);
            gx = fma(nm, w[1], gx);
            gy = fma(nm, w[2], gy);
            gz = fma(nm, w[3], gz);
          }
      const long t = (F.base[l] + nd) * 512 + c;
      for (long e = poff[t]; e < poff[t + 1]; ++e) {
        int sd;
        long si, sj, sk;
        skey_decode(pent[e].s, &sd, &si, &sj, &sk);
        if (cnt) {
          p += 1.0;
          continue;
        }
        const double nm = -momp(&F, sd, si, sj, sk)[0];
        double w[4];
        tmo_grav_p2p_geom(centre(i, d) - centre(si, sd), centre(j, d) - centre(sj, sd),
                          centre(k, d) - centre(sk, sd), w);
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
  PHASE("l2p+p2p");
  if (flags & 1) { /* tmo_grav_am_correct, per-slot pair trees in parallel (same tree) */
    long P = 1;
    while (P < nleaves) P <<= 1;
    double* S = (double*)calloc((size_t)P * 16, sizeof(double));
    if (!S) return -1;
#pragma omp parallel
    {
      double* v = (double*)malloc(512 * 16 * sizeof(double));
#pragma omp for schedule(static)
      for (long s = 0; s < nleaves; ++s) {
        const int d = leaves[4 * s] + 3;
        for (int c = 0; c < 512; ++c) {
          const long o = s * 512 + c;
          const double x = centre(8L * leaves[4 * s + 1] + (c & 7), d),
                       y = centre(8L * leaves[4 * s + 2] + ((c >> 3) & 7), d),
                       z = centre(8L * leaves[4 * s + 3] + (c >> 6), d);
          const double m = mass[o], gx = g[o], gy = g[ncell + o], gz = g[2 * ncell + o];
          double* w = v + c * 16;
          w[0] = m;
          w[1] = m * x;
          w[2] = m * y;
          w[3] = m * z;
          w[4] = m * gx;
          w[5] = m * gy;
          w[6] = m * gz;
          w[7] = m * (y * gz - z * gy);
          w[8] = m * (z * gx - x * gz);
          w[9] = m * (x * gy - y * gx);
          w[10] = w[1] * x;
          w[11] = w[1] * y;
          w[12] = w[1] * z;
          w[13] = w[2] * y;
          w[14] = w[2] * z;
          w[15] = w[3] * z;
        }
        for (long st = 1; st < 512; st <<= 1)
          for (long c = 0; c + st < 512; c += 2 * st)
            for (int q = 0; q < 16; ++q) v[c * 16 + q] = v[c * 16 + q] + v[(c + st) * 16 + q];
        memcpy(S + s * 16, v, 16 * sizeof(double));
      }
      free(v);
    }
    for (long st = 1; st < P; st <<= 1)
      for (long c = 0; c + st < P; c += 2 * st)
        for (int q = 0; q < 16; ++q) S[c * 16 + q] = S[c * 16 + q] + S[(c + st) * 16 + q];
    double R[3], w[3];
    tmo_grav_am_solve(S, R, w);
    free(S);
#pragma omp parallel for schedule(static)
    for (long s = 0; s < nleaves; ++s) {
      const int d = leaves[4 * s] + 3;
      for (int c = 0; c < 512; ++c) {
        const long o = s * 512 + c;
        const double dx = centre(8L * leaves[4 * s + 1] + (c & 7), d) - R[0],
                     dy = centre(8L * leaves[4 * s + 2] + ((c >> 3) & 7), d) - R[1],
                     dz = centre(8L * leaves[4 * s + 3] + (c >> 6), d) - R[2];
        g[o] = g[o] + (w[1] * dz - w[2] * dy);
        g[ncell + o] = g[ncell + o] + (w[2] * dx - w[0] * dz);
        g[2 * ncell + o] = g[2 * ncell + o] + (w[0] * dy - w[1] * dx);
      }
    }
    PHASE("am");
  }
  return 0;
}

int tmo_grav_amr_sparse(long nleaves, const int* leaves, const double* mass, int flags, double* phi,
                        double* g, long* counts) {
  int rc = 0;
  tmo_grav_plan* P = tmo_grav_plan_create(nleaves, leaves, &rc);
  if (!P) return rc;
  rc = tmo_grav_plan_solve(P, mass, flags, phi, g, counts);
  tmo_grav_plan_destroy(P);
  return rc;
}
