// AMR cell-level FMM gravity over a forest (rows a12/a13 of SURVEY.md §8).
//
// Our specification (the reference has no gravity code), restated
// in oracle/gravity_amr_oracle.c and matched bitwise (-fmad=false): the
// classic adaptive FMM (U, V, W, X lists) on the cell tree of the forest,
// with the operators of the uniform solver (gravity_common.cuh). Layout: every
// forest node (leaf or internal) at level l is one 8^3 patch of cells at cell
// depth l + 3, AoS [node*512 + (k*8+j)*8+i][10] moments / locals per level;
// cell depths 0..2 are three tiny dense levels above the root patch.
//
//   amr_p2m     leaf cells: (m, 0, 0)                      one launch
//   amr_m2m     internal patches from their 8 child patches, per level
//   dense       depths 2..0: M2M, depth-2 M2L, depth-3 L2L (uniform kernels)
//   amr_m2l     per level, 4 CTAs per patch (8x4x4 targets each): the 12x8x8
//               source window gathered from the 27 neighbour patches into
//               shared memory (missing neighbours = zero moments), the 189-cell
//               V stencil with tabulated geometry, then the
//               target's W/X pairs (CSR) — fused, one write of the locals
//   amr_l2l     per level, parent local shifted + own M2L sum
//   amr_l2p     leaf cells: L2P + same-depth P2P over the 26 neighbours that
//               are leaf cells + cross-depth U pairs (CSR)
//   am_*        angular-momentum correction (our rigid-rotation
//               specification, tmo_grav_am_correct): per-slot adjacent-pair
//               tree (shuffles + shared memory), one-CTA tree over slots,
//               3x3 solve, apply
#include <cstring>
#include <string>
#include <vector>

#include "gravity_amr_plan.h"
#include "gravity_common.cuh"

namespace tmgpu {

struct GLv {
  double* mom;
  double* loc;
  const int* ijk;
  const int* nbr;
  const int* child;
  const int* parent;
  const int* leaf_slot;
  const long long* moff;
  const long long* ment;
  const long long* poff;
  const long long* pent;
};

namespace {

__device__ __forceinline__ double centre(long long gi, int d) {
  return ((double)gi + 0.5) / (double)(1LL << d);
}

__global__ void amr_mass_kernel(const double* __restrict__ arena, int V, long long nslots,
                                const int* __restrict__ slot_level, double* __restrict__ mass) {
  const long long total = nslots * 512;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long s = t >> 9;
    const int c = (int)(t & 511);
    const int i = c & 7, j = (c >> 3) & 7, k = c >> 6;
    const double h = 1.0 / (double)(8LL << slot_level[s]);
    const double dV = h * h * h;
    mass[t] = arena[s * V * 1728 + ((k + 2) * 12 + (j + 2)) * 12 + (i + 2)] * dV;
  }
}

__global__ void amr_p2m_kernel(const double* __restrict__ mass, long long nslots,
                               const int* __restrict__ slot_level, const int* __restrict__ slot_node,
                               const GLv* __restrict__ L) {
  const long long total = nslots * 512;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long s = t >> 9;
    const int c = (int)(t & 511);
    double* o = L[slot_level[s]].mom + ((long long)slot_node[s] * 512 + c) * 10;
    o[0] = mass[t];
#pragma unroll
    for (int q = 1; q < 10; ++q) o[q] = 0.0;
  }
}

__global__ void amr_m2m_kernel(const GLv* __restrict__ L, int l, const int* __restrict__ internal,
                               long long n_int) {
  const GLv P = L[l], Ch = L[l + 1];
  const double hc = 1.0 / (double)(1LL << (l + 4));
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n_int * 512;
       t += (long long)gridDim.x * blockDim.x) {
    const int n = internal[t >> 9];
    const int c = (int)(t & 511);
    const int I = c & 7, J = (c >> 3) & 7, K = c >> 6;
    const int cn = P.child[n * 8 + ((K >> 2) * 2 + (J >> 2)) * 2 + (I >> 2)];
    const double* base = Ch.mom + (long long)cn * 512 * 10;
    double o[10];
#pragma unroll
    for (int q = 0; q < 10; ++q) o[q] = 0.0;
    for (int cc = 0; cc < 2; ++cc)
      for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 2; ++a) {
          const double s[3] = {(a - 0.5) * hc, (b - 0.5) * hc, (cc - 0.5) * hc};
          const int ci = ((2 * I) & 7) + a, cj = ((2 * J) & 7) + b, ck = ((2 * K) & 7) + cc;
          const double* ch = base + ((ck * 8 + cj) * 8 + ci) * 10;
          const double M = ch[0];
          o[0] += M;
#pragma unroll
          for (int i = 0; i < 3; ++i) o[1 + i] += ch[1 + i] + M * s[i];
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = i; j < 3; ++j)
              o[4 + s2(i, j)] += ch[4 + s2(i, j)] + ch[1 + i] * s[j] + s[i] * ch[1 + j] + M * s[i] * s[j];
        }
    double* out = P.mom + ((long long)n * 512 + c) * 10;
#pragma unroll
    for (int q = 0; q < 10; ++q) out[q] = o[q];
  }
}

// M2L of one level: CTA = (patch, z-half of 8x8x4 targets), 256 threads.
// Warp w owns the 32 targets of one parity class (a, b, c) = (w&1, w>>1&1,
// w>>2): lane (I, J, K) -> target (2I+a, 2J+b, z0+2K+c). Every lane of a warp
// then walks the same stencil offsets (no divergence; the tabulated geometry
// is a warp-uniform broadcast load). The 12x12x8 source window (27-patch
// neighbourhood, missing patches = zero moments) is stored de-interleaved by
// parity: 8 sub-grids of 6x6x4 cells with row pitch 6 and plane pitch 40, so a
// warp's 32 source loads of any offset hit 32 distinct banks (2 wavefronts).
constexpr int kSubPitchY = 6, kSubPitchZ = 40, kSub = 4 * kSubPitchZ, kWin = 8 * kSub;  // 1280

__device__ __forceinline__ int win_index(int wx, int wy, int wz) {
  return ((((wz & 1) * 2 + (wy & 1)) * 2 + (wx & 1)) * kSub) + (wz >> 1) * kSubPitchZ +
         (wy >> 1) * kSubPitchY + (wx >> 1);
}

__global__ void __launch_bounds__(256, 2) amr_m2l_kernel(const GLv* __restrict__ Lv, int l,
                                                         const double* __restrict__ tab) {
  extern __shared__ double sm[];  // [10][kWin] doubles = 102,400 B
  const GLv L = Lv[l];
  const int n = blockIdx.x >> 1;
  const int z0 = (blockIdx.x & 1) * 4;
  const int* nb27 = L.nbr + (long long)n * 27;
  for (int q = threadIdx.x; q < 12 * 12 * 8; q += blockDim.x) {
    const int wx = q % 12, wy = (q / 12) % 12, wz = q / 144;
    int lx = wx - 2, ly = wy - 2, lz = z0 + wz - 2;
    const int ox = lx < 0 ? -1 : (lx > 7 ? 1 : 0), oy = ly < 0 ? -1 : (ly > 7 ? 1 : 0),
              oz = lz < 0 ? -1 : (lz > 7 ? 1 : 0);
    lx -= 8 * ox, ly -= 8 * oy, lz -= 8 * oz;
    const int nb = nb27[((oz + 1) * 3 + (oy + 1)) * 3 + ox + 1];
    const double* src = L.mom + ((long long)(nb < 0 ? 0 : nb) * 512 + (lz * 8 + ly) * 8 + lx) * 10;
    const int w = win_index(wx, wy, wz);
#pragma unroll
    for (int c = 0; c < 10; ++c) sm[c * kWin + w] = nb >= 0 ? src[c] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = warp & 1, b = (warp >> 1) & 1, c = warp >> 2;
  // half-warps take J even / J odd: with the (6, 40) sub-grid pitches every
  // half-warp's 16 doubles then fall in 16 distinct banks for every offset
  const int I = lane & 3, K = (lane >> 2) & 1, J = ((lane >> 3) & 1) * 2 + (lane >> 4);
  const int i = 2 * I + a, j = 2 * J + b, k = z0 + 2 * K + c;
  const int lane_off = K * kSubPitchZ + J * kSubPitchY + I;
  double o[10];
#pragma unroll
  for (int q = 0; q < 10; ++q) o[q] = 0.0;
  for (int dz = -2 - c; dz <= 3 - c; ++dz)
    for (int dy = -2 - b; dy <= 3 - b; ++dy)
      for (int dx = -2 - a; dx <= 3 - a; ++dx) {
        if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1) continue;
        // window coordinates of the source: (t + d) + 2 (z relative to z0)
        const int sx = a + dx + 2, sy = b + dy + 2, sz = c + dz + 2;  // + 2*(I, J, K)
        const int q = ((((sz & 1) * 2 + (sy & 1)) * 2 + (sx & 1)) * kSub) + (sz >> 1) * kSubPitchZ +
                      (sy >> 1) * kSubPitchY + (sx >> 1) + lane_off;
        double mom_q[10];
#pragma unroll
        for (int cc = 0; cc < 10; ++cc) mom_q[cc] = sm[cc * kWin + q];
        m2l_tab10(mom_q, tab + (((dz + 3) * kOff + (dy + 3)) * kOff + (dx + 3)) * kTab10, o);
      }
  const long long flat = (long long)n * 512 + (k * 8 + j) * 8 + i;
  const long long e0 = L.moff[flat], e1 = L.moff[flat + 1];
  if (e0 < e1) {  // W/X pairs (AMR level jumps), sorted by source
    const int d = l + 3;
    const double cx = centre(8LL * L.ijk[3 * n] + i, d), cy = centre(8LL * L.ijk[3 * n + 1] + j, d),
                 cz = centre(8LL * L.ijk[3 * n + 2] + k, d);
    for (long long e = e0; e < e1; ++e) {
      const long long enc = L.ment[e];
      const int sl = (int)(enc >> 40);
      const long long sf = enc & ((1LL << 40) - 1);
      const GLv S = Lv[sl];
      const long long sn = sf >> 9;
      const int sc = (int)(sf & 511);
      const int sd = sl + 3;
      const double sx = centre(8LL * S.ijk[3 * sn] + (sc & 7), sd),
                   sy = centre(8LL * S.ijk[3 * sn + 1] + ((sc >> 3) & 7), sd),
                   sz = centre(8LL * S.ijk[3 * sn + 2] + (sc >> 6), sd);
      m2l_direct(S.mom + sf * 10, cx - sx, cy - sy, cz - sz, o);
    }
  }
  double* out = L.loc + flat * 10;
#pragma unroll
  for (int q = 0; q < 10; ++q) out[q] = o[q];
}

__global__ void amr_l2l_kernel(const GLv* __restrict__ Lv, int l, long long nnodes) {
  const GLv L = Lv[l], P = Lv[l - 1];
  const double h = 1.0 / (double)(1LL << (l + 3));
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nnodes * 512;
       t += (long long)gridDim.x * blockDim.x) {
    const long long n = t >> 9;
    const int c = (int)(t & 511);
    const int i = c & 7, j = (c >> 3) & 7, k = c >> 6;
    const int pn = L.parent[n];
    const int pi = (L.ijk[3 * n] & 1) * 4 + (i >> 1), pj = (L.ijk[3 * n + 1] & 1) * 4 + (j >> 1),
              pk = (L.ijk[3 * n + 2] & 1) * 4 + (k >> 1);
    const double* Lp = P.loc + ((long long)pn * 512 + (pk * 8 + pj) * 8 + pi) * 10;
    const double s[3] = {((i & 1) - 0.5) * h, ((j & 1) - 0.5) * h, ((k & 1) - 0.5) * h};
    double Lm[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) Lm[a][b] = Lp[4 + s2(a, b)];
    double t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) t1 += Lp[1 + a] * s[a];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) t2 += Lm[a][b] * s[a] * s[b];
    double sh[10];
    sh[0] = Lp[0] + t1 + 0.5 * t2;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double u = 0.0;
#pragma unroll
      for (int b = 0; b < 3; ++b) u += Lm[a][b] * s[b];
      sh[1 + a] = Lp[1 + a] + u;
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) sh[4 + q] = Lp[4 + q];
    double* out = L.loc + t * 10;
#pragma unroll
    for (int q = 0; q < 10; ++q) out[q] = sh[q] + out[q];
  }
}

// L2P + P2P at the leaf cells, output by canonical slot: phi[s*512 + c],
// g[q*ncell + s*512 + c]
__global__ void amr_l2p_kernel(const GLv* __restrict__ Lv, long long nslots,
                               const int* __restrict__ slot_level, const int* __restrict__ slot_node,
                               double* __restrict__ phi, double* __restrict__ g) {
  const long long ncell = nslots * 512;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ncell;
       t += (long long)gridDim.x * blockDim.x) {
    const long long s = t >> 9;
    const int c = (int)(t & 511);
    const int i = c & 7, j = (c >> 3) & 7, k = c >> 6;
    const int l = slot_level[s], n = slot_node[s];
    const GLv L = Lv[l];
    const int d = l + 3;
    const double h = 1.0 / (double)(1LL << d);
    const long long flat = (long long)n * 512 + c;
    const double* Lc = L.loc + flat * 10;
    double p = Lc[0], gx = -Lc[1], gy = -Lc[2], gz = -Lc[3];
    const int* nb27 = L.nbr + (long long)n * 27;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (!dx && !dy && !dz) continue;
          int lx = i + dx, ly = j + dy, lz = k + dz;
          const int ox = lx < 0 ? -1 : (lx > 7 ? 1 : 0), oy = ly < 0 ? -1 : (ly > 7 ? 1 : 0),
                    oz = lz < 0 ? -1 : (lz > 7 ? 1 : 0);
          lx -= 8 * ox, ly -= 8 * oy, lz -= 8 * oz;
          const int nb = nb27[((oz + 1) * 3 + (oy + 1)) * 3 + ox + 1];
          if (nb < 0 || L.leaf_slot[nb] < 0) continue;
          const double ms = L.mom[((long long)nb * 512 + (lz * 8 + ly) * 8 + lx) * 10];
          const double Rx = -(double)dx * h, Ry = -(double)dy * h, Rz = -(double)dz * h;
          const double r2 = Rx * Rx + Ry * Ry + Rz * Rz;
          const double ir = 1.0 / sqrt(r2);
          const double ir3 = ir * ir * ir;
          p -= ms * ir;
          gx -= ms * Rx * ir3;
          gy -= ms * Ry * ir3;
          gz -= ms * Rz * ir3;
        }
    const long long e0 = L.poff[flat], e1 = L.poff[flat + 1];
    if (e0 < e1) {
      const double cx = centre(8LL * L.ijk[3 * n] + i, d), cy = centre(8LL * L.ijk[3 * n + 1] + j, d),
                   cz = centre(8LL * L.ijk[3 * n + 2] + k, d);
      for (long long e = e0; e < e1; ++e) {
        const long long enc = L.pent[e];
        const int sl = (int)(enc >> 40);
        const long long sf = enc & ((1LL << 40) - 1);
        const GLv S = Lv[sl];
        const long long sn = sf >> 9;
        const int sc = (int)(sf & 511);
        const int sd = sl + 3;
        const double ms = S.mom[sf * 10];
        const double Rx = cx - centre(8LL * S.ijk[3 * sn] + (sc & 7), sd),
                     Ry = cy - centre(8LL * S.ijk[3 * sn + 1] + ((sc >> 3) & 7), sd),
                     Rz = cz - centre(8LL * S.ijk[3 * sn + 2] + (sc >> 6), sd);
        const double r2 = Rx * Rx + Ry * Ry + Rz * Rz;
        const double ir = 1.0 / sqrt(r2);
        const double ir3 = ir * ir * ir;
        p -= ms * ir;
        gx -= ms * Rx * ir3;
        gy -= ms * Ry * ir3;
        gz -= ms * Rz * ir3;
      }
    }
    phi[t] = p;
    g[t] = gx;
    g[ncell + t] = gy;
    g[2 * ncell + t] = gz;
  }
}

// ---- angular-momentum correction (tmo_grav_am_correct) ---------------------

__device__ __forceinline__ void cell_pos(const GLv* __restrict__ Lv, int l, int n, int c, double x[3]) {
  const GLv L = Lv[l];
  const int d = l + 3;
  x[0] = centre(8LL * L.ijk[3 * n] + (c & 7), d);
  x[1] = centre(8LL * L.ijk[3 * n + 1] + ((c >> 3) & 7), d);
  x[2] = centre(8LL * L.ijk[3 * n + 2] + (c >> 6), d);
}

// one CTA (512 threads) per slot: adjacent-pair tree over its 512 cells
__global__ void __launch_bounds__(512) am_slot_kernel(const GLv* __restrict__ Lv, long long nslots,
                                                      const int* __restrict__ slot_level,
                                                      const int* __restrict__ slot_node,
                                                      const double* __restrict__ mass,
                                                      const double* __restrict__ g,
                                                      double* __restrict__ part) {
  __shared__ double red[16][16];  // [warp][value]
  const long long s = blockIdx.x;
  const int c = threadIdx.x;
  const long long ncell = nslots * 512, t = s * 512 + c;
  double x[3];
  cell_pos(Lv, slot_level[s], slot_node[s], c, x);
  const double m = mass[t], gx = g[t], gy = g[ncell + t], gz = g[2 * ncell + t];
  double v[16];
  v[0] = m;
  v[1] = m * x[0];
  v[2] = m * x[1];
  v[3] = m * x[2];
  v[4] = m * gx;
  v[5] = m * gy;
  v[6] = m * gz;
  v[7] = m * (x[1] * gz - x[2] * gy);
  v[8] = m * (x[2] * gx - x[0] * gz);
  v[9] = m * (x[0] * gy - x[1] * gx);
  v[10] = v[1] * x[0];
  v[11] = v[1] * x[1];
  v[12] = v[1] * x[2];
  v[13] = v[2] * x[1];
  v[14] = v[2] * x[2];
  v[15] = v[3] * x[2];
  const int lane = c & 31, warp = c >> 5;
#pragma unroll
  for (int st = 1; st < 32; st <<= 1)
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const double o = __shfl_down_sync(0xffffffffu, v[q], st);
      if ((lane & (2 * st - 1)) == 0) v[q] = v[q] + o;
    }
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 16; ++q) red[warp][q] = v[q];
  __syncthreads();
  if (c < 16) {  // thread q: tree over the 16 warps for value q
    double w[16];
#pragma unroll
    for (int a = 0; a < 16; ++a) w[a] = red[a][c];
#pragma unroll
    for (int st = 1; st < 16; st <<= 1)
#pragma unroll
      for (int a = 0; a < 16; a += 2 * st) w[a] = w[a] + w[a + st];
    part[s * 16 + c] = w[0];
  }
}

// adjacent-pair tree over n (power of two) entries of 16 sums: each CTA
// reduces a chunk of min(n, 256) consecutive entries (the first levels of the
// global tree) into out[blockIdx.x]
__global__ void __launch_bounds__(256) am_tree_pass_kernel(const double* __restrict__ in,
                                                           double* __restrict__ out, long long n) {
  __shared__ double v[256][17];
  const int chunk = n < 256 ? (int)n : 256;
  const long long base = (long long)blockIdx.x * chunk;
  const int t = threadIdx.x;
  if (t < chunk)
#pragma unroll
    for (int q = 0; q < 16; ++q) v[t][q] = in[(base + t) * 16 + q];
  __syncthreads();
  for (int st = 1; st < chunk; st <<= 1) {
    if (t < chunk && (t & (2 * st - 1)) == 0)
#pragma unroll
      for (int q = 0; q < 16; ++q) v[t][q] = v[t][q] + v[t + st][q];
    __syncthreads();
  }
  if (t < 16) out[(long long)blockIdx.x * 16 + t] = v[0][t];
}

// the 3x3 solve of tmo_grav_am_solve on the total sums S -> rw = (R, w, S)
__global__ void am_solve_kernel(const double* __restrict__ part, double* __restrict__ rw) {
  if (threadIdx.x != 0) return;
  const double* S = part;
  double R[3], w[3];
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
  } else {
    const double b0 = -tau[0], b1 = -tau[1], b2 = -tau[2];
    w[0] = ((a00 * b0 + a01 * b1) + a02 * b2) / det;
    w[1] = ((a01 * b0 + a11 * b1) + a12 * b2) / det;
    w[2] = ((a02 * b0 + a12 * b1) + a22 * b2) / det;
  }
  for (int q = 0; q < 3; ++q) rw[q] = R[q], rw[3 + q] = w[q];
  for (int q = 0; q < 16; ++q) rw[6 + q] = S[q];
}

__global__ void am_apply_kernel(const GLv* __restrict__ Lv, long long nslots,
                                const int* __restrict__ slot_level, const int* __restrict__ slot_node,
                                const double* __restrict__ rw, double* __restrict__ g) {
  const long long ncell = nslots * 512;
  const double R0 = rw[0], R1 = rw[1], R2 = rw[2], w0 = rw[3], w1 = rw[4], w2 = rw[5];
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ncell;
       t += (long long)gridDim.x * blockDim.x) {
    const long long s = t >> 9;
    double x[3];
    cell_pos(Lv, slot_level[s], slot_node[s], (int)(t & 511), x);
    const double dx = x[0] - R0, dy = x[1] - R1, dz = x[2] - R2;
    g[t] = g[t] + (w1 * dz - w2 * dy);
    g[ncell + t] = g[ncell + t] + (w2 * dx - w0 * dz);
    g[2 * ncell + t] = g[2 * ncell + t] + (w0 * dy - w1 * dx);
  }
}

template <class T>
cudaError_t upload(const std::vector<T>& v, T** out) {
  *out = nullptr;
  if (v.empty()) return cudaSuccess;
  cudaError_t e = cudaMalloc(out, v.size() * sizeof(T));
  if (e == cudaSuccess) e = cudaMemcpy(*out, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

}  // namespace

struct GravAmrWork {
  GravPlan plan;
  std::vector<GLv> host_lv;
  std::vector<void*> allocs;
  GLv* dev_lv = nullptr;
  int* slot_level = nullptr;
  int* slot_node = nullptr;
  std::vector<int*> internal;
  double* dmom[3] = {nullptr, nullptr, nullptr};
  double* dloc[3] = {nullptr, nullptr, nullptr};
  double* tab = nullptr;
  double* tab10 = nullptr;
  double* mass = nullptr;
  double* part = nullptr;   // [P][16] + rw[22]
  double* part2 = nullptr;  // [P/256 + 1][16] tree scratch
  long long nslots = 0, P = 1;
  long long nodes = 0;
};

}  // namespace tmgpu

using namespace tmgpu;

struct tmgpu_gravity_amr {
  GravAmrWork w;
};

extern "C" {

void tmgpu_gravity_amr_destroy(tmgpu_gravity_amr* G) {
  if (!G) return;
  for (void* p : G->w.allocs)
    if (p) cudaFree(p);
  delete G;
}

tmgpu_gravity_amr* tmgpu_gravity_amr_create(const int* leaves, long long nleaves, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  auto* G = new tmgpu_gravity_amr;
  GravAmrWork& w = G->w;
  std::string why;
  if (!build_grav_plan(leaves, nleaves, w.plan, &why)) {
    set_err(err, TMGPU_ERR_INVALID, why.c_str());
    delete G;
    return nullptr;
  }
  const GravPlan& P = w.plan;
  w.nslots = nleaves;
  while (w.P < nleaves) w.P <<= 1;
  cudaError_t e = cudaSuccess;
  auto track = [&](void* p) { w.allocs.push_back(p); };
  w.host_lv.resize(P.nlevels);
  w.internal.assign(P.nlevels, nullptr);
  for (int l = 0; l < P.nlevels && e == cudaSuccess; ++l) {
    const GravLevel& L = P.lv[l];
    GLv& g = w.host_lv[l];
    std::memset(&g, 0, sizeof(g));
    const size_t ncell = (size_t)L.n * 512;
    w.nodes += L.n;
    e = cudaMalloc(&g.mom, ncell * 10 * sizeof(double));
    track(g.mom);
    if (e == cudaSuccess) e = cudaMalloc(&g.loc, ncell * 10 * sizeof(double)), track(g.loc);
    int *ijk, *nbr, *child, *parent, *slot, *inter;
    long long *moff, *ment, *poff, *pent;
    if (e == cudaSuccess) e = upload(L.ijk, &ijk), track(ijk);
    if (e == cudaSuccess) e = upload(L.nbr, &nbr), track(nbr);
    if (e == cudaSuccess) e = upload(L.child, &child), track(child);
    if (e == cudaSuccess) e = upload(L.parent, &parent), track(parent);
    if (e == cudaSuccess) e = upload(L.leaf_slot, &slot), track(slot);
    if (e == cudaSuccess) e = upload(L.internal, &inter), track(inter);
    static_assert(sizeof(long long) == sizeof(int64_t), "int64");
    if (e == cudaSuccess)
      e = upload(reinterpret_cast<const std::vector<long long>&>(L.moff), &moff), track(moff);
    if (e == cudaSuccess)
      e = upload(reinterpret_cast<const std::vector<long long>&>(L.ment), &ment), track(ment);
    if (e == cudaSuccess)
      e = upload(reinterpret_cast<const std::vector<long long>&>(L.poff), &poff), track(poff);
    if (e == cudaSuccess)
      e = upload(reinterpret_cast<const std::vector<long long>&>(L.pent), &pent), track(pent);
    if (e != cudaSuccess) break;
    g.ijk = ijk, g.nbr = nbr, g.child = child, g.parent = parent, g.leaf_slot = slot;
    g.moff = moff, g.ment = ment, g.poff = poff, g.pent = pent;
    w.internal[l] = inter;
  }
  if (e == cudaSuccess) e = cudaMalloc(&w.dev_lv, P.nlevels * sizeof(GLv)), track(w.dev_lv);
  if (e == cudaSuccess)
    e = cudaMemcpy(w.dev_lv, w.host_lv.data(), P.nlevels * sizeof(GLv), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = upload(P.slot_level, &w.slot_level), track(w.slot_level);
  if (e == cudaSuccess) e = upload(P.slot_node, &w.slot_node), track(w.slot_node);
  for (int d = 0; d < 3 && e == cudaSuccess; ++d) {
    const size_t n3 = (size_t)1 << (3 * d);
    e = cudaMalloc(&w.dmom[d], n3 * 10 * sizeof(double));
    track(w.dmom[d]);
    if (e == cudaSuccess) e = cudaMalloc(&w.dloc[d], n3 * 10 * sizeof(double)), track(w.dloc[d]);
  }
  const int Dmax = P.nlevels - 1 + 3;
  if (e == cudaSuccess) e = cudaMalloc(&w.tab, (size_t)(Dmax + 1) * kOff3 * kTab * sizeof(double)), track(w.tab);
  if (e == cudaSuccess) e = cudaMalloc(&w.tab10, (size_t)(Dmax + 1) * kOff3 * kTab10 * sizeof(double)), track(w.tab10);
  if (e == cudaSuccess) e = cudaMalloc(&w.mass, (size_t)w.nslots * 512 * sizeof(double)), track(w.mass);
  if (e == cudaSuccess) e = cudaMalloc(&w.part, ((size_t)w.P * 16 + 22) * sizeof(double)), track(w.part);
  if (e == cudaSuccess) e = cudaMalloc(&w.part2, ((size_t)w.P / 256 + 1) * 16 * sizeof(double)), track(w.part2);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(amr_m2l_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(10 * kWin * sizeof(double)));
  if (e == cudaSuccess) {
    stencil_table_kernel<<<((Dmax + 1) * kOff3 + 127) / 128, 128>>>(w.tab, Dmax);
    table10_kernel<<<((Dmax + 1) * kOff3 + 127) / 128, 128>>>(w.tab, w.tab10, (Dmax + 1) * kOff3);
    g_launches.fetch_add(2, std::memory_order_relaxed);
    e = cudaDeviceSynchronize();
  }
  if (e != cudaSuccess) {
    cuda_err(err, e, "tmgpu_gravity_amr_create");
    tmgpu_gravity_amr_destroy(G);
    return nullptr;
  }
  return G;
}

int tmgpu_gravity_amr_info(const tmgpu_gravity_amr* G, long long* out) {
  if (!G || !out) return TMGPU_ERR_INVALID;
  out[0] = G->w.plan.nlevels;
  out[1] = G->w.nodes;
  out[2] = G->w.plan.m_entries;
  out[3] = G->w.plan.p_entries;
  return TMGPU_OK;
}

// Host-only: build the plan and report info[4] without touching the GPU.
int tmgpu_gravity_amr_plan_info(const int* leaves, long long nleaves, long long* out,
                                tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  GravPlan P;
  std::string why;
  if (!build_grav_plan(leaves, nleaves, P, &why)) return set_err(err, TMGPU_ERR_INVALID, why.c_str());
  long long nodes = 0;
  for (const auto& L : P.lv) nodes += L.n;
  out[0] = P.nlevels;
  out[1] = nodes;
  out[2] = P.m_entries;
  out[3] = P.p_entries;
  return TMGPU_OK;
}

int tmgpu_gravity_amr_mass_from_arena(tmgpu_gravity_amr* G, const double* arena, int vars,
                                      void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  GravAmrWork& w = G->w;
  cudaStream_t st = as_stream(stream);
  amr_mass_kernel<<<grid_for(w.nslots * 512), 128, 0, st>>>(arena, vars, w.nslots, w.slot_level, w.mass);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_err(err, cudaGetLastError(), "tmgpu_gravity_amr_mass_from_arena");
}

int tmgpu_gravity_amr_solve(tmgpu_gravity_amr* G, const double* mass, double* phi, double* g,
                            int flags, void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  GravAmrWork& w = G->w;
  const GravPlan& P = w.plan;
  cudaStream_t st = as_stream(stream);
  const long long ncell = w.nslots * 512;
  const bool host = (flags & TMGPU_HOST_PTRS) != 0;
  cudaError_t e = cudaSuccess;
  double *dphi = phi, *dg = g;
  if (mass)
    e = cudaMemcpyAsync(w.mass, mass, ncell * sizeof(double),
                        host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st);
  if (host && e == cudaSuccess) {
    e = cudaMallocAsync(&dphi, ncell * sizeof(double), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&dg, 3 * ncell * sizeof(double), st);
  }
  if (e == cudaSuccess) {
    long long launches = 0;
    amr_p2m_kernel<<<grid_for(ncell), 128, 0, st>>>(w.mass, w.nslots, w.slot_level, w.slot_node, w.dev_lv);
    ++launches;
    for (int l = P.nlevels - 2; l >= 0; --l) {
      const long long ni = (long long)P.lv[l].internal.size();
      if (!ni) continue;
      amr_m2m_kernel<<<grid_for(ni * 512), 128, 0, st>>>(w.dev_lv, l, w.internal[l], ni);
      ++launches;
    }
    m2m_kernel<<<1, 128, 0, st>>>(w.host_lv[0].mom, w.dmom[2], 4, 1.0 / 8.0);
    m2m_kernel<<<1, 128, 0, st>>>(w.dmom[2], w.dmom[1], 2, 1.0 / 4.0);
    m2m_kernel<<<1, 128, 0, st>>>(w.dmom[1], w.dmom[0], 1, 1.0 / 2.0);
    m2l_kernel<<<1, 128, 0, st>>>(w.dmom[2], w.dloc[2], 4, w.tab + 2LL * kOff3 * kTab);
    launches += 4;
    for (int l = 0; l < P.nlevels; ++l) {
      amr_m2l_kernel<<<(unsigned)(P.lv[l].n * 2), 256, 10 * kWin * sizeof(double), st>>>(
          w.dev_lv, l, w.tab10 + (long long)(l + 3) * kOff3 * kTab10);
      ++launches;
    }
    l2l_kernel<<<grid_for(512), 128, 0, st>>>(w.dloc[2], w.host_lv[0].loc, 8, 1.0 / 8.0);
    ++launches;
    for (int l = 1; l < P.nlevels; ++l) {
      amr_l2l_kernel<<<grid_for((long long)P.lv[l].n * 512), 128, 0, st>>>(w.dev_lv, l, P.lv[l].n);
      ++launches;
    }
    amr_l2p_kernel<<<grid_for(ncell), 128, 0, st>>>(w.dev_lv, w.nslots, w.slot_level, w.slot_node,
                                                    dphi, dg);
    ++launches;
    if (flags & TMGPU_GRAV_AM) {
      e = cudaMemsetAsync(w.part, 0, (size_t)w.P * 16 * sizeof(double), st);
      am_slot_kernel<<<(unsigned)w.nslots, 512, 0, st>>>(w.dev_lv, w.nslots, w.slot_level, w.slot_node,
                                                         w.mass, dg, w.part);
      double* bufs[2] = {w.part, w.part2};
      int cur = 0;
      for (long long n = w.P; n > 1;) {
        const long long chunk = n < 256 ? n : 256;
        am_tree_pass_kernel<<<(unsigned)(n / chunk), 256, 0, st>>>(bufs[cur], bufs[cur ^ 1], n);
        n /= chunk;
        cur ^= 1;
        ++launches;
      }
      am_solve_kernel<<<1, 32, 0, st>>>(bufs[cur], w.part + w.P * 16);
      am_apply_kernel<<<grid_for(ncell), 128, 0, st>>>(w.dev_lv, w.nslots, w.slot_level, w.slot_node,
                                                       w.part + w.P * 16, dg);
      launches += 3;
    }
    g_launches.fetch_add(launches, std::memory_order_relaxed);
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  if (host) {
    if (e == cudaSuccess) e = cudaMemcpyAsync(phi, dphi, ncell * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g, dg, 3 * ncell * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (dphi && dphi != phi) cudaFreeAsync(dphi, st);
    if (dg && dg != g) cudaFreeAsync(dg, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = e2;
  } else if (!(flags & TMGPU_ASYNC)) {
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = e2;
  }
  return cuda_err(err, e, "tmgpu_gravity_amr_solve");
}

// AM-correction sums of the last solve with TMGPU_GRAV_AM: out[0..2] centre of
// mass, [3..5] w, [6..21] the 16 sums (tests).
int tmgpu_gravity_amr_am_stats(tmgpu_gravity_amr* G, double* out) {
  if (!G || !out) return TMGPU_ERR_INVALID;
  return cudaMemcpy(out, G->w.part + G->w.P * 16, 22 * sizeof(double), cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? TMGPU_OK
             : TMGPU_ERR_CUDA;
}

// Leaf-cell masses currently in the workspace ([slot][512], device pointer).
const double* tmgpu_gravity_amr_mass_ptr(const tmgpu_gravity_amr* G) { return G ? G->w.mass : nullptr; }

}  // extern "C"
