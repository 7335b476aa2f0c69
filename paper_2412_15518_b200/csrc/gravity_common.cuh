// Device helpers shared by the uniform (gravity.cu) and AMR (gravity_amr.cu)
// FMM solvers: the operators of our gravity specification
// (oracle/gravity_oracle.c), with its exact operation order (-fmad=false).
#pragma once

#include "tmgpu_internal.h"

namespace tmgpu {
namespace {

__device__ __forceinline__ int s2(int i, int j) {
  return (i == 0) ? j : (i == 1) ? (j == 0 ? 1 : 2 + j) : (j == 0 ? 2 : 3 + j);
}

// The stencil approach: on a uniform level R depends only on
// the integer offset, so the geometry of each of the 7^3 offsets is computed
// once per level (tmo_grav_geom's exact operations) and the per-pair M2L
// reduces to the 28-FMA contraction. Entry: [ir, D1 x y z, D2 xx xy xz yy yz
// zz, D2/2 xx yy zz] = 13 doubles.
constexpr int kOff = 7, kOff3 = 343, kTab = 13;

__device__ __forceinline__ void m2l_geom(double x, double y, double z, double* __restrict__ e) {
  const double r2 = x * x + y * y + z * z;
  const double r = sqrt(r2);
  const double ir = 1.0 / r;
  const double ir2 = ir * ir;
  const double ir3 = ir * ir2, ir5 = ir3 * ir2;
  const double R[3] = {x, y, z};
  e[0] = ir;
#pragma unroll
  for (int i = 0; i < 3; ++i) e[1 + i] = -R[i] * ir3;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) e[4 + s2(i, j)] = 3.0 * R[i] * R[j] * ir5 - (i == j ? ir3 : 0.0);
  e[10] = 0.5 * e[4];
  e[11] = 0.5 * e[7];
  e[12] = 0.5 * e[9];
}

__global__ void stencil_table_kernel(double* __restrict__ tab, int D) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (D + 1) * kOff3) return;
  const int l = t / kOff3, o = t % kOff3;
  const int dx = o % kOff - 3, dy = (o / kOff) % kOff - 3, dz = o / (kOff * kOff) - 3;
  double* e = tab + (long long)t * kTab;
  if (dx == 0 && dy == 0 && dz == 0) {
    for (int q = 0; q < kTab; ++q) e[q] = 0.0;
    return;
  }
  const double h = 1.0 / (double)(1LL << l);
  m2l_geom(-(double)dx * h, -(double)dy * h, -(double)dz * h, e);
}

// One M2L term with known geometry, operation for operation tmo_grav_m2l_geom:
// the L0 increment is formed on its own and then added (27 FMAs, 1 mul, 1 add).
// nM = -M and nQ = -Q (negation is exact, and fma(-a, b, c) is the same
// correctly rounded operation either way).
__device__ __forceinline__ void m2l_acc(double nM, double Dx, double Dy, double Dz, double nQxx,
                                        double nQxy, double nQxz, double nQyy, double nQyz,
                                        double nQzz, const double* __restrict__ e, double out[10]) {
  double o = nM * e[0];
  o = fma(Dx, e[1], o);
  o = fma(Dy, e[2], o);
  o = fma(Dz, e[3], o);
  o = fma(nQxx, e[10], o);
  o = fma(nQxy, e[5], o);
  o = fma(nQxz, e[6], o);
  o = fma(nQyy, e[11], o);
  o = fma(nQyz, e[8], o);
  o = fma(nQzz, e[12], o);
  out[0] = out[0] + o;
  // D2 rows: x (xx xy xz) = e4 e5 e6, y (xy yy yz) = e5 e7 e8, z (xz yz zz) = e6 e8 e9
  out[1] = fma(Dz, e[6], fma(Dy, e[5], fma(Dx, e[4], fma(nM, e[1], out[1]))));
  out[2] = fma(Dz, e[8], fma(Dy, e[7], fma(Dx, e[5], fma(nM, e[2], out[2]))));
  out[3] = fma(Dz, e[9], fma(Dy, e[8], fma(Dx, e[6], fma(nM, e[3], out[3]))));
#pragma unroll
  for (int q = 0; q < 6; ++q) out[4 + q] = fma(nM, e[4 + q], out[4 + q]);
}

// m2l_acc without the L_ij terms (leaf targets: L2P reads only L0 and L_i;
// the other components' operations are unchanged)
__device__ __forceinline__ void m2l_tab4(const double* __restrict__ mom, const double* __restrict__ e,
                                         double out[4]) {
  const double nM = -mom[0], Dx = mom[1], Dy = mom[2], Dz = mom[3];
  double o = nM * e[0];
  o = fma(Dx, e[1], o);
  o = fma(Dy, e[2], o);
  o = fma(Dz, e[3], o);
  o = fma(-mom[4], e[10], o);
  o = fma(-mom[5], e[5], o);
  o = fma(-mom[6], e[6], o);
  o = fma(-mom[7], e[11], o);
  o = fma(-mom[8], e[8], o);
  o = fma(-mom[9], e[12], o);
  out[0] = out[0] + o;
  out[1] = fma(Dz, e[6], fma(Dy, e[5], fma(Dx, e[4], fma(nM, e[1], out[1]))));
  out[2] = fma(Dz, e[8], fma(Dy, e[7], fma(Dx, e[5], fma(nM, e[2], out[2]))));
  out[3] = fma(Dz, e[9], fma(Dy, e[8], fma(Dx, e[6], fma(nM, e[3], out[3]))));
}

__device__ __forceinline__ void m2l_tab(const double* __restrict__ mom, const double* __restrict__ e,
                                        double out[10]) {
  m2l_acc(-mom[0], mom[1], mom[2], mom[3], -mom[4], -mom[5], -mom[6], -mom[7], -mom[8], -mom[9], e,
          out);
}

// P2P geometry (tmo_grav_p2p_geom): w = [1/r, R/r^3]
__device__ __forceinline__ void p2p_geom(double Rx, double Ry, double Rz, double w[4]) {
  const double r2 = Rx * Rx + Ry * Ry + Rz * Rz;
  const double ir = 1.0 / sqrt(r2);
  const double ir3 = ir * ir * ir;
  w[0] = ir;
  w[1] = Rx * ir3;
  w[2] = Ry * ir3;
  w[3] = Rz * ir3;
}

__device__ __forceinline__ long long cidx(long long n, long long i, long long j, long long k) {
  return (k * n + j) * n + i;
}

// M2L with the geometry computed from R (tmo_grav_m2l), for the AMR W/X list
// pairs, whose offsets are not on the same-level stencil
__device__ __forceinline__ void m2l_direct(const double* __restrict__ mom, double x, double y,
                                           double z, double out[10]) {
  double e[kTab];
  m2l_geom(x, y, z, e);
  m2l_tab(mom, e, out);
}

// M2M of dense cell p of an n^3 level from its 8 children (level 2n)
__device__ __forceinline__ void m2m_cell(const double* __restrict__ child, double* __restrict__ parent,
                                         long long n, double hc, long long p) {
  {
    const long long I = p % n, J = (p / n) % n, K = p / (n * n);
    double o[10];
#pragma unroll
    for (int q = 0; q < 10; ++q) o[q] = 0.0;
    for (int c = 0; c < 2; ++c)
      for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 2; ++a) {
          const double s[3] = {(a - 0.5) * hc, (b - 0.5) * hc, (c - 0.5) * hc};
          const double* ch = child + cidx(2 * n, 2 * I + a, 2 * J + b, 2 * K + c) * 10;
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
    double* out = parent + p * 10;
#pragma unroll
    for (int q = 0; q < 10; ++q) out[q] = o[q];
  }
}

__global__ void m2m_kernel(const double* __restrict__ child, double* __restrict__ parent, long long n,
                           double hc) {
  const long long n3 = n * n * n;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n3;
       p += (long long)gridDim.x * blockDim.x)
    m2m_cell(child, parent, n, hc, p);
}

__global__ void __launch_bounds__(128) m2l_kernel(const double* __restrict__ mom,
                                                  double* __restrict__ loc, long long m,
                                                  const double* __restrict__ tab) {
  const long long n3 = m * m * m;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n3;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t % m, j = (t / m) % m, k = t / (m * m);
    double o[2][10];  // lower / upper three source planes (tmo_grav_solve)
#pragma unroll
    for (int q = 0; q < 10; ++q) o[0][q] = o[1][q] = 0.0;
    for (long long dz = -2 - (k & 1); dz <= 3 - (k & 1); ++dz)
      for (long long dy = -2 - (j & 1); dy <= 3 - (j & 1); ++dy)
        for (int pe = 0; pe < 2; ++pe)  /* even source x, then odd */
              for (long long dx = -2 - (i & 1) + pe; dx <= 3 - (i & 1); dx += 2) {
          if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1) continue;
          const long long si = i + dx, sj = j + dy, sk = k + dz;
          if (si < 0 || sj < 0 || sk < 0 || si >= m || sj >= m || sk >= m) continue;
          m2l_tab(mom + cidx(m, si, sj, sk) * 10,
                  tab + (((dz + 3) * kOff + (dy + 3)) * kOff + (dx + 3)) * kTab,
                  o[dz + (k & 1) >= 1]);
        }
    double* out = loc + t * 10;
#pragma unroll
    for (int q = 0; q < 10; ++q) out[q] = o[0][q] + o[1][q];
  }
}

__global__ void l2l_kernel(const double* __restrict__ parent, double* __restrict__ loc, long long m,
                           double h) {
  const long long n3 = m * m * m;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n3;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t % m, j = (t / m) % m, k = t / (m * m);
    const double s[3] = {((i & 1) - 0.5) * h, ((j & 1) - 0.5) * h, ((k & 1) - 0.5) * h};
    const double* L = parent + cidx(m / 2, i >> 1, j >> 1, k >> 1) * 10;
    double Lm[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) Lm[a][b] = L[4 + s2(a, b)];
    double t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) t1 += L[1 + a] * s[a];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) t2 += Lm[a][b] * s[a] * s[b];
    double sh[10];
    sh[0] = L[0] + t1 + 0.5 * t2;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double u = 0.0;
#pragma unroll
      for (int b = 0; b < 3; ++b) u += Lm[a][b] * s[b];
      sh[1 + a] = L[1 + a] + u;
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) sh[4 + q] = L[4 + q];
    double* out = loc + t * 10;
#pragma unroll
    for (int q = 0; q < 10; ++q) out[q] = sh[q] + out[q];
  }
}

unsigned grid_for(long long n) {
  long long b = (n + 127) / 128;
  if (b < 1) b = 1;
  if (b > 148 * 64) b = 148 * 64;
  return (unsigned)b;
}


}  // namespace
}  // namespace tmgpu
