// Aggregated hydro stage kernel for sm_100a, FP64.
//
// Restates reference proj/src/hydro/stage.cpp:93-218 (stage_impl) with
// euler.hpp:27-137 (MUSCL-minmod "PPM slot" + Rusanov/KT flux) for
// E=8, G=2 (S=12) sub-grids; one CTA = one sub-grid, any number of
// sub-grids (slices) per launch (the paper's kernel aggregation).
//
// Data flow per CTA
//   1. TMA (cp.async.bulk.tensor, 5-D map over [slice][var][z][y][x]) stages
//      exactly the cells the stage reads: the 12x8x8 x-pencil box plus four
//      8x2x8 / 8x8x2 face-ghost slabs = 1280 cells x V vars (51.2 KB at V=5).
//      Edge/corner ghosts are never read by the reference stage (its
//      pencils are tangential-interior, stage.cpp:131-140), so never loaded.
//   2. cons -> prim in place, once per staged cell (the reference converts
//      every pencil cell per axis, stage.cpp:141-153; each cell's primitive
//      is a pure function of its own conserved values, so converting once is
//      bitwise identical). Interior conserved values seed the accumulator.
//   3. per axis x,y,z: 64 pencils x 9 faces; each of 192 lanes evaluates 3
//      consecutive faces of one pencil; the 9th-face neighbour flux comes
//      from the next lane by warp shuffle; the lane applies
//      acc -= cdt*(F[c0+1]-F[c0]) to its cells after a block barrier, so per
//      cell the update order is x, then y, then z exactly as stage.cpp:166-183.
//   4. epilogue per cell: floors (stage.cpp:187-208), non-finite check
//      (stage.cpp:209-216), optional SSP-RK3 combine (rk3.hpp:18-27), store.
//
// BITWISE (compiled with -fmad=false): every + - * / sqrt is one IEEE
// round-to-nearest op in the reference's association order; fmax/fmin are not
// used (vmax is `x > f ? x : f`, std::max is `(a < b) ? b : a`).
// FAST: reciprocal reuse + FMA; parity within 1e-10 of the per-variable scale.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tmgpu_internal.h"

namespace tmgpu {

constexpr int kE = 8, kG = 2, kS = 12;
constexpr int kE2 = 64, kE3 = 512;
constexpr int kStageThreads = 256;  // 8 warps: the face passes use 7 (30 lanes x 7 >= 64 pencils x 3 segments), the cell phases all 8
constexpr double kRhoFloor = 1e-10;       // euler.hpp:15
constexpr double kPressureFloor = 1e-12;  // euler.hpp:16

// Staged smem layout (doubles), var-major inside each TMA box:
//   B0 [V][8 z][8 y][10 x]  x in [2,12): interior plus two never-read columns,
//                           so the 80-byte row stride spreads the pencil loads
//                           of neighbouring lanes over the banks (the box start
//                           stays 16-byte aligned)
//   XL [V][8 z][8 y][2 x]  x in {0,1}     XH  x in {10,11}
//   YL [V][8 z][2 y][8 x]  y in {0,1}     YH  y in {10,11}
//   ZL [V][2 z][8 y][8 x]  z in {0,1}     ZH  z in {10,11}
// Each face slab is TMA-loaded either from the leaf's own ghost cells or,
// for a same-level neighbour, straight from the neighbour's interior
// (StageLaunch::face_src): the same-level ghost copy is fused into the load.
// Accumulator layout: x rows of 8 cells at a pitch of 9 doubles, so the x-axis
// update (lanes on consecutive (y, z) pencils) hits distinct banks instead of
// the two a row pitch of 8 would give; y and z updates stay unit-stride.
constexpr int kAccV = 64 * 9;  // per var
__device__ __forceinline__ int acc_at(int c) { return (c >> 3) * 9 + (c & 7); }

template <int V>
struct Lay {
  static constexpr int B0 = 0;
  static constexpr int XL = V * 640;
  static constexpr int XH = XL + V * 128;
  static constexpr int YL = XH + V * 128;
  static constexpr int YH = YL + V * 128;
  static constexpr int ZL = YH + V * 128;
  static constexpr int ZH = ZL + V * 128;
  static constexpr int kStaged = ZH + V * 128;  // = V*1408 doubles
  static constexpr int kAcc = kStaged;          // accumulator [V][64 rows][9] (acc_at)
  // RK3 u0 block [V][E^3]: bulk-copied over the x and y face slabs (XL..YH,
  // exactly V*512 doubles, contiguous) once the y pass has read them
  static constexpr int kU0 = XL;
  static_assert(YH + V * 128 - XL == V * kE3, "u0 fits the x/y face slabs");
  // the leaf's gravity field g[3][E^3] (Euler with gravity), bulk-copied at
  // the start on its own mbarrier and read by the epilogue
  static constexpr int kGv = kAcc + V * kAccV;
  static constexpr int kDoubles = kGv + (V == 5 ? 3 * kE3 : 0);
  static constexpr int kBytes = kDoubles * 8 + 64;  // + mbarriers/scratch
  static constexpr uint32_t kTxBytes = (uint32_t)(V * 1408 * 8);
};

// StageLaunch is declared in tmgpu_internal.h


// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3), "r"(c4)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_5d(const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                                int c4) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}

__device__ __forceinline__ void bulk_prefetch(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(src)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------------ arithmetic
// lanes.hpp:109-113 vmax and std::max, exactly (NaN / signed-zero behaviour).
__device__ __forceinline__ double vmax_(double x, double f) { return x > f ? x : f; }
__device__ __forceinline__ double stdmax_(double a, double b) { return (a < b) ? b : a; }

// limiter.hpp:18-26 lane minmod: select(a*b > 0, select(|a|<|b|, a, b), 0)
__device__ __forceinline__ double minmod_lane(double a, double b) {
  double sm = fabs(a) < fabs(b) ? a : b;
  return (a * b) > 0.0 ? sm : 0.0;
}

// Correctly rounded a / b from y = RN(1/b) (Markstein): q = RN(a*y),
// r = a - b*q (exact via FMA), RN(q + r*y) == RN(a/b) when no operand or
// result is near over/underflow; outside [2^-900, 2^901) (and for 0, inf,
// NaN) it falls back to the IEEE division, so the result is bitwise the
// reference's `a / b` for every input. Lets one reciprocal serve several
// quotients with the same divisor (cons->prim) and a per-slice constant
// divisor (gamma - 1) cost 3 FP64 ops instead of a full division sequence.
__device__ __forceinline__ bool exp_ok(double x) {
  const unsigned e = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;
  return (e - 123u) < 1800u;
}
__device__ __forceinline__ double div_rn(double a, double b, double y, bool b_ok) {
  const double q = a * y;
  const double r = fma(-q, b, a);
  const double q2 = fma(r, y, q);
  return (b_ok && exp_ok(a) && exp_ok(q2)) ? q2 : a / b;
}
// The same with a divisor of moderate magnitude: b and y = RN(1/b) in
// [2^-60, 2^61) (b_narrow, checked once per divisor) and a in [2^-900, 2^900)
// keep q, r and q2 in (2^-961, 2^961) — no over/underflow anywhere — so the
// quotient's own range check is implied and dropped. Used for the gamma - 1
// divisions (per launch) and the cons -> prim divisions by rho (per cell).
__device__ __forceinline__ bool exp_narrow(double x) {
  const unsigned e = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;
  return (e - 963u) < 121u;
}
__device__ __forceinline__ double div_rn_n(double a, double b, double y, bool b_narrow) {
  const double q = a * y;
  const double r = fma(-q, b, a);
  const double q2 = fma(r, y, q);
  return (b_narrow && exp_ok(a)) ? q2 : a / b;
}

// euler.hpp:27-35
__device__ __forceinline__ void recon(double um1, double u0, double up1, double up2, double& l,
                                      double& r) {
  l = u0 + 0.5 * minmod_lane(u0 - um1, up1 - u0);
  r = up1 - 0.5 * minmod_lane(up1 - u0, up2 - up1);
}

// Rusanov / KT central flux between primitive face states (euler.hpp:116-137
// with euler_flux :96-114, prim_to_cons :78-89, sound_speed :91-94).
// prim_to_cons is evaluated once per side: the reference evaluates it twice
// (inside euler_flux and again for U) with identical operands, so sharing the
// value is bitwise neutral.
template <int AXIS, bool FAST>
__device__ __forceinline__ void rusanov(const double (&ql)[5], const double (&qr)[5], double gamma,
                                        double gm1, double inv_gm1, bool gm1_ok, double (&f)[5]) {
  double cl, cr, el, er;
  if constexpr (!FAST) {
    cl = sqrt(gamma * ql[4] / ql[0]);
    cr = sqrt(gamma * qr[4] / qr[0]);
    el = div_rn_n(ql[4], gm1, inv_gm1, gm1_ok) +
         0.5 * ql[0] * (ql[1] * ql[1] + ql[2] * ql[2] + ql[3] * ql[3]);
    er = div_rn_n(qr[4], gm1, inv_gm1, gm1_ok) +
         0.5 * qr[0] * (qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3]);
  } else {
    cl = sqrt(gamma * ql[4] * __drcp_rn(ql[0]));
    cr = sqrt(gamma * qr[4] * __drcp_rn(qr[0]));
    el = fma(ql[4], inv_gm1,
             0.5 * ql[0] * fma(ql[1], ql[1], fma(ql[2], ql[2], ql[3] * ql[3])));
    er = fma(qr[4], inv_gm1,
             0.5 * qr[0] * fma(qr[1], qr[1], fma(qr[2], qr[2], qr[3] * qr[3])));
  }
  const double unl = ql[1 + AXIS], unr = qr[1 + AXIS];
  const double smax = vmax_(fabs(unl) + cl, fabs(unr) + cr);
  const double hs = 0.5 * smax;
  // conserved states
  const double ul[5] = {ql[0], ql[0] * ql[1], ql[0] * ql[2], ql[0] * ql[3], el};
  const double ur[5] = {qr[0], qr[0] * qr[1], qr[0] * qr[2], qr[0] * qr[3], er};
  double fl[5], fr[5];
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    fl[v] = ul[v] * unl;
    fr[v] = ur[v] * unr;
  }
  fl[1 + AXIS] = fl[1 + AXIS] + ql[4];
  fr[1 + AXIS] = fr[1 + AXIS] + qr[4];
  fl[4] = (el + ql[4]) * unl;
  fr[4] = (er + qr[4]) * unr;
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    if constexpr (!FAST)
      f[v] = 0.5 * (fl[v] + fr[v]) - hs * (ur[v] - ul[v]);
    else
      f[v] = fma(-hs, ur[v] - ul[v], 0.5 * (fl[v] + fr[v]));
  }
}

// Address (var 0) and var stride of storage position `pos` along AXIS for the
// pencil with tangential interior indices (c1 on axis AXIS+1, c2 on AXIS+2).
template <int V, int AXIS>
__device__ __forceinline__ void pos_addr(int pos, int c1, int c2, int& a, int& vs) {
  using L = Lay<V>;
  if constexpr (AXIS == 0) {  // y = c1, z = c2 interior
    const int row = c2 * 8 + c1;
    if (pos < 2) {
      a = L::XL + row * 2 + pos;
      vs = 128;
    } else if (pos >= 10) {
      a = L::XH + row * 2 + (pos - 10);
      vs = 128;
    } else {
      a = L::B0 + row * 10 + (pos - 2);
      vs = 640;
    }
  } else if constexpr (AXIS == 1) {  // z = c1, x = c2 interior
    if (pos < 2) {
      a = L::YL + (c1 * 2 + pos) * 8 + c2;
      vs = 128;
    } else if (pos >= 10) {
      a = L::YH + (c1 * 2 + pos - 10) * 8 + c2;
      vs = 128;
    } else {
      a = L::B0 + (c1 * 8 + pos - 2) * 10 + c2;
      vs = 640;
    }
  } else {  // x = c1, y = c2 interior
    if (pos < 2) {
      a = L::ZL + (pos * 8 + c2) * 8 + c1;
      vs = 128;
    } else if (pos >= 10) {
      a = L::ZH + ((pos - 10) * 8 + c2) * 8 + c1;
      vs = 128;
    } else {
      a = L::B0 + ((pos - 2) * 8 + c2) * 10 + c1;
      vs = 640;
    }
  }
}

// Lane -> (pencil, segment) map for the face phase. Returns false for idle
// lanes. nb = lane holding segment r+1 of the same pencil.
template <int AXIS>
__device__ __forceinline__ bool face_map(int tid, int& c1, int& c2, int& r, int& nb) {
  (void)AXIS;
  const int warp = tid >> 5, lane = tid & 31;
  // segments 10 lanes apart: the 10 lanes of one segment walk consecutive
  // pencils, which the B0 row stride maps to distinct banks
  const int j = lane % 10;
  r = lane / 10;
  nb = lane + 10;
  const int p = warp * 10 + j;
  if constexpr (AXIS == 1) {
    c2 = p & 7;
    c1 = p >> 3;
  } else {
    c1 = p & 7;
    c2 = p >> 3;
  }
  return lane < 30 && p < 64;
}

__device__ __forceinline__ int interior_index(int axis, int c0, int c1, int c2) {
  int cc[3];
  cc[axis] = c0;
  cc[(axis + 1) % 3] = c1;
  cc[(axis + 2) % 3] = c2;
  return (cc[2] * kE + cc[1]) * kE + cc[0];
}

// One axis of the stage: fluxes of 3 faces per lane, boundary-face record,
// then (after the barrier) the divergence update of the lane's cells.
// After the y pass's barrier the x/y face slabs are dead: `u0_src` (when
// non-null) is bulk-copied over them on `u0_bar`, in flight during the z pass.
template <int V, int AXIS, bool FAST, bool EULER>
__device__ __forceinline__ void axis_pass(const double* __restrict__ sm, double* __restrict__ acc,
                                          int tid, double gamma, double gm1, double inv_gm1,
                                          bool gm1_ok, double a_vel, double cdt,
                                          double* faces_out, const double* u0_src = nullptr,
                                          uint64_t* u0_bar = nullptr) {
  int c1, c2, r, nb;
  const bool active = face_map<AXIS>(tid, c1, c2, r, nb);
  double F[3][V];
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int v = 0; v < V; ++v) F[k][v] = 0.0;
  if (active) {
    // Stencil window: positions 3r..3r+5 along the axis serve faces 3r..3r+2.
    // Each cell's limited slope m[j] = minmod(d[j-1], d[j]) is computed once
    // and shared by the right state of face j-2 and the left state of face
    // j-1 (the reference evaluates the identical expression twice,
    // euler.hpp:32-33).
    const int base = 3 * r;
    int a[6], vs[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) pos_addr<V, AXIS>(base + s, c1, c2, a[s], vs[s]);
    constexpr int NV = EULER ? 5 : 1;
    double ql[3][NV], qr[3][NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double c[6], d[5], m[5];
#pragma unroll
      for (int s = 0; s < 6; ++s) c[s] = sm[a[s] + v * vs[s]];
#pragma unroll
      for (int i = 0; i < 5; ++i) d[i] = c[i + 1] - c[i];
#pragma unroll
      for (int j = 1; j < 5; ++j) m[j] = minmod_lane(d[j - 1], d[j]);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        ql[k][v] = c[k + 1] + 0.5 * m[k + 1];
        qr[k][v] = c[k + 2] - 0.5 * m[k + 2];
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if constexpr (EULER) {
        double l5[5], r5[5], f[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          l5[v] = ql[k][v];
          r5[v] = qr[k][v];
        }
        // stage.cpp:80-83 face floors
        l5[0] = vmax_(l5[0], kRhoFloor);
        r5[0] = vmax_(r5[0], kRhoFloor);
        l5[4] = vmax_(l5[4], kPressureFloor);
        r5[4] = vmax_(r5[4], kPressureFloor);
        rusanov<AXIS, FAST>(l5, r5, gamma, gm1, inv_gm1, gm1_ok, f);
#pragma unroll
        for (int v = 0; v < 5; ++v) F[k][v] = f[v];
      } else {
        // stage.cpp:44-55 scalar advection on var 0; other vars keep zero flux
        const double l = ql[k][0], rr = qr[k][0];
        F[k][0] = 0.5 * (a_vel * l + a_vel * rr) - 0.5 * fabs(a_vel) * (rr - l);
      }
    }
    // boundary-face record (stage.cpp:180-182): F[0] -> side 0, F[E] -> side 1
    if (faces_out) {
      const int fo = c2 * kE + c1;
      if (r == 0) {
#pragma unroll
        for (int v = 0; v < V; ++v) faces_out[(2 * AXIS) * V * kE2 + v * kE2 + fo] = F[0][v];
      } else if (r == 2) {
#pragma unroll
        for (int v = 0; v < V; ++v) faces_out[(2 * AXIS + 1) * V * kE2 + v * kE2 + fo] = F[2][v];
      }
    }
  }
  // F[3] = first face of the next segment (warp shuffle; all lanes take part)
  double D[3][V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double nxt = __shfl_sync(0xffffffffu, F[0][v], nb & 31);
    D[0][v] = F[1][v] - F[0][v];
    D[1][v] = F[2][v] - F[1][v];
    D[2][v] = nxt - F[2][v];
  }
  __syncthreads();  // previous axis' updates of every cell are complete
  if (AXIS == 1 && u0_src && tid == 0) {
    // the slabs' last generic reads are ordered before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(u0_bar, (uint32_t)(V * kE3 * 8));
    bulk_load(const_cast<double*>(sm) + Lay<V>::kU0, u0_src, V * kE3 * 8, u0_bar);
  }
  if (active) {
    const int ncell = r == 2 ? 2 : 3;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k < ncell) {
        const int ci = interior_index(AXIS, 3 * r + k, c1, c2);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          double& o = acc[v * kAccV + acc_at(ci)];
          if constexpr (FAST)
            o = fma(-cdt, D[k][v], o);
          else
            o -= cdt * D[k][v];
        }
      }
    }
  }
}

// ------------------------------------------------------------------ epilogue
// Gravity source (our spec): after the z update, before the
// floors, with the stage input's primitives (oracle tmo_stage_subgrid_grav).
__device__ __forceinline__ void grav_apply(double (&u)[5], double dt, double rho, double iu, double iv, double iw,
                                           double gx, double gy, double gz) {
  u[1] = u[1] + dt * (rho * gx);
  u[2] = u[2] + dt * (rho * gy);
  u[3] = u[3] + dt * (rho * gz);
  u[4] = u[4] + dt * (rho * ((iu * gx + iv * gy) + iw * gz));
}
__device__ __forceinline__ void grav_source(double (&u)[5], const StageLaunch& p, int slot, int c, double dt,
                                            double rho, double iu, double iv, double iw) {
  const double* gq = p.grav + (long long)slot * kE3 + c;
  const double gx = gq[0], gy = gq[p.grav_stride], gz = gq[2 * p.grav_stride];
  grav_apply(u, dt, rho, iu, iv, iw, gx, gy, gz);
}

// stage.cpp:187-208 density and pressure floors; returns the floor hits
template <bool FAST>
__device__ __forceinline__ unsigned euler_floors(double (&u)[5], double gm1) {
  unsigned hits = 0;
  if (u[0] < kRhoFloor) {
    u[0] = kRhoFloor;
    ++hits;
  }
  double ke;
  if constexpr (!FAST) {
    ke = 0.5 * (u[1] * u[1] + u[2] * u[2] + u[3] * u[3]) / u[0];
  } else {
    ke = 0.5 * fma(u[1], u[1], fma(u[2], u[2], u[3] * u[3])) * __drcp_rn(u[0]);
  }
  const double pr = gm1 * (u[4] - ke);
  if (pr < kPressureFloor) {
    u[4] = kPressureFloor / gm1 + ke;
    ++hits;
  }
  return hits;
}

// finiteness (stage.cpp:209-216), provisional density, RK3 combine
// (rk3.hpp:18-27) with u0p [V][E^3] (or none), store
template <int V>
__device__ __forceinline__ void finish_cell(double (&u)[V], const StageLaunch& p, int slot, int c,
                                            const double* u0p, double* outp, unsigned& bad) {
#pragma unroll
  for (int v = 0; v < V; ++v)
    if (!isfinite(u[v])) bad = min(bad, (unsigned)(v * kE3 + c));
  if (p.rho_save) p.rho_save[(long long)slot * kE3 + c] = u[0];
  const int z = c >> 6, y = (c >> 3) & 7, x = c & 7;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    double o = u[v];
    if (u0p) {
      const double a0 = u0p[v * kE3 + c];
      if (p.rk_stage == 2)
        o = a0 + 0.25 * (o - a0);
      else if (p.rk_stage == 3)
        o = a0 + (2.0 / 3.0) * (o - a0);
    }
    if (p.out_ghosted)
      outp[((v * kS + z + 2) * kS + y + 2) * kS + x + 2] = o;
    else
      outp[v * kE3 + c] = o;
    if (p.out_compact) p.out_compact[((long long)slot * V + v) * kE3 + c] = o;
  }
}

template <int V, bool FAST>
__global__ void __launch_bounds__(kStageThreads, 2)
    stage_kernel(const __grid_constant__ CUtensorMap tm_i, const __grid_constant__ CUtensorMap tm_x,
                 const __grid_constant__ CUtensorMap tm_y, const __grid_constant__ CUtensorMap tm_z,
                 const StageLaunch p) {
  using L = Lay<V>;
  extern __shared__ __align__(128) double smem[];
  double* sm = smem;
  double* acc = smem + L::kAcc;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kDoubles);
  unsigned int& s_hits = *reinterpret_cast<unsigned int*>(smem + L::kDoubles + 1);
  unsigned int& s_bad = *(reinterpret_cast<unsigned int*>(smem + L::kDoubles + 1) + 1);
  uint64_t* bar_u0 = reinterpret_cast<uint64_t*>(smem + L::kDoubles + 2);
  uint64_t* bar_g = reinterpret_cast<uint64_t*>(smem + L::kDoubles + 3);
  const bool want_g = V == 5 && p.grav && !p.defer;
  const bool want_u0 = p.u0 && p.rk_stage >= 2 && !p.defer;

  const int tid = threadIdx.x;
  const int s = blockIdx.x;
  const int slot = p.index ? p.index[s] : s;  // per-slice outputs are indexed by slot

  if (tid == 0) {
    s_hits = 0;
    s_bad = 0xffffffffu;
    mbar_init(bar, 1);
    mbar_init(bar_u0, 1);
    if constexpr (V == 5) {
      if (want_g) {  // g[3][E^3] of this leaf, needed only by the epilogue
        mbar_init(bar_g, 1);
        mbar_expect_tx(bar_g, 3 * kE3 * 8);
#pragma unroll
        for (int q = 0; q < 3; ++q)
          bulk_load(smem + L::kGv + q * kE3, p.grav + q * p.grav_stride + (long long)slot * kE3, kE3 * 8, bar_g);
      }
    }
    mbar_expect_tx(bar, L::kTxBytes);
    tma_load_5d(sm + L::B0, &tm_i, bar, 2, 2, 2, 0, slot);
    // face f = 2*axis + side; own ghost layer or the same-level neighbour's
    // adjacent interior layers (ghost.cpp:40-68 same-slab, fused)
    const CUtensorMap* fm[3] = {&tm_x, &tm_y, &tm_z};
    const int off[6] = {L::XL, L::XH, L::YL, L::YH, L::ZL, L::ZH};
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int axis = f >> 1, side = f & 1;
      int src = slot, ca;
      const int code = p.face_src ? p.face_src[(long long)slot * 6 + f] : (slot << 1);
      if (code & 1) {
        src = code >> 1;
        ca = side ? kG : kE;  // neighbour interior layers next to the shared face
      } else {
        ca = side ? kG + kE : 0;  // own ghost layers
      }
      int c[3] = {kG, kG, kG};
      c[axis] = ca;
      tma_load_5d(sm + off[f], fm[axis], bar, c[0], c[1], c[2], 0, src);
    }
    // the same boxes of the CTA one resident wave ahead, into L2
    if (p.prefetch_ahead > 0 && s + p.prefetch_ahead < p.count) {
      const int sa = s + p.prefetch_ahead;
      const int slot_a = p.index ? p.index[sa] : sa;
      if (want_u0) bulk_prefetch(p.u0 + (long long)slot_a * p.u0_stride, V * kE3 * 8);
      tma_prefetch_5d(&tm_i, 2, 2, 2, 0, slot_a);
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        const int axis = f >> 1, side = f & 1;
        int src = slot_a, ca;
        const int code = p.face_src ? p.face_src[(long long)slot_a * 6 + f] : (slot_a << 1);
        if (code & 1) {
          src = code >> 1;
          ca = side ? kG : kE;
        } else {
          ca = side ? kG + kE : 0;
        }
        int c[3] = {kG, kG, kG};
        c[axis] = ca;
        tma_prefetch_5d(fm[axis], c[0], c[1], c[2], 0, src);
      }
    }
  }

  // header (decode_header stage.cpp:21-29)
  double mode, dx, dt, gamma, ax, ay, az;
  if (p.hdr) {
    const double* h = p.hdr + (long long)slot * p.hdr_stride;
    mode = h[0];
    dx = h[1];
    dt = h[2];
    gamma = h[3];
    ax = h[4];
    ay = h[5];
    az = h[6];
  } else {
    mode = p.g_mode;
    dx = p.leaf_dx[slot];
    dt = p.dt_ptr ? *p.dt_ptr : p.g_dt;
    gamma = p.g_gamma;
    ax = p.g_ax;
    ay = p.g_ay;
    az = p.g_az;
  }
  const bool euler = mode != 0.0;
  const double cdt = dt / dx;
  const double gm1 = gamma - 1.0;
  const double inv_gm1 = 1.0 / gm1;  // RN(1/(gamma-1)) for div_rn
  const bool gm1_ok = exp_narrow(gm1) && exp_narrow(inv_gm1);  // div_rn_n's divisor condition

  __syncthreads();  // barrier init visible
  mbar_wait(bar, 0);

  // ---- phase 2: accumulator seed + cons -> prim in place (stage.cpp:141-153)
  for (int c = tid; c < 1280; c += kStageThreads) {
    int a, vs;
    const bool interior = c < kE3;
    if (interior) {  // compact (k,j,i) == acc index
      a = L::B0 + (c >> 3) * 10 + (c & 7);
      vs = 640;
    } else {
      const int q = c - kE3;
      a = L::XL + (q >> 7) * V * 128 + (q & 127);
      vs = 128;
    }
    double u[V];
#pragma unroll
    for (int v = 0; v < V; ++v) u[v] = sm[a + v * vs];
    if (interior) {
      const int ci = c;
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v * kAccV + acc_at(ci)] = u[v];
      if (p.u0_save) {
        double* u0s = p.u0_save + (long long)slot * p.u0_save_stride;
#pragma unroll
        for (int v = 0; v < V; ++v) u0s[v * kE3 + ci] = u[v];
      }
    }
    if constexpr (V == 5) {
      if (euler) {
        const double rho = stdmax_(u[0], kRhoFloor);
        double iu, iv, iw, ke, pr;
        if constexpr (!FAST) {
          const double yr = __drcp_rn(rho);  // RN(1/rho)
          const bool rok = exp_narrow(rho) && exp_narrow(yr);
          iu = div_rn_n(u[1], rho, yr, rok);
          iv = div_rn_n(u[2], rho, yr, rok);
          iw = div_rn_n(u[3], rho, yr, rok);
          ke = 0.5 * rho * (iu * iu + iv * iv + iw * iw);
          pr = stdmax_(gm1 * (u[4] - ke), kPressureFloor);
        } else {
          const double ir = __drcp_rn(rho);
          iu = u[1] * ir;
          iv = u[2] * ir;
          iw = u[3] * ir;
          ke = 0.5 * rho * fma(iu, iu, fma(iv, iv, iw * iw));
          pr = stdmax_(gm1 * (u[4] - ke), kPressureFloor);
        }
        sm[a] = rho;
        sm[a + vs] = iu;
        sm[a + 2 * vs] = iv;
        sm[a + 3 * vs] = iw;
        sm[a + 4 * vs] = pr;
      }
    }
  }
  __syncthreads();

  // ---- phase 3: x, y, z passes
  double* faces_out = p.faces ? p.faces + (long long)slot * p.faces_stride : nullptr;
  const double* u0_src = want_u0 ? p.u0 + (long long)slot * p.u0_stride : nullptr;
  if (V == 5 && euler) {
    axis_pass<V, 0, FAST, (V == 5)>(sm, acc, tid, gamma, gm1, inv_gm1, gm1_ok, 0.0, cdt, faces_out);
    axis_pass<V, 1, FAST, (V == 5)>(sm, acc, tid, gamma, gm1, inv_gm1, gm1_ok, 0.0, cdt, faces_out, u0_src,
                                    bar_u0);
    axis_pass<V, 2, FAST, (V == 5)>(sm, acc, tid, gamma, gm1, inv_gm1, gm1_ok, 0.0, cdt, faces_out);
  } else {
    axis_pass<V, 0, FAST, false>(sm, acc, tid, gamma, gm1, inv_gm1, gm1_ok, ax, cdt, faces_out);
    axis_pass<V, 1, FAST, false>(sm, acc, tid, gamma, gm1, inv_gm1, gm1_ok, ay, cdt, faces_out, u0_src, bar_u0);
    axis_pass<V, 2, FAST, false>(sm, acc, tid, gamma, gm1, inv_gm1, gm1_ok, az, cdt, faces_out);
  }
  __syncthreads();

  // ---- phase 4: floors, finiteness, RK3 combine, store
  double* outp = p.out + (long long)slot * p.out_stride;
  if (p.defer) {  // split step: the raw update; stage_epilogue_kernel finishes it
    for (int c = tid; c < kE3; c += kStageThreads) {
      const int z = c >> 6, y = (c >> 3) & 7, x = c & 7;
#pragma unroll
      for (int v = 0; v < V; ++v) outp[((v * kS + z + 2) * kS + y + 2) * kS + x + 2] = acc[v * kAccV + acc_at(c)];
    }
    return;
  }
  unsigned int hits = 0, bad = 0xffffffffu;
  const double* u0p = want_u0 ? smem + L::kU0 : nullptr;
  if (want_u0) mbar_wait(bar_u0, 0);
  if (want_g) mbar_wait(bar_g, 0);
  for (int c = tid; c < kE3; c += kStageThreads) {
    double u[V];
#pragma unroll
    for (int v = 0; v < V; ++v) u[v] = acc[v * kAccV + acc_at(c)];
    if constexpr (V == 5) {
      if (euler && p.grav) {  // gravity source with the stage input's primitives
        const double* pq = sm + L::B0 + (c >> 3) * 10 + (c & 7);
        const double* sg = smem + L::kGv + c;
        grav_apply(u, dt, pq[0], pq[640], pq[1280], pq[1920], sg[0], sg[kE3], sg[2 * kE3]);
      }
      if (euler) hits += euler_floors<FAST>(u, gm1);
    }
    finish_cell<V>(u, p, slot, c, u0p, outp, bad);
  }
  // block reductions (integer counts: order-free, exact as double)
  if (hits) atomicAdd(&s_hits, hits);
  if (bad != 0xffffffffu) atomicMin(&s_bad, bad);
  __syncthreads();
  if (tid == 0) {
    if (p.diag) p.diag[(long long)slot * p.diag_stride] = (double)s_hits;
    if (s_bad != 0xffffffffu && p.err)
      atomicMin(p.err, ((unsigned long long)slot << 32) | s_bad);
  }
}

// Second half of a split stage (the gravity step: the update of every cell is
// computed by stage_kernel with p.defer while the stage's gravity solve runs,
// and finished here once the field exists): gravity source with the stage
// input's primitives (recomputed from the input arena by the stage kernel's own
// cons -> prim operations), floors, finiteness, provisional density, RK3
// combine, store — stage_kernel's phase 4 bit for bit. One CTA per slot.
template <bool FAST>
__global__ void __launch_bounds__(256) stage_epilogue_kernel(const double* __restrict__ in_arena,
                                                             const StageLaunch p) {
  __shared__ unsigned int s_hits, s_bad;
  const int tid = threadIdx.x;
  const int slot = p.index ? p.index[blockIdx.x] : blockIdx.x;
  if (tid == 0) s_hits = 0, s_bad = 0xffffffffu;
  const double dt = p.dt_ptr ? *p.dt_ptr : p.g_dt;
  const double gm1 = p.g_gamma - 1.0;
  const double* inp = in_arena + (long long)slot * p.out_stride;
  double* outp = p.out + (long long)slot * p.out_stride;
  const double* u0p = (p.u0 && p.rk_stage >= 2) ? p.u0 + (long long)slot * p.u0_stride : nullptr;
  __syncthreads();
  unsigned int hits = 0, bad = 0xffffffffu;
  for (int c = tid; c < kE3; c += blockDim.x) {
    const int z = c >> 6, y = (c >> 3) & 7, x = c & 7;
    const long long q = ((long long)(z + 2) * kS + y + 2) * kS + x + 2;
    double u[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = outp[v * kS * kS * kS + q];
    if (p.grav) {
      const double rho = stdmax_(inp[q], kRhoFloor);
      const double m1 = inp[kS * kS * kS + q], m2 = inp[2 * kS * kS * kS + q], m3 = inp[3 * kS * kS * kS + q];
      double iu, iv, iw;
      if constexpr (!FAST) {
        const double yr = __drcp_rn(rho);
        const bool rok = exp_ok(rho) && exp_ok(yr);
        iu = div_rn(m1, rho, yr, rok);
        iv = div_rn(m2, rho, yr, rok);
        iw = div_rn(m3, rho, yr, rok);
      } else {
        const double ir = __drcp_rn(rho);
        iu = m1 * ir;
        iv = m2 * ir;
        iw = m3 * ir;
      }
      grav_source(u, p, slot, c, dt, rho, iu, iv, iw);
    }
    hits += euler_floors<FAST>(u, gm1);
    finish_cell<5>(u, p, slot, c, u0p, outp, bad);
  }
  if (hits) atomicAdd(&s_hits, hits);
  if (bad != 0xffffffffu) atomicMin(&s_bad, bad);
  __syncthreads();
  if (tid == 0) {
    if (p.diag) p.diag[(long long)slot * p.diag_stride] = (double)s_hits;
    if (s_bad != 0xffffffffu && p.err) atomicMin(p.err, ((unsigned long long)slot << 32) | s_bad);
  }
}

}  // namespace tmgpu
