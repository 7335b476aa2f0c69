// Time-centred gravity source of one RK stage (the 6-solve cadence of
// tmgpu_forest_set_gravity_solver; our specification — the paper states only
// that a step runs "six (instead of three) iterations of the FMM solver",
// PAPER.md:240-241, and the reference has no gravity).
//
// The stage kernel applied dt*S(u, g_a) with g_a solved on the stage input u.
// A second solve on the stage's provisional density gives g_b; this kernel
// moves the source to the trapezoid dt*rho*(g_a + g_b)/2 (a predictor-corrector
// source, as grid codes do for self-gravity), scaled by the stage's RK3 weight
// w (1, 1/4, 2/3) because it runs after the combine:
//   m_q += w * ((0.5*dt) * (rho * (gb_q - ga_q)))
//   E   += w * ((0.5*dt) * (rho * ((u*dgx + v*dgy) + w*dgz)))
// with rho = max(rho_in, 1e-10) and u = m_in/rho the stage input's primitives
// (the ones the stage kernel's source used). Oracle: the composition in
// tests/test_gravity_cadence_gpu.py (numpy, same association).
#include <algorithm>

#include "tmgpu_internal.h"

namespace tmgpu {
namespace {

constexpr double kRhoFloorSrc = 1e-10;  // euler.hpp:15, as the stage kernel

__global__ void grav_correct_kernel(const double* __restrict__ in, double* __restrict__ out,
                                    long long nslots, const double* __restrict__ ga,
                                    const double* __restrict__ gb, long long gstride,
                                    const double* __restrict__ dt_ptr, double g_dt, double w) {
  const double dt = dt_ptr ? *dt_ptr : g_dt;
  const double hdt = 0.5 * dt;
  const long long total = nslots * 512;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long s = t >> 9;
    const int c = (int)(t & 511);
    const int i = c & 7, j = (c >> 3) & 7, k = c >> 6;
    const long long q = s * 5 * 1728 + ((k + 2) * 12 + (j + 2)) * 12 + (i + 2);
    const double r = in[q];
    const double rho = (r < kRhoFloorSrc) ? kRhoFloorSrc : r;  // std::max(r, floor)
    const double iu = in[q + 1728] / rho, iv = in[q + 2 * 1728] / rho, iw = in[q + 3 * 1728] / rho;
    const double dgx = gb[t] - ga[t], dgy = gb[gstride + t] - ga[gstride + t],
                 dgz = gb[2 * gstride + t] - ga[2 * gstride + t];
    out[q + 1728] = out[q + 1728] + w * (hdt * (rho * dgx));
    out[q + 2 * 1728] = out[q + 2 * 1728] + w * (hdt * (rho * dgy));
    out[q + 3 * 1728] = out[q + 3 * 1728] + w * (hdt * (rho * dgz));
    out[q + 4 * 1728] = out[q + 4 * 1728] + w * (hdt * (rho * ((iu * dgx + iv * dgy) + iw * dgz)));
  }
}

}  // namespace

cudaError_t launch_grav_correct(const double* in_arena, double* out_arena, long long nslots, const double* ga,
                                const double* gb, long long gstride, const double* dt_ptr, double g_dt,
                                double w, cudaStream_t st) {
  if (nslots <= 0) return cudaSuccess;
  const long long total = nslots * 512;
  const unsigned grid = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 16);
  grav_correct_kernel<<<grid, 256, 0, st>>>(in_arena, out_arena, nslots, ga, gb, gstride, dt_ptr, g_dt, w);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace tmgpu
