// Flux-register reflux at refinement jumps. The
// reference declares the FluxRegister (proj/include/taskmesh/amr/
// flux_register.hpp:21-63) but ships no definition; SPEC.md:383-391 gives the
// operation: every coarse cell next to a finer face is corrected by
//   (sum fine_flux * fine_area - coarse_flux * coarse_area) * dt / volume
// = (fine_mean - coarse_flux) * w / dx,  applied with the sign -dir
// (flux_register.hpp:4-9), w = stage coefficient * dt, fine_mean the 2x2
// arithmetic mean of the covering fine face fluxes (restrict_face), entries
// in sorted (leaf, axis, dir) order. Our restatement: oracle tmo_reflux_apply
// (parity unpinned beyond that formula; conservation is the test).
//
// One CTA per coarse leaf with finer faces: its faces in (axis, dir) order,
// a barrier between faces (edge cells are touched by two or three faces and
// the corrections must be applied in that order), threads over (var, c2, c1).
#include "tmgpu_internal.h"

namespace tmgpu {
namespace {

__global__ void __launch_bounds__(320) reflux_kernel(double* __restrict__ arena, long long slot_stride,
                                                     const double* __restrict__ flux, long long flux_stride,
                                                     const int* __restrict__ leaf_slot,
                                                     const int* __restrict__ face_off,
                                                     const int* __restrict__ face_ad,
                                                     const int* __restrict__ fine,
                                                     const double* __restrict__ leaf_dx,
                                                     const double* __restrict__ dt_ptr, double g_dt,
                                                     double coef, int V, const double* __restrict__ rflux) {
  const int slot = leaf_slot[blockIdx.x];
  const double dt = dt_ptr ? *dt_ptr : g_dt;
  const double w = coef * dt;
  const double cw = w / leaf_dx[slot];
  const int nE2 = 64;
  for (int f = face_off[blockIdx.x]; f < face_off[blockIdx.x + 1]; ++f) {
    const int axis = face_ad[2 * f], dir = face_ad[2 * f + 1];
    const int side_c = dir > 0 ? 1 : 0, side_f = 1 - side_c;
    for (int t = threadIdx.x; t < V * nE2; t += blockDim.x) {
      const int v = t >> 6, c = t & 63, c1 = c & 7, c2 = c >> 3;
      const int fs = fine[4 * f + (c2 >> 2) * 2 + (c1 >> 2)];
      const int f1 = 2 * (c1 & 3), f2 = 2 * (c2 & 3);
      // a fine leaf on another GPU (fs < 0): its face block came with the
      // stage's flux exchange, [V][E^2] at entry -fs - 1 of rflux
      const double* Ff = fs >= 0 ? flux + (long long)fs * flux_stride + ((2 * axis + side_f) * V + v) * nE2
                                 : rflux + ((long long)(-fs - 1) * V + v) * nE2;
      const double a00 = Ff[f2 * 8 + f1], a10 = Ff[f2 * 8 + f1 + 1], a01 = Ff[(f2 + 1) * 8 + f1],
                   a11 = Ff[(f2 + 1) * 8 + f1 + 1];
      const double mean = (((a00 + a10) + a01) + a11) * 0.25;
      const double coarse = flux[(long long)slot * flux_stride + ((2 * axis + side_c) * V + v) * nE2 + c];
      const double delta = mean - coarse;
      int x[3];
      x[axis] = side_c ? 7 : 0;
      x[(axis + 1) % 3] = c1;
      x[(axis + 2) % 3] = c2;
      double& u = arena[(long long)slot * slot_stride + ((v * 12 + x[2] + 2) * 12 + x[1] + 2) * 12 + x[0] + 2];
      u = dir > 0 ? u - cw * delta : u + cw * delta;
    }
    __syncthreads();
  }
}

// the face flux blocks other GPUs' coarse leaves need: entry e copies face
// item[e].y of local slot item[e].x ([V][E^2]) to out + e * V * E^2
__global__ void __launch_bounds__(320) flux_pack_kernel(const double* __restrict__ flux, long long flux_stride,
                                                        const int2* __restrict__ item, double* __restrict__ out,
                                                        int V) {
  const int2 it = item[blockIdx.x];
  const double* src = flux + (long long)it.x * flux_stride + (long long)it.y * V * 64;
  double* dst = out + (long long)blockIdx.x * V * 64;
  for (int t = threadIdx.x; t < V * 64; t += blockDim.x) dst[t] = src[t];
}

}  // namespace

cudaError_t launch_flux_pack(const double* flux, int V, const int2* items, long long n, double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  flux_pack_kernel<<<(unsigned)n, 320, 0, st>>>(flux, (long long)6 * V * 64, items, out, V);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_reflux(double* arena, int V, const double* flux, const int* leaf_slot,
                          const int* face_off, const int* face_ad, const int* fine, long long nleaves,
                          const double* leaf_dx, const double* dt_ptr, double g_dt, double coef,
                          cudaStream_t st, const double* rflux) {
  if (nleaves <= 0) return cudaSuccess;
  reflux_kernel<<<(unsigned)nleaves, 320, 0, st>>>(arena, (long long)V * 1728, flux,
                                                   (long long)6 * V * 64, leaf_slot, face_off, face_ad,
                                                   fine, leaf_dx, dt_ptr, g_dt, coef, V, rflux);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace tmgpu
