// Device ghost-shell exchange over the leaf arena [slot][V][S][S][S]
// (S = 12, x fastest), reference-exact: restates proj/src/amr/ghost.cpp
// fill_ghosts_sync (:282-296) — three sequential axis passes; per pass the
// prolonged (coarse->fine) slabs are extracted first from the pre-pass state
// (phase 1, the reference's `staged` map), then every fill of the pass is
// applied (phase 2). Within phase 2 all fills write disjoint ghost cells and
// read interior-along-axis cells only, so one CTA per fill in any order is
// bitwise identical to the reference's sequential loop (test_amr.cpp:300-347
// proves the reference itself is fill-order independent).
//
// Per-element arithmetic follows the reference exactly:
//   same        copy                                 ghost.cpp:40-68
//   prolonged   c +/- 0.25*minmod(c+ - c, c - c-)    ghost.cpp:70-111, limiter.hpp:13-16
//   restricted  (sum of 8 in dn,d1,d2 order)*0.125   ghost.cpp:113-149
//   reflective  sign * mirrored interior             ghost.cpp:151-166
#include "ghost.h"
#include "tmgpu_internal.h"

namespace tmgpu {
namespace {

constexpr int E = 8, G = 2, S = 12, S3 = S * S * S;

__device__ __forceinline__ double minmod_scalar(double a, double b) {
  if (a * b <= 0.0) return 0.0;
  return fabs(a) < fabs(b) ? a : b;
}

__device__ __forceinline__ int at(int var, int x, int y, int z) {
  return var * S3 + (z * S + y) * S + x;
}

// Compose (x,y,z) from (coordinate along axis, tangential t1, tangential t2).
__device__ __forceinline__ void compose(int axis, int na, int v1, int v2, int& x, int& y, int& z) {
  int c[3];
  c[axis] = na;
  c[(axis + 1) % 3] = v1;
  c[(axis + 2) % 3] = v2;
  x = c[0];
  y = c[1];
  z = c[2];
}

// Phase 1: one CTA per prolonged fill; staged slab in ghost.cpp:161-186 order
// n = ((var*E + f2)*E + f1)*G + dd.
__global__ void __launch_bounds__(128) prolong_extract_kernel(const double* __restrict__ arena,
                                                              const GhostFill* __restrict__ fills,
                                                              const int* __restrict__ which, int V,
                                                              double* __restrict__ staged) {
  const GhostFill f = fills[which[blockIdx.x]];
  const double* src = arena + (long long)f.src * V * S3;
  double* out = staged + (long long)blockIdx.x * V * E * E * G;
  const int axis = f.axis, dir = f.dir;
  const int n_el = V * E * E * G;
  for (int n = threadIdx.x; n < n_el; n += blockDim.x) {
    const int dd = n % G, f1 = (n / G) % E, f2 = (n / (G * E)) % E, var = n / (G * E * E);
    const int cd = dd / 2, sub = dd - 2 * cd;
    const int na = dir > 0 ? G + cd : G + E - 1 - cd;
    const int ct1 = G + f.qt1 * (E / 2) + f1 / 2;
    const int ct2 = G + f.qt2 * (E / 2) + f2 / 2;
    int x, y, z, xm, ym, zm, xp, yp, zp;
    compose(axis, na, ct1, ct2, x, y, z);
    compose(axis, na - 1, ct1, ct2, xm, ym, zm);
    compose(axis, na + 1, ct1, ct2, xp, yp, zp);
    const double c = src[at(var, x, y, z)];
    const double s = minmod_scalar(src[at(var, xp, yp, zp)] - c, c - src[at(var, xm, ym, zm)]);
    const double off = 0.25 * s;
    const int sign = dir > 0 ? (sub == 0 ? -1 : +1) : (sub == 0 ? +1 : -1);
    out[n] = sign > 0 ? c + off : c - off;
  }
}

// Phase 2: one CTA per fill of the pass.
__global__ void __launch_bounds__(128) apply_kernel(double* __restrict__ arena,
                                                    const GhostFill* __restrict__ fills,
                                                    const int* __restrict__ staged_of, int V,
                                                    const double* __restrict__ staged) {
  const GhostFill f = fills[blockIdx.x];
  double* dst = arena + (long long)f.dst * V * S3;
  const int axis = f.axis, dir = f.dir;
  switch (f.kind) {
    case 0:    // same level: G layers, full S x S tangential extent
    case 3: {  // reflective wall (boundary)
      const bool refl = f.kind == 3;
      const double* src = refl ? dst : arena + (long long)f.src * V * S3;
      const int nmv = (refl && V == 5) ? 1 + axis : -1;
      const int n_el = V * S * S * G;
      for (int n = threadIdx.x; n < n_el; n += blockDim.x) {
        // enumerate the ghost box in storage order (x fastest) for coalescing
        int e[3] = {S, S, S};
        e[axis] = G;
        const int lx = n % e[0], ly = (n / e[0]) % e[1], lz = (n / (e[0] * e[1])) % e[2];
        const int var = n / (e[0] * e[1] * e[2]);
        int p[3] = {lx, ly, lz};
        p[axis] += dir > 0 ? G + E : 0;  // destination ghost layer
        int q[3] = {p[0], p[1], p[2]};
        if (refl)
          q[axis] = dir > 0 ? 2 * (G + E) - 1 - p[axis] : 2 * G - 1 - p[axis];
        else
          q[axis] = dir > 0 ? p[axis] - E : p[axis] + E;
        const double v = src[at(var, q[0], q[1], q[2])];
        dst[at(var, p[0], p[1], p[2])] = refl ? (var == nmv ? -1.0 : 1.0) * v : v;
      }
      break;
    }
    case 1: {  // coarser neighbour: staged prolonged slab
      const double* in = staged + (long long)staged_of[blockIdx.x] * V * E * E * G;
      const int n_el = V * E * E * G;
      for (int n = threadIdx.x; n < n_el; n += blockDim.x) {
        const int dd = n % G, f1 = (n / G) % E, f2 = (n / (G * E)) % E, var = n / (G * E * E);
        const int na = dir > 0 ? G + E + dd : G - 1 - dd;
        int x, y, z;
        compose(axis, na, G + f1, G + f2, x, y, z);
        dst[at(var, x, y, z)] = in[n];
      }
      break;
    }
    case 2: {  // finer neighbour: restricted quadrant
      const double* src = arena + (long long)f.src * V * S3;
      const int h = E / 2, n_el = V * h * h * G;
      for (int n = threadIdx.x; n < n_el; n += blockDim.x) {
        const int dd = n % G, c1 = (n / G) % h, c2 = (n / (G * h)) % h, var = n / (G * h * h);
        double acc = 0.0;
        for (int dn = 0; dn < 2; ++dn)
          for (int d1 = 0; d1 < 2; ++d1)
            for (int d2 = 0; d2 < 2; ++d2) {
              const int fn = dir > 0 ? G + 2 * dd + dn : G + E - 1 - (2 * dd + dn);
              int x, y, z;
              compose(axis, fn, G + 2 * c1 + d1, G + 2 * c2 + d2, x, y, z);
              acc += src[at(var, x, y, z)];
            }
        const int na = dir > 0 ? G + E + dd : G - 1 - dd;
        int x, y, z;
        compose(axis, na, G + f.qt1 * h + c1, G + f.qt2 * h + c2, x, y, z);
        dst[at(var, x, y, z)] = acc * 0.125;
      }
      break;
    }
  }
}

// compact [slot][V][E^3] (k,j,i order) <-> arena interior
__global__ void interior_copy_kernel(double* __restrict__ arena, double* __restrict__ compact,
                                     int V, long long nslots, int to_arena) {
  const long long total = nslots * V * (E * E * E);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % (E * E * E));
    const long long sv = i / (E * E * E);  // slot*V + var
    const int x = G + (c & 7), y = G + ((c >> 3) & 7), z = G + (c >> 6);
    double* a = arena + sv * S3 + (z * S + y) * S + x;
    if (to_arena)
      *a = compact[i];
    else
      compact[i] = *a;
  }
}

}  // namespace

cudaError_t ghost_pass(double* arena, int V, const GhostPassDev& pass, double* staged,
                       cudaStream_t st) {
  if (pass.n_prolong > 0) {
    prolong_extract_kernel<<<pass.n_prolong, 128, 0, st>>>(arena, pass.fills, pass.prolong_fills,
                                                           V, staged);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  if (pass.n_fills > 0) {
    apply_kernel<<<pass.n_fills, 128, 0, st>>>(arena, pass.fills, pass.staged_of, V, staged);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  return cudaGetLastError();
}

cudaError_t interior_copy(double* arena, double* compact, int V, long long nslots, bool to_arena,
                          cudaStream_t st) {
  if (nslots <= 0) return cudaSuccess;
  long long total = nslots * V * 512;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  interior_copy_kernel<<<(unsigned)blocks, 256, 0, st>>>(arena, compact, V, nslots, to_arena ? 1 : 0);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace tmgpu
