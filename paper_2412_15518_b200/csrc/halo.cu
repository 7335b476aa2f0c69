// Pack / pull kernels of the one-round face exchange (see halo.h).
#include "halo.h"
#include "peer.cuh"
#include "tmgpu_internal.h"

namespace tmgpu {
namespace {

constexpr int E = 8, G = 2, S = 12, S3 = S * S * S, H = E / 2;

__device__ __forceinline__ double minmod_scalar(double a, double b) {  // limiter.hpp:13-16
  if (a * b <= 0.0) return 0.0;
  return fabs(a) < fabs(b) ? a : b;
}

__device__ __forceinline__ int at(int var, int x, int y, int z) {
  return var * S3 + (z * S + y) * S + x;
}

__device__ __forceinline__ void compose(int axis, int na, int v1, int v2, int& x, int& y, int& z) {
  int c[3];
  c[axis] = na;
  c[(axis + 1) % 3] = v1;
  c[(axis + 2) % 3] = v2;
  x = c[0];
  y = c[1];
  z = c[2];
}

// One CTA per pack item. Slab layouts (n = flat index):
//   same       ((var*E + f2)*E + f1)*G + la   value for destination ghost layer la
//   prolonged  ((var*E + f2)*E + f1)*G + dd   ghost.cpp:161-186 order
//   restricted ((var*H + c2)*H + c1)*G + dd   ghost.cpp:204-224 order
__device__ __forceinline__ void pack_item(const double* __restrict__ arena,
                                          const double* __restrict__ prev, int V,
                                          const PackItem& it, double* out) {
  const double* src = arena + (long long)it.src * V * S3;
  const double* gsrc = prev + (long long)it.src * V * S3;
  const int axis = it.axis, dir = it.dir;
  if (it.kind == 0) {
    for (int n = threadIdx.x; n < V * E * E * G; n += blockDim.x) {
      const int la = n % G, f1 = (n / G) % E, f2 = (n / (G * E)) % E, var = n / (G * E * E);
      int x, y, z;
      compose(axis, dir > 0 ? G + la : E + la, G + f1, G + f2, x, y, z);
      out[n] = src[at(var, x, y, z)];
    }
  } else if (it.kind == 1) {
    for (int n = threadIdx.x; n < V * E * E * G; n += blockDim.x) {
      const int dd = n % G, f1 = (n / G) % E, f2 = (n / (G * E)) % E, var = n / (G * E * E);
      const int cd = dd / 2, sub = dd - 2 * cd;
      const int na = dir > 0 ? G + cd : G + E - 1 - cd;
      const int ct1 = G + it.qt1 * H + f1 / 2, ct2 = G + it.qt2 * H + f2 / 2;
      int x, y, z, xm, ym, zm, xp, yp, zp;
      compose(axis, na, ct1, ct2, x, y, z);
      compose(axis, na - 1, ct1, ct2, xm, ym, zm);
      compose(axis, na + 1, ct1, ct2, xp, yp, zp);
      const double c = src[at(var, x, y, z)];
      // the tap beyond the face is the source's ghost from the previous exchange
      const double cp = dir > 0 ? src[at(var, xp, yp, zp)] : gsrc[at(var, xp, yp, zp)];
      const double cm = dir > 0 ? gsrc[at(var, xm, ym, zm)] : src[at(var, xm, ym, zm)];
      const double off = 0.25 * minmod_scalar(cp - c, c - cm);
      const int sign = dir > 0 ? (sub == 0 ? -1 : +1) : (sub == 0 ? +1 : -1);
      out[n] = sign > 0 ? c + off : c - off;
    }
  } else {
    for (int n = threadIdx.x; n < V * H * H * G; n += blockDim.x) {
      const int dd = n % G, c1 = (n / G) % H, c2 = (n / (G * H)) % H, var = n / (G * H * H);
      double acc = 0.0;
#pragma unroll
      for (int dn = 0; dn < 2; ++dn)
#pragma unroll
        for (int d1 = 0; d1 < 2; ++d1)
#pragma unroll
          for (int d2 = 0; d2 < 2; ++d2) {
            const int fn = dir > 0 ? G + 2 * dd + dn : G + E - 1 - (2 * dd + dn);
            int x, y, z;
            compose(axis, fn, G + 2 * c1 + d1, G + 2 * c2 + d2, x, y, z);
            acc += src[at(var, x, y, z)];
          }
      out[n] = acc * 0.125;
    }
  }
}

__global__ void __launch_bounds__(128) pack_kernel(const double* __restrict__ arena,
                                                   const double* __restrict__ prev, int V,
                                                   const PackItem* __restrict__ items,
                                                   double* __restrict__ slabs) {
  const PackItem it = items[blockIdx.x];
  pack_item(arena, prev, V, it, slabs + it.out);
}

template <int AXIS>
__device__ __forceinline__ void pull_face(double* __restrict__ arena, int V, int slot, int dir,
                                          const FaceSrc& fs, const double* __restrict__ slabs) {
  double* dst = arena + (long long)slot * V * S3;
  constexpr int t1 = (AXIS + 1) % 3, t2 = (AXIS + 2) % 3;
  constexpr int ex = AXIS == 0 ? G : E, ey = AXIS == 1 ? G : E, ez = AXIS == 2 ? G : E;
  const int per_face = V * G * E * E;
  for (int m = threadIdx.x; m < per_face; m += blockDim.x) {
    const int lx = m % ex, ly = (m / ex) % ey, lz = (m / (ex * ey)) % ez, var = m / (ex * ey * ez);
    int p[3] = {G + lx, G + ly, G + lz};
    const int la = AXIS == 0 ? lx : AXIS == 1 ? ly : lz;
    p[AXIS] = (dir > 0 ? G + E : 0) + la;
    const int dd = dir > 0 ? la : G - 1 - la;
    const int f1 = p[t1] - G, f2 = p[t2] - G;
    double v;
    switch (fs.kind) {
      case 0:  // same level (ghost.cpp:40-68)
        if (fs.src[0] >= 0) {
          int q[3] = {p[0], p[1], p[2]};
          q[AXIS] = dir > 0 ? p[AXIS] - E : p[AXIS] + E;
          v = arena[(long long)fs.src[0] * V * S3 + at(var, q[0], q[1], q[2])];
        } else {
          v = slabs[fs.off[0] + ((var * E + f2) * E + f1) * G + la];
        }
        break;
      case 3: {  // reflective wall (ghost.cpp:151-166)
        int q[3] = {p[0], p[1], p[2]};
        q[AXIS] = dir > 0 ? 2 * (G + E) - 1 - p[AXIS] : 2 * G - 1 - p[AXIS];
        const double sgn = (V == 5 && var == 1 + AXIS) ? -1.0 : 1.0;
        v = sgn * dst[at(var, q[0], q[1], q[2])];
        break;
      }
      case 1:  // coarser: prolonged slab (ghost.cpp:98-111)
        v = slabs[fs.off[0] + ((var * E + f2) * E + f1) * G + dd];
        break;
      default: {  // finer: restricted quadrant (ghost.cpp:135-149)
        const int qt1 = f1 / H, qt2 = f2 / H, c1 = f1 % H, c2 = f2 % H, q = qt2 * 2 + qt1;
        if (fs.src[q] >= 0) {
          const double* src = arena + (long long)fs.src[q] * V * S3;
          double acc = 0.0;
#pragma unroll
          for (int dn = 0; dn < 2; ++dn)
#pragma unroll
            for (int d1 = 0; d1 < 2; ++d1)
#pragma unroll
              for (int d2 = 0; d2 < 2; ++d2) {
                const int fn = dir > 0 ? G + 2 * dd + dn : G + E - 1 - (2 * dd + dn);
                int x, y, z;
                compose(AXIS, fn, G + 2 * c1 + d1, G + 2 * c2 + d2, x, y, z);
                acc += src[at(var, x, y, z)];
              }
          v = acc * 0.125;
        } else {
          v = slabs[fs.off[q] + ((var * H + c2) * H + c1) * G + dd];
        }
        break;
      }
    }
    dst[at(var, p[0], p[1], p[2])] = v;
  }
}

__device__ __forceinline__ void pull_item(double* __restrict__ arena, int V,
                                          const FaceSrc* __restrict__ faces, int2 it,
                                          const double* __restrict__ slabs) {
  // it = (slot, face = 2*axis + (dir > 0))
  const FaceSrc fs = faces[(long long)it.x * 6 + it.y];
  const int axis = it.y >> 1, dir = (it.y & 1) ? 1 : -1;
  if (axis == 0)
    pull_face<0>(arena, V, it.x, dir, fs, slabs);
  else if (axis == 1)
    pull_face<1>(arena, V, it.x, dir, fs, slabs);
  else
    pull_face<2>(arena, V, it.x, dir, fs, slabs);
}

__global__ void __launch_bounds__(128) pull_kernel(double* __restrict__ arena, int V,
                                                   const FaceSrc* __restrict__ faces,
                                                   const int2* __restrict__ items,
                                                   const double* __restrict__ slabs) {
  pull_item(arena, V, faces, items[blockIdx.x], slabs);
}

// ---- peer-memory exchange (PeerTab in halo.h; flag helpers in peer.cuh) ---

// Pack straight into the destination rank's receive region. Items with
// pad[0] = q + 1 go to peer q: the CTA first waits until q has consumed the
// previous exchange's slabs (WAR), and the last of q's CTAs raises q's
// arrival flag after a system-scope fence.
__global__ void __launch_bounds__(128) pack_peer_kernel(const double* __restrict__ arena,
                                                        const double* __restrict__ prev, int V,
                                                        const PackItem* __restrict__ items,
                                                        double* __restrict__ slabs, PeerTab t) {
  const unsigned long long seq = *t.seqp;  // this round's (seq_bump ran before on the stream)
  const PackItem it = items[blockIdx.x];
  const int q = it.pad[0] - 1;
  if (q < 0) {
    pack_item(arena, prev, V, it, slabs + it.out);
    return;
  }
  if (threadIdx.x == 0) spin_geq(t.mine + t.world + q, seq - 1, t.spin_ns);
  __syncthreads();
  pack_item(arena, prev, V, it, t.slabs[q] + it.out);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* cnt = t.mine + 2 * t.world + q;
    if (atomicAdd(cnt, 1ull) == (unsigned long long)t.n_send[q] - 1) {
      *cnt = 0;
      __threadfence_system();
      st_release_sys(t.flags[q] + t.me, seq);
    }
  }
}

// Pull with items [0, n_local) needing no received slab and [n_local, n) that
// do: those CTAs wait for every sender's arrival flag; the last of them tells
// each sender that its slabs are consumed.
__global__ void __launch_bounds__(128) pull_peer_kernel(double* __restrict__ arena, int V,
                                                        const FaceSrc* __restrict__ faces,
                                                        const int2* __restrict__ items,
                                                        const double* __restrict__ slabs,
                                                        PeerTab t, int n_local, int n_remote) {
  const unsigned long long seq = *t.seqp;
  const bool remote = (int)blockIdx.x >= n_local;
  if (remote) {
    if (threadIdx.x == 0)
      for (int s = 0; s < t.world; ++s)
        if (t.recv_mask >> s & 1u) spin_geq(t.mine + s, seq, t.spin_ns);
    __syncthreads();
  }
  pull_item(arena, V, faces, items[blockIdx.x], slabs);
  if (!remote) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* cnt = t.mine + 3 * t.world;
    if (atomicAdd(cnt, 1ull) == (unsigned long long)n_remote - 1) {
      *cnt = 0;
      __threadfence_system();
      for (int s = 0; s < t.world; ++s)
        if (t.recv_mask >> s & 1u) st_release_sys(t.flags[s] + t.world + t.me, seq);
    }
  }
}

__global__ void seq_bump_kernel(unsigned long long* p) { *p += 1; }

}  // namespace

cudaError_t seq_bump(unsigned long long* p, cudaStream_t st) {
  seq_bump_kernel<<<1, 1, 0, st>>>(p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t halo_pack(const double* arena, const double* prev, int V, const PackItem* items,
                      int n_items, double* slabs, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  pack_kernel<<<n_items, 128, 0, st>>>(arena, prev, V, items, slabs);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t halo_pull(double* arena, int V, const FaceSrc* faces, const int2* items, int n_items,
                      const double* slabs, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  pull_kernel<<<n_items, 128, 0, st>>>(arena, V, faces, items, slabs);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t halo_pack_peer(const double* arena, const double* prev, int V, const PackItem* items,
                           int n_items, double* slabs, const PeerTab& t, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  pack_peer_kernel<<<n_items, 128, 0, st>>>(arena, prev, V, items, slabs, t);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t halo_pull_peer(double* arena, int V, const FaceSrc* faces, const int2* items,
                           int n_local, int n_items, const double* slabs, const PeerTab& t,
                           cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  pull_peer_kernel<<<n_items, 128, 0, st>>>(arena, V, faces, items, slabs, t, n_local,
                                            n_items - n_local);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace tmgpu
