// AMR regrid with data on the device: the reference's
// Tree::refine -> prolong_into_children / prolong_cell and Tree::coarsen ->
// restrict_cells (proj/src/amr/octree.cpp:149-293), and flag_refinement
// (:295-323). Same arithmetic and order, so regridded grids equal the
// reference's bit for bit (tests/test_regrid_gpu.py).
#include "tmgpu_internal.h"

namespace tmgpu {
namespace {

// limiter.hpp:13-16 scalar minmod
__device__ __forceinline__ double minmod_s(double a, double b) {
  if (a * b <= 0.0) return 0.0;
  return fabs(a) < fabs(b) ? a : b;
}

__device__ __forceinline__ long long gidx(int var, int i, int j, int k) {
  return ((long long)(var * 12 + k) * 12 + j) * 12 + i;
}

// octree.cpp:149-198: parent interior cell -> 2x2x2 cells of one child
// (children[b], b = bk*4 + bj*2 + bi, zeroed ghosted blocks)
__global__ void prolong_kernel(const double* __restrict__ pg, double* __restrict__ children, int V) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < V * 512; t += gridDim.x * blockDim.x) {
    const int var = t >> 9, c = t & 511;
    const int pi = c & 7, pj = (c >> 3) & 7, pk = c >> 6;
    const int i = pi + 2, j = pj + 2, k = pk + 2;
    const double cc = pg[gidx(var, i, j, k)];
    const double ox = 0.25 * minmod_s(pg[gidx(var, i + 1, j, k)] - cc, cc - pg[gidx(var, i - 1, j, k)]);
    const double oy = 0.25 * minmod_s(pg[gidx(var, i, j + 1, k)] - cc, cc - pg[gidx(var, i, j - 1, k)]);
    const double oz = 0.25 * minmod_s(pg[gidx(var, i, j, k + 1)] - cc, cc - pg[gidx(var, i, j, k - 1)]);
    const int bi = pi >= 4, bj = pj >= 4, bk = pk >= 4;
    double* cg = children + (long long)(bk * 4 + bj * 2 + bi) * V * 1728;
    const int fi = 2 + 2 * pi - bi * 8, fj = 2 + 2 * pj - bj * 8, fk = 2 + 2 * pk - bk * 8;
#pragma unroll
    for (int dk = 0; dk < 2; ++dk)
#pragma unroll
      for (int dj = 0; dj < 2; ++dj)
#pragma unroll
        for (int di = 0; di < 2; ++di) {
          double v = cc + (di ? ox : -ox);
          v += dj ? oy : -oy;
          v += dk ? oz : -oz;
          cg[gidx(var, fi + di, fj + dj, fk + dk)] = v;
        }
  }
}

struct Ptr8 {
  const double* p[8];
};

// octree.cpp:236-293 + restrict_cells: parent interior cell = mean of the
// 8 fine cells, summed in (dk, dj, di) order from 0.0, times 0.125
__global__ void restrict_kernel(Ptr8 ch, double* __restrict__ pg, int V) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < V * 512; t += gridDim.x * blockDim.x) {
    const int var = t >> 9, c = t & 511;
    const int pi = c & 7, pj = (c >> 3) & 7, pk = c >> 6;
    const int bi = pi >= 4, bj = pj >= 4, bk = pk >= 4;
    const double* cg = ch.p[bk * 4 + bj * 2 + bi];
    const int fi = 2 + 2 * pi - bi * 8, fj = 2 + 2 * pj - bj * 8, fk = 2 + 2 * pk - bk * 8;
    double acc = 0.0;
#pragma unroll
    for (int dk = 0; dk < 2; ++dk)
#pragma unroll
      for (int dj = 0; dj < 2; ++dj)
#pragma unroll
        for (int di = 0; di < 2; ++di) acc += cg[gidx(var, fi + di, fj + dj, fk + dk)];
    pg[gidx(var, pi + 2, pj + 2, pk + 2)] = acc * 0.125;
  }
}

// whole ghosted blocks src[s] -> dst + s*stride
__global__ void gather_blocks_kernel(const double* const* __restrict__ src, double* __restrict__ dst,
                                     long long stride) {
  const double* s = src[blockIdx.y];
  double* d = dst + (long long)blockIdx.y * stride;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < stride;
       q += (long long)gridDim.x * blockDim.x)
    d[q] = s[q];
}

// octree.cpp:295-323 flag_refinement: any interior cell with
// |grad rho| / max(rho, floor) > theta (centred differences, undivided)
__global__ void __launch_bounds__(512) flag_kernel(const double* __restrict__ arena, long long stride,
                                                   double theta, double rho_floor, int* __restrict__ flag) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  const double* g = arena + (long long)blockIdx.x * stride;
  const int c = threadIdx.x;
  const int i = (c & 7) + 2, j = ((c >> 3) & 7) + 2, k = (c >> 6) + 2;
  const double gx = 0.5 * (g[gidx(0, i + 1, j, k)] - g[gidx(0, i - 1, j, k)]);
  const double gy = 0.5 * (g[gidx(0, i, j + 1, k)] - g[gidx(0, i, j - 1, k)]);
  const double gz = 0.5 * (g[gidx(0, i, j, k + 1)] - g[gidx(0, i, j, k - 1)]);
  const double mag = sqrt(gx * gx + gy * gy + gz * gz);
  const double r0 = g[gidx(0, i, j, k)];
  const double rho = (r0 < rho_floor) ? rho_floor : r0;  // std::max(r0, floor)
  if (mag / rho > theta) any = 1;
  __syncthreads();
  if (threadIdx.x == 0) flag[blockIdx.x] = any;
}

}  // namespace

cudaError_t launch_prolong(const double* parent, double* children8, int V, cudaStream_t st) {
  prolong_kernel<<<10, 256, 0, st>>>(parent, children8, V);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_restrict(const double* const* children, double* parent, int V, cudaStream_t st) {
  Ptr8 p;
  for (int b = 0; b < 8; ++b) p.p[b] = children[b];
  restrict_kernel<<<10, 256, 0, st>>>(p, parent, V);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_gather_blocks(const double* const* src_dev, long long n, double* dst, long long stride,
                                 cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  for (long long b = 0; b < n; b += 65535) {
    const long long m = n - b < 65535 ? n - b : 65535;
    gather_blocks_kernel<<<dim3(8, (unsigned)m), 256, 0, st>>>(src_dev + b, dst + b * stride, stride);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  return cudaGetLastError();
}

cudaError_t launch_flag(const double* arena, long long stride, long long n, double theta, double rho_floor,
                        int* flag, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  flag_kernel<<<(unsigned)n, 512, 0, st>>>(arena, stride, theta, rho_floor, flag);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace tmgpu
