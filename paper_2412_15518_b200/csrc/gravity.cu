// Cell-level FMM gravity on a uniform octree level (rows a12/a13 of SURVEY.md §8).
//
// The reference has no gravity code (prose only, PAPER.md:120,
// 233,238,241,347), so the specification is ours and is restated operation by
// operation in oracle/gravity_oracle.c; these kernels follow
// the same operation order and are bitwise equal to it (-fmad=false).
//
//   P2M   masses m = rho * h^3 of the finest cells (from the leaf arena)
//   M2M   order-2 Cartesian moments (M, D_i, Q_ij) per cell of every level
//   M2L   per level, each cell sums its 189-cell interaction list ("stencil
//         approach"): children of the parent's 27 neighbours that
//         are not its own neighbours; Dehnen truncation |alpha|+|beta| <= 2,
//         which makes every mutual pair force exactly opposite (linear
//         momentum conserved to round-off)
//   L2L   local expansions shifted down the levels
//   P2P   monopole near field over the 26 neighbours at the finest level,
//         fused with L2P (phi = L0, g = -L_i at the cell centre)
#include <cstring>
#include <vector>

#include "gravity_common.cuh"

namespace tmgpu {
namespace {

__global__ void p2m_kernel(const double* __restrict__ mass, double* __restrict__ mom, long long n3) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n3;
       c += (long long)gridDim.x * blockDim.x) {
    double* o = mom + c * 10;
    o[0] = mass[c];
#pragma unroll
    for (int q = 1; q < 10; ++q) o[q] = 0.0;
  }
}

// arena (uniform level, leaf slot = canonical Morton order) -> finest masses (k,j,i)
__global__ void arena_mass_kernel(const double* __restrict__ arena, const int* __restrict__ leaf_ijk,
                                  long long nleaves, int V, double dV, long long N,
                                  double* __restrict__ mass) {
  const long long total = nleaves * 512;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long s = t >> 9;
    const int c = (int)(t & 511);
    const int i = c & 7, j = (c >> 3) & 7, k = c >> 6;
    const double rho = arena[s * V * 1728 + ((k + 2) * 12 + (j + 2)) * 12 + (i + 2)];
    const long long gi = leaf_ijk[3 * s] * 8LL + i, gj = leaf_ijk[3 * s + 1] * 8LL + j,
                    gk = leaf_ijk[3 * s + 2] * 8LL + k;
    mass[cidx(N, gi, gj, gk)] = rho * dV;
  }
}

// Tiled M2L for levels with m >= 8: a CTA owns an 8x4x4 block of targets
// (128 threads, one target each); the union of their interaction lists is the
// 12x8x8 source box [x0-2, x0+9] x [y0-2, y0+5] x [z0-2, z0+5], staged once in
// shared memory (SoA by component) and reused by all 128 targets. Per-target
// loop order and arithmetic are those of m2l_kernel (bitwise identical).
constexpr int TBX = 8, TBY = 4, TBZ = 4;
constexpr int SBX = TBX + 4, SBY = TBY + 4, SBZ = TBZ + 4, SB3 = SBX * SBY * SBZ;

__global__ void __launch_bounds__(128) m2l_tiled_kernel(const double* __restrict__ mom,
                                                        double* __restrict__ loc, long long m,
                                                        const double* __restrict__ tab) {
  extern __shared__ double sm[];  // 10 x SB3 doubles = 61,440 B (dynamic)
  const long long nbx = m / TBX, nby = m / TBY;
  const long long b = blockIdx.x;
  const long long x0 = (b % nbx) * TBX, y0 = ((b / nbx) % nby) * TBY, z0 = (b / (nbx * nby)) * TBZ;
  for (int q = threadIdx.x; q < SB3; q += blockDim.x) {
    const long long sx = x0 - 2 + q % SBX, sy = y0 - 2 + (q / SBX) % SBY, sz = z0 - 2 + q / (SBX * SBY);
    const bool in = sx >= 0 && sy >= 0 && sz >= 0 && sx < m && sy < m && sz < m;
    const double* src = mom + cidx(m, in ? sx : 0, in ? sy : 0, in ? sz : 0) * 10;
#pragma unroll
    for (int c = 0; c < 10; ++c) sm[c * SB3 + q] = in ? src[c] : 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x % TBX, ty = (threadIdx.x / TBX) % TBY, tz = threadIdx.x / (TBX * TBY);
  const long long i = x0 + tx, j = y0 + ty, k = z0 + tz;
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
        const int q = (int)(((sk - z0 + 2) * SBY + (sj - y0 + 2)) * SBX + (si - x0 + 2));
        double mom_q[10];
#pragma unroll
        for (int c = 0; c < 10; ++c) mom_q[c] = sm[c * SB3 + q];
        m2l_tab(mom_q, tab + (((dz + 3) * kOff + (dy + 3)) * kOff + (dx + 3)) * kTab,
                o[dz + (k & 1) >= 1]);
      }
  double* out = loc + cidx(m, i, j, k) * 10;
#pragma unroll
  for (int q = 0; q < 10; ++q) out[q] = o[0][q] + o[1][q];
}

__global__ void p2p_kernel(const double* __restrict__ mass, const double* __restrict__ loc,
                           long long N, double h, double* __restrict__ phi, double* __restrict__ g) {
  const long long n3 = N * N * N;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n3;
       c += (long long)gridDim.x * blockDim.x) {
    const long long i = c % N, j = (c / N) % N, k = c / (N * N);
    const double* L = loc + c * 10;
    double p = L[0], gx = -L[1], gy = -L[2], gz = -L[3];
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (!dx && !dy && !dz) continue;
          const long long si = i + dx, sj = j + dy, sk = k + dz;
          if (si < 0 || sj < 0 || sk < 0 || si >= N || sj >= N || sk >= N) continue;
          const double nm = -mass[cidx(N, si, sj, sk)];
          double w[4];
          p2p_geom(-(double)dx * h, -(double)dy * h, -(double)dz * h, w);
          p = fma(nm, w[0], p);
          gx = fma(nm, w[1], gx);
          gy = fma(nm, w[2], gy);
          gz = fma(nm, w[3], gz);
        }
    phi[c] = p;
    g[c] = gx;
    g[n3 + c] = gy;
    g[2 * n3 + c] = gz;
  }
}

}  // namespace

struct GravityWork {
  int D = 0;
  std::vector<double*> mom, loc;
  double* mass = nullptr;
  double* tab = nullptr;  // [level][343][13] stencil geometry
};

}  // namespace tmgpu

using namespace tmgpu;

struct tmgpu_gravity {
  GravityWork w;
};

extern "C" {

// Workspace for a uniform cell level D (N = 2^D cells per axis).
tmgpu_gravity* tmgpu_gravity_create(int D, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (D < 2 || D > 11) {
    set_err(err, TMGPU_ERR_INVALID, "gravity: cell level must be in [2, 11]");
    return nullptr;
  }
  auto* g = new tmgpu_gravity;
  g->w.D = D;
  cudaError_t e = cudaSuccess;
  for (int l = 0; l <= D && e == cudaSuccess; ++l) {
    const size_t n3 = (size_t)1 << (3 * l);
    double *m = nullptr, *L = nullptr;
    e = cudaMalloc(&m, n3 * 10 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&L, n3 * 10 * sizeof(double));
    g->w.mom.push_back(m);
    g->w.loc.push_back(L);
  }
  if (e == cudaSuccess) e = cudaMalloc(&g->w.mass, ((size_t)1 << (3 * D)) * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&g->w.tab, (size_t)(D + 1) * kOff3 * kTab * sizeof(double));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(m2l_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(10 * SB3 * sizeof(double)));
  if (e == cudaSuccess) {
    stencil_table_kernel<<<((D + 1) * kOff3 + 127) / 128, 128>>>(g->w.tab, D);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = cudaDeviceSynchronize();
  }
  if (e != cudaSuccess) {
    cuda_err(err, e, "tmgpu_gravity_create");
    for (auto p : g->w.mom)
      if (p) cudaFree(p);
    for (auto p : g->w.loc)
      if (p) cudaFree(p);
    delete g;
    return nullptr;
  }
  return g;
}

void tmgpu_gravity_destroy(tmgpu_gravity* g) {
  if (!g) return;
  for (auto p : g->w.mom) cudaFree(p);
  for (auto p : g->w.loc) cudaFree(p);
  if (g->w.mass) cudaFree(g->w.mass);
  if (g->w.tab) cudaFree(g->w.tab);
  delete g;
}

// Solve from finest-level masses ((k,j,i), x fastest). mass == NULL: use the
// workspace masses (filled by tmgpu_gravity_mass_from_forest). Device pointers
// unless TMGPU_HOST_PTRS. phi: N^3, g: 3 x N^3.
int tmgpu_gravity_solve(tmgpu_gravity* G, const double* mass, double* phi, double* g, int flags,
                        void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  cudaStream_t st = as_stream(stream);
  GravityWork& w = G->w;
  const int D = w.D;
  const long long N = 1LL << D, n3 = N * N * N;
  const bool host = (flags & TMGPU_HOST_PTRS) != 0;
  cudaError_t e = cudaSuccess;
  double *dphi = phi, *dg = g;
  if (mass) {
    e = cudaMemcpyAsync(w.mass, mass, n3 * sizeof(double),
                        host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st);
  }
  if (host && e == cudaSuccess) {
    e = cudaMallocAsync(&dphi, n3 * sizeof(double), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&dg, 3 * n3 * sizeof(double), st);
  }
  if (e == cudaSuccess) {
    p2m_kernel<<<grid_for(n3), 128, 0, st>>>(w.mass, w.mom[D], n3);
    for (int l = D - 1; l >= 0; --l)
      m2m_kernel<<<grid_for(1LL << (3 * l)), 128, 0, st>>>(w.mom[l + 1], w.mom[l], 1LL << l,
                                                          1.0 / (double)(1LL << (l + 1)));
    for (int l = 2; l <= D; ++l) {
      const long long m = 1LL << l;
      if (m >= TBX)
        m2l_tiled_kernel<<<(unsigned)(m * m * m / (TBX * TBY * TBZ)), 128,
                           10 * SB3 * sizeof(double), st>>>(
            w.mom[l], w.loc[l], m, w.tab + (long long)l * kOff3 * kTab);
      else
        m2l_kernel<<<grid_for(m * m * m), 128, 0, st>>>(w.mom[l], w.loc[l], m,
                                                         w.tab + (long long)l * kOff3 * kTab);
    }
    for (int l = 3; l <= D; ++l)
      l2l_kernel<<<grid_for(1LL << (3 * l)), 128, 0, st>>>(w.loc[l - 1], w.loc[l], 1LL << l,
                                                          1.0 / (double)(1LL << l));
    p2p_kernel<<<grid_for(n3), 128, 0, st>>>(w.mass, w.loc[D], N, 1.0 / (double)N, dphi, dg);
    g_launches.fetch_add(2 + D + 2 * (D - 1), std::memory_order_relaxed);
    e = cudaGetLastError();
  }
  if (host) {
    if (e == cudaSuccess) e = cudaMemcpyAsync(phi, dphi, n3 * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g, dg, 3 * n3 * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (dphi && dphi != phi) cudaFreeAsync(dphi, st);
    if (dg && dg != g) cudaFreeAsync(dg, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = e2;
  } else if (!(flags & TMGPU_ASYNC)) {
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = e2;
  }
  return cuda_err(err, e, "tmgpu_gravity_solve");
}

// Finest-level masses from a device leaf arena of a UNIFORM forest: leaf s
// covers cells 8*leaf_ijk[3s..3s+2] + (i,j,k); mass = rho * dV.
int tmgpu_gravity_mass_from_arena(tmgpu_gravity* G, const double* arena, const int* leaf_ijk_dev,
                                  long long nleaves, int vars, double dV, void* stream,
                                  tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  const long long N = 1LL << G->w.D;
  if (nleaves * 512 != N * N * N) return set_err(err, TMGPU_ERR_INVALID, "gravity: leaves do not tile the level");
  cudaStream_t st = as_stream(stream);
  arena_mass_kernel<<<grid_for(nleaves * 512), 128, 0, st>>>(arena, leaf_ijk_dev, nleaves, vars, dV,
                                                             N, G->w.mass);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_err(err, cudaGetLastError(), "tmgpu_gravity_mass_from_arena");
}

}  // extern "C"
