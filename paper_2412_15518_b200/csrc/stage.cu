// Stage-kernel instantiations, TMA map encoding and the small hydro kernels
// (max_wavespeed, rk3_combine). Compiled with -fmad=false: the BITWISE
// kernels must not have their multiply/add pairs contracted (reference
// CMakeLists.txt:12-14 builds with -ffp-contract=off); the FAST kernels use
// explicit fma() instead.
#include <cudaTypedefs.h>

#include <mutex>

#include <cstdlib>

#include "stage_kernel.cuh"
#include "tmgpu_internal.h"

namespace tmgpu {

std::atomic<uint64_t> g_launches{0};

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

template <int V, bool FAST>
cudaError_t launch_stage_t(const StageMaps& m, const StageLaunch& p, cudaStream_t stream) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(stage_kernel<V, FAST>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, Lay<V>::kBytes);
  });
  if (attr_err != cudaSuccess) return attr_err;
  if (p.count <= 0) return cudaSuccess;
  static const int ahead = [] {  // two resident CTAs per SM: one wave ahead
    if (const char* v = std::getenv("TMGPU_STAGE_PREFETCH")) return std::atoi(v);
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return 2 * sms;
  }();
  StageLaunch q = p;
  q.prefetch_ahead = ahead;
  stage_kernel<V, FAST><<<p.count, kStageThreads, Lay<V>::kBytes, stream>>>(m.i, m.x, m.y, m.z, q);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// stage.cpp:248-272 max_wavespeed, one CTA per slot; block max of
// |v| + sqrt(gamma p / rho) with the reference's floors and divisions.
__global__ void __launch_bounds__(256) max_wavespeed_kernel(const double* __restrict__ in,
                                                            long long slot_stride,
                                                            const double* __restrict__ hdr,
                                                            long long hdr_stride,
                                                            const double* __restrict__ leaf_dx,
                                                            double g_gamma, int V,
                                                            double* __restrict__ result) {
  (void)leaf_dx;
  const int s = blockIdx.x;
  double gamma = g_gamma, mode = 1.0, ax = 0, ay = 0, az = 0;
  if (hdr) {
    const double* h = hdr + (long long)s * hdr_stride;
    mode = h[0];
    gamma = h[3];
    ax = h[4];
    ay = h[5];
    az = h[6];
  }
  __shared__ double red[8];
  if (mode == 0.0) {
    if (threadIdx.x == 0) result[s] = sqrt(ax * ax + ay * ay + az * az);
    return;
  }
  const double* g = in + (long long)s * slot_stride;
  const int s3 = kS * kS * kS;
  double smax = 0.0;
  for (int c = threadIdx.x; c < kE3; c += blockDim.x) {
    const int i = kG + (c & 7), j = kG + ((c >> 3) & 7), k = kG + (c >> 6);
    const int o = (k * kS + j) * kS + i;
    const double rho = stdmax_(g[o], kRhoFloor);
    const double iu = g[s3 + o] / rho, iv = g[2 * s3 + o] / rho, iw = g[3 * s3 + o] / rho;
    const double ke = 0.5 * rho * (iu * iu + iv * iv + iw * iw);
    const double pr = stdmax_((gamma - 1.0) * (g[4 * s3 + o] - ke), kPressureFloor);
    const double sp = sqrt(iu * iu + iv * iv + iw * iw) + sqrt(gamma * pr / rho);
    smax = stdmax_(smax, sp);
  }
  (void)V;
  for (int off = 16; off > 0; off >>= 1) smax = stdmax_(smax, __shfl_xor_sync(0xffffffffu, smax, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = smax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = stdmax_(m, red[w]);
    result[s] = m;
  }
}

// The step's first pass when its input arrives as compact interiors
// [slot][V][E^3] (tmgpu_forest_step_io): each CTA copies its slot's interior
// into the ghosted arena (the scatter of tmgpu_forest_interior) and, from the
// same registers, computes max_wavespeed exactly as max_wavespeed_kernel
// (Euler; the reference's floors and divisions): one read of the input
// instead of a scatter pass plus a wavespeed pass over the arena.
__global__ void __launch_bounds__(256) scatter_wavespeed_kernel(const double* __restrict__ compact,
                                                                double* __restrict__ arena,
                                                                long long slot_stride, double gamma,
                                                                double* __restrict__ result) {
  const int s = blockIdx.x;
  __shared__ double red[8];
  const double* src = compact + (long long)s * 5 * kE3;
  double* g = arena + (long long)s * slot_stride;
  const int s3 = kS * kS * kS;
  double smax = 0.0;
  for (int c = threadIdx.x; c < kE3; c += blockDim.x) {
    const int i = kG + (c & 7), j = kG + ((c >> 3) & 7), k = kG + (c >> 6);
    const int o = (k * kS + j) * kS + i;
    double u[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      u[v] = src[v * kE3 + c];
      g[v * s3 + o] = u[v];
    }
    const double rho = stdmax_(u[0], kRhoFloor);
    const double iu = u[1] / rho, iv = u[2] / rho, iw = u[3] / rho;
    const double ke = 0.5 * rho * (iu * iu + iv * iv + iw * iw);
    const double pr = stdmax_((gamma - 1.0) * (u[4] - ke), kPressureFloor);
    const double sp = sqrt(iu * iu + iv * iv + iw * iw) + sqrt(gamma * pr / rho);
    smax = stdmax_(smax, sp);
  }
  for (int off = 16; off > 0; off >>= 1) smax = stdmax_(smax, __shfl_xor_sync(0xffffffffu, smax, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = smax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = stdmax_(m, red[w]);
    result[s] = m;
  }
}

// rk3.hpp:18-27
__global__ void rk3_combine_kernel(int stage, const double* __restrict__ u0,
                                   const double* __restrict__ v, double* __restrict__ out,
                                   long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double a = u0[i], b = v[i];
    out[i] = stage == 1 ? b : stage == 2 ? a + 0.25 * (b - a) : a + (2.0 / 3.0) * (b - a);
  }
}

// dt = cfl * min_leaf(dx_leaf / smax_leaf) (min over cells
// of dx/s equals dx / max s because IEEE division is monotone). One block.
__global__ void __launch_bounds__(1024) cfl_reduce_kernel(const double* __restrict__ speeds,
                                                          const double* __restrict__ leaf_dx,
                                                          long long n, double cfl,
                                                          double* __restrict__ dt) {
  __shared__ double red[32];
  double m = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double s = speeds[i];
    if (s > 0.0) {
      const double q = leaf_dx[i] / s;
      m = q < m ? q : m;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, m, off);
    m = o < m ? o : m;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = red[w] < m ? red[w] : m;
    dt[0] = cfl * m;
  }
}

}  // namespace

cudaError_t launch_cfl_reduce(const double* speeds, const double* leaf_dx, long long n, double cfl,
                              double* dt, cudaStream_t stream) {
  cfl_reduce_kernel<<<1, 1024, 0, stream>>>(speeds, leaf_dx, n, cfl, dt);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

int make_stage_maps(const double* base, int V, long long slot_stride, long long count,
                    StageMaps* maps, std::string* why) {
  auto fn = encode_fn();
  if (!fn) {
    if (why) *why = "cuTensorMapEncodeTiled unavailable";
    return TMGPU_ERR_CUDA;
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || ((slot_stride * 8) & 15) != 0) {
    if (why) *why = "TMA needs 16-byte aligned sub-grid blocks";
    return TMGPU_ERR_INVALID;
  }
  cuuint64_t dims[5] = {12, 12, 12, (cuuint64_t)V, (cuuint64_t)(count > 0 ? count : 1)};
  cuuint64_t strides[4] = {12 * 8, 144 * 8, 1728 * 8, (cuuint64_t)slot_stride * 8};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const cuuint32_t boxes[4][5] = {{10, 8, 8, (cuuint32_t)V, 1},
                                  {2, 8, 8, (cuuint32_t)V, 1},
                                  {8, 2, 8, (cuuint32_t)V, 1},
                                  {8, 8, 2, (cuuint32_t)V, 1}};
  CUtensorMap* out[4] = {&maps->i, &maps->x, &maps->y, &maps->z};
  for (int b = 0; b < 4; ++b) {
    CUresult r = fn(out[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(base), dims,
                    strides, boxes[b], estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      if (why) *why = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
      return TMGPU_ERR_CUDA;
    }
  }
  return TMGPU_OK;
}

cudaError_t launch_stage(int V, bool fast, const StageMaps& m, const StageLaunch& p,
                         cudaStream_t stream) {
  if (V == 5) return fast ? launch_stage_t<5, true>(m, p, stream) : launch_stage_t<5, false>(m, p, stream);
  if (V == 1) return fast ? launch_stage_t<1, true>(m, p, stream) : launch_stage_t<1, false>(m, p, stream);
  return cudaErrorInvalidValue;
}

cudaError_t launch_stage_epilogue(bool fast, const double* in_arena, const StageLaunch& p, cudaStream_t stream) {
  if (p.count <= 0) return cudaSuccess;
  if (fast)
    stage_epilogue_kernel<true><<<p.count, 256, 0, stream>>>(in_arena, p);
  else
    stage_epilogue_kernel<false><<<p.count, 256, 0, stream>>>(in_arena, p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_max_wavespeed(const double* in, long long slot_stride, const double* hdr,
                                 long long hdr_stride, const double* leaf_dx, double g_gamma,
                                 int V, long long count, double* result, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  max_wavespeed_kernel<<<(unsigned)count, 256, 0, stream>>>(in, slot_stride, hdr, hdr_stride,
                                                            leaf_dx, g_gamma, V, result);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_scatter_wavespeed(const double* compact, double* arena, long long slot_stride, double gamma,
                                     long long count, double* result, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  scatter_wavespeed_kernel<<<(unsigned)count, 256, 0, stream>>>(compact, arena, slot_stride, gamma, result);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_rk3_combine(int stage, const double* u0, const double* v, double* out,
                               long long n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  rk3_combine_kernel<<<(unsigned)blocks, 256, 0, stream>>>(stage, u0, v, out, n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace tmgpu
