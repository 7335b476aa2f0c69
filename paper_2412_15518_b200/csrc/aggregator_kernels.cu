// Device kernels of the aggregation executor that are not the hydro stage:
// the reference tests' toy fusable kernel y = 2x + 1 (test_aggregator.cpp:17-29),
// used to replay the reference's aggregation tests on the device.
#include "tmgpu_internal.h"

namespace tmgpu {
namespace {
__global__ void affine_kernel(const double* __restrict__ in, double* __restrict__ out,
                              long long in_slice, long long out_slice, long long count) {
  const long long n = count * in_slice;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long s = i / in_slice, k = i % in_slice;
    if (k < out_slice) out[s * out_slice + k] = 2.0 * in[i] + 1.0;
  }
}
}  // namespace

cudaError_t launch_affine(const double* in, double* out, long long in_slice, long long out_slice,
                          long long count, cudaStream_t st) {
  const long long n = count * in_slice;
  long long blocks = (n + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 1184) blocks = 1184;
  affine_kernel<<<(unsigned)blocks, 256, 0, st>>>(in, out, in_slice, out_slice, count);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}
}  // namespace tmgpu
