// NOT PRODUCT CODE (tools/probes -> libtmprobe.so): the reference tests' toy
// fusable kernel y = 2x + 1 (test_aggregator.cpp:17-29) as a custom device
// kernel (tmgpu_region_create_kernel), used by tests/test_aggregator.py to
// replay the reference's aggregation tests on the device.
#include <cstddef>

#include <cuda_runtime.h>

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

// tmgpu_device_kernel (include/tmgpu.h)
extern "C" int tmprobe_affine_launch(const double* in, double* out, size_t in_slice, size_t out_slice,
                                     size_t count, void* stream, void* /*user*/) {
  const long long n = (long long)(count * in_slice);
  long long blocks = (n + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 1184) blocks = 1184;
  affine_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      in, out, (long long)in_slice, (long long)out_slice, (long long)count);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
