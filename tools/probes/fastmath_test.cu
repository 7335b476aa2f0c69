// NOT PRODUCT CODE (tools/probes -> libtmprobe.so, loaded by tests/test_fastmath_gpu.py):
// device self-test of the product's fastmath.cuh: bitwise comparison of the branch-free
// division / square root with the IEEE operators over random operands.
#include <cstdint>

#include "fastmath.cuh"
#include "tmgpu_internal.h"  // error codes, cuda_err (product header, -I)

namespace tmgpu {
namespace {

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ double u01(uint64_t x) { return (double)(x >> 11) * 0x1p-53; }

__device__ __forceinline__ double loguni(uint64_t x, double lo, double hi) {
  return exp(log(lo) + (log(hi) - log(lo)) * u01(x));
}

__global__ void fm_selftest_kernel(uint64_t seed, long long n, int mode,
                                   unsigned long long* bad, unsigned long long* checked,
                                   double* first) {
  unsigned long long nb = 0, nc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t r1 = splitmix(seed ^ (uint64_t)i * 2), r2 = splitmix(seed ^ ((uint64_t)i * 2 + 1));
    double a = 0, b = 1, want, got;
    bool ok = true;
    if (mode <= 2) {
      if (mode == 0) {
        a = __longlong_as_double((long long)r1);
        b = __longlong_as_double((long long)r2);
      } else if (mode == 1) {  // stage operands: gamma*p / rho and p / (gamma-1)
        a = loguni(r1, 1e-12, 1e7) * ((r1 & 1) ? 1.0 : -1.0);
        b = loguni(r2, 1e-10, 1e6);
      } else {  // divisors with near all-ones significands
        const long long bits = 0x3ffffffffffff000ll | (long long)(r2 & 0xfff);
        b = ldexp(__longlong_as_double(bits), (int)(r2 >> 52) % 80 - 40);
        a = loguni(r1, 1e-20, 1e20);
      }
      want = a / b;
      got = fm_div(a, b, ok);
    } else {
      if (mode == 3)
        a = fabs(__longlong_as_double((long long)r1));
      else
        a = loguni(r1, 1e-14, 1e12);
      want = sqrt(a);
      got = fm_sqrt(a, ok);
    }
    if (!ok) continue;  // out of the fast path's range: the caller falls back
    ++nc;
    if (__double_as_longlong(want) != __double_as_longlong(got)) {
      ++nb;
      first[0] = a;
      first[1] = b;
    }
  }
  atomicAdd(bad, nb);
  atomicAdd(checked, nc);
}

}  // namespace
}  // namespace tmgpu

extern "C" int tmgpu_selftest_fastmath(int mode, long long n, uint64_t seed,
                                       unsigned long long* mismatches,
                                       unsigned long long* checked, double* first_bad,
                                       tmgpu_error* err) {
  using namespace tmgpu;
  unsigned long long* d = nullptr;
  double* f = nullptr;
  cudaError_t e = cudaMalloc(&d, 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&f, 2 * sizeof(double));
  if (e == cudaSuccess) e = cudaMemset(d, 0, 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(f, 0, 2 * sizeof(double));
  if (e == cudaSuccess) {
    fm_selftest_kernel<<<148 * 16, 256>>>(seed, n, mode, d, d + 1, f);
    e = cudaDeviceSynchronize();
  }
  unsigned long long h[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(first_bad, f, 2 * sizeof(double), cudaMemcpyDeviceToHost);
  if (d) cudaFree(d);
  if (f) cudaFree(f);
  *mismatches = h[0];
  *checked = h[1];
  return cuda_err(err, e, "tmgpu_selftest_fastmath");
}
