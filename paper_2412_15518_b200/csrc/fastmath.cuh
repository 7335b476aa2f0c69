// Branch-free correctly rounded FP64 division and square root for the stage
// kernel's hot loop.
//
// CUDA's IEEE `/` and `sqrt` are multi-instruction sequences with an
// out-of-line slow path for special operands; each one ends a basic block, so
// the compiler cannot interleave independent face computations across them.
// Here the common case is straight-line code:
//   reciprocal / rsqrt seed (MUFU) -> Newton refinements (DFMA) ->
//   Markstein correction  q = RN(a*y); r = a - b*q (exact, FMA); q' = RN(q + r*y)
//                         s = RN(x*y); r = x - s*s (exact, FMA); s' = RN(s + r*y/2)
// which returns the IEEE round-to-nearest result whenever every operand and
// result lies in [2^-900, 2^901) (no over/underflow in any intermediate).
// Callers AND the per-operation `ok` flags and re-evaluate with the IEEE
// operators when any lane of the warp saw an operand outside that range
// (zero, subnormal, inf, NaN, extreme exponents), so results are bitwise the
// reference's for every input. The equivalence on the safe range is checked
// on the device over billions of random operands (tmgpu_selftest_fastmath,
// tests/test_fastmath_gpu.py) besides the end-to-end memcmp parity tests.
#pragma once

#include <cuda_runtime.h>

namespace tmgpu {

__device__ __forceinline__ bool fm_range_ok(double x) {
  const unsigned e = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;  // biased exponent
  return (e - 123u) < 1800u;                                       // 2^-900 <= |x| < 2^901
}

__device__ __forceinline__ double fm_rcp_seed(double b) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
  return y;
}

__device__ __forceinline__ double fm_rsqrt_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// ~correctly rounded reciprocal: seed + 3 Newton steps (error well below 1 ulp)
__device__ __forceinline__ double fm_rcp(double b) {
  double y = fm_rcp_seed(b);
  double e = fma(-b, y, 1.0);
  y = fma(y, e, y);
  e = fma(-b, y, 1.0);
  y = fma(y, e, y);
  e = fma(-b, y, 1.0);
  y = fma(y, e, y);
  return y;
}

// a / b given y ~ 1/b (Markstein correction)
__device__ __forceinline__ double fm_div_y(double a, double b, double y) {
  const double q = a * y;
  const double r = fma(-b, q, a);
  return fma(r, y, q);
}

__device__ __forceinline__ double fm_div(double a, double b, bool& ok) {
  const double q = fm_div_y(a, b, fm_rcp(b));
  ok = ok && fm_range_ok(a) && fm_range_ok(b) && fm_range_ok(q);
  return q;
}

__device__ __forceinline__ double fm_sqrt(double x, bool& ok) {
  double y = fm_rsqrt_seed(x);
  // Newton for 1/sqrt: y <- y + y/2 * (1 - x y^2)
  double e = fma(-x, y * y, 1.0);
  y = fma(0.5 * y, e, y);
  e = fma(-x, y * y, 1.0);
  y = fma(0.5 * y, e, y);
  e = fma(-x, y * y, 1.0);
  y = fma(0.5 * y, e, y);
  const double s = x * y;
  const double r = fma(-s, s, x);
  const double out = fma(r, 0.5 * y, s);
  ok = ok && fm_range_ok(x) && fm_range_ok(out);
  return out;
}

}  // namespace tmgpu
