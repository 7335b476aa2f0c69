// NOT PRODUCT CODE (tools/probes -> tools/probes/libtmprobe.so, loaded by bench.py and
// tools/*): FP64 pipe peak microbenchmark (roofline denominator: MEASURED_PEAKS.json has
// no FP64 entry). Each thread runs 8 independent DFMA chains; FLOP = 2 per FMA.
#include "tmgpu_internal.h"  // error codes, cuda_err (product header, -I)

namespace tmgpu {
namespace {
__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // never true; keeps the chains live
}
// latency/occupancy probe: C independent DFMA chains per thread
template <int C>
__global__ void dfma_chains_kernel(double* out, int iters, double a, double b) {
  double x[C];
#pragma unroll
  for (int k = 0; k < C; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < C; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < C; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}
// register-operand probe: each DFMA reads three registers no earlier
// instruction just read (x = fma(y, z, x) over rotating y, z): the operand
// bandwidth of the register file, not the pipe, is then the limit
template <int C>
__global__ void dfma3_kernel(double* out, int iters, double a, double b) {
  double x[C], y[C], z[C];
#pragma unroll
  for (int k = 0; k < C; ++k)
    x[k] = threadIdx.x * 1e-3 + k, y[k] = a + k * 1e-9 + threadIdx.x * 1e-12, z[k] = b - k * 1e-9 - threadIdx.x * 1e-12;
  for (int i = 0; i < iters; i += C) {
#pragma unroll
    for (int r = 0; r < C; ++r)
#pragma unroll
      for (int k = 0; k < C; ++k) x[k] = fma(y[(k + r) % C], z[(k + 3 * r + 1) % C], x[k]);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < C; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

// FP64 tensor-core probe: C independent m8n8k4 DMMA accumulators per warp
template <int C>
__global__ void dmma_kernel(double* out, int iters, double a0, double b0) {
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  double c[C][2];
#pragma unroll
  for (int k = 0; k < C; ++k) c[k][0] = c[k][1] = k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < C; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < C; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}
}  // namespace
}  // namespace tmgpu

// Diagnostics: FP64 tensor-core (DMMA m8n8k4) TFLOP/s with `warps` warps per
// SM and `chains` independent accumulators per warp (2*8*8*4 flop per MMA).
extern "C" int tmgpu_dfma3_probe(int warps, int iters, double* tflops) {
  using namespace tmgpu;
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double)) != cudaSuccess) return TMGPU_ERR_CUDA;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  dfma3_kernel<8><<<sms, 32 * warps>>>(d, iters / 10 + 1, 0.999999, 1e-7);
  cudaEventRecord(t0);
  dfma3_kernel<8><<<sms, 32 * warps>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(t1);
  cudaError_t e = cudaEventSynchronize(t1);
  float msf = 0;
  cudaEventElapsedTime(&msf, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(d);
  if (e != cudaSuccess) return TMGPU_ERR_CUDA;
  *tflops = 2.0 * 8 * (double)iters * sms * 32.0 * warps / (msf * 1e-3) / 1e12;
  return TMGPU_OK;
}

extern "C" int tmgpu_dmma_probe(int warps, int chains, int iters, double* tflops) {
  using namespace tmgpu;
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double)) != cudaSuccess) return TMGPU_ERR_CUDA;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto launch = [&](int it) {
    if (chains <= 1) { dmma_kernel<1><<<sms, 32 * warps>>>(d, it, 0.999, 1e-7); chains = 1; }
    else if (chains <= 2) { dmma_kernel<2><<<sms, 32 * warps>>>(d, it, 0.999, 1e-7); chains = 2; }
    else if (chains <= 4) { dmma_kernel<4><<<sms, 32 * warps>>>(d, it, 0.999, 1e-7); chains = 4; }
    else { dmma_kernel<8><<<sms, 32 * warps>>>(d, it, 0.999, 1e-7); chains = 8; }
  };
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  launch(iters / 10 + 1);
  cudaEventRecord(t0);
  launch(iters);
  cudaEventRecord(t1);
  cudaError_t e = cudaEventSynchronize(t1);
  float msf = 0;
  cudaEventElapsedTime(&msf, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(d);
  if (e != cudaSuccess) return TMGPU_ERR_CUDA;
  *tflops = 2.0 * 8 * 8 * 4 * chains * (double)iters * sms * warps / (msf * 1e-3) / 1e12;
  return TMGPU_OK;
}

// Diagnostics: DFMA TFLOP/s with `warps` warps per SM (one CTA per SM) and
// `chains` (1, 2, 4, 8, 16) independent FMA chains per thread.
extern "C" int tmgpu_fp64_probe(int warps, int chains, int iters, double* tflops) {
  using namespace tmgpu;
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double)) != cudaSuccess) return TMGPU_ERR_CUDA;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto launch = [&](int it) {
    switch (chains) {
      case 1: dfma_chains_kernel<1><<<sms, 32 * warps>>>(d, it, 0.999999, 1e-7); break;
      case 2: dfma_chains_kernel<2><<<sms, 32 * warps>>>(d, it, 0.999999, 1e-7); break;
      case 4: dfma_chains_kernel<4><<<sms, 32 * warps>>>(d, it, 0.999999, 1e-7); break;
      case 8: dfma_chains_kernel<8><<<sms, 32 * warps>>>(d, it, 0.999999, 1e-7); break;
      default: dfma_chains_kernel<16><<<sms, 32 * warps>>>(d, it, 0.999999, 1e-7); chains = 16;
    }
  };
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  launch(iters / 10 + 1);
  cudaEventRecord(t0);
  launch(iters);
  cudaEventRecord(t1);
  cudaError_t e = cudaEventSynchronize(t1);
  float msf = 0;
  cudaEventElapsedTime(&msf, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(d);
  if (e != cudaSuccess) return TMGPU_ERR_CUDA;
  *tflops = 2.0 * chains * (double)iters * sms * 32.0 * warps / (msf * 1e-3) / 1e12;
  return TMGPU_OK;
}

extern "C" int tmgpu_fp64_peak(int iters, double* tflops, double* ms, tmgpu_error* err) {
  using namespace tmgpu;
  double* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(double));
  if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_fp64_peak");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  dfma_kernel<<<blocks, threads>>>(d, iters / 10 + 1, 0.999999, 1e-7);  // warm-up
  cudaEventRecord(t0);
  dfma_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(t1);
  e = cudaEventSynchronize(t1);
  float msf = 0;
  cudaEventElapsedTime(&msf, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_fp64_peak");
  const double flops = 2.0 * 8.0 * (double)iters * blocks * threads;
  *ms = msf;
  *tflops = flops / (msf * 1e-3) / 1e12;
  return TMGPU_OK;
}
