/* tools/probes/libtmprobe.so — diagnostics, not the product ABI (include/tmgpu.h). */
#ifndef TMPROBE_H
#define TMPROBE_H
#include <stdint.h>
#include "../../include/tmgpu.h"
#ifdef __cplusplus
extern "C" {
#endif
/* bitwise self-test of fastmath.cuh's branch-free division / sqrt against IEEE */
int tmgpu_selftest_fastmath(int mode, long long n, uint64_t seed, unsigned long long* mismatches,
                            unsigned long long* checked, double* first_bad, tmgpu_error* err);
/* FP64 DFMA throughput microbenchmark (roofline denominator) */
int tmgpu_fp64_peak(int iters, double* tflops, double* ms, tmgpu_error* err);
/* DFMA TFLOP/s with `warps` warps per SM and `chains` independent chains per thread */
int tmgpu_fp64_probe(int warps, int chains, int iters, double* tflops);
/* FP64 tensor-core (mma m8n8k4 f64) TFLOP/s, `warps` per SM, `chains` accumulators */
int tmgpu_dmma_probe(int warps, int chains, int iters, double* tflops);
/* DFMA TFLOP/s when every FMA reads three fresh registers (8 chains per thread) */
int tmgpu_dfma3_probe(int warps, int iters, double* tflops);
#ifdef __cplusplus
}
#endif
#endif
