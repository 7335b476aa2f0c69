/* tmgpu — B200-native (sm_100a, FP64) per-subgrid hot path behind the
 * reference mini-app's subgrid-kernel API (taskmesh, arXiv 2412.15518).
 *
 * C ABI: plain pointers and sizes, no torch/CUDA types in the signatures
 * (streams are passed as void* = cudaStream_t). Every entry point names the
 * reference interface it replaces (paths relative to /root/reference/proj).
 * All functions are thread-safe; the stage entry points may be called
 * concurrently from several scheduler workers (reference aggregator.cpp:147-157).
 *
 * Return value: TMGPU_OK (0) or a negative/positive error code; details in
 * the optional tmgpu_error record.
 */
#ifndef TMGPU_H
#define TMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- errors */
enum {
  TMGPU_OK = 0,
  TMGPU_ERR_SOLVER = 1,      /* non-finite state (reference hydro::SolverError, stage.cpp:209-216) */
  TMGPU_ERR_INVALID = 2,     /* bad argument / unsupported geometry */
  TMGPU_ERR_CUDA = 3,        /* CUDA runtime failure (message holds cudaGetErrorString) */
  TMGPU_ERR_AMR = 4,         /* reference amr::AmrError analog (morton/partition/tree) */
  TMGPU_ERR_AGG = 5          /* reference agg::AggError analog (aggregator.cpp) */
};

typedef struct tmgpu_error {
  int code;
  int cell[3];               /* solver errors: interior cell (i,j,k) of the first bad value */
  int64_t slice;             /* solver errors: first failing slice (launch order) */
  char message[256];         /* solver errors carry the reference's exact text */
} tmgpu_error;

/* ---------------------------------------------------------------- flags */
#define TMGPU_HOST_PTRS 0x1  /* in/out are host memory: H2D, kernel, D2H inside the call */
#define TMGPU_FAST 0x2       /* FMA/reciprocal arithmetic: parity within 1e-10 (scaled), not bitwise */

/* ---------------------------------------------------------------- hydro
 * Slice contract (reference stage.hpp:8-12, 39-66):
 *   in  slice = [8-double header | vars * S^3 ghosted state], S = edge + 2*ghost
 *   out slice = [vars*E^3 interior | 6 face-flux blocks of vars*E^2 | 1 floor-hit count]
 * Header = [mode (0 scalar, else Euler), dx, dt, gamma, ax, ay, az, 0]
 *   (reference stage.cpp:10-29 encode_header/decode_header).
 */
size_t tmgpu_in_slice(int edge, int ghost, int vars);   /* StageGeom::in_slice  stage.hpp:54 */
size_t tmgpu_out_slice(int edge, int ghost, int vars);  /* StageGeom::out_slice stage.hpp:65 */

/* Replaces the body of hydro::make_stage_kernel's KernelFn
 * (reference src/hydro/stage.cpp:229-246; KernelFn type aggregator.hpp:96-99):
 * one fused launch over `count` slices packed at in + s*in_slice /
 * out + s*out_slice. Bitwise equal to the reference unless TMGPU_FAST.
 * Device pointers (default) run on `stream` (NULL = per-thread default) and
 * the call returns after the stream reaches the end of the launch; with
 * TMGPU_HOST_PTRS the call stages through device memory itself.
 * Supported geometry: edge 8, ghost 2, vars 1 (scalar) or 5 (Euler or scalar). */
int tmgpu_stage_fused(const double* in, double* out, size_t in_slice, size_t out_slice,
                      size_t count, int edge, int ghost, int vars, int flags,
                      void* stream, tmgpu_error* err);

/* Replaces hydro::stage_subgrid (reference stage.hpp:68-71, stage.cpp:222-227)
 * for one sub-grid: header8 + ghosted state -> out slice. lane_width is
 * accepted for API parity and ignored (output is W-invariant, stage.hpp:69). */
int tmgpu_stage_subgrid(const double* header8, int edge, int ghost, int vars,
                        unsigned lane_width, const double* in_ghosted, double* out,
                        int flags, void* stream, tmgpu_error* err);

/* Replaces hydro::max_wavespeed (reference stage.cpp:248-272) over `count`
 * slices (same slice layout as tmgpu_stage_fused); result[s] per slice. */
int tmgpu_max_wavespeed(const double* in, size_t in_slice, size_t count, int edge, int ghost,
                        int vars, double* result, int flags, void* stream, tmgpu_error* err);

/* hydro::rk3_combine (reference include/taskmesh/hydro/rk3.hpp:18-34) on n values. */
int tmgpu_rk3_combine(int stage, const double* u0, const double* v, double* out, size_t n,
                      int flags, void* stream, tmgpu_error* err);

/* ---------------------------------------------------------------- build info */
const char* tmgpu_version(void);
/* number of kernels launched by this library since load (bench/gpu_launches) */
uint64_t tmgpu_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TMGPU_H */
