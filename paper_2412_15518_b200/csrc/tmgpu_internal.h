// Internal C++ interfaces shared by the CUDA translation units and the C ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/tmgpu.h"

// gravity_amr.cu: may a CUDA graph capture this solver's solve (no host-side
// state per call: not timing)?
extern "C" bool tmgpu_gravity_amr_graph_safe(const tmgpu_gravity_amr* G);
// ... and the solver's configuration version (distribute / set_peer bump it)
extern "C" unsigned long long tmgpu_gravity_amr_version(const tmgpu_gravity_amr* G);

namespace tmgpu {

// Per-launch arguments of the aggregated stage kernel (stage_kernel.cuh).
struct StageLaunch {
  // headers: slice mode reads hdr + s*hdr_stride; arena mode (hdr == nullptr)
  // uses leaf_dx[slot] and the launch-wide fields below.
  const double* hdr;
  long long hdr_stride;
  const double* leaf_dx;
  double g_mode, g_dt, g_gamma, g_ax, g_ay, g_az;
  const double* dt_ptr;  // arena mode: dt read from device memory when non-null
  // interior destination
  double* out;
  long long out_stride;
  int out_ghosted;  // 1: write interior positions of a ghosted S^3 block
  // optional outputs
  double* faces;  // [6][V][E^2] per slice
  long long faces_stride;
  double* diag;  // floor hits per slice
  long long diag_stride;
  // optional SSP-RK3 combine: out = rk3_combine(rk_stage, u0, v)
  const double* u0;
  long long u0_stride;
  int rk_stage;
  double* u0_save;  // optional: interior state before the update -> compact [V][E^3]
  long long u0_save_stride;
  const int* index;  // optional: tensor slot of CTA b = index[b]
  // optional [slot][6] face sources (face = 2*axis + side): (slot << 1) loads
  // the leaf's own ghost layers, (nbr << 1) | 1 the same-level neighbour's
  // adjacent interior layers. nullptr: own ghosts everywhere.
  const int* face_src;
  // optional gravity source (our spec; not in the reference):
  // g[q*grav_stride + slot*512 + c]; after the z update, before the floors:
  // m_q += dt*(rho*g_q), E += dt*(rho*((u*gx + v*gy) + w*gz)) with the stage
  // input's primitives (oracle tmo_stage_subgrid_grav)
  const double* grav;
  long long grav_stride;
  // optional [slot][E^3]: the stage update's density after the floors and
  // before the RK3 combine (the provisional state a second gravity solve of
  // the 6-solve cadence reads; tmgpu_forest_set_gravity_solver)
  double* rho_save;
  // split stage (gravity step): store the raw update only; the floors, the
  // source, finiteness and the combine follow in stage_epilogue_kernel
  int defer;
  // optional second output: the final values also as compact interiors
  // [slot][V][E^3] (tmgpu_forest_step_io's output, fused into the last stage)
  double* out_compact;
  unsigned long long* err;  // atomicMin of (slice << 32 | var-major interior index)
  int count;
  // L2 prefetch distance in CTAs (set by launch_stage_t): CTA b also prefetches
  // the boxes of CTA b + prefetch_ahead, which starts about one resident wave
  // later, so its TMA loads hit L2 (0: off)
  int prefetch_ahead;
};

// Number of kernels this library launched since load.
extern std::atomic<uint64_t> g_launches;

struct StageMaps {
  CUtensorMap i, x, y, z;  // boxes 10x8x8, 2x8x8, 8x2x8, 8x8x2 over [slot][var][z][y][x]
};

// Encode the three TMA maps for `count` ghosted 12^3 blocks of V vars whose
// var-0 element of slot s sits at base + s*slot_stride (doubles). base must be
// 16-byte aligned and slot_stride*8 a multiple of 16.
int make_stage_maps(const double* base, int V, long long slot_stride, long long count,
                    StageMaps* maps, std::string* why);

cudaError_t launch_stage(int V, bool fast, const StageMaps& maps, const StageLaunch& p,
                         cudaStream_t stream);

// the second half of a split stage (stage_kernel.cuh stage_epilogue_kernel)
cudaError_t launch_stage_epilogue(bool fast, const double* in_arena, const StageLaunch& p, cudaStream_t stream);

cudaError_t launch_max_wavespeed(const double* in, long long slot_stride, const double* hdr,
                                 long long hdr_stride, const double* leaf_dx, double g_gamma,
                                 int V, long long count, double* result, cudaStream_t stream);

// compact interiors [slot][5][E^3] -> arena + max_wavespeed per slot (the step_io input pass)
cudaError_t launch_scatter_wavespeed(const double* compact, double* arena, long long slot_stride, double gamma,
                                     long long count, double* result, cudaStream_t stream);

cudaError_t launch_cfl_reduce(const double* speeds, const double* leaf_dx, long long n, double cfl,
                              double* dt, cudaStream_t stream);

// Reflux of the stage output at the coarse side of refinement jumps (reflux.cu).
cudaError_t launch_reflux(double* arena, int V, const double* flux, const int* leaf_slot,
                          const int* face_off, const int* face_ad, const int* fine, long long nleaves,
                          const double* leaf_dx, const double* dt_ptr, double g_dt, double coef,
                          cudaStream_t st, const double* rflux = nullptr);
// distributed reflux: pack the face flux blocks other GPUs need (reflux.cu)
cudaError_t launch_flux_pack(const double* flux, int V, const int2* items, long long n, double* out,
                             cudaStream_t st);

// regrid.cu: octree.cpp:149-323 data operations
cudaError_t launch_prolong(const double* parent, double* children8, int V, cudaStream_t st);
cudaError_t launch_restrict(const double* const* children, double* parent, int V, cudaStream_t st);
cudaError_t launch_gather_blocks(const double* const* src_dev, long long n, double* dst, long long stride,
                                 cudaStream_t st);
cudaError_t launch_flag(const double* arena, long long stride, long long n, double theta, double rho_floor,
                        int* flag, cudaStream_t st);

// 6-solve cadence: the stage's gravity source moved to the trapezoid of the
// solves on the stage input (ga) and on its provisional density (gb); after
// the RK3 combine, scaled by the stage weight w (grav_source.cu)
cudaError_t launch_grav_correct(const double* in_arena, double* out_arena, long long nslots, const double* ga,
                                const double* gb, long long gstride, const double* dt_ptr, double g_dt,
                                double w, cudaStream_t st);

cudaError_t launch_rk3_combine(int stage, const double* u0, const double* v, double* out,
                               long long n, cudaStream_t stream);

inline int set_err(tmgpu_error* err, int code, const char* msg) {
  if (err) {
    err->code = code;
    std::snprintf(err->message, sizeof(err->message), "%s", msg);
  }
  return code;
}

inline int cuda_err(tmgpu_error* err, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return TMGPU_OK;
  if (err) {
    err->code = TMGPU_ERR_CUDA;
    std::snprintf(err->message, sizeof(err->message), "%s: %s", where, cudaGetErrorString(e));
  }
  return TMGPU_ERR_CUDA;
}

// Flag-wait limit of the peer-memory exchanges (peer.cuh spin_geq), read at
// peer setup: TMGPU_PEER_TIMEOUT_S seconds, default 20, 0 = wait forever.
inline unsigned long long peer_spin_ns() {
  const char* v = std::getenv("TMGPU_PEER_TIMEOUT_S");
  if (!v || !*v) return 20000000000ull;
  const double s = std::atof(v);
  return s <= 0.0 ? 0ull : (unsigned long long)(s * 1e9);
}

inline cudaStream_t as_stream(void* s) {
  return s ? static_cast<cudaStream_t>(s) : cudaStreamPerThread;
}

}  // namespace tmgpu
