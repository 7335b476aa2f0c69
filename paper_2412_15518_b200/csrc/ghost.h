// Device ghost exchange interfaces (ghost.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tmgpu {

// One fill of an axis pass on the device (ghost.hpp:53-61 by leaf slot).
struct alignas(16) GhostFill {
  int32_t dst;
  int32_t src;  // -1 for boundary fills
  int8_t kind;  // 0 same, 1 coarser (prolonged), 2 finer (restricted), 3 boundary
  int8_t axis, dir, qt1, qt2;
  int8_t pad[3];
};

// Device arrays describing one axis pass.
struct GhostPassDev {
  const GhostFill* fills = nullptr;   // n_fills, plan order
  const int* staged_of = nullptr;     // per fill: index into the staged slabs (coarser fills)
  const int* prolong_fills = nullptr; // n_prolong: fill indices of the coarser fills
  int n_fills = 0;
  int n_prolong = 0;
};

// Phase 1 (prolonged snapshot) + phase 2 (apply) of one axis pass.
cudaError_t ghost_pass(double* arena, int V, const GhostPassDev& pass, double* staged,
                       cudaStream_t st);

// compact [slot][V][E^3] <-> arena interior positions.
cudaError_t interior_copy(double* arena, double* compact, int V, long long nslots, bool to_arena,
                          cudaStream_t st);

}  // namespace tmgpu
