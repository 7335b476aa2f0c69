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

// Per destination leaf and face (2*axis + (dir>0)): where its face ghosts come
// from in the one-round exchange.
struct alignas(16) FaceSrc {
  int32_t src[4];  // same/coarser: src[0]; finer: quadrant (qt2*2+qt1); boundary: unused
  int32_t staged;  // coarser: index of the snapshot slab
  int8_t kind;     // 0 same, 1 coarser, 2 finer, 3 boundary
  int8_t pad[11];
};

// One-round, face-only exchange: snapshot every prolonged slab of all three
// axes from the pre-exchange state, then one CTA per (leaf, face) item pulls
// that face's E x E x G ghost slab. Bitwise identical to the reference on
// every ghost the stage reads; edge/corner ghosts untouched.
// items = all 6 faces of every leaf (full face exchange) or only the
// coarse-fine / boundary faces (the step: same-level faces are read by the
// stage kernel straight from the neighbour, see StageLaunch::face_src).
// `prev` holds the ghosts of the previous exchange (== arena when in place).
cudaError_t ghost_exchange_faces(double* arena, const double* prev, int V, const FaceSrc* faces,
                                 const int2* items, int n_items, const GhostFill* prolong_fills,
                                 int n_prolong, double* staged, cudaStream_t st);

// Phase 1 (prolonged snapshot) + phase 2 (apply) of one axis pass.
cudaError_t ghost_pass(double* arena, int V, const GhostPassDev& pass, double* staged,
                       cudaStream_t st);

// compact [slot][V][E^3] <-> arena interior positions.
cudaError_t interior_copy(double* arena, double* compact, int V, long long nslots, bool to_arena,
                          cudaStream_t st);

}  // namespace tmgpu
