// Header-only drop-in adapter for the reference mini-app (taskmesh).
// Include from code that already includes the reference headers; link
// libtmgpu.so. Replaces hydro::make_stage_kernel (proj/src/hydro/stage.cpp:229-246)
// with a KernelSpec whose fn is ONE aggregated sm_100a launch (tmgpu_stage_fused).
#pragma once

#include <stdexcept>

#include "taskmesh/aggregator.hpp"
#include "taskmesh/hydro/stage.hpp"
#include "tmgpu.h"

namespace taskmesh::hydro {

inline agg::KernelSpec make_stage_kernel_gpu(const StageGeom& geom, std::uint32_t kernel_id,
                                             bool fast = false) {
  agg::KernelSpec spec;
  spec.id = kernel_id;
  spec.in_slice = geom.in_slice();
  spec.out_slice = geom.out_slice();
  spec.fn = [geom, fast](const double* in, double* out, std::size_t in_slice,
                         std::size_t out_slice, std::size_t count) {
    tmgpu_error err;
    const int rc = tmgpu_stage_fused(in, out, in_slice, out_slice, count, geom.edge, geom.ghost,
                                     geom.vars, TMGPU_HOST_PTRS | (fast ? TMGPU_FAST : 0),
                                     nullptr, &err);
    if (rc == TMGPU_ERR_SOLVER) throw SolverError(err.message);  // stage.cpp:209-216 text
    if (rc != TMGPU_OK) throw std::runtime_error(err.message);
  };
  return spec;
}

}  // namespace taskmesh::hydro
