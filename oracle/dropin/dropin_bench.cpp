// TEST INFRASTRUCTURE (benchmark): the drop-in timed INSIDE the unmodified
// reference. The reference's own AggregationRegion + task::Scheduler +
// ExecutorPool + BufferPool (proj/src/aggregator.cpp:106-172) aggregate
// `count` Euler slices (the C3 leaf count by default) through
//   make_stage_kernel       the reference CPU kernel (stage.cpp:229-246), and
//   make_stage_kernel_gpu   include/tmgpu_taskmesh.hpp: one sm_100a launch per
//                           batch over the region's host buffers
// for several max_slices, all host threads as workers; plus the fused kernel on
// slices already resident in HBM (tmgpu_stage_fused with device pointers).
// Prints one JSON object per configuration (cell-stage/s, slice bytes/s).
// Built by oracle/Makefile into oracle/_ref/dropin_bench.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "taskmesh/aggregator.hpp"
#include "taskmesh/bufferpool.hpp"
#include "taskmesh/hydro/stage.hpp"
#include "taskmesh/taskgraph.hpp"
#include "tmgpu_taskmesh.hpp"

using namespace taskmesh;
using clk = std::chrono::steady_clock;

static void fill_slice(const hydro::StageGeom& g, std::mt19937_64& rng, double dx, double* s) {
  std::uniform_real_distribution<double> pos(0.2, 2.0), vel(-0.5, 0.5);
  hydro::StageParams p;
  p.mode = hydro::Mode::euler;
  p.dx = dx;
  p.dt = 0.2 * dx;
  hydro::encode_header(p, {s, hydro::kHeaderDoubles});
  const std::size_t s3 = (g.in_slice() - hydro::kHeaderDoubles) / 5;
  double* st = s + hydro::kHeaderDoubles;
  for (std::size_t c = 0; c < s3; ++c) {
    const double rho = pos(rng), u = vel(rng), v = vel(rng), w = vel(rng), pr = pos(rng);
    st[c] = rho;
    st[s3 + c] = rho * u;
    st[2 * s3 + c] = rho * v;
    st[3 * s3 + c] = rho * w;
    st[4 * s3 + c] = pr / 0.4 + 0.5 * rho * (u * u + v * v + w * w);
  }
}

static double region_seconds(const agg::KernelSpec& spec, const std::vector<double>& slices, std::size_t n,
                             std::size_t max_slices, unsigned workers, std::uint64_t* launches) {
  task::Scheduler sched(workers);
  agg::ExecutorPool execs(workers);
  mem::BufferPool pool;
  agg::AggCounters cnt;
  const auto t0 = clk::now();
  agg::AggregationRegion region(sched, execs, pool, spec, max_slices, n, &cnt);
  std::vector<task::Future<agg::SliceOutput>> futs;
  futs.reserve(n);
  for (std::size_t s = 0; s < n; ++s)
    futs.push_back(region.submit_slice({slices.data() + s * spec.in_slice, spec.in_slice}));
  region.flush();
  auto outs = sched.run_until(task::when_all(sched, std::move(futs)));
  const double sec = std::chrono::duration<double>(clk::now() - t0).count();
  if (launches) *launches = cnt.launches.load();
  return sec;
}

int main(int argc, char** argv) {
  const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 5888;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 3;
  unsigned workers = std::thread::hardware_concurrency();
  if (workers == 0) workers = 8;
  hydro::StageGeom g;
  g.vars = 5;
  std::vector<double> slices(n * g.in_slice());
  std::mt19937_64 rng(2412518);
  for (std::size_t s = 0; s < n; ++s) fill_slice(g, rng, (1.0 / 256) * (1 + s % 2), slices.data() + s * g.in_slice());
  const double cells = (double)n * 512.0;
  const double slice_bytes = (double)(g.in_slice() + g.out_slice()) * 8.0 * n;  // 205.1 B per cell
  auto cpu = hydro::make_stage_kernel(g, 1, 1);
  auto gpu = hydro::make_stage_kernel_gpu(g, 2);
  // warm-up: CUDA context, per-thread staging buffers
  { std::uint64_t l; region_seconds(gpu, slices, std::min<std::size_t>(n, 512), 64, workers, &l); }
  for (const char* which : {"gpu", "cpu"}) {
    const auto& spec = which[0] == 'g' ? gpu : cpu;
    for (std::size_t ms : {8u, 64u, 512u}) {
      double best = 1e30;
      std::uint64_t launches = 0;
      for (int r = 0; r < (which[0] == 'g' ? reps : 1); ++r)
        best = std::min(best, region_seconds(spec, slices, n, ms, workers, &launches));
      std::printf("{\"path\": \"%s\", \"api\": \"AggregationRegion(%s)\", \"max_slices\": %zu, \"slices\": %zu, "
                  "\"workers\": %u, \"launches\": %llu, \"seconds\": %.6f, \"cell_stage_per_s\": %.6e, "
                  "\"slice_GBps\": %.3f}\n",
                  which, which[0] == 'g' ? "make_stage_kernel_gpu" : "make_stage_kernel", ms, n, workers,
                  (unsigned long long)launches, best, cells / best, slice_bytes / best / 1e9);
      std::fflush(stdout);
    }
  }
  // the fused kernel alone on slices resident in HBM (the slice contract's HBM roofline)
  double *d_in = nullptr, *d_out = nullptr;
  if (cudaMalloc(&d_in, slices.size() * 8) == cudaSuccess && cudaMalloc(&d_out, n * g.out_slice() * 8) == cudaSuccess) {
    cudaMemcpy(d_in, slices.data(), slices.size() * 8, cudaMemcpyHostToDevice);
    tmgpu_error err;
    cudaStream_t st;
    cudaStreamCreate(&st);
    tmgpu_stage_fused(d_in, d_out, g.in_slice(), g.out_slice(), n, 8, 2, 5, 0, st, &err);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int K = 20;
    cudaEventRecord(a, st);
    for (int k = 0; k < K; ++k) tmgpu_stage_fused(d_in, d_out, g.in_slice(), g.out_slice(), n, 8, 2, 5, 0, st, &err);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double sec = ms * 1e-3 / K;
    std::printf("{\"path\": \"gpu-resident\", \"api\": \"tmgpu_stage_fused(device pointers)\", \"slices\": %zu, "
                "\"seconds\": %.6f, \"cell_stage_per_s\": %.6e, \"slice_GBps\": %.3f}\n",
                n, sec, cells / sec, slice_bytes / sec / 1e9);
  }
  return 0;
}
