// TEST INFRASTRUCTURE: the drop-in exercised INSIDE the unmodified reference.
// The reference's own AggregationRegion + task::Scheduler drive
// make_stage_kernel_gpu (include/tmgpu_taskmesh.hpp); outputs must equal the
// reference make_stage_kernel bitwise for every batching, and a non-finite
// state must fail every promise of its batch with the reference's message.
// Built by oracle/Makefile into oracle/_ref/dropin_test; run by
// tests/test_dropin_gpu.py on a B200.
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "taskmesh/aggregator.hpp"
#include "taskmesh/bufferpool.hpp"
#include "taskmesh/hydro/stage.hpp"
#include "taskmesh/taskgraph.hpp"
#include "tmgpu_taskmesh.hpp"

using namespace taskmesh;

static std::vector<double> random_slice(const hydro::StageGeom& g, std::mt19937_64& rng,
                                        double dx) {
  std::uniform_real_distribution<double> pos(0.2, 2.0), vel(-0.5, 0.5);
  std::vector<double> s(g.in_slice());
  hydro::StageParams p;
  p.mode = hydro::Mode::euler;
  p.dx = dx;
  p.dt = 0.2 * dx;
  hydro::encode_header(p, {s.data(), hydro::kHeaderDoubles});
  const std::size_t s3 = (g.in_slice() - hydro::kHeaderDoubles) / 5;
  double* st = s.data() + hydro::kHeaderDoubles;
  for (std::size_t c = 0; c < s3; ++c) {
    double rho = pos(rng), u = vel(rng), v = vel(rng), w = vel(rng), pr = pos(rng);
    st[c] = rho;
    st[s3 + c] = rho * u;
    st[2 * s3 + c] = rho * v;
    st[3 * s3 + c] = rho * w;
    st[4 * s3 + c] = pr / 0.4 + 0.5 * rho * (u * u + v * v + w * w);
  }
  return s;
}

int main() {
  hydro::StageGeom g;
  g.vars = 5;
  std::mt19937_64 rng(2412);
  const std::size_t n = 40;
  std::vector<std::vector<double>> slices;
  for (std::size_t s = 0; s < n; ++s) slices.push_back(random_slice(g, rng, 0.01 / (1 + s % 3)));
  auto cpu = hydro::make_stage_kernel(g, 1, 1);
  auto gpu = hydro::make_stage_kernel_gpu(g, 2);
  int failures = 0;
  for (std::size_t max_slices : {1u, 3u, 8u, 40u}) {
    task::Scheduler sched(4);
    agg::ExecutorPool execs(4);
    mem::BufferPool pool;
    agg::AggCounters ca, cb;
    agg::AggregationRegion ra(sched, execs, pool, cpu, max_slices, n, &ca);
    agg::AggregationRegion rb(sched, execs, pool, gpu, max_slices, n, &cb);
    std::vector<task::Future<agg::SliceOutput>> fa, fb;
    for (auto& s : slices) {
      fa.push_back(ra.submit_slice(s));
      fb.push_back(rb.submit_slice(s));
    }
    ra.flush();
    rb.flush();
    auto oa = sched.run_until(task::when_all(sched, std::move(fa)));
    auto ob = sched.run_until(task::when_all(sched, std::move(fb)));
    for (std::size_t s = 0; s < n; ++s) {
      auto a = oa[s].values(), b = ob[s].values();
      if (std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) != 0) {
        std::printf("MISMATCH max_slices=%zu slice=%zu\n", max_slices, s);
        ++failures;
      }
    }
    std::printf("max_slices=%zu gpu launches=%llu fused=%llu\n", max_slices,
                (unsigned long long)cb.launches.load(), (unsigned long long)cb.fused_slices.load());
  }
  // error path: NaN in one slice of a fused batch, GPU and CPU kernels
  std::string msgs[2];
  for (int which = 0; which < 2; ++which) {
    task::Scheduler sched(2);
    agg::ExecutorPool execs(1);
    mem::BufferPool pool;
    auto busy = execs.acquire();  // keep the executor busy so the 4 slices fuse
    agg::AggregationRegion rb(sched, execs, pool, which ? cpu : gpu, 4, 4);
    std::vector<task::Future<agg::SliceOutput>> fb;
    for (std::size_t s = 0; s < 4; ++s) {
      auto x = slices[s];
      if (s == 2) x[hydro::kHeaderDoubles + 1728 * 2 + 5 * 144 + 6 * 12 + 7] = 0.0 / 0.0;
      fb.push_back(rb.submit_slice(x));
    }
    busy.reset();
    int thrown = 0;
    for (auto& f : fb) {
      try {
        sched.run_until(f);
      } catch (const hydro::SolverError& e) {
        ++thrown;
        msgs[which] = e.what();
      }
    }
    std::printf("%s error batch: %d/4 promises failed: %s\n", which ? "cpu" : "gpu", thrown,
                msgs[which].c_str());
    if (thrown != 4) ++failures;
  }
  if (msgs[0] != msgs[1]) ++failures;
  std::printf(failures ? "DROPIN_FAIL\n" : "DROPIN_OK\n");
  return failures ? 1 : 0;
}
