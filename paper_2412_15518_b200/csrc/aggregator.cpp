// GPU kernel-aggregation executor: the reference's ExecutorPool +
// AggregationRegion (proj/src/aggregator.cpp, include/taskmesh/aggregator.hpp)
// with CUDA streams as the executors.
//
// Semantics kept from the reference (and its tests, test_aggregator.cpp):
//  * ExecutorPool: per-executor in-flight counters; acquire picks a minimal
//    counter, ties broken round-robin from a cursor (aggregator.cpp:24-49);
//    acquire_at pins a slot on a given executor; leases release slots.
//  * AggregationRegion: slices are packed at index*slice; a batch launches
//    when it reaches max_slices or when the pinned executor is idle at submit
//    time; flush() launches the remainder and finalises the region (idempotent;
//    submitting afterwards is an error); counters launches / fused_slices /
//    solo_launches; after every launch the region re-pins to the least-loaded
//    executor (aggregator.cpp:106-172).
// B200-native execution: a launch is one asynchronous sequence on the pinned
// executor's stream — H2D of the batch's packed slices (pinned host staging),
// ONE aggregated kernel over the batch, D2H of the outputs — followed by a
// host callback that retires the in-flight slot and settles the batch's
// futures. A kernel error (non-finite state) fails every slice of the batch,
// as the reference's catch-all does (aggregator.cpp:164-167).
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "tmgpu_internal.h"

namespace tmgpu {

namespace {

struct Pool {
  explicit Pool(size_t n) : in_flight(n, 0) {}
  std::mutex mu;
  std::vector<uint64_t> in_flight;
  size_t next = 0;
  std::vector<cudaStream_t> streams;  // created lazily (first launch)

  size_t select_locked() {  // aggregator.cpp:24-37
    uint64_t best = in_flight[next % in_flight.size()];
    for (uint64_t v : in_flight) best = std::min(best, v);
    const size_t n = in_flight.size();
    for (size_t k = 0; k < n; ++k) {
      const size_t i = (next + k) % n;
      if (in_flight[i] == best) {
        next = i + 1;
        return i;
      }
    }
    return 0;
  }
  cudaError_t stream(size_t i, cudaStream_t* s) {
    std::lock_guard<std::mutex> lk(mu);
    if (streams.empty()) {
      streams.resize(in_flight.size(), nullptr);
      for (auto& x : streams) {
        cudaError_t e = cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
        if (e != cudaSuccess) return e;
      }
    }
    *s = streams[i];
    return cudaSuccess;
  }
  ~Pool() {
    for (auto s : streams)
      if (s) cudaStreamDestroy(s);
  }
};

struct Batch {
  size_t first = 0, count = 0;
  bool done = false;
  int code = TMGPU_OK;
  tmgpu_error err{};
};

}  // namespace
}  // namespace tmgpu

using namespace tmgpu;

struct tmgpu_execpool {
  explicit tmgpu_execpool(size_t n) : p(n) {}
  Pool p;
};

struct tmgpu_region {
  tmgpu_execpool* pool = nullptr;
  int kind = 0;  // 0 custom device kernel (fn, user), 1 hydro stage
  tmgpu_device_kernel fn = nullptr;
  void* user = nullptr;
  int edge = 8, ghost = 2, vars = 5, flags = 0;
  size_t in_slice = 0, out_slice = 0, max_slices = 1, capacity = 0;
  uint64_t* counters = nullptr;  // [launches, fused_slices, solo_launches]
  std::mutex mu;
  std::condition_variable cv;
  double *h_in = nullptr, *h_out = nullptr;  // pinned
  double *d_in = nullptr, *d_out = nullptr;
  unsigned long long* d_err = nullptr;       // one word per batch slot (capacity)
  std::vector<std::shared_ptr<Batch>> batch_of;  // per slice
  std::vector<std::shared_ptr<Batch>> batches;
  size_t pinned = 0, total = 0, batch_first = 0, open = 0;
  bool launched = false;
  size_t outstanding = 0;  // launched batches not yet retired
};

namespace {

struct Retire {
  tmgpu_region* r;
  std::shared_ptr<Batch> b;
  size_t exec;
  unsigned long long* word;  // host-visible error word of the batch
};

void CUDART_CB on_done(void* arg) {
  std::unique_ptr<Retire> rt(static_cast<Retire*>(arg));
  tmgpu_region* r = rt->r;
  {
    std::lock_guard<std::mutex> lk(r->pool->p.mu);
    r->pool->p.in_flight[rt->exec] -= 1;  // launched work settles before results
  }
  std::lock_guard<std::mutex> lk(r->mu);
  rt->b->done = true;
  r->outstanding -= 1;
  r->cv.notify_all();
}

int launch_locked(tmgpu_region* r, tmgpu_error* err) {  // aggregator.cpp:132-172
  const size_t first = r->batch_first, count = r->open;
  r->batch_first = first + count;
  r->open = 0;
  auto b = std::make_shared<Batch>();
  b->first = first;
  b->count = count;
  for (size_t s = first; s < first + count; ++s) r->batch_of[s] = b;
  r->batches.push_back(b);
  if (r->counters) {
    r->counters[0] += 1;
    r->counters[1] += count;
    if (count == 1) r->counters[2] += 1;
  }
  const size_t exec = r->pinned;
  {
    std::lock_guard<std::mutex> lk(r->pool->p.mu);
    r->pool->p.in_flight.at(exec) += 1;  // acquire_at(pinned)
  }
  cudaStream_t st;
  cudaError_t e = r->pool->p.stream(exec, &st);
  const size_t ib = r->in_slice * sizeof(double), ob = r->out_slice * sizeof(double);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(r->d_in + first * r->in_slice, r->h_in + first * r->in_slice, count * ib,
                        cudaMemcpyHostToDevice, st);
  unsigned long long* word = r->d_err + first;  // batch error word lives at its first slot
  if (e == cudaSuccess) e = cudaMemsetAsync(word, 0xff, sizeof(unsigned long long), st);
  if (e == cudaSuccess) {
    if (r->kind == 0) {  // KernelSpec::fn of a registered kernel (aggregator.hpp:94-106)
      const int rc = r->fn(r->d_in + first * r->in_slice, r->d_out + first * r->out_slice, r->in_slice,
                           r->out_slice, count, st, r->user);
      if (rc != 0) e = cudaErrorLaunchFailure;
    } else {
      StageMaps maps;
      std::string why;
      const double* in = r->d_in + first * r->in_slice;
      if (make_stage_maps(in + 8, r->vars, (long long)r->in_slice, (long long)count, &maps, &why) !=
          TMGPU_OK) {
        e = cudaErrorInvalidValue;
      } else {
        StageLaunch p{};
        double* out = r->d_out + first * r->out_slice;
        const size_t e3 = (size_t)r->vars * 512;
        p.hdr = in;
        p.hdr_stride = (long long)r->in_slice;
        p.out = out;
        p.out_stride = (long long)r->out_slice;
        p.faces = out + e3;
        p.faces_stride = (long long)r->out_slice;
        p.diag = out + e3 + 6 * (size_t)r->vars * 64;
        p.diag_stride = (long long)r->out_slice;
        p.err = word;
        p.count = (int)count;
        e = launch_stage(r->vars, (r->flags & TMGPU_FAST) != 0, maps, p, st);
      }
    }
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(r->h_out + first * r->out_slice, r->d_out + first * r->out_slice,
                        count * ob, cudaMemcpyDeviceToHost, st);
  r->outstanding += 1;
  if (e == cudaSuccess) {
    auto* rt = new Retire{r, b, exec, word};
    e = cudaLaunchHostFunc(st, on_done, rt);
    if (e != cudaSuccess) delete rt;
  }
  if (e != cudaSuccess) {  // settle synchronously with the failure
    {
      std::lock_guard<std::mutex> lk(r->pool->p.mu);
      r->pool->p.in_flight[exec] -= 1;
    }
    b->done = true;
    b->code = cuda_err(&b->err, e, "aggregated launch");
    r->outstanding -= 1;
    r->cv.notify_all();
    if (err) *err = b->err;
  }
  {  // re-pin to the least-loaded executor (aggregator.cpp:170-171)
    std::lock_guard<std::mutex> lk(r->pool->p.mu);
    r->pinned = r->pool->p.select_locked();
  }
  return TMGPU_OK;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------- ExecutorPool
// ExecutorPool(count) (aggregator.hpp:57-85); count 0 is an error (AggError).
tmgpu_execpool* tmgpu_execpool_create(size_t count, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (count == 0) {
    set_err(err, TMGPU_ERR_AGG, "executor pool must be non-empty");
    return nullptr;
  }
  return new tmgpu_execpool(count);
}
void tmgpu_execpool_destroy(tmgpu_execpool* p) { delete p; }
size_t tmgpu_execpool_size(tmgpu_execpool* p) { return p->p.in_flight.size(); }
// acquire(): least-loaded, round-robin ties; returns the executor index (a lease)
size_t tmgpu_execpool_acquire(tmgpu_execpool* p) {
  std::lock_guard<std::mutex> lk(p->p.mu);
  const size_t i = p->p.select_locked();
  p->p.in_flight[i] += 1;
  return i;
}
size_t tmgpu_execpool_pick_index(tmgpu_execpool* p) {
  std::lock_guard<std::mutex> lk(p->p.mu);
  return p->p.select_locked();
}
int tmgpu_execpool_acquire_at(tmgpu_execpool* p, size_t index, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  std::lock_guard<std::mutex> lk(p->p.mu);
  if (index >= p->p.in_flight.size()) return set_err(err, TMGPU_ERR_AGG, "executor index out of range");
  p->p.in_flight[index] += 1;
  return TMGPU_OK;
}
void tmgpu_execpool_release(tmgpu_execpool* p, size_t index) {
  std::lock_guard<std::mutex> lk(p->p.mu);
  if (index < p->p.in_flight.size() && p->p.in_flight[index] > 0) p->p.in_flight[index] -= 1;
}
uint64_t tmgpu_execpool_in_flight(tmgpu_execpool* p, size_t index) {
  std::lock_guard<std::mutex> lk(p->p.mu);
  return index < p->p.in_flight.size() ? p->p.in_flight[index] : 0;
}

// ------------------------------------------------------------- AggregationRegion
// kind 1: hydro::make_stage_kernel(geom) (stage.cpp:229-246) on the device;
// any other registered kernel through tmgpu_region_create_kernel.
// counters: optional uint64[3] {launches, fused_slices, solo_launches}
// (AggCounters, aggregator.hpp:87-92), updated under the region lock.
namespace {
tmgpu_region* region_new(tmgpu_execpool* pool, int kind, size_t in_slice, size_t out_slice, int edge, int ghost,
                         int vars, int flags, size_t max_slices, size_t capacity, uint64_t* counters,
                         tmgpu_device_kernel fn, void* user, tmgpu_error* err) {
  if (!pool) {
    set_err(err, TMGPU_ERR_AGG, "null executor pool");
    return nullptr;
  }
  if (max_slices == 0) {
    set_err(err, TMGPU_ERR_AGG, "max_slices must be positive");
    return nullptr;
  }
  if (capacity == 0) {
    set_err(err, TMGPU_ERR_AGG, "region capacity must be positive");
    return nullptr;
  }
  if (kind == 1) {
    if (edge != 8 || ghost != 2 || (vars != 1 && vars != 5)) {
      set_err(err, TMGPU_ERR_INVALID, "unsupported geometry (need edge 8, ghost 2, vars 1|5)");
      return nullptr;
    }
    in_slice = tmgpu_in_slice(edge, ghost, vars);
    out_slice = tmgpu_out_slice(edge, ghost, vars);
  }
  auto* r = new tmgpu_region;
  r->pool = pool;
  r->kind = kind;
  r->fn = fn;
  r->user = user;
  r->edge = edge;
  r->ghost = ghost;
  r->vars = vars;
  r->flags = flags;
  r->in_slice = in_slice;
  r->out_slice = out_slice;
  r->max_slices = max_slices;
  r->capacity = capacity;
  r->counters = counters;
  r->batch_of.resize(capacity);
  cudaError_t e = cudaMallocHost(&r->h_in, capacity * in_slice * sizeof(double));
  if (e == cudaSuccess) e = cudaMallocHost(&r->h_out, capacity * out_slice * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&r->d_in, capacity * in_slice * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&r->d_out, capacity * out_slice * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&r->d_err, capacity * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    cuda_err(err, e, "tmgpu_region_create");
    if (r->h_in) cudaFreeHost(r->h_in);
    if (r->h_out) cudaFreeHost(r->h_out);
    if (r->d_in) cudaFree(r->d_in);
    if (r->d_out) cudaFree(r->d_out);
    delete r;
    return nullptr;
  }
  std::memset(r->h_out, 0, capacity * out_slice * sizeof(double));  // zeroed lease
  std::lock_guard<std::mutex> lk(pool->p.mu);
  r->pinned = pool->p.select_locked();  // pick_index (aggregator.cpp:98)
  return r;
}
}  // namespace

tmgpu_region* tmgpu_region_create(tmgpu_execpool* pool, int kind, size_t in_slice,
                                  size_t out_slice, int edge, int ghost, int vars, int flags,
                                  size_t max_slices, size_t capacity, uint64_t* counters,
                                  tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (kind != 1) {
    set_err(err, TMGPU_ERR_INVALID, "region kind must be 1 (hydro stage); use tmgpu_region_create_kernel");
    return nullptr;
  }
  return region_new(pool, kind, in_slice, out_slice, edge, ghost, vars, flags, max_slices, capacity, counters,
                    nullptr, nullptr, err);
}

// submit_slice (aggregator.cpp:106-124): returns the slice ticket (>= 0) or -1.
// A region over any device kernel (the reference's KernelRegistry holds
// arbitrary KernelSpecs, aggregator.hpp:94-116): fn(d_in, d_out, in_slice,
// out_slice, count, stream, user) launches one aggregated kernel over `count`
// packed device slices on `stream` and returns 0 (else the batch fails).
tmgpu_region* tmgpu_region_create_kernel(tmgpu_execpool* pool, tmgpu_device_kernel fn, void* user,
                                         size_t in_slice, size_t out_slice, size_t max_slices,
                                         size_t capacity, uint64_t* counters, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!fn) {
    set_err(err, TMGPU_ERR_AGG, "null kernel function");
    return nullptr;
  }
  if (in_slice == 0 || out_slice == 0) {
    set_err(err, TMGPU_ERR_AGG, "slice sizes must be positive");
    return nullptr;
  }
  return region_new(pool, 0, in_slice, out_slice, 0, 0, 0, 0, max_slices, capacity, counters, fn, user, err);
}

long long tmgpu_region_submit(tmgpu_region* r, const double* input, size_t len, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  std::lock_guard<std::mutex> lk(r->mu);
  if (r->launched) {
    set_err(err, TMGPU_ERR_AGG, "submit_slice after final flush");
    return -1;
  }
  if (len != r->in_slice) {
    set_err(err, TMGPU_ERR_AGG, "slice length does not match the region's slice size");
    return -1;
  }
  if (r->total == r->capacity) {
    set_err(err, TMGPU_ERR_AGG, "region capacity exhausted");
    return -1;
  }
  const size_t idx = r->total++;
  std::memcpy(r->h_in + idx * r->in_slice, input, len * sizeof(double));
  r->open += 1;
  const bool full = r->open == r->max_slices;
  bool idle;
  {
    std::lock_guard<std::mutex> pl(r->pool->p.mu);
    idle = r->pool->p.in_flight[r->pinned] == 0;
  }
  if (full || idle) launch_locked(r, err);
  return (long long)idx;
}

// flush (aggregator.cpp:126-130): launch the remainder, finalise; idempotent.
int tmgpu_region_flush(tmgpu_region* r, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  std::lock_guard<std::mutex> lk(r->mu);
  if (r->open) launch_locked(r, err);
  r->launched = true;
  return TMGPU_OK;
}

// Wait for the batch holding `ticket`; 0 ok, else the batch's error (every slice
// of a failed batch reports it). Unlaunched tickets return TMGPU_ERR_AGG.
int tmgpu_region_wait(tmgpu_region* r, long long ticket, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  std::unique_lock<std::mutex> lk(r->mu);
  if (ticket < 0 || (size_t)ticket >= r->total)
    return set_err(err, TMGPU_ERR_AGG, "unknown slice ticket");
  auto b = r->batch_of[ticket];
  if (!b) return set_err(err, TMGPU_ERR_AGG, "slice not launched yet (flush the region)");
  r->cv.wait(lk, [&] { return b->done; });
  if (b->code == TMGPU_OK && r->kind == 1) {
    unsigned long long word = ~0ull;
    lk.unlock();
    cudaMemcpy(&word, r->d_err + b->first, sizeof(word), cudaMemcpyDeviceToHost);
    lk.lock();
    if (word != ~0ull && b->code == TMGPU_OK) {  // the batch fails for every slice
      const unsigned cell = (unsigned)(word & 0xffffffffu) % 512u;
      b->code = TMGPU_ERR_SOLVER;
      b->err.code = TMGPU_ERR_SOLVER;
      b->err.slice = (int64_t)b->first + (int64_t)(word >> 32);
      b->err.cell[0] = (int)(cell % 8);
      b->err.cell[1] = (int)(cell / 8 % 8);
      b->err.cell[2] = (int)(cell / 64);
      std::snprintf(b->err.message, sizeof(b->err.message),
                    "non-finite state after stage at cell (%d,%d,%d)", b->err.cell[0],
                    b->err.cell[1], b->err.cell[2]);
    }
  }
  if (b->code != TMGPU_OK && err) *err = b->err;
  return b->code;
}

// Pointer to slice `ticket`'s output (SliceOutput::values, aggregator.hpp:127-136);
// valid after tmgpu_region_wait and until the region is destroyed.
const double* tmgpu_region_output(tmgpu_region* r, long long ticket) {
  return r->h_out + (size_t)ticket * r->out_slice;
}

size_t tmgpu_region_submitted(tmgpu_region* r) {
  std::lock_guard<std::mutex> lk(r->mu);
  return r->total;
}

void tmgpu_region_destroy(tmgpu_region* r) {
  if (!r) return;
  {
    std::unique_lock<std::mutex> lk(r->mu);
    r->cv.wait(lk, [&] { return r->outstanding == 0; });
  }
  cudaFreeHost(r->h_in);
  cudaFreeHost(r->h_out);
  cudaFree(r->d_in);
  cudaFree(r->d_out);
  cudaFree(r->d_err);
  delete r;
}

}  // extern "C"
