// C ABI: hydro stage entry points (include/tmgpu.h). Host-side only; the
// kernels live in stage.cu.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "tmgpu_internal.h"

using namespace tmgpu;

namespace {

constexpr int kHeader = 8;  // stage.hpp:39 kHeaderDoubles

bool geometry_ok(int edge, int ghost, int vars) {
  return edge == 8 && ghost == 2 && (vars == 1 || vars == 5);
}

int solver_error(tmgpu_error* err, unsigned long long word) {
  const long long slot = (long long)(word >> 32);
  const unsigned idx = (unsigned)(word & 0xffffffffu);
  const unsigned cell = idx % 512u;
  const int i = (int)(cell % 8), j = (int)(cell / 8 % 8), k = (int)(cell / 64);
  if (err) {
    err->code = TMGPU_ERR_SOLVER;
    err->slice = slot;
    err->cell[0] = i;
    err->cell[1] = j;
    err->cell[2] = k;
    // identical text to hydro::SolverError (reference stage.cpp:211-215)
    std::snprintf(err->message, sizeof(err->message),
                  "non-finite state after stage at cell (%d,%d,%d)", i, j, k);
  }
  return TMGPU_ERR_SOLVER;
}

// Stream-ordered allocations are served from the device's default memory pool;
// keep freed blocks cached in the pool (release threshold = max) so repeated
// calls do not remap memory.
void keep_pool_warm() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  });
}

// Device-pointer fused stage over packed slices; synchronises `st`.
int stage_fused_device(const double* in, double* out, size_t in_slice, size_t out_slice,
                       size_t count, int vars, bool fast, cudaStream_t st, tmgpu_error* err) {
  if (count == 0) return TMGPU_OK;
  StageMaps maps;
  std::string why;
  int rc = make_stage_maps(in + kHeader, vars, (long long)in_slice, (long long)count, &maps, &why);
  if (rc != TMGPU_OK) return set_err(err, rc, why.c_str());
  keep_pool_warm();
  unsigned long long* d_err = nullptr;
  cudaError_t e = cudaMallocAsync(&d_err, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return cuda_err(err, e, "cudaMallocAsync");
  e = cudaMemsetAsync(d_err, 0xff, sizeof(unsigned long long), st);
  const size_t e3 = (size_t)vars * 512;
  StageLaunch p{};
  p.hdr = in;
  p.hdr_stride = (long long)in_slice;
  p.out = out;
  p.out_stride = (long long)out_slice;
  p.out_ghosted = 0;
  p.faces = out + e3;
  p.faces_stride = (long long)out_slice;
  p.diag = out + e3 + 6 * (size_t)vars * 64;
  p.diag_stride = (long long)out_slice;
  p.err = d_err;
  p.count = (int)count;
  if (e == cudaSuccess) e = launch_stage(vars, fast, maps, p, st);
  unsigned long long word = ~0ull;
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&word, d_err, sizeof(word), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_err, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_stage_fused");
  if (word != ~0ull) return solver_error(err, word);
  return TMGPU_OK;
}

// ---- host-pointer path (the drop-in's KernelFn over RegionBuffers) --------
// The reference calls KernelFn with its region's host buffers (pageable heap,
// bufferpool.cpp) from arbitrary scheduler workers, concurrently. Each calling
// thread keeps a context: two streams, device slice buffers and pinned bounce
// buffers for a chunk of slices each, allocated once and grown on demand. A
// call is chunked: while the GPU runs chunk c (H2D, the fused stage, D2H on
// stream c % 2) the thread copies chunk c + 1 into the other pinned buffer and
// chunk c - 1's results out of it — one cudaMemcpyAsync per direction per
// chunk, no allocation, no pageable DMA.
constexpr size_t kChunkSlices = 64;

struct HostCtx {
  cudaStream_t st[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  double *d_in[2] = {}, *d_out[2] = {}, *h_in[2] = {}, *h_out[2] = {};
  unsigned long long *d_err = nullptr, *h_err = nullptr;  // 2 words
  size_t cap_in = 0, cap_out = 0;  // doubles per buffer
  bool ok = false;
  ~HostCtx() {
    for (int b = 0; b < 2; ++b) {
      if (st[b]) cudaStreamSynchronize(st[b]);
      if (done[b]) cudaEventDestroy(done[b]);
      if (st[b]) cudaStreamDestroy(st[b]);
      cudaFree(d_in[b]);
      cudaFree(d_out[b]);
      cudaFreeHost(h_in[b]);
      cudaFreeHost(h_out[b]);
    }
    cudaFree(d_err);
    cudaFreeHost(h_err);
  }
  cudaError_t reserve(size_t in_doubles, size_t out_doubles) {
    cudaError_t e = cudaSuccess;
    if (!ok) {
      for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        e = cudaStreamCreateWithFlags(&st[b], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
      }
      if (e == cudaSuccess) e = cudaMalloc(&d_err, 2 * sizeof(unsigned long long));
      if (e == cudaSuccess) e = cudaMallocHost(&h_err, 2 * sizeof(unsigned long long));
      if (e != cudaSuccess) return e;
      ok = true;
    }
    if (in_doubles > cap_in) {
      for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        cudaFree(d_in[b]);
        cudaFreeHost(h_in[b]);
        d_in[b] = h_in[b] = nullptr;
        e = cudaMalloc(&d_in[b], in_doubles * sizeof(double));
        if (e == cudaSuccess) e = cudaMallocHost(&h_in[b], in_doubles * sizeof(double));
      }
      cap_in = e == cudaSuccess ? in_doubles : 0;
    }
    if (e == cudaSuccess && out_doubles > cap_out) {
      for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        cudaFree(d_out[b]);
        cudaFreeHost(h_out[b]);
        d_out[b] = h_out[b] = nullptr;
        e = cudaMalloc(&d_out[b], out_doubles * sizeof(double));
        if (e == cudaSuccess) e = cudaMallocHost(&h_out[b], out_doubles * sizeof(double));
      }
      cap_out = e == cudaSuccess ? out_doubles : 0;
    }
    return e;
  }
};

HostCtx& host_ctx() {
  thread_local HostCtx ctx;
  return ctx;
}

// enqueue one chunk of `n` slices (already in h_in[b]) on stream b
cudaError_t enqueue_chunk(HostCtx& C, int b, size_t n, size_t in_slice, size_t out_slice, int vars, bool fast,
                          std::string* why) {
  cudaStream_t st = C.st[b];
  cudaError_t e = cudaMemcpyAsync(C.d_in[b], C.h_in[b], n * in_slice * sizeof(double), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(C.d_err + b, 0xff, sizeof(unsigned long long), st);
  StageMaps maps;
  if (e == cudaSuccess && make_stage_maps(C.d_in[b] + kHeader, vars, (long long)in_slice, (long long)n, &maps, why) !=
                              TMGPU_OK)
    e = cudaErrorInvalidValue;
  if (e == cudaSuccess) {
    const size_t e3 = (size_t)vars * 512;
    double* out = C.d_out[b];
    StageLaunch p{};
    p.hdr = C.d_in[b];
    p.hdr_stride = (long long)in_slice;
    p.out = out;
    p.out_stride = (long long)out_slice;
    p.faces = out + e3;
    p.faces_stride = (long long)out_slice;
    p.diag = out + e3 + 6 * (size_t)vars * 64;
    p.diag_stride = (long long)out_slice;
    p.err = C.d_err + b;
    p.count = (int)n;
    e = launch_stage(vars, fast, maps, p, st);
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(C.h_out[b], C.d_out[b], n * out_slice * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(C.h_err + b, C.d_err + b, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaEventRecord(C.done[b], st);
  return e;
}

int stage_fused_host(const double* in, double* out, size_t in_slice, size_t out_slice, size_t count, int vars,
                     bool fast, tmgpu_error* err) {
  HostCtx& C = host_ctx();
  const size_t K = std::min(count, kChunkSlices);
  cudaError_t e = C.reserve(K * in_slice, K * out_slice);
  if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_stage_fused host staging");
  const size_t nch = (count + K - 1) / K;
  std::string why;
  unsigned long long first_bad = ~0ull;  // (global slice << 32 | index) of the first failure
  auto retire = [&](size_t c) -> cudaError_t {  // results of chunk c out of its pinned buffer
    const int b = (int)(c & 1);
    cudaError_t r = cudaEventSynchronize(C.done[b]);
    if (r != cudaSuccess) return r;
    const size_t n = std::min(K, count - c * K);
    std::memcpy(out + c * K * out_slice, C.h_out[b], n * out_slice * sizeof(double));
    const unsigned long long w = C.h_err[b];
    if (w != ~0ull && first_bad == ~0ull)
      first_bad = (((unsigned long long)(c * K) + (w >> 32)) << 32) | (w & 0xffffffffull);
    return cudaSuccess;
  };
  for (size_t c = 0; c < nch && e == cudaSuccess; ++c) {
    const int b = (int)(c & 1);
    if (c >= 2) e = retire(c - 2);  // frees buffer b (the GPU has moved on to chunk c - 1)
    if (e != cudaSuccess) break;
    const size_t n = std::min(K, count - c * K);
    std::memcpy(C.h_in[b], in + c * K * in_slice, n * in_slice * sizeof(double));
    e = enqueue_chunk(C, b, n, in_slice, out_slice, vars, fast, &why);
  }
  for (size_t c = nch >= 2 ? nch - 2 : 0; c < nch && e == cudaSuccess; ++c) e = retire(c);
  if (e != cudaSuccess) {
    cudaStreamSynchronize(C.st[0]);
    cudaStreamSynchronize(C.st[1]);
    if (!why.empty()) return set_err(err, TMGPU_ERR_INVALID, why.c_str());
    return cuda_err(err, e, "tmgpu_stage_fused");
  }
  if (first_bad != ~0ull) return solver_error(err, first_bad);
  return TMGPU_OK;
}

}  // namespace

extern "C" {

size_t tmgpu_in_slice(int edge, int ghost, int vars) {
  size_t s = (size_t)(edge + 2 * ghost);
  return kHeader + (size_t)vars * s * s * s;
}

size_t tmgpu_out_slice(int edge, int ghost, int vars) {
  (void)ghost;
  size_t e = (size_t)edge;
  return (size_t)vars * e * e * e + 6 * (size_t)vars * e * e + 1;
}

int tmgpu_stage_fused(const double* in, double* out, size_t in_slice, size_t out_slice,
                      size_t count, int edge, int ghost, int vars, int flags, void* stream,
                      tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!geometry_ok(edge, ghost, vars))
    return set_err(err, TMGPU_ERR_INVALID, "unsupported geometry (need edge 8, ghost 2, vars 1|5)");
  if (in_slice < tmgpu_in_slice(edge, ghost, vars) || out_slice < tmgpu_out_slice(edge, ghost, vars))
    return set_err(err, TMGPU_ERR_INVALID, "slice length smaller than the stage geometry");
  if (count == 0) return TMGPU_OK;
  if (!in || !out) return set_err(err, TMGPU_ERR_INVALID, "null buffer");
  const bool fast = (flags & TMGPU_FAST) != 0;
  cudaStream_t st = as_stream(stream);
  if (!(flags & TMGPU_HOST_PTRS))
    return stage_fused_device(in, out, in_slice, out_slice, count, vars, fast, st, err);

  return stage_fused_host(in, out, in_slice, out_slice, count, vars, fast, err);
}

int tmgpu_stage_subgrid(const double* header8, int edge, int ghost, int vars, unsigned lane_width,
                        const double* in_ghosted, double* out, int flags, void* stream,
                        tmgpu_error* err) {
  (void)lane_width;  // output is lane-width invariant (reference stage.hpp:69)
  if (err) std::memset(err, 0, sizeof(*err));
  if (!geometry_ok(edge, ghost, vars))
    return set_err(err, TMGPU_ERR_INVALID, "unsupported geometry (need edge 8, ghost 2, vars 1|5)");
  const size_t ins = tmgpu_in_slice(edge, ghost, vars), outs = tmgpu_out_slice(edge, ghost, vars);
  cudaStream_t st = as_stream(stream);
  if (flags & TMGPU_HOST_PTRS) {
    // one packed host slice
    double* slice = new double[ins];
    std::memcpy(slice, header8, kHeader * sizeof(double));
    std::memcpy(slice + kHeader, in_ghosted, (ins - kHeader) * sizeof(double));
    int rc = tmgpu_stage_fused(slice, out, ins, outs, 1, edge, ghost, vars, flags, stream, err);
    delete[] slice;
    return rc;
  }
  // device pointers: pack header + state into one aligned device slice
  double* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, ins * sizeof(double), st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d, header8, kHeader * sizeof(double), cudaMemcpyDefault, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d + kHeader, in_ghosted, (ins - kHeader) * sizeof(double),
                        cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) {
    if (d) cudaFreeAsync(d, st);
    return cuda_err(err, e, "tmgpu_stage_subgrid");
  }
  int rc = stage_fused_device(d, out, ins, outs, 1, vars, (flags & TMGPU_FAST) != 0, st, err);
  cudaFreeAsync(d, st);
  cudaStreamSynchronize(st);
  return rc;
}

int tmgpu_max_wavespeed(const double* in, size_t in_slice, size_t count, int edge, int ghost,
                        int vars, double* result, int flags, void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!geometry_ok(edge, ghost, vars))
    return set_err(err, TMGPU_ERR_INVALID, "unsupported geometry (need edge 8, ghost 2, vars 1|5)");
  if (count == 0) return TMGPU_OK;
  cudaStream_t st = as_stream(stream);
  const double* d_in = in;
  double* d_res = result;
  double* tmp_in = nullptr;
  double* tmp_res = nullptr;
  cudaError_t e = cudaSuccess;
  if (flags & TMGPU_HOST_PTRS) {
    e = cudaMallocAsync(&tmp_in, count * in_slice * sizeof(double), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&tmp_res, count * sizeof(double), st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(tmp_in, in, count * in_slice * sizeof(double), cudaMemcpyHostToDevice, st);
    d_in = tmp_in;
    d_res = tmp_res;
  }
  if (e == cudaSuccess)
    e = launch_max_wavespeed(d_in + kHeader, (long long)in_slice, d_in, (long long)in_slice,
                             nullptr, 1.4, vars, (long long)count, d_res, st);
  if (e == cudaSuccess && (flags & TMGPU_HOST_PTRS))
    e = cudaMemcpyAsync(result, tmp_res, count * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (tmp_in) cudaFreeAsync(tmp_in, st);
  if (tmp_res) cudaFreeAsync(tmp_res, st);
  cudaError_t e2 = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = e2;
  return cuda_err(err, e, "tmgpu_max_wavespeed");
}

int tmgpu_rk3_combine(int stage, const double* u0, const double* v, double* out, size_t n,
                      int flags, void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (stage < 1 || stage > 3) return set_err(err, TMGPU_ERR_INVALID, "stage must be 1, 2 or 3");
  if (n == 0) return TMGPU_OK;
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaSuccess;
  if (flags & TMGPU_HOST_PTRS) {
    double *a = nullptr, *b = nullptr;
    const size_t bytes = n * sizeof(double);
    e = cudaMallocAsync(&a, bytes, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&b, bytes, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(a, u0, bytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(b, v, bytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = launch_rk3_combine(stage, a, b, b, (long long)n, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, b, bytes, cudaMemcpyDeviceToHost, st);
    if (a) cudaFreeAsync(a, st);
    if (b) cudaFreeAsync(b, st);
  } else {
    e = launch_rk3_combine(stage, u0, v, out, (long long)n, st);
  }
  cudaError_t e2 = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = e2;
  return cuda_err(err, e, "tmgpu_rk3_combine");
}

const char* tmgpu_version(void) { return "tmgpu 0.1 (sm_100a, FP64)"; }

uint64_t tmgpu_launch_count(void) { return g_launches.load(); }

}  // extern "C"
