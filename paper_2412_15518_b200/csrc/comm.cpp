// NCCL binding (see comm.h). Everything is stream-ordered: no host syncs.
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "tmgpu_internal.h"

namespace {

struct Api {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.Send = (decltype(a.Send))sym("ncclSend");
    a.Recv = (decltype(a.Recv))sym("ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
    a.Broadcast = (decltype(a.Broadcast))sym("ncclBroadcast");
    a.AllGather = (decltype(a.AllGather))sym("ncclAllGather");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
    if (!a.GetUniqueId || !a.CommInitRank || !a.Send || !a.Recv || !a.GroupStart || !a.GroupEnd ||
        !a.AllReduce || !a.Broadcast || !a.AllGather)
      a.error = "libnccl.so.2 lacks required symbols";
  });
  return a;
}

std::string nerr(ncclResult_t r) {
  return api().GetErrorString ? api().GetErrorString(r) : ("nccl error " + std::to_string((int)r));
}

}  // namespace

struct tmgpu_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
};

namespace tmgpu {

int comm_rank(const tmgpu_comm* c) { return c ? c->rank : 0; }
int comm_world(const tmgpu_comm* c) { return c ? c->world : 1; }

int comm_exchange(tmgpu_comm* c, const double* send, const std::vector<long long>& send_off,
                  const std::vector<long long>& send_cnt, double* recv,
                  const std::vector<long long>& recv_off, const std::vector<long long>& recv_cnt,
                  cudaStream_t st, std::string* why) {
  Api& a = api();
  ncclResult_t r = a.GroupStart();
  for (int p = 0; p < c->world && r == ncclSuccess; ++p) {
    if (p == c->rank) continue;
    if (send_cnt[p] > 0)
      r = a.Send(send + send_off[p], (size_t)send_cnt[p], ncclDouble, p, c->comm, st);
    if (r == ncclSuccess && recv_cnt[p] > 0)
      r = a.Recv(recv + recv_off[p], (size_t)recv_cnt[p], ncclDouble, p, c->comm, st);
  }
  ncclResult_t r2 = a.GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) {
    if (why) *why = "halo exchange: " + nerr(r);
    return TMGPU_ERR_CUDA;
  }
  return TMGPU_OK;
}

int comm_allreduce_min(tmgpu_comm* c, double* buf, size_t n, cudaStream_t st, std::string* why) {
  ncclResult_t r = api().AllReduce(buf, buf, n, ncclDouble, ncclMin, c->comm, st);
  if (r != ncclSuccess) {
    if (why) *why = "dt allreduce: " + nerr(r);
    return TMGPU_ERR_CUDA;
  }
  return TMGPU_OK;
}

int comm_barrier(tmgpu_comm* c, std::string* why) {
  if (!c || comm_world(c) < 2) return TMGPU_OK;
  double* d = nullptr;
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMalloc(&d, sizeof(double));
  if (e == cudaSuccess) e = cudaMemset(d, 0, sizeof(double));
  if (e != cudaSuccess) {
    if (why) *why = std::string("barrier: ") + cudaGetErrorString(e);
    return TMGPU_ERR_CUDA;
  }
  int rc = comm_allreduce_min(c, d, 1, nullptr, why);
  e = cudaDeviceSynchronize();
  cudaFree(d);
  if (rc == TMGPU_OK && e != cudaSuccess) {
    if (why) *why = std::string("barrier: ") + cudaGetErrorString(e);
    rc = TMGPU_ERR_CUDA;
  }
  return rc;
}

int comm_allgather(tmgpu_comm* c, const double* send, double* recv, size_t count, cudaStream_t st,
                   std::string* why) {
  ncclResult_t r = api().AllGather(send, recv, count, ncclDouble, c->comm, st);
  if (r != ncclSuccess) {
    if (why) *why = "allgather: " + nerr(r);
    return TMGPU_ERR_CUDA;
  }
  return TMGPU_OK;
}

int comm_allgatherv(tmgpu_comm* c, double* buf, const std::vector<long long>& off,
                    const std::vector<long long>& cnt, cudaStream_t st, std::string* why) {
  Api& a = api();
  ncclResult_t r = a.GroupStart();
  for (int p = 0; p < c->world && r == ncclSuccess; ++p)
    if (cnt[p] > 0) r = a.Broadcast(buf + off[p], buf + off[p], (size_t)cnt[p], ncclDouble, p, c->comm, st);
  ncclResult_t r2 = a.GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) {
    if (why) *why = "allgatherv: " + nerr(r);
    return TMGPU_ERR_CUDA;
  }
  return TMGPU_OK;
}

}  // namespace tmgpu

using namespace tmgpu;

extern "C" {

int tmgpu_comm_unique_id(unsigned char* id128, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  Api& a = api();
  if (!a.error.empty()) return set_err(err, TMGPU_ERR_CUDA, a.error.c_str());
  ncclUniqueId id;
  ncclResult_t r = a.GetUniqueId(&id);
  if (r != ncclSuccess) return set_err(err, TMGPU_ERR_CUDA, nerr(r).c_str());
  std::memcpy(id128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return TMGPU_OK;
}

tmgpu_comm* tmgpu_comm_create(int rank, int world, const unsigned char* id128, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  Api& a = api();
  if (!a.error.empty()) {
    set_err(err, TMGPU_ERR_CUDA, a.error.c_str());
    return nullptr;
  }
  ncclUniqueId id;
  std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
  auto* c = new tmgpu_comm;
  c->rank = rank;
  c->world = world;
  ncclResult_t r = a.CommInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    set_err(err, TMGPU_ERR_CUDA, nerr(r).c_str());
    delete c;
    return nullptr;
  }
  return c;
}

void tmgpu_comm_destroy(tmgpu_comm* c) {
  if (!c) return;
  if (c->comm && api().CommDestroy) api().CommDestroy(c->comm);
  delete c;
}

}  // extern "C"
