// NCCL communicator for the cross-GPU halo and the CFL reduction (comm.cpp).
// NCCL is bound at run time (dlopen of libnccl.so.2: the copy torch already
// loaded, else the system library), so the library has no link-time NCCL
// dependency and single-GPU use never touches it.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

struct tmgpu_comm;

namespace tmgpu {

int comm_rank(const tmgpu_comm* c);
int comm_world(const tmgpu_comm* c);
// Grouped point-to-point: for every peer p with a nonzero count, send
// send[send_off[p] .. +send_cnt[p]) and receive into recv[recv_off[p] ..).
int comm_exchange(tmgpu_comm* c, const double* send, const std::vector<long long>& send_off,
                  const std::vector<long long>& send_cnt, double* recv,
                  const std::vector<long long>& recv_off, const std::vector<long long>& recv_cnt,
                  cudaStream_t st, std::string* why);
// ncclAllGather of `count` doubles per rank into recv[world * count].
int comm_allgather(tmgpu_comm* c, const double* send, double* recv, size_t count, cudaStream_t st,
                   std::string* why);
// In-place all-gather of variable segments: rank p contributes
// buf[off[p] .. +cnt[p]) (grouped ncclBroadcast, root p), every rank ends with all.
int comm_allgatherv(tmgpu_comm* c, double* buf, const std::vector<long long>& off,
                    const std::vector<long long>& cnt, cudaStream_t st, std::string* why);
// Barrier over the communicator (a one-double all-reduce, synchronised on the
// host): every rank's earlier device work is complete when it returns.
int comm_barrier(tmgpu_comm* c, std::string* why);
// In-place min-allreduce of n doubles (the global CFL dt).
int comm_allreduce_min(tmgpu_comm* c, double* buf, size_t n, cudaStream_t st, std::string* why);

}  // namespace tmgpu
