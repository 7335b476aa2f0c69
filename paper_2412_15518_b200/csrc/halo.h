// One-round face exchange with cross-GPU halos (halo.cu).
//
// Every directed face fill of the reference plan (ghost.cpp:168-210) is
// executed once per exchange as
//   pack   — on the SOURCE leaf's GPU: the slab the destination needs
//            (same-level: 2 interior layers; prolonged: ghost.cpp:70-96 with
//            the coarse source's ghost tap read from the previous exchange;
//            restricted: ghost.cpp:113-131 2x2x2 means), into a slab buffer;
//   move   — when source and destination GPUs differ, the slab travels in
//            one grouped NCCL send/recv per peer (comm.cpp);
//   pull   — on the DESTINATION leaf's GPU: one CTA per (leaf, face) writes
//            the E x E x G face-ghost slab from a local leaf, a slab, or the
//            reflective mirror (ghost.cpp:151-166).
// Same-level fills between leaves on the same GPU are neither packed nor
// pulled: the stage kernel TMA-loads the neighbour's interior directly.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tmgpu {

// kind: 0 same, 1 coarser source (prolonged), 2 finer source (restricted)
struct alignas(16) PackItem {
  int32_t src;  // local slot of the source leaf
  int32_t out;  // offset (doubles) into the slab buffer
  int8_t kind, axis, dir, qt1, qt2;
  int8_t pad[3];  // peer exchange: pad[0] = destination rank + 1 (0 = this rank)
};

// Where a destination face gets its ghosts. kind as NeighborKind (0 same,
// 1 coarser, 2 finer, 3 boundary). Per source q (finer: quadrant qt2*2+qt1;
// otherwise q = 0): src[q] >= 0 a local leaf slot, else off[q] is the slab
// buffer offset of a packed slab (coarser fills always use a slab).
struct alignas(16) FaceSrc {
  int32_t src[4];
  int32_t off[4];
  int8_t kind;
  int8_t pad[15];
};

// Slab sizes in doubles per kind (V vars).
inline int slab_doubles(int kind, int V) { return kind == 2 ? V * 2 * 4 * 4 : V * 2 * 8 * 8; }

// Peer-memory exchange (opt-in, tmgpu_forest_set_peer): senders pack straight
// into the receivers' slab buffers (CUDA IPC over NVLink/NVSwitch) and
// synchronise through flag words instead of NCCL send/recv.
constexpr int kMaxPeers = 8;
struct PeerTab {
  double* slabs[kMaxPeers];               // peers' slab buffers (IPC-mapped; [me] unused)
  unsigned long long* flags[kMaxPeers];   // peers' flag words
  // this rank's flag words: [0,w) arrival seq from sender s, [w,2w) consumption
  // seq by receiver q, [2w,3w) per-peer pack CTA counters, [3w] pull counter
  unsigned long long* mine;
  int n_send[kMaxPeers];                  // pack items (CTAs) per destination peer
  int me, world;
  unsigned recv_mask;                     // peers this rank receives slabs from
  unsigned long long spin_ns;             // flag-wait limit (peer_spin_ns(); 0 = none)
  // this rank's exchange sequence number in device memory ([3w + 1] of its
  // flag words): bumped by seq_bump() at the start of every exchange and read
  // by the exchange's kernels, so a captured step (CUDA graph) replays correctly
  unsigned long long* seqp;
};

// *p += 1 on the stream (one thread): the next exchange round's sequence number
cudaError_t seq_bump(unsigned long long* p, cudaStream_t st);

cudaError_t halo_pack_peer(const double* arena, const double* prev, int V, const PackItem* items,
                           int n_items, double* slabs, const PeerTab& t, cudaStream_t st);
cudaError_t halo_pull_peer(double* arena, int V, const FaceSrc* faces, const int2* items,
                           int n_local, int n_items, const double* slabs, const PeerTab& t,
                           cudaStream_t st);

cudaError_t halo_pack(const double* arena, const double* prev, int V, const PackItem* items,
                      int n_items, double* slabs, cudaStream_t st);
cudaError_t halo_pull(double* arena, int V, const FaceSrc* faces, const int2* items, int n_items,
                      const double* slabs, cudaStream_t st);

}  // namespace tmgpu
