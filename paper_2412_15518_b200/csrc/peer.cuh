// Device helpers of the peer-memory exchanges (halo.cu, gravity_amr.cu): flag
// words are monotonic sequence numbers stored with release / loaded with
// acquire semantics at system scope; a wait that does not see its value within
// kPeerSpinNs (20 s) traps (a loud failure instead of a hung GPU).
#pragma once

#include <cstdio>

namespace tmgpu {

constexpr unsigned long long kPeerSpinNs = 20000000000ull;  // 20 s

__device__ __forceinline__ unsigned long long peer_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

static __device__ __noinline__ void spin_geq(const unsigned long long* p, unsigned long long v) {
  if (ld_acquire_sys(p) >= v) return;
  const unsigned long long t0 = peer_globaltimer();
  while (ld_acquire_sys(p) < v) {
    __nanosleep(100);
    if (peer_globaltimer() - t0 > kPeerSpinNs) {
      printf("tmgpu peer exchange: timeout waiting for flag %p >= %llu\n", (const void*)p, v);
      __trap();
    }
  }
}

}  // namespace tmgpu
