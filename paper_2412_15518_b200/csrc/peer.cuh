// Device helpers of the peer-memory exchanges (halo.cu, gravity_amr.cu): flag
// words are monotonic sequence numbers stored with release / loaded with
// acquire semantics at system scope. A wait that does not see its value within
// the exchange's spin limit traps: continuing would compute on a peer's stale
// slabs, so the failure is made loud. The limit comes from TMGPU_PEER_TIMEOUT_S
// at peer setup (default 20 s; 0 = wait forever, e.g. under a debugger or ncu
// replay where a peer can legitimately stall for long).
#pragma once

#include <cstdio>

namespace tmgpu {

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

static __device__ __noinline__ void spin_geq(const unsigned long long* p, unsigned long long v,
                                             unsigned long long limit_ns) {
  if (ld_acquire_sys(p) >= v) return;
  const unsigned long long t0 = peer_globaltimer();
  while (ld_acquire_sys(p) < v) {
    __nanosleep(100);
    if (limit_ns && peer_globaltimer() - t0 > limit_ns) {
      printf("tmgpu peer exchange: timeout waiting for flag %p >= %llu\n", (const void*)p, v);
      __trap();
    }
  }
}

}  // namespace tmgpu
