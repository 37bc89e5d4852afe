// dist_sync.cuh -- cross-GPU flag wait / signal folded into kernels
// (sharded step, dist.cu).  Flags live in the receiver's IPC arena and hold
// the step epoch; see DESIGN.md §6 for the memory-ordering argument.
#pragma once

#include "rs_host.hpp"
#include "rs_internal.cuh"

namespace rs {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// Bounded spin (~20 s at 2 GHz) on one flag; a dead peer sets *error instead
// of hanging the GPU.
__device__ __forceinline__ void spin_flag(const unsigned long long* f, unsigned long long e,
                                          unsigned long long* error) {
  const long long t0 = clock64();
  while (ld_acquire_sys(f) < e) {
    if (clock64() - t0 > 40000000000ll) {
      if (error) *error = 1;
      break;
    }
    __nanosleep(64);
  }
}

// Prologue: the block proceeds once every wait flag reached the epoch.
__device__ __forceinline__ void dist_wait(const rs_dist_sync& s) {
  if (!s.wait_flags) return;
  const unsigned long long e = *s.epoch;
  for (uint32_t r = threadIdx.x; r < s.wait_n; r += blockDim.x) spin_flag(s.wait_flags + r, e, s.error);
  __syncthreads();
}

// Epilogue (every thread of every block): grid-level arrival; the last of
// sig_total blocks raises the flags with release semantics at system scope.
__device__ __forceinline__ void dist_arrive(const rs_dist_sync& s) {
  if (!s.sig_flags) return;
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(s.sig_done) : "memory");
    last = old == s.sig_total - 1;
    if (last) fence_sys();
  }
  __syncthreads();
  if (!last) return;
  const unsigned long long e = *s.epoch;
  for (uint32_t r = threadIdx.x; r < s.sig_n; r += blockDim.x) st_release_sys(s.sig_flags[r], e);
  if (threadIdx.x == 0) *s.sig_done = 0;
}

}  // namespace rs
