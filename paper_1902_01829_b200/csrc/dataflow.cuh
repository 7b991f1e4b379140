// Dataflow synchronisation of the fused sweep launches (k_hmv.cu, k_hmv_mv.cu).
//
// A sweep launch lists the nodes of several tree levels in dependency order; a
// warp claims the next item with an atomic ticket, waits on the completion
// flags of the nodes it reads, computes, and publishes its own node's flag.
// Claimed items only wait for items claimed earlier, whose warps are already
// running, so the launch is deadlock-free at any residency.  Flags hold an
// epoch (2e: up done, 2e + 1: down done, one epoch per mat-vec) and are never
// cleared.  Node vectors written by other SMs are read with ld.cg.
#pragma once

#include <cstdint>

namespace h2b {
namespace df {

// Global node id of level-local node i (complete binary tree, BFS order).
__device__ __forceinline__ int64_t node_id(int level, int64_t i) { return (int64_t(1) << level) - 1 + i; }

__device__ __forceinline__ void wait_flag(const uint32_t* f, uint32_t want) {
  if ((threadIdx.x & 31) == 0) {
    uint32_t v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (v >= want) break;
      __nanosleep(64);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void set_flag(uint32_t* f, uint32_t v) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
  }
}

__device__ __forceinline__ int64_t claim(unsigned long long* ticket) {
  unsigned long long t = 0;
  if ((threadIdx.x & 31) == 0) t = atomicAdd(ticket, 1ull);
  return int64_t(__shfl_sync(0xffffffffu, t, 0));
}

}  // namespace df
}  // namespace h2b
