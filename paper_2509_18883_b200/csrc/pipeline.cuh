// Warp-specialised TMA ring used by the streaming kernels: one producer lane issues cp.async.bulk
// copies into `nstages` shared-memory slots; kCWarps consumer warps wait on `full`, read, and
// release on `empty` (one arrival per consumer warp).
#pragma once
#include "common.cuh"

namespace rlk {

constexpr int kCWarps = 8;
constexpr int kCThreads = kCWarps * 32;
constexpr int kThreads = kCThreads + 32;

__device__ __forceinline__ void cbar_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kCThreads) : "memory"); }

// K3 fast path consumer warps (8: more forces <= 128 registers and spills)
#ifndef RLK_FAST_CWARPS
#define RLK_FAST_CWARPS 16
#endif
constexpr int kFastCWarps = RLK_FAST_CWARPS;
constexpr int kFastCThreads = kFastCWarps * 32;
constexpr int kFastThreads = kFastCThreads + 32;

// Position in the ring: slot and the mbarrier phase parity of the current lap (no runtime division).
struct RingPos {
  uint32_t s = 0, ph = 0;
  __device__ __forceinline__ void next(uint32_t n) {
    if (++s == n) {
      s = 0;
      ph ^= 1u;
    }
  }
};

struct Ring {
  uint8_t* buf;
  uint64_t* full;
  uint64_t* empty;
  uint32_t stage_bytes;
  uint32_t nstages;
};

__device__ __forceinline__ Ring ring_setup(uint8_t* smem, uint32_t stage_bytes, uint32_t nstages,
                                           uint32_t consumer_warps = kCWarps) {
  Ring r;
  r.full = reinterpret_cast<uint64_t*>(smem);
  r.empty = r.full + nstages;
  r.buf = smem + 1024;  // barriers live in the first 1 KiB
  r.stage_bytes = stage_bytes;
  r.nstages = nstages;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < nstages; ++s) {
      mbar_init(&r.full[s], 1);
      mbar_init(&r.empty[s], consumer_warps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  return r;
}

}  // namespace rlk
