// Shared device helpers for the rolloutlab B200 kernels (sm_100a only).
//
//  * SplitMix64 (bit-exact with rolloutlab core.py:42-49 `_mix64` and core.py:69-75 `next_u64`)
//  * bf16 / f32 / f64 element loads and stores, f64 -> bf16 round-to-nearest-even without double rounding
//  * mbarrier + cp.async.bulk (TMA bulk copy, SASS UBLKCP) ring-pipeline primitives
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/rlk.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "rolloutlab kernels are written for sm_100a only"
#endif

namespace rlk {

// ---------------------------------------------------------------- checked builds
// RLK_CHECKED (tools/build_variant.py checked -DRLK_CHECKED): device-side bounds / alignment asserts on
// every TMA copy and shared-memory index of the streaming kernels, and a poll limit on every mbarrier
// wait (a lost arrival traps instead of hanging the GPU).  This pool disables compute-sanitizer; the
// GPU test suite runs against this build instead (tests/test_gpu_checked.py).  Release builds: no-ops.
#ifdef RLK_CHECKED
#define RLK_DCHECK(cond)                                                                             \
  do {                                                                                               \
    if (!(cond)) {                                                                                   \
      printf("RLK_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,        \
             (int)blockIdx.x, (int)threadIdx.x);                                                     \
      __trap();                                                                                      \
    }                                                                                                \
  } while (0)
#else
#define RLK_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

// ---------------------------------------------------------------- SplitMix64 (core.py:26-33, 42-49)
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= kMix1;
  z ^= z >> 27;
  z *= kMix2;
  z ^= z >> 31;
  return z;
}

// Keep decision for draw j of a child stream: core.py:69-75 (counter += gamma; mix64) and
// fusion.py:113 (`rng.uniform() >= p`).  uniform = (u64 >> 11) * 2^-53, so `uniform >= p` is exactly
// `(u64 >> 11) >= ceil(p * 2^53)` = thresh (computed exactly on the host).
__device__ __forceinline__ bool keep_draw(uint64_t child_seed, uint64_t j, uint64_t thresh) {
  return (mix64(child_seed + (j + 1ull) * kGamma) >> 11) >= thresh;
}

// ---------------------------------------------------------------- element types
template <int DT> struct Elem;
template <> struct Elem<RLK_BF16> { using T = __nv_bfloat16; static constexpr int size = 2; };
template <> struct Elem<RLK_F32> { using T = float; static constexpr int size = 4; };
template <> struct Elem<RLK_F64> { using T = double; static constexpr int size = 8; };

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// Round a double to bf16 with a single rounding (round-to-nearest-even).  Round to odd at f32
// precision first (24 bits >= 8 + 2), after which the f32 -> bf16 RNE step is exact-equivalent.
__device__ __forceinline__ uint16_t f64_to_bf16_rne(double x) {
  float f = __double2float_rz(x);
  if ((double)f != x && !isnan(x) && !isinf(f)) {
    uint32_t u = __float_as_uint(f) | 1u;  // sticky bit (round-to-odd)
    f = __uint_as_float(u);
  }
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}
__device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}
// f64 -> f32 with a single rounding (hardware cvt.rn.f32.f64 is correctly rounded).
__device__ __forceinline__ float f64_to_f32_rn(double x) { return __double2float_rn(x); }

template <int DT> __device__ __forceinline__ double load_f64(const void* p, uint64_t i) {
  if constexpr (DT == RLK_BF16) {
    uint16_t u = reinterpret_cast<const uint16_t*>(p)[i];
    return (double)__uint_as_float(((uint32_t)u) << 16);
  } else if constexpr (DT == RLK_F32) {
    return (double)reinterpret_cast<const float*>(p)[i];
  } else {
    return reinterpret_cast<const double*>(p)[i];
  }
}
template <int DT> __device__ __forceinline__ void store_from_f64(void* p, uint64_t i, double v) {
  if constexpr (DT == RLK_BF16) {
    reinterpret_cast<uint16_t*>(p)[i] = f64_to_bf16_rne(v);
  } else if constexpr (DT == RLK_F32) {
    reinterpret_cast<float*>(p)[i] = f64_to_f32_rn(v);
  } else {
    reinterpret_cast<double*>(p)[i] = v;
  }
}

// ---------------------------------------------------------------- mbarrier / bulk-copy PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
#ifdef RLK_CHECKED
  for (uint64_t polls = 0;; ++polls) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    RLK_DCHECK(polls < (1ull << 26));  // each try_wait suspends up to a hardware time limit: ~seconds
  }
#endif
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 1-D TMA bulk copy global -> shared, completion signalled on `bar` (complete_tx::bytes).
// dst / src / bytes must be 16-byte aligned / multiples of 16.
__device__ __forceinline__ uint32_t total_smem_bytes() {
  uint32_t r;
  asm("mov.u32 %0, %%total_smem_size;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t dynamic_smem_bytes() {
  uint32_t r;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  RLK_DCHECK(bytes > 0 && bytes % 16 == 0 && ((uintptr_t)src & 15u) == 0 && (smem_u32(dst) & 15u) == 0);
  // the CTA's offset in its shared window (a cluster CTA's window carries its rank above bit 24), within
  // the CTA's allocation (+ the 1 KiB system reservation)
  RLK_DCHECK((smem_u32(dst) & 0x00ffffffu) + bytes <= total_smem_bytes() + 1024u);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ void stg128_stream(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace rlk
