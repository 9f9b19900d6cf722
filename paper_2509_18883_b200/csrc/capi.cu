// C-ABI plumbing: thread-local last error, device queries, and small utility kernels
// (finite check for ParamTable, toy_env.py:71-72; ascent_step add, objective.py:286-293).
#include "common.cuh"
#include "capi_internal.h"

namespace rlk {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return RLK_OK;
  set_error("%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
  return RLK_ERR_CUDA;
}

int launch_status(const char* where) { return cuda_status(cudaGetLastError(), where); }

int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

template <int DT>
__global__ void k_nonfinite(const void* __restrict__ x, uint64_t n, unsigned long long* count) {
  uint64_t local = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double v = load_f64<DT>(x, i);
    local += !isfinite(v);
  }
  unsigned int c = (unsigned int)local;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

template <int DT>
__global__ void k_scaled_add(const void* __restrict__ a, const void* __restrict__ b, double alpha,
                             void* __restrict__ out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    // objective.py:293: params.logits + lr * gradient (two f64 roundings, no FMA contraction)
    double v = __dadd_rn(load_f64<DT>(a, i), __dmul_rn(alpha, load_f64<DT>(b, i)));
    store_from_f64<DT>(out, i, v);
  }
}

}  // namespace rlk

using namespace rlk;

extern "C" {

const char* rlk_last_error(void) { return g_last_error; }

int rlk_abi_version(void) { return 2; }  // 2: rlk_fusion_merge takes exact_path

int rlk_device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}

int rlk_nonfinite_count(const void* x, int dtype, uint64_t n, unsigned long long* count, void* stream) {
  RLK_REQUIRE(count != nullptr, "rlk_nonfinite_count: count is NULL");
  if (n == 0) return RLK_OK;
  RLK_REQUIRE(x != nullptr, "rlk_nonfinite_count: x is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t blocks = (n + 255) / 256;
  int grid = (int)(blocks < (uint64_t)sm_count() * 8 ? blocks : (uint64_t)sm_count() * 8);
  switch (dtype) {
    case RLK_BF16: k_nonfinite<RLK_BF16><<<grid, 256, 0, s>>>(x, n, count); break;
    case RLK_F32: k_nonfinite<RLK_F32><<<grid, 256, 0, s>>>(x, n, count); break;
    case RLK_F64: k_nonfinite<RLK_F64><<<grid, 256, 0, s>>>(x, n, count); break;
    default: set_error("rlk_nonfinite_count: bad dtype %d", dtype); return RLK_ERR_INVALID;
  }
  return launch_status("rlk_nonfinite_count");
}

int rlk_scaled_add(const void* a, const void* b, double alpha, void* out, int dtype, uint64_t n,
                   void* stream) {
  if (n == 0) return RLK_OK;
  RLK_REQUIRE(a && b && out, "rlk_scaled_add: NULL pointer");
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t blocks = (n + 255) / 256;
  int grid = (int)(blocks < (uint64_t)sm_count() * 8 ? blocks : (uint64_t)sm_count() * 8);
  switch (dtype) {
    case RLK_BF16: k_scaled_add<RLK_BF16><<<grid, 256, 0, s>>>(a, b, alpha, out, n); break;
    case RLK_F32: k_scaled_add<RLK_F32><<<grid, 256, 0, s>>>(a, b, alpha, out, n); break;
    case RLK_F64: k_scaled_add<RLK_F64><<<grid, 256, 0, s>>>(a, b, alpha, out, n); break;
    default: set_error("rlk_scaled_add: bad dtype %d", dtype); return RLK_ERR_INVALID;
  }
  return launch_status("rlk_scaled_add");
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// Synthetic parameters for benchmarks / tests: out[i] = RN_dtype(base[i] + std * N(0,1)), where the
// normal deviate is a Box-Muller transform of mix64(seed ^ mix64(j0 + i)).  Counter-based, so a slice
// [j0, j0 + n) has the same values at any world size / piece split.
namespace rlk {
template <int DT, int BT>
__global__ void k_synth(void* __restrict__ out, uint64_t n, uint64_t j0, uint64_t seed, double stdv,
                        const void* __restrict__ base) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h = mix64(seed ^ mix64(j0 + i + 1));
    const float u1 = ((uint32_t)(h >> 40) + 0.5f) * (1.0f / 16777216.0f);
    const float u2 = (uint32_t)(h & 0xffffffu) * (1.0f / 16777216.0f);
    const float z = sqrtf(-2.0f * __logf(u1)) * __cosf(6.283185307f * u2);
    const double b = base ? load_f64<BT>(base, i) : 0.0;
    store_from_f64<DT>(out, i, b + stdv * (double)z);
  }
}
}  // namespace rlk

extern "C" int rlk_synth_normal(void* out, int dtype, uint64_t n, uint64_t j0, uint64_t seed, double stdv,
                                const void* base, void* stream) {
  if (n == 0) return RLK_OK;
  RLK_REQUIRE(out != nullptr, "rlk_synth_normal: out is NULL");
  RLK_REQUIRE(dtype >= 0 && dtype <= 2, "rlk_synth_normal: bad dtype %d", dtype);
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t blocks = (n + 255) / 256;
  const int grid = (int)(blocks < (uint64_t)sm_count() * 8 ? blocks : (uint64_t)sm_count() * 8);
  // base (if any) has the same dtype as out
  switch (dtype) {
    case RLK_BF16: k_synth<RLK_BF16, RLK_BF16><<<grid, 256, 0, s>>>(out, n, j0, seed, stdv, base); break;
    case RLK_F32: k_synth<RLK_F32, RLK_F32><<<grid, 256, 0, s>>>(out, n, j0, seed, stdv, base); break;
    default: k_synth<RLK_F64, RLK_F64><<<grid, 256, 0, s>>>(out, n, j0, seed, stdv, base); break;
  }
  return launch_status("rlk_synth_normal");
}

// ---------------------------------------------------------------------------------------------
// Checkpoint checksum (checkpoint.py): sum over 64-bit words w_i at global word index o + i of
// mix64(w_i ^ ((o + i + 1) * GAMMA)) mod 2^64.  Position-keyed (detects permutations) and a plain
// modular sum (so chunks can be checksummed independently and added, in any order).
namespace rlk {
__global__ void k_checksum64(const uint64_t* __restrict__ w, uint64_t n, uint64_t off, unsigned long long* out) {
  uint64_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    acc += mix64(w[i] ^ ((off + i + 1) * kGamma));
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}
}  // namespace rlk

extern "C" int rlk_checksum64(const void* data, uint64_t n_words, uint64_t word_offset, unsigned long long* out,
                              void* stream) {
  RLK_REQUIRE(out != nullptr, "rlk_checksum64: out is NULL");
  if (n_words == 0) return RLK_OK;
  RLK_REQUIRE(data != nullptr && ((uintptr_t)data & 7u) == 0, "rlk_checksum64: data must be 8-byte aligned");
  const uint64_t blocks = (n_words + 255) / 256;
  const int grid = (int)(blocks < (uint64_t)sm_count() * 8 ? blocks : (uint64_t)sm_count() * 8);
  k_checksum64<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint64_t*)data, n_words, word_offset, out);
  return launch_status("rlk_checksum64");
}
