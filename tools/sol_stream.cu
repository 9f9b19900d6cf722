// Speed-of-light for the fusion kernels' HBM access patterns (not product code):
//   r4   : read 4 streams, reduce (K1's pattern: base + 3 experts)
//   r4w1 : read 4 streams, write 1 (K3's pattern)
//   r1w1 : copy
// Plain 16-byte vector loads, grid-stride, several loads in flight per thread.
// Usage: sol_stream [n_elems_per_stream (bf16), default 8.03e9]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stcs(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}

template <int U>
__global__ void __launch_bounds__(512) k_r4w1(const uint4* a, const uint4* b, const uint4* c, const uint4* d, uint4* o, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 va[U], vb[U], vc[U], vd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < n) { va[u] = ldnc(a + j); vb[u] = ldnc(b + j); vc[u] = ldnc(c + j); vd[u] = ldnc(d + j); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < n) stcs(o + j, make_uint4(va[u].x ^ vb[u].x ^ vc[u].x ^ vd[u].x, va[u].y ^ vb[u].y ^ vc[u].y ^ vd[u].y,
                                         va[u].z ^ vb[u].z ^ vc[u].z ^ vd[u].z, va[u].w ^ vb[u].w ^ vc[u].w ^ vd[u].w));
    }
  }
}

template <int U>
__global__ void __launch_bounds__(512) k_r4(const uint4* a, const uint4* b, const uint4* c, const uint4* d, unsigned* o, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  unsigned acc = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 va[U], vb[U], vc[U], vd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < n) { va[u] = ldnc(a + j); vb[u] = ldnc(b + j); vc[u] = ldnc(c + j); vd[u] = ldnc(d + j); }
      else { va[u] = vb[u] = vc[u] = vd[u] = make_uint4(0, 0, 0, 0); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += va[u].x ^ vb[u].y ^ vc[u].z ^ vd[u].w ^ va[u].w ^ vd[u].x;
  }
  if (acc == 0x12345678u) o[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(512) k_r1w1(const uint4* a, uint4* o, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 va[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t j = i + (size_t)u * blockDim.x; if (j < n) va[u] = ldnc(a + j); }
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t j = i + (size_t)u * blockDim.x; if (j < n) stcs(o + j, va[u]); }
  }
}

int main(int argc, char** argv) {
  size_t n_el = argc > 1 ? strtoull(argv[1], 0, 10) : 8030261248ull;
  size_t n = n_el / 8;  // uint4 per stream
  uint4 *a, *b, *c, *d, *o;
  unsigned* sink;
  CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16)); CK(cudaMalloc(&c, n * 16)); CK(cudaMalloc(&d, n * 16));
  CK(cudaMalloc(&o, n * 16)); CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(a, 1, n * 16)); CK(cudaMemset(b, 2, n * 16)); CK(cudaMemset(c, 3, n * 16)); CK(cudaMemset(d, 4, n * 16));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto time = [&](const char* name, double bytes, auto launch) {
    for (int w = 0; w < 2; ++w) launch();
    CK(cudaEventRecord(e0));
    const int R = 5;
    for (int r = 0; r < R; ++r) launch();
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= R;
    printf("%-22s %8.3f ms  %7.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  for (int bpsm : {1, 2, 4}) {
    for (int thr : {256, 512}) {
      char nm[64];
      int grid = sms * bpsm * (512 / thr);
      snprintf(nm, 64, "r4w1 U2 g%d t%d", grid, thr);
      time(nm, n * 16.0 * 5, [&] { k_r4w1<2><<<grid, thr>>>(a, b, c, d, o, n); });
      snprintf(nm, 64, "r4w1 U4 g%d t%d", grid, thr);
      time(nm, n * 16.0 * 5, [&] { k_r4w1<4><<<grid, thr>>>(a, b, c, d, o, n); });
      snprintf(nm, 64, "r4 U2 g%d t%d", grid, thr);
      time(nm, n * 16.0 * 4, [&] { k_r4<2><<<grid, thr>>>(a, b, c, d, sink, n); });
      snprintf(nm, 64, "r4 U4 g%d t%d", grid, thr);
      time(nm, n * 16.0 * 4, [&] { k_r4<4><<<grid, thr>>>(a, b, c, d, sink, n); });
      snprintf(nm, 64, "r1w1 U4 g%d t%d", grid, thr);
      time(nm, n * 16.0 * 2, [&] { k_r1w1<4><<<grid, thr>>>(a, o, n); });
    }
  }
  CK(cudaGetLastError());
  return 0;
}
