// Pipe-throughput microbenchmarks for design decisions (not product code).
// Measures per-SM throughput of: F2F.F64.F32, DFMA, MUFU.EX2, 64-bit mul (SplitMix64 draw), FFMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
__global__ void k_f2f(float* out, float seed) {
  float a = seed + threadIdx.x; double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  float b = a * 1.5f, c = a * 0.5f, d = a + 3.f;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    acc0 += (double)a; acc1 += (double)b; acc2 += (double)c; acc3 += (double)d;
    a += 1.0f; b += 1.0f; c += 1.0f; d += 1.0f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(acc0 + acc1 + acc2 + acc3);
}
__global__ void k_dfma(double* out, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const double m = 0.999999, c = 1e-7;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_ex2(float* out, float seed) {
  float a0 = seed * threadIdx.x * 1e-6f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    s0 += exp2f(a0); s1 += exp2f(a1); s2 += exp2f(a2); s3 += exp2f(a3);
    a0 -= 1e-7f; a1 -= 1e-7f; a2 -= 1e-7f; a3 -= 1e-7f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; z ^= z >> 31; return z;
}
__global__ void k_mix(uint64_t* out, uint64_t seed) {
  uint64_t c = seed + threadIdx.x; uint32_t cnt = 0;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    c += 0x9E3779B97F4A7C15ull;
    cnt += (mix64(c) >> 11) >= 4503599627370496ull;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = cnt;
}
__global__ void k_ffma(float* out, float seed) {
  float a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const float m = 0.999999f, c = 1e-7f;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
    a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_copy(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
__global__ void k_read(const int4* __restrict__ a, int* out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  int x = 0;
  for (; i < n; i += st) { int4 v = a[i]; x ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (x == 0x12345678) out[0] = x;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock(kHz) %d\n", sms, clk);
  void* buf; cudaMalloc(&buf, 64 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  double nthr = (double)blocks * threads;
  auto report = [&](const char* name, double ops_per_iter_thread, auto launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double ops = nthr * ITERS * ops_per_iter_thread;
    printf("%-10s %8.3f ms  %8.2f Gop/s  %7.1f op/clk/SM (at %d MHz nominal)\n", name, ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  };
  report("f2f.f64", 4, [&] { k_f2f<<<blocks, threads>>>((float*)buf, 1.f); });
  report("dfma", 8, [&] { k_dfma<<<blocks, threads>>>((double*)buf, 1.0); });
  report("ex2", 4, [&] { k_ex2<<<blocks, threads>>>((float*)buf, 1.f); });
  report("mix64", 1, [&] { k_mix<<<blocks, threads>>>((uint64_t*)buf, 1); });
  report("ffma", 8, [&] { k_ffma<<<blocks, threads>>>((float*)buf, 1.f); });
  size_t bytes = (size_t)8 << 30; void *a, *b;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMemset(a, 1, bytes);
  size_t n = bytes / 16;
  for (int bl : {sms * 4, sms * 8, sms * 16}) {
    k_copy<<<bl, 512>>>((int4*)a, (int4*)b, n); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k_copy<<<bl, 512>>>((int4*)a, (int4*)b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("copy grid %d: %.1f GB/s\n", bl, 2.0 * bytes / ms / 1e6);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k_read<<<bl, 512>>>((int4*)a, (int*)buf, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("read grid %d: %.1f GB/s\n", bl, 1.0 * bytes / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
