// Microbenchmark: per-SM throughput of cvt.rn.bf16x2.f32 (F2FP), MUFU.EX2, and their mix.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t cvt2(float a, float b) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }
template <int MODE>
__global__ void k(uint32_t* out, int iters, float a) {
  float v[16]; uint32_t acc = 0;
  for (int i = 0; i < 16; ++i) v[i] = a * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) { acc ^= cvt2(v[i], v[i + 1]); v[i] += 1.0f; }                 // F2FP only
      if (MODE == 1) { v[i] = ex2(v[i]); v[i + 1] = ex2(v[i + 1]); }                 // 2 EX2
      if (MODE == 2) { v[i] = ex2(v[i]); v[i + 1] = ex2(v[i + 1]); acc ^= cvt2(v[i], v[i + 1]); }  // 2 EX2 + 1 F2FP
    }
  }
  uint32_t s = acc; for (int i = 0; i < 16; ++i) s += __float_as_uint(v[i]);
  if (s == 12345u) out[threadIdx.x] = s;
}
int main() {
  uint32_t* d; cudaMalloc(&d, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[3] = {"f2fp(pairs)", "ex2", "ex2x2+f2fp"};
  const double per_iter[3] = {8, 16, 16};    // counted ops per thread-iteration (pairs / exps)
  for (int mode = 0; mode < 3; ++mode) {
    int threads = 512, iters = 2048;
    auto launch = [&] {
      if (mode == 0) k<0><<<sms * 2, threads>>>(d, iters, 1e-3f);
      if (mode == 1) k<1><<<sms * 2, threads>>>(d, iters, 1e-3f);
      if (mode == 2) k<2><<<sms * 2, threads>>>(d, iters, 1e-3f);
    };
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = double(sms) * 2 * threads * iters * per_iter[mode];
    printf("%-12s %.3f ms  %.2f ops/clk/SM (max clock %d MHz)\n", names[mode], ms, ops / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000);
  }
  return 0;
}
