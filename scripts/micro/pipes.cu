// Microbenchmark: per-SM throughput of MUFU.EX2, FFMA, FFMA2 and the polynomial exp2 on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int MODE>
__global__ void k(float* out, int iters, float a) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = a * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) v[i] = ex2(v[i]) * -0.5f;            // MUFU + FMUL
      if (MODE == 1) v[i] = fmaf(v[i], 0.999f, 0.001f);    // FFMA
      if (MODE == 2) { asm volatile("{.reg .b64 t; mov.b64 t, {%0,%1}; fma.rn.f32x2 t, t, t, t; mov.b64 {%0,%1}, t;}" : "+f"(v[i]), "+f"(v[(i+1)&7])); }
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
int main() {
  float* d; cudaMalloc(&d, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[3] = {"ex2+fmul", "ffma", "ffma2(pair)"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int threads : {128, 256, 512, 1024}) {
      int iters = 4096;
      auto launch = [&] {
        if (mode == 0) k<0><<<sms * 2, threads>>>(d, iters, 1e-3f);
        if (mode == 1) k<1><<<sms * 2, threads>>>(d, iters, 1e-3f);
        if (mode == 2) k<2><<<sms * 2, threads>>>(d, iters, 1e-3f);
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = double(sms) * 2 * threads * iters * 8;   // per-element ops (pairs count once)
      double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
      printf("%-12s threads/CTA=%4d  %.2f ms  %.1f ops/clk/SM (at max clock %d MHz)\n", names[mode], threads, ms, per_clk_sm, clk / 1000);
    }
  }
  return 0;
}
