// Microbenchmark: two warps per sub-partition alternate exp passes under a named-barrier token
// (the pair attention kernel's softmax schedule) with the softmax's other per-tile work (TMEM
// load of S, x = s*c - m) in between, no MMA / TMA / epilogue.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_2511_21095_b200/csrc -o exp_token exp_token.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace gesr;

__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1,
                                      float c0, float c1) {
  asm("{\n .reg .b64 a, b, c, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n"
      " mov.b64 c, {%6, %7};\n fma.rn.f32x2 d, a, b, c;\n mov.b64 {%0, %1}, d;\n}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void fadd2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n .reg .b64 a, b, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n"
      " add.rn.f32x2 d, a, b;\n mov.b64 {%0, %1}, d;\n}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

template <int WORK>
__global__ void __launch_bounds__(288, 1) k(long long* clk, int iters, float sl2) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) { tmem_alloc(&slot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 8) {
    // WORK >= 2: a tcgen05 MMA stream (SS M=128 N=128 K=16, operands in smem at 96 KB+) for the
    // duration, as the attention kernel's tensor pipe runs beside its softmax
    if (WORK >= 2 && lane == 0) {
      const uint32_t sa = smem_u32(smem + 98304), sb = smem_u32(smem + 98304 + 32768);
      const uint32_t idesc = make_idesc_bf16(128, 128, 0, 0);
      __shared__ __align__(8) uint64_t mb;
      mbar_init(&mb, 1);
      fence_mbar_init();
      for (int rep = 0; rep < iters * 4; ++rep) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          mma_ss(tmem + 384, make_sdesc(sa + (ks / 4) * 16384 + (ks % 4) * 32, 16, 1024, 2),
                 make_sdesc(sb + (ks / 4) * 16384 + (ks % 4) * 32, 16, 1024, 2), idesc, 1u);
        mma_commit(&mb);
        mbar_wait(&mb, rep & 1);
      }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
    return;
  }
  const int g = warp / 4, sub = warp & 3;
  const uint32_t tS = tmem + ((sub * 32) << 16) + g * 128;
  const uint32_t prow = smem_u32(smem) + g * 32768 + (sub * 32 + lane) * 128;
  const uint32_t tok_mine = (g == 0 ? 1u : 5u) + sub, tok_other = (g == 0 ? 5u : 1u) + sub;
  uint32_t r[128];
  float m = 0.25f, l = 0.f;
  long long texp = 0;
  for (int it = 0; it < iters; ++it) {
    const int j = 2 * it + g;
    if (WORK) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, r + c * 32);
      tmem_ld_wait();
#pragma unroll
      for (int kk = 0; kk < 64; ++kk) {
        float x0, x1;
        ffma2(x0, x1, __uint_as_float(r[2 * kk]) * 1e-30f, __uint_as_float(r[2 * kk + 1]) * 1e-30f, sl2, sl2, -m, -m);
        r[2 * kk] = __float_as_uint(x0);
        r[2 * kk + 1] = __float_as_uint(x1);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < 128; ++kk) r[kk] = __float_as_uint(-0.01f * (kk + lane));
    }
    if (j > 0) named_bar_sync(tok_mine, 64);
    const long long t0 = clock64();
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      uint32_t pw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = q * 4 + u;
        const float p0 = ex2(__uint_as_float(r[2 * kk])), p1 = ex2(__uint_as_float(r[2 * kk + 1]));
        const int a = (kk & 3) * 2;
        fadd2(acc[a], acc[a + 1], acc[a], acc[a + 1], p0, p1);
        pw[u] = pack_bf16x2(p0, p1);
      }
      st_shared_v4(prow + (q >> 3) * 16384 + (((q & 7) ^ (lane & 7)) << 4), pw[0], pw[1], pw[2], pw[3]);
    }
    const float tsum = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    const bool over = !(tsum <= 4096.f);
    if (__any_sync(0xffffffffu, over)) l += 1.f;
    const long long t1 = clock64();
    texp += t1 - t0;
    if (it + 1 < iters || g == 0) named_bar_arrive(tok_other, 64);
    l += tsum;
    fence_proxy_async_smem();
    __syncwarp();
  }
  if (threadIdx.x == 0) clk[blockIdx.x * 2] = texp / iters;
  if (threadIdx.x == 0 && l == 1.2345f) clk[1] = 1;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* c;
  cudaMalloc(&c, 4096 * 8);
  for (int work = 0; work < 3; ++work) {
    const int iters = 300;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    auto launch = [&] {
      if (work == 2) k<2><<<148, 288, 200000>>>(c, iters, 0.1f);
      else if (work) k<1><<<148, 288, 200000>>>(c, iters, 0.1f); else k<0><<<148, 288, 200000>>>(c, iters, 0.1f);
    };
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    int clkr;
    cudaDeviceGetAttribute(&clkr, cudaDevAttrClockRate, 0);
    printf("token-alternating exp passes, %s: exp window %lld clk; period per tile %.0f clk (at max clock) (%s)\n",
           work == 2 ? "S load + x pass + MMA stream" : work ? "with S load + x pass between" : "no other work", h,
           ms * 1e-3 * clkr * 1e3 / (2.0 * iters), cudaGetErrorString(e));
  }
  return 0;
}
