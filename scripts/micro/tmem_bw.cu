// Microbenchmark: tcgen05.ld (32x32b.x32) / tcgen05.st throughput per SM vs resident warps.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tmem_bw tmem_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"

__device__ __forceinline__ void ld32(uint32_t a, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(a));
}
__device__ __forceinline__ void st32(uint32_t a, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

template <int MODE>
__global__ void k(uint32_t* out, unsigned long long* clk, int iters);

// tcgen05.ld (x16, like the attention epilogue) latency + throughput from warps 4.., with and
// without a concurrent MMA stream (SS M=128 N=128 K=16 into columns 256..383) from warp 0.
template <int WITH_MMA>
__global__ void k_mma(unsigned long long* clk, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32;
  if (warp == 0) { gesr::tmem_alloc(&slot, 512); gesr::tmem_relinquish(); }
  if (threadIdx.x == 0) { gesr::mbar_init(&bar, 1); gesr::fence_mbar_init(); stop = 0; }
  gesr::tc_fence_before();
  __syncthreads();
  gesr::tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    if (WITH_MMA && threadIdx.x == 0) {
      const uint32_t sa = gesr::smem_u32(smem), sb = gesr::smem_u32(smem + 32768);
      const uint32_t idesc = gesr::make_idesc_bf16(128, 128, 0, 0);
      int n = 0;
      while (!stop && n < 200000) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          gesr::mma_ss(tmem + 256, gesr::make_sdesc(sa + (ks / 4) * 16384 + (ks % 4) * 32, 16, 1024, 2),
                       gesr::make_sdesc(sb + (ks / 4) * 16384 + (ks % 4) * 32, 16, 1024, 2), idesc, 1u);
        ++n;
        if ((n & 15) == 0) { gesr::mma_commit(&bar); gesr::mbar_wait(&bar, ((n >> 4) - 1) & 1); }
      }
    }
  } else if (warp >= 4) {
    const uint32_t taddr = tmem + (((warp & 3) * 32) << 16) + ((warp / 4) - 1) * 64;
    uint32_t a[16], b[16], acc = 0;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      gesr::tmem_ld16(taddr + (it & 1) * 16, a);
      gesr::tmem_ld16(taddr + 32 + (it & 1) * 16, b);
      gesr::tmem_ld_wait();
      acc += a[0] ^ b[15] ^ a[7];
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 128) clk[blockIdx.x] = t1 - t0;
    if (acc == 0x1234567u) clk[1000] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) stop = 1;
  gesr::tc_fence_before();
  __syncthreads();
  if (warp == 0) { gesr::tc_fence_after(); gesr::tmem_dealloc(tmem, 512); }
}

template <int MODE>
__global__ void k(uint32_t* out, unsigned long long* clk, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        static_cast<uint32_t>(__cvta_generic_to_shared(&slot))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot + (((warp & 3) * 32) << 16) + (warp / 4) * 128 % 512;
  uint32_t r[32], acc = 0;
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * i;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {   // 4 loads (128 columns) then one wait
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        ld32(t + c * 32, r);
        asm volatile("" ::: "memory");
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= r[it & 31];
    } else {           // 2 stores (64 columns) then one wait
      st32(t, r);
      st32(t + 32, r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      r[it & 31] += 1;
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  if (acc == 0x12345u) out[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
  uint32_t* d;
  unsigned long long* c;
  cudaMalloc(&d, 4096);
  cudaMalloc(&c, 148 * 8);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode) {
    for (int warps : {4, 8, 16}) {
      auto launch = [&] {
        if (mode == 0) k<0><<<148, warps * 32>>>(d, c, iters);
        else k<1><<<148, warps * 32>>>(d, c, iters);
      };
      launch();
      cudaDeviceSynchronize();
      launch();
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
      double bytes = double(warps) * 32 * iters * (mode == 0 ? 128 : 64) * 4;
      printf("%s warps=%2d  %.1f B/clk/SM  (%s)\n", mode == 0 ? "tcgen05.ld" : "tcgen05.st", warps,
             bytes / double(h[0]), cudaGetErrorString(e));
    }
  }
  unsigned long long* c2;
  cudaMalloc(&c2, 2048 * 8);
  for (int mma = 0; mma < 2; ++mma) {
    for (int warps : {1, 4}) {
      const int iters = 2000;
      const int threads = (4 + warps) * 32;
      if (mma) { cudaFuncSetAttribute(k_mma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024); k_mma<1><<<148, threads, 80 * 1024>>>(c2, iters); }
      else { cudaFuncSetAttribute(k_mma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024); k_mma<0><<<148, threads, 80 * 1024>>>(c2, iters); }
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h;
      cudaMemcpy(&h, c2, 8, cudaMemcpyDeviceToHost);
      printf("2 x tcgen05.ld x16 + wait, %d loader warp(s)%s: %.0f clk per iteration (%s)\n", warps,
             mma ? ", MMA stream running" : "", double(h) / iters, cudaGetErrorString(e));
    }
  }
  return 0;
}
