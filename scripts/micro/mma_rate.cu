// Microbenchmark: tcgen05.mma kind::f16 (bf16 -> fp32) issue rate per SM for the attention
// shapes: SS (A, B in smem, K-major SW128) and TS (A in TMEM) with M = 128 and N = 64/128/256.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_2511_21095_b200/csrc -o mma_rate mma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace gesr;

template <int N, int TS>
__global__ void k(unsigned long long* clk, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (warp == 0) { tmem_alloc(&slot, 512); tmem_relinquish(); }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    const uint32_t idesc = make_idesc_bf16(128, N, 0, 0);
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint64_t bd = make_sdesc(sb + (ks / 4) * (N * 128) + (ks % 4) * 32, 16, 1024, 2);
        if (TS) {
          mma_ts(tmem + 256, tmem + ks * 8, bd, idesc, 1u);
        } else {
          const uint64_t ad = make_sdesc(sa + (ks / 4) * 16384 + (ks % 4) * 32, 16, 1024, 2);
          mma_ss(tmem + 256, ad, bd, idesc, 1u);
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    clk[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// same MMA stream (SS, N, K=16 steps) while warps 4..7 write 16-byte st.shared at full rate
template <int N>
__global__ void k_sts(unsigned long long* clk, int reps, int sts_iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) { tmem_alloc(&slot, 512); tmem_relinquish(); }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    const uint32_t idesc = make_idesc_bf16(128, N, 0, 0);
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint64_t bd = make_sdesc(sb + (ks / 4) * (N * 128) + (ks % 4) * 32, 16, 1024, 2);
        const uint64_t ad = make_sdesc(sa + (ks / 4) * 16384 + (ks % 4) * 32, 16, 1024, 2);
        mma_ss(tmem + 256, ad, bd, idesc, 1u);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    clk[blockIdx.x] = t1 - t0;
  } else if (warp >= 4) {
    const uint32_t dst = smem_u32(smem + 98304) + (threadIdx.x - 128) * 16;
    const unsigned long long t0 = clock64();
    uint32_t v0 = threadIdx.x;
    for (int i = 0; i < sts_iters; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(dst + ((u & 1) * 2048)), "r"(v0) : "memory");
        v0 += 1;
      }
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 128) clk[gridDim.x + blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N>
void run_sts(unsigned long long* c, int sts_iters) {
  const int reps = 2000;
  cudaFuncSetAttribute(k_sts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  k_sts<N><<<148, 256, 120 * 1024>>>(c, reps, sts_iters);
  k_sts<N><<<148, 256, 120 * 1024>>>(c, reps, sts_iters);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[296];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const double per = double(h[0]) / (reps * 8.0);
  const double sts_bpc = sts_iters ? 128.0 * 8 * 16 * sts_iters / double(h[148]) : 0.0;
  printf("SS N=%3d + STS(iters %6d): MMA %.1f clk/instr; STS %.1f B/clk over %llu clk (MMA span %llu) (%s)\n",
         N, sts_iters, per, sts_bpc, h[148], h[0], cudaGetErrorString(e));
}

template <int N, int TS>
void run(unsigned long long* c) {
  const int reps = 2000;
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<N, TS><<<148, 128, 100 * 1024>>>(c, reps);
  k<N, TS><<<148, 128, 100 * 1024>>>(c, reps);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double per = double(h) / (reps * 8.0);
  const double flop_clk = 2.0 * 128 * N * 16 / per;
  printf("%s M=128 N=%3d K=16: %.1f clk/instr  %.0f flop/clk/SM  (%s)\n", TS ? "TS" : "SS", N, per,
         flop_clk, cudaGetErrorString(e));
}

int main() {
  unsigned long long* c;
  cudaMalloc(&c, 296 * 8);
  run<64, 0>(c);
  run<128, 0>(c);
  run<256, 0>(c);
  run<64, 1>(c);
  run<128, 1>(c);
  run<256, 1>(c);
  for (int it : {0, 1000, 4000, 16000}) run_sts<128>(c, it);
  for (int it : {0, 1000, 4000, 16000}) run_sts<64>(c, it);
  return 0;
}
