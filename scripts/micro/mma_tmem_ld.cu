// Microbenchmark: does an epilogue's TMEM traffic slow a tcgen05.mma stream?  One CTA per SM:
// thread 0 issues SS M=128 N=256 K=16 MMAs into TMEM columns [0, 256) back to back while W
// "epilogue" warps loop tcgen05.ld 32x32b.x32 (+ wait) over columns [256, 512) (their lane
// quarter).  Reports MMA cycles per instruction for W = 0, 4, 8, 16.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_2511_21095_b200/csrc -o mma_tmem_ld mma_tmem_ld.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace gesr;

__global__ void __launch_bounds__(640, 1) k(unsigned long long* clk, unsigned long long* ldcnt, int reps, int nld) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (warp == 0) { tmem_alloc(&slot, 512); tmem_relinquish(); }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); done = 0; }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 16384);
    const uint32_t idesc = make_idesc_bf16(128, 256, 0, 0);
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t ad = make_sdesc(sa + ks * 32, 16, 1024, 2);
        const uint64_t bd = make_sdesc(sb + ks * 32, 16, 1024, 2);
        mma_ss(tmem, ad, bd, idesc, 1u);
      }
      if ((r & 63) == 63) { mma_commit(&bar); mbar_wait(&bar, (r >> 6) & 1); }
    }
    mma_commit(&bar);
    mbar_wait(&bar, (reps >> 6) & 1);
    const unsigned long long t1 = clock64();
    clk[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (warp >= 4 && warp < 4 + nld) {
    const uint32_t sub = warp & 3;
    unsigned long long n = 0;
    uint32_t acc = 0;
    while (!done) {
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + ((sub * 32) << 16) + 256 + c * 32, r);
        tmem_ld_wait();
        acc += r[0] ^ r[31];
        ++n;
      }
    }
    if ((threadIdx.x & 31) == 0) atomicAdd(ldcnt, n + (acc == 12345 ? 1 : 0));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long *clk, *ldc;
  cudaMalloc(&clk, 148 * 8);
  cudaMalloc(&ldc, 8);
  const int smem = 64 * 1024 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 20000;
  for (int nld : {0, 4, 8, 16}) {
    cudaMemset(ldc, 0, 8);
    k<<<148, 640, smem>>>(clk, ldc, reps, nld);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148], L = 0;
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    cudaMemcpy(&L, ldc, 8, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += h[i];
    mean /= 148;
    printf("MMA M=128 N=256 K=16 with %2d TMEM-loader warps: %.1f clk/MMA, %.1f B/clk/SM loaded (%s)\n",
           nld, mean / (reps * 4.0), L * 32.0 * 32 * 4 / 148 / mean, cudaGetErrorString(e));
  }
  return 0;
}
