// TMA tile::gather4 probe (sm_100a): which tensor-map box and smem placement give four gathered
// 128-byte rows in the same 128B-swizzled layout a 128-row tile load produces?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2511_21095_b200/csrc \
//        scripts/micro/gather4_probe.cu -o /tmp/g4 -lcuda && /tmp/g4
//
// E [1024 rows, 64 cols] bf16 with E[r][c] = r * 64 + c (as a 16-bit pattern).  One thread
// issues 32 gather4 loads (rows idx[4i..4i+3]) into smem rows 4i..4i+3 of a 128 x 64 tile; the
// tile is compared, 16-byte chunk by chunk, with the 128B swizzle (chunk j of row r at chunk
// j ^ (r & 7)).  Prints, per box height tried, the number of mismatching chunks.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "ptx.cuh"

__global__ void probe(const __grid_constant__ CUtensorMap map, const int* idx, uint16_t* out,
                      int cta_group2) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    gesr::mbar_init(&bar, 1);
    gesr::fence_mbar_init();
    gesr::mbar_arrive_expect_tx(&bar, 128 * 128);
    for (int i = 0; i < 32; ++i) {
      const uint32_t dst = gesr::smem_u32(smem + i * 4 * 128);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(gesr::smem_u32(&bar)), "r"(0),
          "r"(idx[4 * i]), "r"(idx[4 * i + 1]), "r"(idx[4 * i + 2]), "r"(idx[4 * i + 3])
          : "memory");
    }
    gesr::mbar_wait(&bar, 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x)
    out[i] = reinterpret_cast<const uint16_t*>(smem)[i];
}

int main() {
  const int R = 1024, C = 64;
  std::vector<uint16_t> hE(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) hE[r * C + c] = static_cast<uint16_t>(r * 64 + c);
  std::vector<int> hidx(128);
  for (int i = 0; i < 128; ++i) hidx[i] = (i * 397 + 11) % R;
  void *dE, *dIdx, *dOut;
  cudaMalloc(&dE, R * C * 2);
  cudaMalloc(&dIdx, 128 * 4);
  cudaMalloc(&dOut, 128 * 64 * 2);
  cudaMemcpy(dE, hE.data(), R * C * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dIdx, hidx.data(), 128 * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  for (int boxh : {1, 4}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(R)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(C * 2)};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(boxh)};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dE, dims,
                                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                         CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
      printf("box height %d: encode failed (%d)\n", boxh, static_cast<int>(cr));
      continue;
    }
    cudaMemset(dOut, 0xff, 128 * 64 * 2);
    probe<<<1, 128, 32 * 1024>>>(map, static_cast<const int*>(dIdx),
                                  static_cast<uint16_t*>(dOut), 0);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("box height %d: kernel error %s\n", boxh, cudaGetErrorString(e));
      return 1;
    }
    std::vector<uint16_t> hout(128 * 64);
    cudaMemcpy(hout.data(), dOut, 128 * 64 * 2, cudaMemcpyDeviceToHost);
    int bad_swz = 0, bad_lin = 0;
    for (int r = 0; r < 128; ++r)
      for (int j = 0; j < 8; ++j) {
        const uint16_t* want = &hE[hidx[r] * C + j * 8];
        const uint16_t* got_swz = &hout[r * 64 + ((j ^ (r & 7)) * 8)];
        const uint16_t* got_lin = &hout[r * 64 + j * 8];
        if (memcmp(want, got_swz, 16) != 0) ++bad_swz;
        if (memcmp(want, got_lin, 16) != 0) ++bad_lin;
      }
    printf("box height %d: mismatching 16-byte chunks vs 128B swizzle %d / 1024, vs linear %d / 1024\n",
           boxh, bad_swz, bad_lin);
  }
  return 0;
}
