// debug.cu -- opt-in device validation of jagged offsets (GESR_DEBUG=1; include/gesr.h,
// SURVEY.md s8(b)): offsets[0] == 0, nondecreasing, offsets[n] == total (total < 0: unknown, not checked).  A violation traps, so
// the caller's stream reports a launch failure instead of the kernels reading out of bounds.
#include <cstdio>

#include "kernels.h"

namespace gesr {
namespace {

__global__ void check_offsets_kernel(const int64_t* offsets, int64_t n, int64_t total, int tag) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= n;
       i += stride) {
    const int64_t v = offsets[i];
    bool bad = (i == 0 && v != 0) || v < 0 || (total >= 0 && ((i == n && v != total) || v > total));
    if (i > 0 && offsets[i - 1] > v) bad = true;
    if (bad) {
      printf("gesr debug: offsets array %d invalid at index %lld (value %lld, n %lld, total %lld)\n",
             tag, static_cast<long long>(i), static_cast<long long>(v), static_cast<long long>(n),
             static_cast<long long>(total));
      __trap();
    }
  }
}

}  // namespace

cudaError_t launch_check_offsets(const int64_t* offsets, int64_t n, int64_t total, int tag,
                                 cudaStream_t stream) {
  if (offsets == nullptr) return cudaSuccess;
  int64_t blocks = (n + 1 + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  check_offsets_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(offsets, n, total, tag);
  count_launch();
  return cudaGetLastError();
}

}  // namespace gesr
