// nro.cu -- NRO cross attention's query gate (PAPER.md:373-380 s3.4.3; SPEC.md
// 316-324; reading R16).
//
// Slot s of the j query slots attends over the user's RO rows with its own key/value
// projections (the slots are heads of gesr_kv_project / gesr_tasa_score) and a learned
// elementwise gate g_s on the candidate query input:  q_s = act((x (.) g_s) W_{Q,s}^T + b_s).
// Because (x (.) g) W^T = x (W diag(g))^T, the gate folds into the query weight once per call:
//   W'[s*d + i][k] = W_q[s*d + i][k] * g[s][k]   (rounded to bf16, RNE),
// and the slots then run on the target-aware attention path unchanged (q projection, attention
// over the cached K/V of the request's history).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace gesr {

namespace {

__global__ void fold_gate_kernel(const __nv_bfloat16* __restrict__ W, const float* __restrict__ g,
                                 __nv_bfloat16* __restrict__ out, int64_t n_rows, int D_in, int d) {
  const int64_t pairs = n_rows * D_in / 2;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < pairs;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = 2 * i;
    const int64_t row = e / D_in;
    const int k = static_cast<int>(e - row * D_in);   // even: D_in is a multiple of 8
    const float* gs = g + (row / d) * D_in + k;
    const __nv_bfloat162 w = reinterpret_cast<const __nv_bfloat162*>(W)[i];
    const float2 wf = __bfloat1622float2(w);
    reinterpret_cast<__nv_bfloat162*>(out)[i] = __floats2bfloat162_rn(wf.x * gs[0], wf.y * gs[1]);
  }
}

}  // namespace

cudaError_t launch_fold_gate(const void* W_q, const float* gate, void* out, int j, int d, int D_in,
                             cudaStream_t stream) {
  const int64_t pairs = static_cast<int64_t>(j) * d * D_in / 2;
  if (pairs == 0) return cudaSuccess;
  int64_t blocks = (pairs + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  fold_gate_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(W_q), gate, static_cast<__nv_bfloat16*>(out),
      static_cast<int64_t>(j) * d, D_in, d);
  return cudaGetLastError();
}

}  // namespace gesr
