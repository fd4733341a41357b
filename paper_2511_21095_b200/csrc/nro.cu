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

// RO cross attention queries: row b*i + s = seed s (+ the request's context
// token ctx[b][s]) in bf16, and the candidate offsets of the i query rows per request.
__global__ void ro_queries_kernel(const __nv_bfloat16* __restrict__ seeds,
                                  const __nv_bfloat16* __restrict__ ctx,
                                  __nv_bfloat16* __restrict__ X, int64_t* __restrict__ offs,
                                  int64_t B, int i, int D_in) {
  const int64_t n = B * i * D_in;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = e / D_in;
    const int k = static_cast<int>(e - row * D_in);
    const int s = static_cast<int>(row % i);
    float v = __bfloat162float(seeds[static_cast<int64_t>(s) * D_in + k]);
    if (ctx != nullptr) v += __bfloat162float(ctx[e]);
    X[e] = __float2bfloat16_rn(v);
  }
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b <= B;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x)
    offs[b] = b * i;
}

// U_cross[b][s*d + j] = O_full[b*i + s][s*d + j]: query row s of request b keeps slot s's output
__global__ void ro_gather_kernel(const float* __restrict__ O_full, void* __restrict__ out,
                                 int o_bf16, int64_t B, int i, int d) {
  const int64_t n = B * i * d;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = e / (static_cast<int64_t>(i) * d);
    const int sj = static_cast<int>(e - b * i * d);          // s * d + j
    const int s = sj / d;
    const float v = O_full[(b * i + s) * static_cast<int64_t>(i) * d + sj];
    if (o_bf16) static_cast<__nv_bfloat16*>(out)[e] = __float2bfloat16_rn(v);
    else static_cast<float*>(out)[e] = v;
  }
}

}  // namespace

cudaError_t launch_ro_queries(const void* seeds, const void* ctx, void* X, int64_t* offs,
                              int64_t B, int i, int D_in, cudaStream_t stream) {
  ro_queries_kernel<<<148 * 4, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(seeds),
                                                 static_cast<const __nv_bfloat16*>(ctx),
                                                 static_cast<__nv_bfloat16*>(X), offs, B, i, D_in);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_ro_gather(const float* O_full, void* out, int o_bf16, int64_t B, int i, int d,
                             cudaStream_t stream) {
  ro_gather_kernel<<<148 * 4, 256, 0, stream>>>(O_full, out, o_bf16, B, i, d);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_fold_gate(const void* W_q, const float* gate, void* out, int j, int d, int D_in,
                             cudaStream_t stream) {
  const int64_t pairs = static_cast<int64_t>(j) * d * D_in / 2;
  if (pairs == 0) return cudaSuccess;
  int64_t blocks = (pairs + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  fold_gate_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(W_q), gate, static_cast<__nv_bfloat16*>(out),
      static_cast<int64_t>(j) * d, D_in, d);
  count_launch();
  return cudaGetLastError();
}

}  // namespace gesr
