// stu.cu -- K-STU: normalisation and gating of the attention output.
//
// The STU layer's candidate row after the attention (the paper defers STU
// internals to HSTU; reading R15):
//   Z[t] = (LayerNorm(O[t]) * gamma + beta) (.) G[t],   LayerNorm over the D = H*d features of
//   the concatenated heads (population variance, eps inside the square root).
// G (the gating branch SiLU(T W_g^T + b_g)) and the output projection Z W_o^T + b_o + residual
// run on the K-PROJ GEMM (proj.cu); this kernel is the HBM-bound step between them.
//
// B200 design: one warp per row, 16-byte vector loads (8 bf16 / 2x4 fp32 per chunk, chunk q of
// a row at lane q mod 32: every warp instruction reads 512 contiguous bytes), two-pass mean and
// variance in fp32 from the row held in registers (D <= 1024) or re-read through L1 (larger D),
// the gate chunks loaded together with O (one DRAM round trip per row), Z written in place over
// G as bf16 (RNE).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace gesr {

namespace {

constexpr int kWarpsPerCta = 8;

__device__ __forceinline__ void load8(const void* O, int o_bf16, int64_t idx, float* x) {
  if (o_bf16) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(O) + idx));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      x[2 * e] = __uint_as_float(w[e] << 16);
      x[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
    }
  } else {
    const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(O) + idx);
    const float4 a = __ldg(src), b = __ldg(src + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// z = (x - mean) * rstd * gamma + beta, times the gate gu (8 bf16, loaded by the caller);
// 8 features at column c, written over the gate
__device__ __forceinline__ void emit8(const float* x, float mean, float rstd, const float* gamma,
                                      const float* beta, __nv_bfloat16* G, int64_t gidx, int c,
                                      const uint4 gu) {
  uint4* gp = reinterpret_cast<uint4*>(G + gidx);
  const uint32_t gw[4] = {gu.x, gu.y, gu.z, gu.w};
  const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + c));
  const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + c) + 1);
  const float4 b0 = __ldg(reinterpret_cast<const float4*>(beta + c));
  const float4 b1 = __ldg(reinterpret_cast<const float4*>(beta + c) + 1);
  const float ga[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
  const float be[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
  uint32_t out[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float gate0 = __uint_as_float(gw[e] << 16);
    const float gate1 = __uint_as_float(gw[e] & 0xFFFF0000u);
    const float z0 = ((x[2 * e] - mean) * rstd * ga[2 * e] + be[2 * e]) * gate0;
    const float z1 = ((x[2 * e + 1] - mean) * rstd * ga[2 * e + 1] + be[2 * e + 1]) * gate1;
    const __nv_bfloat162 h = __floats2bfloat162_rn(z0, z1);
    out[e] = *reinterpret_cast<const uint32_t*>(&h);
  }
  *gp = make_uint4(out[0], out[1], out[2], out[3]);
}

// kRegChunks: 8-feature chunks per lane held in registers (rows with D <= 256 kRegChunks);
// longer rows take the three-pass path
template <int kRegChunks>
__global__ void __launch_bounds__(kWarpsPerCta * 32, kRegChunks <= 2 ? 5 : 3)
    ln_gate_kernel(const void* __restrict__ O, int o_bf16, __nv_bfloat16* __restrict__ G,
                   const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
                   int64_t C, int D) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kWarpsPerCta + (threadIdx.x >> 5);
  if (row >= C) return;
  const int nch = D >> 3;                   // 8-feature chunks per row
  const int64_t base = row * D;
  const float inv_d = 1.0f / static_cast<float>(D);
  if (nch <= 32 * kRegChunks) {
    float x[kRegChunks][8];
    uint4 gq[kRegChunks];
    float s = 0.f;
    // the row's gate chunks are loaded together with O, so the row costs one DRAM round trip
#pragma unroll
    for (int k = 0; k < kRegChunks; ++k) {
      const int q = lane + 32 * k;
      if (q < nch) {
        load8(O, o_bf16, base + 8 * q, x[k]);
        gq[k] = *reinterpret_cast<const uint4*>(G + base + 8 * q);
      }
    }
#pragma unroll
    for (int k = 0; k < kRegChunks; ++k) {
      const int q = lane + 32 * k;
      if (q < nch) {
#pragma unroll
        for (int e = 0; e < 8; ++e) s += x[k][e];
      }
    }
    const float mean = warp_sum(s) * inv_d;
    float v = 0.f;
#pragma unroll
    for (int k = 0; k < kRegChunks; ++k) {
      const int q = lane + 32 * k;
      if (q < nch) {
#pragma unroll
        for (int e = 0; e < 8; ++e) { const float t = x[k][e] - mean; v += t * t; }
      }
    }
    const float rstd = rsqrtf(warp_sum(v) * inv_d + eps);
#pragma unroll
    for (int k = 0; k < kRegChunks; ++k) {
      const int q = lane + 32 * k;
      if (q < nch) emit8(x[k], mean, rstd, gamma, beta, G, base + 8 * q, 8 * q, gq[k]);
    }
    return;
  }
  // long rows: three passes, the re-reads hit L1
  float s = 0.f, x[8];
  for (int q = lane; q < nch; q += 32) {
    load8(O, o_bf16, base + 8 * q, x);
#pragma unroll
    for (int e = 0; e < 8; ++e) s += x[e];
  }
  const float mean = warp_sum(s) * inv_d;
  float v = 0.f;
  for (int q = lane; q < nch; q += 32) {
    load8(O, o_bf16, base + 8 * q, x);
#pragma unroll
    for (int e = 0; e < 8; ++e) { const float t = x[e] - mean; v += t * t; }
  }
  const float rstd = rsqrtf(warp_sum(v) * inv_d + eps);
  for (int q = lane; q < nch; q += 32) {
    load8(O, o_bf16, base + 8 * q, x);
    emit8(x, mean, rstd, gamma, beta, G, base + 8 * q, 8 * q,
          *reinterpret_cast<const uint4*>(G + base + 8 * q));
  }
}

// Plain row LayerNorm of bf16 rows (the STU layer's input normalisation, "normalize
// input"; R18): Y[r] = (X[r] - mean) / sqrt(var + eps) * gamma + beta, bf16 out.
// One warp per row, 16-byte loads, fp32 two-pass statistics from registers (D <= 1024) or
// through L1 (larger D).
template <int kRegChunks>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    layer_norm_kernel(const __nv_bfloat16* __restrict__ X, __nv_bfloat16* __restrict__ Y,
                      const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
                      int64_t rows, int D) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kWarpsPerCta + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int nch = D >> 3;
  const int64_t base = row * D;
  const float inv_d = 1.0f / static_cast<float>(D);
  const uint4 ones = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);  // bf16 1.0
  auto emit = [&](const float* x, float mean, float rstd, int q) {
    // emit8 multiplies by a gate: a gate of ones (exact) leaves (x - mean) rstd gamma + beta
    emit8(x, mean, rstd, gamma, beta, Y, base + 8 * q, 8 * q, ones);
  };
  if (nch <= 32 * kRegChunks) {
    float x[kRegChunks][8];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kRegChunks; ++k) {
      const int q = lane + 32 * k;
      if (q < nch) load8(X, 1, base + 8 * q, x[k]);
    }
#pragma unroll
    for (int k = 0; k < kRegChunks; ++k)
      if (lane + 32 * k < nch) {
#pragma unroll
        for (int e = 0; e < 8; ++e) s += x[k][e];
      }
    const float mean = warp_sum(s) * inv_d;
    float v = 0.f;
#pragma unroll
    for (int k = 0; k < kRegChunks; ++k)
      if (lane + 32 * k < nch) {
#pragma unroll
        for (int e = 0; e < 8; ++e) { const float t = x[k][e] - mean; v += t * t; }
      }
    const float rstd = rsqrtf(warp_sum(v) * inv_d + eps);
#pragma unroll
    for (int k = 0; k < kRegChunks; ++k)
      if (lane + 32 * k < nch) emit(x[k], mean, rstd, lane + 32 * k);
    return;
  }
  float s = 0.f, x[8];
  for (int q = lane; q < nch; q += 32) {
    load8(X, 1, base + 8 * q, x);
#pragma unroll
    for (int e = 0; e < 8; ++e) s += x[e];
  }
  const float mean = warp_sum(s) * inv_d;
  float v = 0.f;
  for (int q = lane; q < nch; q += 32) {
    load8(X, 1, base + 8 * q, x);
#pragma unroll
    for (int e = 0; e < 8; ++e) { const float t = x[e] - mean; v += t * t; }
  }
  const float rstd = rsqrtf(warp_sum(v) * inv_d + eps);
  for (int q = lane; q < nch; q += 32) {
    load8(X, 1, base + 8 * q, x);
    emit(x, mean, rstd, q);
  }
}

}  // namespace

cudaError_t launch_ln_gate(const void* O, int o_bf16, __nv_bfloat16* G, const float* gamma,
                           const float* beta, float eps, int64_t C, int D, cudaStream_t stream) {
  if (C <= 0) return cudaSuccess;
  const int64_t blocks = (C + kWarpsPerCta - 1) / kWarpsPerCta;
  if (D <= 512)
    ln_gate_kernel<2><<<static_cast<unsigned>(blocks), kWarpsPerCta * 32, 0, stream>>>(
        O, o_bf16, G, gamma, beta, eps, C, D);
  else
    ln_gate_kernel<4><<<static_cast<unsigned>(blocks), kWarpsPerCta * 32, 0, stream>>>(
        O, o_bf16, G, gamma, beta, eps, C, D);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_layer_norm(const void* X, void* Y, const float* gamma, const float* beta,
                              float eps, int64_t rows, int D, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  const int64_t blocks = (rows + kWarpsPerCta - 1) / kWarpsPerCta;
  const auto* x = static_cast<const __nv_bfloat16*>(X);
  auto* y = static_cast<__nv_bfloat16*>(Y);
  if (D <= 512)
    layer_norm_kernel<2><<<static_cast<unsigned>(blocks), kWarpsPerCta * 32, 0, stream>>>(
        x, y, gamma, beta, eps, rows, D);
  else
    layer_norm_kernel<4><<<static_cast<unsigned>(blocks), kWarpsPerCta * 32, 0, stream>>>(
        x, y, gamma, beta, eps, rows, D);
  count_launch();
  return cudaGetLastError();
}

}  // namespace gesr
