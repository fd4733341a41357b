// kernels.h -- internal launch interface between capi.cpp (validation, tensor maps) and the
// sm_100a kernels.  Not part of the public ABI (include/gesr.h).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace gesr {

// ---------------------------------------------------------------- launch bookkeeping (capi.cpp)
// Raise `fn`'s dynamic shared-memory limit to `bytes` on the CURRENT device, once per (device,
// kernel): the attribute belongs to each device's context, so a process driving several GPUs
// sets it on each.  Thread-safe.
cudaError_t ensure_smem_attr(const void* fn, int bytes);
// Per-device cached value of a launch-configuration query (e.g. the occupancy in CTA pairs):
// slot in [0, 8); returns 0 if not yet stored on this device.
int device_cached(int slot);
void device_cache_store(int slot, int value);
// Every kernel launch of the library is counted (gesr_launch_count(): the bench's
// gpu_launches claim is read from it, not typed in).
void count_launch();
// Launch with programmatic stream serialisation (PDL, ptx.cuh pdl_wait): the kernel's CTAs may
// be scheduled as soon as every CTA of the previous kernel on the stream has started, and wait
// in pdl_wait() for its completion -- the launch latency and the prologue (barrier init, TMEM
// allocation, tensor-map prefetch) overlap the previous kernel's tail.  Only kernels that call
// pdl_wait() in every CTA before touching global memory are launched this way.  -DGESR_PDL=0
// builds plain stream-ordered launches (A/B).
#ifndef GESR_PDL
#define GESR_PDL 1
#endif
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = GESR_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  count_launch();
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}
// GESR_DEBUG=1: device check of a jagged offsets array [n + 1] (debug.cu); traps if
// offsets[0] != 0, offsets decrease, or offsets[n] != total.  tag names the array in the report.
cudaError_t launch_check_offsets(const int64_t* offsets, int64_t n, int64_t total, int tag,
                                 cudaStream_t stream);

// ---------------------------------------------------------------- K-PROJ (proj.cu)
struct ProjParams {
  int64_t M;          // rows of X
  int K;              // D_in
  int n_split;        // columns < n_split come from W0 (out0), the rest from W1 (out1)
  int d;              // head dim
  int act;            // 0 identity, 1 SiLU
  int num_m_blocks;
  int num_n_blocks;
  int m_major;        // set by launch_proj: tile order (see ProjTiles in proj.cu)
  const float* bias0;
  const float* bias1;
  __nv_bfloat16* out0;   // [H, M, d]
  __nv_bfloat16* out1;   // [H, M, d] or null
  // row-major output (out0 [M, N] through a {N, M, 1} map): columns are not split into heads
  int rowmajor;
  // optional residual added after the activation: out[r][c] += residual[r * res_ld + c]
  const __nv_bfloat16* residual;
  int64_t res_ld;
  // optional row gather (gesr_kv_project_gather): X row m is row gather[m] of the table that
  // map_a describes (box {64, 1}); loaded by TMA tile::gather4, four rows per instruction
  const int32_t* gather;
};

// Tile width: the widest of 256 / 128 / 64 dividing N (the columns of one weight; `ways`
// weights stacked along N) whose (256-row x bn) tiles still give every CTA pair of the device
// one; narrower for few rows (a 512-row chunk: 64, so 16 pairs run the 8-deep K loop and the
// epilogue instead of 4); N not a multiple of 64: 32.
int proj_pick_bn(int64_t M, int N, int ways, int num_sms);
cudaError_t launch_proj(const CUtensorMap& map_a, const CUtensorMap& map_b0,
                        const CUtensorMap& map_b1, const CUtensorMap& map_o0,
                        const CUtensorMap& map_o1, const ProjParams& p, int bn, int num_sms,
                        cudaStream_t stream);

// ---------------------------------------------------------------- K-SCHED + K-ATTN (attn.cu)
struct AttnParams {
  const int64_t* seq_offsets;
  const int64_t* cand_offsets;
  const int4* units;       // work list: {first history row s0, L_b, first candidate row, rows}
  const int* unit_count;
  int64_t total_C;
  int64_t total_L;
  int H;
  float scale_log2;        // scale * log2(e)
  void* O;                 // [total_C, H*d]
  int o_bf16;
  int o_tma;               // bf16 O through the map_o TMA tensor stores
  float* lse;              // [total_C, H] or null
  // split-L (pair kernel): each (unit, head) is cut into `splits` ranges of key tiles; with
  // splits > 1 the kernel writes per-split partials (O_s / l_s fp32 and (m_s, l_s), m in log2
  // units) that launch_attn_combine merges into O / lse
  int splits;
  float* part_o;           // [splits, total_C, H, d]
  float2* part_ml;         // [splits, total_C, H]
  // causal self-attention over the history (gesr_history_attention): the queries are
  // the history rows themselves; a unit {s0, L, first row, rows} covers query rows
  // [L - rows, L) of its request and row r (0-based in the unit) sees keys [0, L - rows + r]
  int causal;
  // HSTU pointwise normalisation (GESR_TASA_HSTU_SILU): O = sum_i SiLU(scale s_i) v_i / L_b
  // (1-CTA kernel only; no lse, one split)
  int hstu;
};

constexpr int kUnitRows = 256;   // candidates per work unit (two 128-row Q tiles)

#ifdef __CUDACC__
// The attention kernels' work list.  p.units == nullptr: one request (B = 1), whose offsets are
// {0, total} by the ABI contract, so unit u follows from total_L / total_C without a
// build_units launch: {0, L, 256 u, rows} (causal: L = 256 u + rows, as build_units_kernel).
__device__ __forceinline__ int unit_count_of(const AttnParams& p) {
  return p.units != nullptr ? __ldg(p.unit_count)
                            : static_cast<int>((p.total_C + kUnitRows - 1) / kUnitRows);
}
__device__ __forceinline__ int4 unit_of(const AttnParams& p, int u) {
  if (p.units != nullptr) return __ldg(p.units + u);
  const int c0 = u * kUnitRows;
  const int left = static_cast<int>(p.total_C) - c0;
  const int rows = left < kUnitRows ? left : kUnitRows;
  return make_int4(0, p.causal ? c0 + rows : static_cast<int>(p.total_L), c0, rows);
}
#endif

// causal = 1: queries are the history rows (cand_offsets == seq_offsets), unit k of request b
// is {s0, 256 k + rows, s0 + 256 k, rows} (keys up to the unit's last query row)
cudaError_t launch_build_units(const int64_t* seq_offsets, const int64_t* cand_offsets, int64_t B,
                               int4* units, int* count, int causal,
                               cudaStream_t stream);
// map_o: bf16 O as [total_C, H, d] (box {32, 1, 32}, 64B swizzle), used when p.o_tma
cudaError_t launch_attn(int d, const CUtensorMap& map_q, const CUtensorMap& map_k,
                        const CUtensorMap& map_v, const CUtensorMap& map_o, const AttnParams& p,
                        int64_t max_units,
                        cudaStream_t stream);
// d = 128: CTA-pair kernel (attn2.cu); K map box {64, 64}, Q / V maps box {64, 128}
cudaError_t launch_attn_pair(const CUtensorMap& map_q, const CUtensorMap& map_kh,
                             const CUtensorMap& map_vh, const CUtensorMap& map_o,
                             const AttnParams& p, int64_t max_units, cudaStream_t stream);
// candidate self key (GESR_TASA_SELF_KEY): merges each row's own key / value into O and lse
// (p.lse must be set): s = scale q.k_self, O' = (O e^lse + v_self e^s) / (e^lse + e^s)
cudaError_t launch_attn_self_merge(const AttnParams& p, const void* Q, const void* K_self,
                                   const void* V_self, int d, float scale, cudaStream_t stream);
// merges split-L partials: O = sum_s w_s O_s / sum_s w_s, w_s = l_s 2^(m_s - max m)
cudaError_t launch_attn_combine(const AttnParams& p, int d, cudaStream_t stream);
cudaError_t launch_attn_empty(const AttnParams& p, int d, cudaStream_t stream);

// ---------------------------------------------------------------- K-STU (stu.cu)
// Z[t][:] = LayerNorm(O[t][:]) * gamma + beta, times G[t][:] (in place over G), D = H*d
// features per row (R15).  O fp32 or bf16 [C, D]; G bf16 [C, D].
cudaError_t launch_ln_gate(const void* O, int o_bf16, __nv_bfloat16* G, const float* gamma,
                           const float* beta, float eps, int64_t C, int D, cudaStream_t stream);

// Y[r] = LayerNorm(X[r]) * gamma + beta over D features, bf16 in / out (stu.cu; R18).
cudaError_t launch_layer_norm(const void* X, void* Y, const float* gamma, const float* beta,
                              float eps, int64_t rows, int D, cudaStream_t stream);

// ---------------------------------------------------------------- NRO query gate (nro.cu)
// out[s*d + i][k] = bf16(W_q[s*d + i][k] * gate[s][k]): the elementwise query gate of NRO
// cross-attention slot s folded into its query weight (R16).
cudaError_t launch_fold_gate(const void* W_q, const float* gate, void* out, int j, int d, int D_in,
                             cudaStream_t stream);

// RO cross attention (nro.cu): query rows X[b*i + s] = seeds[s] (+ ctx[b][s]) and offsets i*b;
// then the diagonal gather U_cross[b][s*d + j] = O_full[b*i + s][s*d + j]
cudaError_t launch_ro_queries(const void* seeds, const void* ctx, void* X, int64_t* offs,
                              int64_t B, int i, int D_in, cudaStream_t stream);
cudaError_t launch_ro_gather(const float* O_full, void* out, int o_bf16, int64_t B, int i, int d,
                             cudaStream_t stream);

// ---------------------------------------------------------------- K-HMA (hma.cu)
struct HmaParams {
  const int64_t* user_ids;
  const int64_t* user_offsets;
  const int64_t* item_ids;
  const int64_t* item_offsets;
  const int64_t* cand_offsets;
  int64_t B;
  int64_t total_C;
  int F;
  int cap;
  int32_t* counts;
  // optional offset embedding: emb[t][f] = E[min(c, cap) + f (cap + 1)], D_h bf16
  const uint4* E;          // [F (cap + 1), D_h] bf16 rows, 16-byte chunks; null = counts only
  int dh_chunks;           // D_h / 8
  uint4* emb;              // [total_C, F D_h] bf16
};

cudaError_t launch_hma(const HmaParams& p, cudaStream_t stream);

}  // namespace gesr
