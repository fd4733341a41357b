// stu_fused.cu -- K-STU fused: the STU candidate-row epilogue's normalisation, gating and output
// projection in one kernel (reading R15):
//   Y[t] = ((LayerNorm(O[t]) * gamma + beta) (.) G[t]) W_o^T + b_o + X_res[t]
// G = SiLU(T W_g^T + b_g) comes from the K-PROJ GEMM (row-major [C, D] bf16).
//
// Opt-in (GESR_STU_FUSED=1): measured 1.79 ms for the whole gesr_stu_output at the headline row
// count against 1.71 ms unfused -- a row block's A production (HBM loads), its MMAs and its
// epilogue run one after another on each pair (A is single-buffered: 128 KB of the 227 KB), so
// neither the loads nor the tensor core are kept busy.  Double-buffering A needs M = 64 rows per
// CTA.
//
// B200 design: persistent CTA PAIRS (cluster of 2, tcgen05 cta_group::2, M = 256 rows per pair,
// N = 256 output columns per MMA tile).  A CTA's 128 rows span the whole reduction dimension
// (K = D = 512), so the A operand of a row block -- the normalised, gated rows -- is produced
// straight into shared memory by the worker warps (one warp per row: 16-byte loads of O and G,
// fp32 two-pass LayerNorm statistics, bf16 RNE, st.shared into the 128B-swizzled K-major layout
// the MMA descriptors read) and stays resident for all D_out / 256 output tiles.  W_o streams
// through a TMA ring.  The same worker warps then drain the double-buffered TMEM accumulator:
// bias + residual in fp32, bf16, 64B-swizzled staging boxes, TMA tensor stores.  The normalised
// rows never touch HBM (the unfused path writes and re-reads them: 2 B x D per row each way).
//   warp 0    TMA producer of W_o (both CTAs; 128 weight rows x 64 per stage per CTA)
//   warp 1    MMA issuer (leader CTA): per row block, per output tile, 8 k-blocks x 4 MMAs
//   warp 2    TMEM allocator (2 x 256 columns)
//   warps 4-19  workers: A production, then the epilogue of each output tile
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace gesr {

namespace {

constexpr int kD = 512;                       // reduction dimension (H*d) of the fused path
constexpr int kBM = 128;                      // rows per CTA
constexpr int kBN = 256;                      // output columns per MMA tile (pair)
constexpr int kBK = 64;
constexpr int kKB = kD / kBK;                 // 8 k-blocks
constexpr int kWorkers = 16;
constexpr int kThreads = (4 + kWorkers) * 32;
constexpr uint32_t kABytes = kBM * kD * 2;            // 128 KB resident A
constexpr uint32_t kAKBBytes = kBM * kBK * 2;         // 16 KB per k-block
constexpr uint32_t kBStage = (kBN / 2) * kBK * 2;     // 16 KB
constexpr int kStages = 4;
constexpr uint32_t kStagingBytes = kWorkers * 2048;
constexpr uint32_t kAOff = 0;
constexpr uint32_t kBOff = kAOff + kABytes;
constexpr uint32_t kStgOff = kBOff + kStages * kBStage;
constexpr uint32_t kBarOff = kStgOff + kStagingBytes;
constexpr uint32_t kSmemBytes = kBarOff + 256 + 1024;
static_assert(kSmemBytes <= 232448, "shared memory budget");

// 16 features (two 16-byte chunks) of row `row` at chunk q -> fp32
__device__ __forceinline__ void load_o8(const void* O, int o_bf16, int64_t idx, float* x) {
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

// wait with cluster-scope acquire: the A operand was written by both CTAs' worker threads
// (generic proxy, then fence.proxy.async) and published with release.cluster arrivals
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(1000000u)
        : "memory");
  }
}

__device__ __forceinline__ float warp_sum32(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    stu_fused_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_y,
                     const StuFusedParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;     // [2]
  uint64_t* tempty_bar = tfull_bar + 2;          // [2] (leader)
  uint64_t* afull_bar = tempty_bar + 2;          // leader: both CTAs' workers
  uint64_t* aempty_bar = afull_bar + 1;          // each CTA: MMAs done reading A
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty_bar + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int nm = static_cast<int>((p.M + 2 * kBM - 1) / (2 * kBM));
  const int nn = p.N / kBN;
  const int my_m = pair < nm ? (nm - 1 - pair) / npairs + 1 : 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_w);
    tma_prefetch_desc(&map_y);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 2 * kWorkers);
    }
    mbar_init(afull_bar, 2 * kWorkers);
    mbar_init(aempty_bar, 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc_pair(tmem_slot, 2 * kBN);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      // ---------------- W_o producer: per row block, per output tile, the 8 k-blocks
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < my_m; ++i) {
        for (int n = 0; n < nn; ++n) {
          const int nb = n * kBN + static_cast<int>(rank) * (kBN / 2);
          for (int kb = 0; kb < kKB; ++kb) {
            mbar_wait_sleep(&empty_bar[stage], phase ^ 1);
            uint8_t* sb = smem + kBOff + stage * kBStage;
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * kBStage);
            tma_load_2d_pair(sb, &map_w, &full_bar[stage], kb * kBK, nb);
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA)
    if (rank == 0) {
      const uint32_t idesc = make_idesc_bf16(2 * kBM, kBN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int tile = 0;
      for (int i = 0; i < my_m; ++i) {
        mbar_wait_acq_cluster(afull_bar, i & 1);   // both CTAs' A of this row block
        tc_fence_after();
        for (int n = 0; n < nn; ++n, ++tile) {
          const uint32_t buf = tile & 1;
          mbar_wait_sleep(&tempty_bar[buf], ((tile >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + buf * kBN;
          for (int kb = 0; kb < kKB; ++kb) {
            mbar_wait_sleep(&full_bar[stage], phase);
            tc_fence_after();
            if (elect_one()) {
              const uint32_t sa = smem_u32(smem + kAOff + kb * kAKBBytes);
              const uint32_t sb = smem_u32(smem + kBOff + stage * kBStage);
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k) {
                const uint64_t ad = make_sdesc(sa + k * 32, 16, 1024, kSwizzle128B);
                const uint64_t bd = make_sdesc(sb + k * 32, 16, 1024, kSwizzle128B);
                mma_ss_pair(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
              }
              mma_commit_pair_mc(&empty_bar[stage], 0x3);
              if (kb == kKB - 1) mma_commit_pair_mc(&tfull_bar[buf], 0x3);
            }
            __syncwarp();
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
        // every MMA of this row block issued: A may be overwritten once they complete
        if (elect_one()) mma_commit_pair_mc(aempty_bar, 0x3);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ---------------- workers
    const int wk = static_cast<int>(warp) - 4;
    const uint32_t sub = warp & 3;                   // TMEM lane quarter of this warp
    const int part = wk >> 2;                        // column part of an output tile
    const uint32_t afull_leader = mapa_shared(smem_u32(afull_bar), 0);
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty_bar[1]), 0);
    const uint32_t a_base = smem_u32(smem + kAOff);
    const uint32_t box_s = smem_u32(smem + kStgOff + wk * 2048);
    uint8_t* box = smem + kStgOff + wk * 2048;
    int tile = 0;
    for (int i = 0; i < my_m; ++i) {
      const int m_blk = pair + i * npairs;
      const int64_t row_cta = static_cast<int64_t>(m_blk) * 2 * kBM + static_cast<int64_t>(rank) * kBM;
      // -- A production: rows wk, wk + 16, ... of this CTA's 128 (warp per row, lane per 2 chunks)
      if (i > 0) mbar_wait_sleep(aempty_bar, (i - 1) & 1);
      for (int r = wk; r < kBM; r += kWorkers) {
        const int64_t row = row_cta + r;
        float x[2][8];
        uint4 gq[2];
        if (row < p.M) {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int q = static_cast<int>(lane) + 32 * k;
            load_o8(p.O, p.o_bf16, row * kD + 8 * q, x[k]);
            gq[k] = __ldg(reinterpret_cast<const uint4*>(p.G + row * kD + 8 * q));
          }
        } else {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
#pragma unroll
            for (int e = 0; e < 8; ++e) x[k][e] = 0.f;
            gq[k] = make_uint4(0, 0, 0, 0);
          }
        }
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int e = 0; e < 8; ++e) s += x[k][e];
        const float mean = warp_sum32(s) * (1.0f / kD);
        float v = 0.f;
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int e = 0; e < 8; ++e) { const float t = x[k][e] - mean; v += t * t; }
        const float rstd = rsqrtf(warp_sum32(v) * (1.0f / kD) + p.eps);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int q = static_cast<int>(lane) + 32 * k;          // 8-feature chunk, col 8q
          const float4 g0 = __ldg(reinterpret_cast<const float4*>(p.gamma + 8 * q));
          const float4 g1 = __ldg(reinterpret_cast<const float4*>(p.gamma + 8 * q) + 1);
          const float4 b0 = __ldg(reinterpret_cast<const float4*>(p.beta + 8 * q));
          const float4 b1 = __ldg(reinterpret_cast<const float4*>(p.beta + 8 * q) + 1);
          const float ga[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
          const float be[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
          const uint32_t gw[4] = {gq[k].x, gq[k].y, gq[k].z, gq[k].w};
          uint32_t z[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float z0 = ((x[k][2 * e] - mean) * rstd * ga[2 * e] + be[2 * e]) *
                             __uint_as_float(gw[e] << 16);
            const float z1 = ((x[k][2 * e + 1] - mean) * rstd * ga[2 * e + 1] + be[2 * e + 1]) *
                             __uint_as_float(gw[e] & 0xFFFF0000u);
            z[e] = pack_bf16x2(z0, z1);
          }
          // K-major 128B-swizzled A: k-block q / 8, 16-byte chunk (q % 8) ^ (r % 8) of row r
          const uint32_t addr = a_base + (q >> 3) * kAKBBytes + r * 128 +
                                ((static_cast<uint32_t>(q & 7) ^ static_cast<uint32_t>(r & 7)) << 4);
          st_shared_v4(addr, z[0], z[1], z[2], z[3]);
        }
      }
      fence_proxy_async_smem();                      // generic-proxy writes -> the tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(afull_leader);      // release: A rows -> leader MMA

      // -- epilogue of each output tile of this row block
      const int64_t row0 = row_cta + static_cast<int64_t>(sub) * 32;
      for (int n = 0; n < nn; ++n, ++tile) {
        const uint32_t buf = tile & 1;
        mbar_wait_sleep(&tfull_bar[buf], (tile >> 1) & 1);
        tc_fence_after();
        const uint32_t tm_row = tmem_base + ((sub * 32) << 16) + buf * kBN;
#pragma unroll 1
        for (int c = 2 * part; c < 2 * part + 2; ++c) {     // 2 chunks of 32 columns
          uint32_t rr[32];
          tmem_ld32(tm_row + c * 32, rr);
          tmem_ld_wait_regs32(rr);
          float v[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(rr[e]);
          const int col = n * kBN + c * 32;
          if (p.b_o != nullptr) {
            const float4* b4 = reinterpret_cast<const float4*>(p.b_o + col);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float4 bb = __ldg(b4 + e);
              v[4 * e] += bb.x; v[4 * e + 1] += bb.y; v[4 * e + 2] += bb.z; v[4 * e + 3] += bb.w;
            }
          }
          const int64_t rr_row = row0 + lane;
          if (p.X_res != nullptr && rr_row < p.M) {
            const uint4* src = reinterpret_cast<const uint4*>(p.X_res + rr_row * p.N + col);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 u = __ldg(src + q);
              const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                v[8 * q + 2 * e] += __uint_as_float(w[e] << 16);
                v[8 * q + 2 * e + 1] += __uint_as_float(w[e] & 0xFFFF0000u);
              }
            }
          }
          uint32_t packed[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) packed[e] = pack_bf16x2(v[2 * e], v[2 * e + 1]);
          if (lane == 0) bulk_wait_group_read<0>();        // the staging box is free again
          __syncwarp();
          const uint32_t rowp = box_s + lane * 64;        // 64B swizzle: chunk q ^ ((lane>>1)&3)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            st_shared_v4(rowp + ((q ^ ((lane >> 1) & 3)) << 4), packed[4 * q], packed[4 * q + 1],
                         packed[4 * q + 2], packed[4 * q + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&map_y, box, col, static_cast<int32_t>(row0), 0);
            bulk_commit_group();
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_relaxed(buf ? tempty_leader1 : tempty_leader0);
      }
    }
    if (lane == 0) bulk_wait_group<0>();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 2 * kBN);
  }
}

}  // namespace

bool stu_fused_supported(int D, int D_out) { return D == kD && D_out % kBN == 0; }

cudaError_t launch_stu_fused(const CUtensorMap& map_w, const CUtensorMap& map_y,
                             const StuFusedParams& p, int num_sms, cudaStream_t stream) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(stu_fused_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int64_t nm = (p.M + 2 * kBM - 1) / (2 * kBM);
  const int pairs = static_cast<int>(nm < num_sms / 2 ? nm : num_sms / 2);
  if (pairs <= 0) return cudaSuccess;
  stu_fused_kernel<<<2 * pairs, kThreads, kSmemBytes, stream>>>(map_w, map_y, p);
  return cudaGetLastError();
}

}  // namespace gesr
