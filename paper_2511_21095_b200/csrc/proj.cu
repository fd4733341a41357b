// proj.cu -- K-PROJ: Y = act(X W^T + b) with a head-major scatter epilogue.
//
// Serves gesr_kv_project (X = U [total_L, D_in], W = [W_k; W_v] as two TMA maps stacked along N,
// outputs K_cache / V_cache [H, total_L, d]) and the Q projection inside gesr_tasa_score
// (X = T, W = W_q, output Q [H, total_C, d] in the workspace).  PAPER.md:335-341 (s3.4.2):
// the [U,T] self-attention layer's projections; projection form act(XW^T+b) per DESIGN.md R3.
//
// B200 design: persistent CTA PAIRS (cluster of 2, tcgen05 cta_group::2), warp-specialised.
// A pair computes a 256 x BN output tile with M=256 MMAs: each CTA stages its own 128 rows of
// X and HALF of the BN weight rows, so every SM receives 16 KB of X plus BN*64 B of W per
// 64-deep K block -- half the weight traffic of a single-CTA 128 x BN tile.  (ncu on the
// single-CTA version: 25.8 GB of L2->SM traffic for the K/V projection, tensor pipe 35%.)
//   warp 0    TMA producer (both CTAs): A 128x64 + B (BN/2)x64 per stage, completion bytes
//             signalled on the leader CTA's full barrier.
//   warp 1    MMA issuer (leader CTA only): tcgen05.mma.cta_group::2.kind::f16, M=256 N=BN
//             K=16, into a double-buffered TMEM accumulator (2*BN columns in each CTA);
//             commits multicast to both CTAs' barriers.
//   warp 2    TMEM allocator (cta_group::2).
//   warps 4-19 epilogue (both CTAs): tcgen05.ld 32x32b (thread = output row), bias + act in
//             fp32 (packed FFMA2 SiLU, one MUFU op per element), RNE to bf16, swizzled 16-byte
//             st.shared into a per-warp staging box, TMA tensor stores into the head-major
//             [H, M, d] output; each warp releases its share of the accumulator with its own
//             arrival on the leader's TMEM-empty barrier (no CTA-wide barrier: the slowest
//             warp no longer holds the others).  (Direct per-thread 16-byte global stores
//             touched 32 rows per instruction and capped the kernel at ~35% tensor-pipe.)
// Gather mode (gesr_kv_project_gather): X row m is table row gather[m]; warp 0
// stages a tile's 128 row ids in shared memory and warps 0, 3 and 2 issue the A operand as TMA
// tile::gather4 loads (four 128-byte table-row slices each, same 128B-swizzled layout).
// The epilogue of tile i overlaps the MMAs of tile i+1.  Tile order is m-major for large M
// (ProjTiles): a pair takes all n-blocks of one 256-row block back to back, so X is read from
// HBM exactly once (ncu: 2.16 GB DRAM reads for the 2.15 GB U, against 3.0 GB interleaved).
#include <cstdlib>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace gesr {

#ifdef GESR_PROJ_PROF
// Wait profile (scripts/proj_prof.py; -DGESR_PROJ_PROF builds only).  Per CTA: [0] producer
// cycles waiting for a free stage, [1] MMA issuer cycles waiting for a loaded stage, [2] MMA
// cycles waiting for a free accumulator, [3] MMA warp total, [4] epilogue warp 4 cycles
// waiting for a full accumulator.
__device__ unsigned long long g_projprof[296][8];
#define PROF_ADD(i, t) atomicAdd(&g_projprof[blockIdx.x][i], static_cast<unsigned long long>(clock64() - (t)))
#define PROF_WAIT(i, call) do { const long long _tw = clock64(); call; if (lane_id() == 0) PROF_ADD(i, _tw); } while (0)
#else
#define PROF_WAIT(i, call) call
#endif

namespace {

constexpr int kBM = 128;             // rows per CTA; a pair tile is 256 rows
constexpr int kBK = 64;              // 64 bf16 = 128 bytes = one 128B-swizzle row
constexpr int kEpiWarps = 16;        // 4 per SM sub-partition: latency hiding by TLP
constexpr int kThreads = (4 + kEpiWarps) * 32;
constexpr uint32_t kABytes = kBM * kBK * 2;   // 16 KB
#ifndef GESR_GATHER_WARPS
#define GESR_GATHER_WARPS 3
#endif
constexpr int kGatherWarps = GESR_GATHER_WARPS;   // warps issuing the gather4 loads (1-3)
constexpr int kBoxes = 1;   // staging boxes per epilogue warp (2 measured slower: one fewer stage)

template <int BN>
struct ProjSmem {
  static constexpr uint32_t kBBytes = (BN / 2) * kBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  // epilogue staging: kBoxes 2 KB boxes (32 rows x 32 columns, 64B swizzle) per epilogue warp
  static constexpr int kChunks = BN / 32;
  static constexpr uint32_t kStagingBytes = kEpiWarps * 2048 * kBoxes;
  static constexpr int kStages = (224 * 1024 - kStagingBytes) / kStageBytes > 8
                                     ? 8 : (224 * 1024 - kStagingBytes) / kStageBytes;
  // accumulator buffers in TMEM: two (the epilogue of tile i overlaps the MMAs of tile i+1),
  // one for BN = 512 (the gather mode's double-width tile: 512 columns fill TMEM)
  static constexpr int kAccBufs = BN >= 512 ? 1 : 2;
  static constexpr uint32_t kTmemCols = (kAccBufs * BN) < 32 ? 32 : kAccBufs * BN;
  static constexpr uint32_t kStagingOffset = kStages * kStageBytes;
  static constexpr uint32_t kBarOffset = kStagingOffset + kStagingBytes;
  static constexpr uint32_t kIdsOffset = kBarOffset + 256;     // gathered row ids of a tile
  static constexpr uint32_t kBytes = kIdsOffset + 512 + 1024;  // + ids + alignment slack
  static_assert(kBytes <= 232448, "shared memory budget");
};

// Tile order of one pair.  m-major (large M): the pair walks all n-blocks of its 256-row block
// back to back, so the X rows are fetched from HBM once and re-read from L2 while hot;
// interleaved (few row blocks): tiles dealt round-robin so every pair has work.
struct ProjTiles {
  int pair, npairs, nm, nn;
  bool m_major;
  __device__ __forceinline__ int count() const {
    if (m_major) return pair < nm ? ((nm - 1 - pair) / npairs + 1) * nn : 0;
    const int tiles = nm * nn;
    return pair < tiles ? (tiles - 1 - pair) / npairs + 1 : 0;
  }
};
// Walks one pair's tiles in ProjTiles order without a division per step.
struct TileCursor {
  int m, n, dm, dn, nn, npairs;
  bool m_major;
  __device__ __forceinline__ explicit TileCursor(const ProjTiles& t)
      : nn(t.nn), npairs(t.npairs), m_major(t.m_major) {
    if (m_major) { m = t.pair; n = 0; dm = 0; dn = 1; }
    else { m = t.pair / t.nn; n = t.pair % t.nn; dm = t.npairs / t.nn; dn = t.npairs % t.nn; }
  }
  __device__ __forceinline__ void next() {
    if (m_major) {
      if (++n == nn) { n = 0; m += npairs; }
    } else {
      n += dn; m += dm;
      if (n >= nn) { n -= nn; ++m; }
    }
  }
};

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    proj_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b0,
                const __grid_constant__ CUtensorMap map_b1, const __grid_constant__ CUtensorMap map_o0,
                const __grid_constant__ CUtensorMap map_o1, const ProjParams p) {
  using S = ProjSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* empty_bar = full_bar + S::kStages;
  uint64_t* tfull_bar = empty_bar + S::kStages;     // [2]
  uint64_t* tempty_bar = tfull_bar + 2;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();          // 0 = leader of the pair
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const ProjTiles tiles{pair, npairs, p.num_m_blocks, p.num_n_blocks, p.m_major != 0};
  const int my_tiles = tiles.count();
  const int num_kb = (p.K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b0);
    tma_prefetch_desc(&map_b1);
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 2 * kEpiWarps);   // one arrival per epilogue warp of the pair
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc_pair(tmem_slot, S::kTmemCols);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();         // the prologue above touched no global memory

  // gather issuers: warp 0, then warps 3 and 2 (idle otherwise; warp 2 only allocates TMEM)
  const int issuer = warp == 0 ? 0 : (warp == 3 ? 1 : (warp == 2 ? 2 : -1));
  if (warp == 0 || (p.gather != nullptr && issuer >= 0 && issuer < kGatherWarps)) {
    // ---------------- TMA producer (both CTAs; one elected lane issues; warp 0 stages a tile's
    // gathered row ids and, with a gather, kGatherWarps warps split its gather4 loads: one
    // thread issuing ~256 gather4 per tile cannot keep up with the MMAs)
    const bool helper = issuer != 0;
    int4* ids = reinterpret_cast<int4*>(smem + S::kIdsOffset);
    int stage = 0;
    uint32_t phase = 0;
    TileCursor cur(tiles);
    for (int i = 0; i < my_tiles; ++i, cur.next()) {
      const int m_blk = cur.m, n_blk = cur.n;
      const int n0 = n_blk * BN;
      // B comes from map_b0 for columns < n_split, else map_b1 (W_k / W_v stacked along N)
      const CUtensorMap* mb = (n0 < p.n_split) ? &map_b0 : &map_b1;
      const int nb = ((n0 < p.n_split) ? n0 : n0 - p.n_split) + static_cast<int>(rank) * (BN / 2);
      const int ma = m_blk * 2 * kBM + static_cast<int>(rank) * kBM;
      if (p.gather != nullptr && !helper) {
        // rows ma + 4 lane .. + 3 of X are table rows gather[...]; rows past M repeat row M - 1
        // (their outputs are clipped by the output map)
        __syncwarp();
        int r[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t m = static_cast<int64_t>(ma) + 4 * lane + q;
          r[q] = __ldg(p.gather + (m < p.M ? m : p.M - 1));
        }
        ids[lane] = make_int4(r[0], r[1], r[2], r[3]);
        __syncwarp();
      }
      if (kGatherWarps > 1 && p.gather != nullptr) named_bar_sync(8, 32 * kGatherWarps);   // ids staged
      if (elect_one()) {
        const int ng = p.gather != nullptr ? kGatherWarps : 1;
        const int g0 = issuer * (kBM / 4) / ng, g1 = (issuer + 1) * (kBM / 4) / ng;
        for (int kb = 0; kb < num_kb; ++kb) {
          PROF_WAIT(0, mbar_wait_sleep(&empty_bar[stage], phase ^ 1));
          uint8_t* sa = smem + stage * S::kStageBytes;
          uint8_t* sb = sa + kABytes;
          if (rank == 0 && !helper) mbar_arrive_expect_tx(&full_bar[stage], 2 * S::kStageBytes);
          if (p.gather != nullptr) {
#pragma unroll 4
            for (int g = g0; g < g1; ++g)
              tma_gather4_pair(sa + g * 4 * kBK * 2, &map_a, &full_bar[stage], kb * kBK, ids[g]);
          } else {
            tma_load_2d_pair(sa, &map_a, &full_bar[stage], kb * kBK, ma);
          }
          if (!helper) {
            if constexpr (BN >= 512) {
              // two 128-row weight boxes per CTA: box j of CTA r holds rows 256 j + 128 r + [0,
              // 128), so the pair MMA j (N = 256) covers columns [256 j, 256 j + 256) in order
              const int nl = nb - static_cast<int>(rank) * (BN / 2) + static_cast<int>(rank) * 128;
              tma_load_2d_pair(sb, mb, &full_bar[stage], kb * kBK, nl);
              tma_load_2d_pair(sb + 128 * kBK * 2, mb, &full_bar[stage], kb * kBK, nl + 256);
            } else {
              tma_load_2d_pair(sb, mb, &full_bar[stage], kb * kBK, nb);
            }
          }
          if (++stage == S::kStages) { stage = 0; phase ^= 1; }
        }
      }
      __syncwarp();
      if (kGatherWarps > 1 && p.gather != nullptr) named_bar_sync(8, 32 * kGatherWarps);   // ids consumed
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA only)
    if (rank == 0) {
      const uint32_t idesc = make_idesc_bf16(2 * kBM, BN >= 512 ? 256 : BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
#ifdef GESR_PROJ_PROF
      const long long tstart = clock64();
#endif
      for (; local < my_tiles; ++local) {
        const uint32_t buf = local % S::kAccBufs;
        const uint32_t aphase = (local / S::kAccBufs) & 1;
        PROF_WAIT(2, mbar_wait_sleep(&tempty_bar[buf], aphase ^ 1));
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          PROF_WAIT(1, mbar_wait_sleep(&full_bar[stage], phase));
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = smem_u32(smem + stage * S::kStageBytes);
            const uint32_t sb = sa + kABytes;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t ad = make_sdesc(sa + k * 32, 16, 1024, kSwizzle128B);
              const uint64_t bd = make_sdesc(sb + k * 32, 16, 1024, kSwizzle128B);
              mma_ss_pair(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
              if constexpr (BN >= 512) {
                const uint64_t bd1 = make_sdesc(sb + 128 * kBK * 2 + k * 32, 16, 1024,
                                                kSwizzle128B);
                mma_ss_pair(d_tmem + 256, ad, bd1, idesc, (kb | k) != 0 ? 1u : 0u);
              }
            }
            mma_commit_pair_mc(&empty_bar[stage], 0x3);
            if (kb == num_kb - 1) mma_commit_pair_mc(&tfull_bar[buf], 0x3);
          }
          __syncwarp();
          if (++stage == S::kStages) { stage = 0; phase ^= 1; }
        }
      }
#ifdef GESR_PROJ_PROF
      if (lane_id() == 0) PROF_ADD(3, tstart);
#endif
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs): TMEM -> regs -> act -> bf16 -> smem -> TMA store
    // 16 warps: warp w reads TMEM lane quarter (w & 3) and column part (w - 4) / 4 of the tile
    // (BN/4 columns = 1-2 chunks of 32).  Each 32x32 chunk goes through the warp's 2 KB
    // 64B-swizzled staging box (conflict-free 16-byte stores) and leaves with one TMA tensor
    // store into the [H, M, d] output (rows >= M are clipped by the tensor map).
    const uint32_t sub = warp & 3;
    const int part = (warp - 4) >> 2;
    constexpr int kPer = S::kChunks >= 4 ? S::kChunks / 4 : 1;
    const int c_begin = part * kPer;
    const int c_end = c_begin + kPer <= S::kChunks ? c_begin + kPer : S::kChunks;
    const uint32_t box_base = smem_u32(smem + S::kStagingOffset + (warp - 4) * 2048 * kBoxes);
    uint32_t bi = 0;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty_bar[1]), 0);
    int local = 0;
    const int dshift = __ffs(p.d) - 1;              // d is 32, 64 or 128
    TileCursor cur(tiles);
    for (; local < my_tiles; ++local, cur.next()) {
      const int m_blk = cur.m, n_blk = cur.n;
      const uint32_t buf = local % S::kAccBufs;
      const uint32_t aphase = (local / S::kAccBufs) & 1;
      const int row0 = m_blk * 2 * kBM + static_cast<int>(rank) * kBM + static_cast<int>(sub) * 32;
      // one warp of each 4-warp column part polls the accumulator's mbarrier and releases the
      // other three through hardware named barrier 1 + part (they wait descheduled): 16 warps
      // polling a try_wait that wakes on every barrier event of the CTA cost issue slots and
      // power for the whole mainloop of every tile
#ifdef GESR_PROJ_PROF
      const long long tw4 = clock64();
#endif
      if (sub == 0) mbar_wait_sleep(&tfull_bar[buf], aphase);
      named_bar_sync(1 + part, 128);
#ifdef GESR_PROJ_PROF
      if (warp == 4 && lane == 0) PROF_ADD(4, tw4);
#endif
      tc_fence_after();
      const uint32_t tm_row = tmem_base + ((sub * 32) << 16) + buf * BN;
#pragma unroll 1
      for (int c = c_begin; c < c_end; ++c) {
        uint32_t r[32];
        tmem_ld32(tm_row + c * 32, r);
        tmem_ld_wait_regs32(r);
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        const int n0 = n_blk * BN + c * 32;   // chunk lies within one head (d >= 32)
        const int which = n0 >= p.n_split ? 1 : 0;
        const int within = n0 - which * p.n_split;
        const float* bias = which ? p.bias1 : p.bias0;
        if (bias != nullptr) {
          const float4* b4 = reinterpret_cast<const float4*>(bias + within);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 bb = __ldg(b4 + i);
            v[4 * i] += bb.x; v[4 * i + 1] += bb.y; v[4 * i + 2] += bb.z; v[4 * i + 3] += bb.w;
          }
        }
        if (p.act == 1) {
#pragma unroll
          for (int i = 0; i < 32; i += 2) silu2(v[i], v[i + 1]);
        }
        if (p.residual != nullptr) {
          // out = act(.) + residual (STU layer output): this lane's row, 32 columns
          const int64_t rr = static_cast<int64_t>(row0) + lane;
          if (rr < p.M) {
            const uint4* src = reinterpret_cast<const uint4*>(p.residual + rr * p.res_ld + within);
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
        }
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) packed[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
        // the staging box must have been read by this warp's TMA store kBoxes chunks ago
        if (lane == 0) bulk_wait_group_read<kBoxes - 1>();
        __syncwarp();
        const uint32_t box_s = box_base + (kBoxes > 1 ? (bi & 1) * 2048 : 0);
        uint8_t* box = smem + S::kStagingOffset + (warp - 4) * 2048 * kBoxes +
                       (kBoxes > 1 ? (bi & 1) * 2048 : 0);
        ++bi;
        // 64B swizzle: 16-byte chunk q of row `lane` goes to slot q ^ ((lane >> 1) & 3)
        const uint32_t rowp = box_s + lane * 64;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_shared_v4(rowp + ((q ^ ((lane >> 1) & 3)) << 4), packed[4 * q], packed[4 * q + 1],
                       packed[4 * q + 2], packed[4 * q + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const int h = p.rowmajor ? 0 : within >> dshift;
          tma_store_3d(which ? &map_o1 : &map_o0, box, within - (h << dshift), row0, h);
          bulk_commit_group();
        }
      }
      // this warp's part of the accumulator is drained
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(buf ? tempty_leader1 : tempty_leader0);
    }
    if (lane == 0) bulk_wait_group<0>();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, S::kTmemCols);
  }
}

template <int BN>
cudaError_t launch_bn(const CUtensorMap& ma, const CUtensorMap& mb0, const CUtensorMap& mb1,
                      const CUtensorMap& mo0, const CUtensorMap& mo1, const ProjParams& p,
                      int num_sms, cudaStream_t stream) {
  using S = ProjSmem<BN>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(proj_kernel<BN>), S::kBytes);
  if (e != cudaSuccess) return e;
  ProjParams q = p;
  q.m_major = p.num_m_blocks >= num_sms / 2 ? 1 : 0;
  const int work = q.m_major ? p.num_m_blocks : p.num_m_blocks * p.num_n_blocks;
  const int pairs = work < num_sms / 2 ? work : num_sms / 2;
  return launch_pdl(proj_kernel<BN>, dim3(2 * pairs), dim3(kThreads), S::kBytes, stream, ma, mb0,
                    mb1, mo0, mo1, q);
}

}  // namespace

#ifdef GESR_PROJ_PROF
extern "C" int gesr_debug_projprof_copy(void* host, int reset) {
  int r = static_cast<int>(cudaMemcpyFromSymbol(host, g_projprof, sizeof(g_projprof)));
  if (reset) {
    static unsigned long long zero[296][8];
    cudaMemcpyToSymbol(g_projprof, zero, sizeof(zero));
  }
  return r;
}
#endif

#ifndef GESR_PROJ_MIN_BN
#define GESR_PROJ_MIN_BN 64
#endif
int proj_pick_bn(int64_t M, int N, int ways, int num_sms) {
  const int64_t m_blocks = (M + 2 * kBM - 1) / (2 * kBM);
  for (int bn = 256; bn > GESR_PROJ_MIN_BN; bn >>= 1)
    if (N % bn == 0 && m_blocks * ways * (N / bn) >= num_sms / 2) return bn;
  for (int bn = GESR_PROJ_MIN_BN; bn >= 32; bn >>= 1)
    if (N % bn == 0) return bn;
  return 32;
}

cudaError_t launch_proj(const CUtensorMap& map_a, const CUtensorMap& map_b0,
                        const CUtensorMap& map_b1, const CUtensorMap& map_o0,
                        const CUtensorMap& map_o1, const ProjParams& p, int bn, int num_sms,
                        cudaStream_t stream) {
  switch (bn) {
    case 512: return launch_bn<512>(map_a, map_b0, map_b1, map_o0, map_o1, p, num_sms, stream);
    case 256: return launch_bn<256>(map_a, map_b0, map_b1, map_o0, map_o1, p, num_sms, stream);
    case 128: return launch_bn<128>(map_a, map_b0, map_b1, map_o0, map_o1, p, num_sms, stream);
    case 64: return launch_bn<64>(map_a, map_b0, map_b1, map_o0, map_o1, p, num_sms, stream);
    case 32: return launch_bn<32>(map_a, map_b0, map_b1, map_o0, map_o1, p, num_sms, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gesr
