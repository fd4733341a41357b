// attn2.cu -- K-ATTN v2 for d = 128: CTA-PAIR (tcgen05 cta_group::2) jagged attention with a
// double-buffered S and P in its own TMEM columns.
//
// Same contract as attn.cu (PAPER.md:341 mask rules (1)-(2): each candidate attends to all L_b
// history keys of its own request and to no other candidate; softmax per DESIGN.md R1).
//
// Why a second design (profiles/r1_attn_trace.txt): in the 1-CTA kernel P aliases S, so S(j+1)
// can only be issued after PV(j) has consumed P(j); the softmax and the MMAs then alternate on
// one critical path (3.8k cycles per 128-key tile instead of ~2k).  Here:
//   * a cluster of 2 CTAs works on one unit (request b, head h, 256 candidates); CTA r owns
//     candidate rows [128 r, 128 r + 128) and its 128 x 128 slice of every S and of O;
//   * the leader issues M=256 MMAs for the pair: S = Q K^T (SS; each CTA stages its Q tile and
//     HALF of each K tile -- 64 keys), O += P V (TS; P from each CTA's TMEM, each CTA stages HALF
//     of each V tile -- 64 of the 128 d-columns).  Per SM, K/V smem traffic and MMA operand reads
//     are half of the 1-CTA kernel's;
//   * TMEM per CTA: S_a [0,128) S_b [128,256) P [256,320) O [320,448): S is double buffered and
//     P is separate, so S(j+2) is issued as soon as both CTAs have LOADED S(j) (s_free), long
//     before P(j) exists, and the softmax of tile j+1 starts right after tile j's: the tensor
//     pipe and the softmax overlap instead of alternating.
// Warp roles per CTA: warp 0 TMA producer (both CTAs), warp 1 TMEM allocator + MMA issuer (leader
// only), warps 4-11 softmax (2 warps per TMEM lane quarter, each owning 64 key columns; row max /
// sum exchanged through smem) + epilogue.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace gesr {

#ifdef GESR_TRACE
__device__ unsigned long long g_trace2[64][32][8];
#define GESR_T2(e, j)                                                                          \
  do {                                                                                         \
    const int _b = blockIdx.x + blockIdx.y * gridDim.x;                                        \
    if (_b < 64 && (j) < 32) g_trace2[_b][(j)][(e)] = clock64();                               \
  } while (0)
#else
#define GESR_T2(e, j) do {} while (0)
#endif

namespace {

constexpr int kD = 128;
#ifndef GESR_PAIR_POLY_EVERY
#define GESR_PAIR_POLY_EVERY 1000   // one pair in N takes the FMA-pipe exp2 on full tiles
#endif
constexpr int kThreads = 384;
constexpr int kKeys = 128;                       // keys per tile (S columns)
constexpr uint32_t kQBytes = 128 * kD * 2;       // 32 KB: Q tile, [2 col blocks][128 rows][64]
constexpr uint32_t kHalfBytes = 16384;           // K half [2][64 keys][64] or V half [128][64]
constexpr int kStages = 8;
constexpr uint32_t kQOff = 0;
constexpr uint32_t kRingOff = kQBytes;
constexpr uint32_t kBarOff = kRingOff + kStages * kHalfBytes;     // 160 KB
constexpr uint32_t kXchOff = kBarOff + 512;
constexpr uint32_t kXchBytes = 2 * 2 * 128 * 4 + 2 * 128 * 4;      // max [half][buf][row], sum
constexpr uint32_t kSmemBytes = kXchOff + kXchBytes + 1024;
// TMEM columns
constexpr uint32_t kTS = 0;          // S_a at 0, S_b at 128
constexpr uint32_t kTP = 256;        // P (bf16 pairs): 64 columns
constexpr uint32_t kTO = 320;        // O: 128 columns
constexpr int kCtrlRegs = 88;
constexpr int kSoftRegs = 208;
static_assert(128 * kCtrlRegs + 256 * kSoftRegs <= 168 * kThreads, "setmaxnreg pool");

__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1,
                                      float c0, float c1) {
  asm("{\n .reg .b64 a, b, c, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n"
      " mov.b64 c, {%6, %7};\n fma.rn.f32x2 d, a, b, c;\n mov.b64 {%0, %1}, d;\n}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
// 2^x for a pair on the FMA/ALU pipes (MUFU offload): round-to-nearest split x = j + f with the
// 1.5*2^23 magic-number add, degree-3 polynomial for 2^f on [-0.5, 0.5] (max rel. error
// 2.1e-4, below the bf16 rounding of P), exponent added in the integer domain; x clamped at -126.
__device__ __forceinline__ void exp2_poly2(float& y0, float& y1, float x0, float x1);

__device__ __forceinline__ void fadd2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n .reg .b64 a, b, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n"
      " add.rn.f32x2 d, a, b;\n mov.b64 {%0, %1}, d;\n}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

__device__ __forceinline__ void exp2_poly2(float& y0, float& y1, float x0, float x1) {
  constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23
  x0 = fmaxf(x0, -126.0f);
  x1 = fmaxf(x1, -126.0f);
  float t0, t1, r0, r1, f0, f1, p0, p1;
  fadd2(t0, t1, x0, x1, kMagic, kMagic);
  fadd2(r0, r1, t0, t1, -kMagic, -kMagic);
  ffma2(f0, f1, r0, r1, -1.0f, -1.0f, x0, x1);
  ffma2(p0, p1, f0, f1, 0.054848f, 0.054848f, 0.24180661f, 0.24180661f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.6932482f, 0.6932482f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.99998866f, 0.99998866f);
  y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

// K-major descriptor (SW128) for a [rows][128] bf16 tile stored as 2 column blocks of
// `block_bytes` each, at K step ks (16 elements).
__device__ __forceinline__ uint64_t kdesc(uint32_t base, uint32_t block_bytes, int ks) {
  const int e = ks * 16;
  return make_sdesc(base + (e >> 6) * block_bytes + (e & 63) * 2, 16, 1024, kSwizzle128B);
}
// MN-major V-half descriptor (one 64-column SW128 atom column, 128 keys) at key step ks.
__device__ __forceinline__ uint64_t vdesc(uint32_t base, int ks) {
  return make_sdesc(base + ks * 16 * 128, 8192, 1024, kSwizzle128B);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap map_q,
                     const __grid_constant__ CUtensorMap map_kh,
                     const __grid_constant__ CUtensorMap map_vh, const AttnParams p) {
  const int u = blockIdx.x >> 1;
  if (u >= __ldg(p.unit_count)) return;   // uniform for the pair
  const uint32_t rank = cluster_ctarank();
  const int h = blockIdx.y;
  const int4 unit = p.units[u];
  const int64_t s0 = unit.x;
  const int L = unit.y;
  const int64_t cbeg = unit.z;
  const int rows_valid = unit.w;
  const int nkv = (L + kKeys - 1) / kKeys;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* q_full = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint64_t* kv_full = q_full + 1;                 // [kStages]  (leader's are used)
  uint64_t* kv_empty = kv_full + kStages;         // [kStages]  (each CTA)
  uint64_t* s_full = kv_empty + kStages;          // [2]        (each CTA)
  uint64_t* s_free = s_full + 2;                  // [2]        (leader; count 2)
  uint64_t* p_full = s_free + 2;                  //            (leader; count 2)
  uint64_t* p_free = p_full + 1;                  //            (each CTA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_free + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_q);
    tma_prefetch_desc(&map_kh);
    tma_prefetch_desc(&map_vh);
    mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 16);     // one arrival per softmax warp of the pair
    }
    mbar_init(p_full, 16);
    mbar_init(p_free, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc_pair(tmem_slot, 512);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sQ = smem_u32(smem + kQOff);
  const uint32_t sRing = smem_u32(smem + kRingOff);

  if (warp < 4) {
    setmaxnreg_dec<kCtrlRegs>();
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer (both CTAs)
      if (nkv > 0 && elect_one()) {
        const int32_t qrow = static_cast<int32_t>(static_cast<int64_t>(h) * p.total_C + cbeg) +
                             static_cast<int32_t>(rank) * 128;
        if (rank == 0) mbar_arrive_expect_tx(q_full, 2 * kQBytes);
        tma_load_2d_pair(smem + kQOff, &map_q, q_full, 0, qrow);
        tma_load_2d_pair(smem + kQOff + kQBytes / 2, &map_q, q_full, 64, qrow);
        const int32_t krow = static_cast<int32_t>(static_cast<int64_t>(h) * p.total_L + s0);
        int stage = 0;
        uint32_t phase = 0;
        // consumption order of the MMA issuer: K0, K1, then per j: V_j, K_{j+2}
        auto load_k = [&](int jj) {
          mbar_wait_sleep(&kv_empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&kv_full[stage], 2 * kHalfBytes);
          uint8_t* dst = smem + kRingOff + stage * kHalfBytes;
          const int32_t row = krow + kKeys * jj + static_cast<int32_t>(rank) * 64;
          tma_load_2d_pair(dst, &map_kh, &kv_full[stage], 0, row);
          tma_load_2d_pair(dst + 8192, &map_kh, &kv_full[stage], 64, row);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        };
        auto load_v = [&](int jj) {
          mbar_wait_sleep(&kv_empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&kv_full[stage], 2 * kHalfBytes);
          uint8_t* dst = smem + kRingOff + stage * kHalfBytes;
          tma_load_2d_pair(dst, &map_vh, &kv_full[stage], static_cast<int32_t>(rank) * 64,
                           krow + kKeys * jj);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        };
        load_k(0);
        if (nkv > 1) load_k(1);
        for (int j = 0; j < nkv; ++j) {
          load_v(j);
          if (j + 2 < nkv) load_k(j + 2);
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer (leader only)
      if (rank == 0 && nkv > 0) {
        const uint32_t idesc_s = make_idesc_bf16(256, kKeys, 0, 0);
        const uint32_t idesc_o = make_idesc_bf16(256, kD, 0, 1);
        int stage = 0;
        uint32_t phase = 0;
        auto take = [&]() {
          const int s = stage;
          mbar_wait_sleep(&kv_full[s], phase);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
          return s;
        };
        auto issue_s = [&](int buf, int slot) {
          const uint32_t kb = sRing + slot * kHalfBytes;
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < kD / 16; ++ks)
              mma_ss_pair(tmem + kTS + buf * kKeys, kdesc(sQ, kQBytes / 2, ks), kdesc(kb, 8192, ks),
                          idesc_s, ks > 0 ? 1u : 0u);
            mma_commit_pair_mc(&s_full[buf], 0x3);
            mma_commit_pair_mc(&kv_empty[slot], 0x3);
          }
          __syncwarp();
        };
        mbar_wait_sleep(q_full, 0);
        issue_s(0, take());
        if (nkv > 1) issue_s(1, take());
        for (int j = 0; j < nkv; ++j) {
          const int vslot = take();
          if (lane == 0) GESR_T2(3, j);
          if (j + 2 < nkv) {
            // S(j+2) reuses S(j)'s buffer: both CTAs must have loaded S(j) into registers
            mbar_wait_sleep(&s_free[j & 1], (j >> 1) & 1);
            if (lane == 0) GESR_T2(4, j);
            issue_s(j & 1, take());
          }
          mbar_wait_sleep(p_full, j & 1);
          if (lane == 0) GESR_T2(5, j);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t vb = sRing + vslot * kHalfBytes;
#pragma unroll
            for (int ks = 0; ks < kKeys / 16; ++ks)
              mma_ts_pair(tmem + kTO, tmem + kTP + ks * 8, vdesc(vb, ks), idesc_o,
                          (j > 0 || ks > 0) ? 1u : 0u);
            mma_commit_pair_mc(p_free, 0x3);
            mma_commit_pair_mc(&kv_empty[vslot], 0x3);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    // Per key tile, one fused pass: p = 2^(s*scale*log2e - m_run) with the running max of the
    // PREVIOUS tiles, the tile's own max reduced alongside (FMNMX beside MUFU), one pair in
    // GESR_PAIR_POLY_EVERY through the FMA-pipe polynomial exp2.  Only if the max grew by more
    // than 2^8 (rare after the first tile) are p recomputed with the new max and O rescaled; the
    // first tile computes its max first.  S(j+1) (double buffer) is loaded from TMEM while tile j's
    // P is handed off, so the TMEM load latency is off the critical path.
    setmaxnreg_inc<kSoftRegs>();
    const int sw = warp - 4;
    const int half = sw >> 2;                   // key-column half of this warp
    const uint32_t sub = warp & 3;              // TMEM lane quarter
    const int rloc = sub * 32 + lane;           // row within this CTA's Q tile
    const int row_in_unit = static_cast<int>(rank) * 128 + rloc;
    float* xmax = reinterpret_cast<float*>(smem + kXchOff);   // [half][buf][row]
    float* xsum = xmax + 2 * 2 * 128;                          // [half][row]
    const uint32_t bar_pair = 3 + sub;          // the two warps of a lane quarter (64 threads)
    const uint32_t lane_addr = (sub * 32) << 16;
    const uint32_t tS = tmem + lane_addr + kTS + half * 64;
    const uint32_t tP = tmem + lane_addr + kTP + half * 32;
    const uint32_t tO = tmem + lane_addr + kTO + half * 64;
    const uint32_t s_free_leader0 = mapa_shared(smem_u32(&s_free[0]), 0);
    const uint32_t s_free_leader1 = mapa_shared(smem_u32(&s_free[1]), 0);
    const uint32_t p_full_leader = mapa_shared(smem_u32(p_full), 0);
    const float sl2 = p.scale_log2;
    float m_run = -INFINITY;
    float l = 0.f;

    auto load_s = [&](int j, uint32_t* r) {       // wait S(j) and start its TMEM load
      mbar_wait_sleep(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      tmem_ld32(tS + (j & 1) * kKeys, r);
      tmem_ld32(tS + (j & 1) * kKeys + 32, r + 32);
    };
    auto release_s = [&](int j) {                 // S(j) landed in registers: free its buffer
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed((j & 1) ? s_free_leader1 : s_free_leader0);
    };
    uint32_t r[64];
    if (nkv > 0) {
      load_s(0, r);
      release_s(0);
    }
    for (int j = 0; j < nkv; ++j) {
      // r holds S(j); S(j+1) is loaded into r once S(j) is dead (completed at the end)
      if (sw == 0 && lane == 0) GESR_T2(0, j);
      const int valid = L - kKeys * j - half * 64;      // valid keys among my 64 columns
      const bool full = valid >= 64;
      if (!full) {
#pragma unroll
        for (int k = 0; k < 64; ++k)
          if (k >= valid) r[k] = __float_as_uint(-INFINITY);
      }
      uint32_t pk[32];
      float acc[8];
      float mx[8];
      auto exp_pass = [&](float m, bool with_max) {
        const float neg_m = -m;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          acc[e] = 0.f;
          mx[e] = -INFINITY;
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float s0v = __uint_as_float(r[2 * k]), s1v = __uint_as_float(r[2 * k + 1]);
          if (with_max) {
            mx[(2 * k) & 7] = fmaxf(mx[(2 * k) & 7], s0v);
            mx[(2 * k + 1) & 7] = fmaxf(mx[(2 * k + 1) & 7], s1v);
          }
          float x0, x1, p0, p1;
          ffma2(x0, x1, s0v, s1v, sl2, sl2, neg_m, neg_m);
          if ((k % GESR_PAIR_POLY_EVERY) == GESR_PAIR_POLY_EVERY - 1 && full) {
            exp2_poly2(p0, p1, x0, x1);
          } else {
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          const int a = (k & 3) * 2;
          fadd2(acc[a], acc[a + 1], acc[a], acc[a + 1], p0, p1);
          pk[k] = pack_bf16x2(p0, p1);
        }
      };
      float mraw;
      if (j == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) mx[e] = -INFINITY;
#pragma unroll
        for (int k = 0; k < 64; ++k) mx[k & 7] = fmaxf(mx[k & 7], __uint_as_float(r[k]));
      } else {
        if (sw == 0 && lane == 0) GESR_T2(1, j);
        exp_pass(m_run, true);     // speculative: assumes the running max still holds
        if (sw == 0 && lane == 0) GESR_T2(7, j);
      }
      mraw = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                   fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      xmax[(half * 2 + (j & 1)) * 128 + rloc] = mraw;
      named_bar_sync(bar_pair, 64);
      mraw = fmaxf(mraw, xmax[((1 - half) * 2 + (j & 1)) * 128 + rloc]);
      const float mt = mraw * sl2;
      if (j == 0) {
        m_run = mt;
        exp_pass(m_run, false);
      } else {
        const bool need = mt > m_run + 8.0f;
        if (__any_sync(0xffffffffu, need)) {
          // O must hold PV(j-1) before it is rescaled
          mbar_wait_sleep(p_free, (j - 1) & 1);
          tc_fence_after();
          float alpha = 1.f;
          if (need) {
            alpha = ex2(m_run - mt);
            m_run = mt;
            l *= alpha;
          }
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st32(tO + c * 32, o);
          }
          tmem_st_wait();
          exp_pass(m_run, false);  // recompute P with the new running max
        }
      }
      // r is dead from here on: start loading S(j+1) so its latency overlaps the P hand-off
      if (j + 1 < nkv) load_s(j + 1, r);
      l += ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
      if (sw == 0 && lane == 0) GESR_T2(6, j);
      // P(j-1) must have been consumed by PV(j-1) before P is overwritten
      if (j > 0) {
        mbar_wait_sleep(p_free, (j - 1) & 1);
        tc_fence_after();
      }
      tmem_st32(tP, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (sw == 0 && lane == 0) GESR_T2(2, j);
      if (lane == 0) mbar_arrive_cluster_relaxed(p_full_leader);
      if (j + 1 < nkv) release_s(j + 1);
    }
    // ---------------- epilogue: O / l for my 64 columns of my rows
    xsum[half * 128 + rloc] = l;
    named_bar_sync(bar_pair, 64);
    l += xsum[(1 - half) * 128 + rloc];
    const bool row_ok = row_in_unit < rows_valid;
    const int64_t row = cbeg + row_in_unit;
    const int64_t HD = static_cast<int64_t>(p.H) * kD;
    if (nkv > 0) {
      mbar_wait_sleep(p_free, (nkv - 1) & 1);
      tc_fence_after();
    }
    const float inv_l = nkv > 0 ? 1.0f / l : 0.f;
    const int64_t col0 = static_cast<int64_t>(h) * kD + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t o[32];
      if (nkv > 0) {
        tmem_ld32(tO + c * 32, o);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0u;
      }
      if (row_ok) {
        if (p.o_bf16) {
          uint32_t pk2[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            pk2[e] = pack_bf16x2(__uint_as_float(o[2 * e]) * inv_l, __uint_as_float(o[2 * e + 1]) * inv_l);
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.O) + row * HD + col0 + c * 32);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            dst[v] = make_uint4(pk2[4 * v], pk2[4 * v + 1], pk2[4 * v + 2], pk2[4 * v + 3]);
        } else {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.O) + row * HD + col0 + c * 32);
#pragma unroll
          for (int v = 0; v < 8; ++v)
            dst[v] = make_float4(__uint_as_float(o[4 * v]) * inv_l, __uint_as_float(o[4 * v + 1]) * inv_l,
                                 __uint_as_float(o[4 * v + 2]) * inv_l, __uint_as_float(o[4 * v + 3]) * inv_l);
        }
      }
    }
    if (row_ok && half == 0 && p.lse != nullptr)
      p.lse[row * p.H + h] = nkv > 0 ? (m_run + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

}  // namespace

#ifdef GESR_TRACE
extern "C" int gesr_debug_trace2_copy(void* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace2, sizeof(g_trace2)));
}
#endif

cudaError_t launch_attn_pair(const CUtensorMap& mq, const CUtensorMap& mkh, const CUtensorMap& mvh,
                             const AttnParams& p, int64_t max_units, cudaStream_t stream) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(attn_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  dim3 grid(static_cast<unsigned>(2 * max_units), static_cast<unsigned>(p.H));
  attn_pair_kernel<<<grid, kThreads, kSmemBytes, stream>>>(mq, mkh, mvh, p);
  return cudaGetLastError();
}

}  // namespace gesr
