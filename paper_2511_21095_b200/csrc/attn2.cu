// attn2.cu -- K-ATTN for d = 128 on a CTA PAIR (tcgen05 cta_group::2), persistent, with two
// softmax warpgroups that take alternate key tiles.
//
// Same contract as attn.cu (PAPER.md:341 mask rules (1)-(2): each candidate attends to all L_b
// history keys of its own request and to no other candidate; softmax per DESIGN.md R1).
//
// Why (profiles/r1_attn_trace.txt): in the 1-CTA kernel the softmax of a Q tile
// and its MMAs form one dependency chain (softmax(j) -> PV(j) -> S(j+1) -> softmax(j+1)), so a
// 128-key tile of two Q tiles takes ~3.8k cycles against ~2k of tensor work.  Here:
//   * a cluster of 2 CTAs works on one unit (request b, head h, 256 candidates); CTA r owns
//     candidate rows [128 r, 128 r + 128).  The leader issues M=256 MMAs for the pair: S = Q K^T
//     (SS; each CTA stages its Q tile and HALF of each K tile -- 64 keys), O += P V (TS; P from
//     each CTA's TMEM, each CTA stages HALF of each V tile -- 64 of the 128 d-columns), so each
//     SM moves half of the 1-CTA kernel's K/V bytes per row;
//   * the key tiles of a unit are dealt alternately to two softmax warpgroups: A takes the even
//     tiles, B the odd ones.  Each has its own S buffer (P aliased into it), its own O
//     accumulator and its own running max / sum; the two partial softmaxes are merged in the
//     epilogue (O = (O_A 2^(m_A-m) + O_B 2^(m_B-m)) / (l_A 2^(m_A-m) + l_B 2^(m_B-m))).  While
//     warpgroup A works on tile j, the tensor pipe runs PV(j-1) and S(j+1) for B: the chain of
//     one warpgroup spans two tiles, and each sub-partition always has a softmax warp with work;
//   * TMEM per CTA (512 columns): S_A [0,128), S_B [128,256), O_A [256,384), O_B [384,512);
//   * persistent: pair c takes work items c, c + G, ... (w -> unit w % U, head w / U), the next
//     unit's Q load and first S MMAs overlap the current unit's epilogue, and full 32-row output
//     slabs leave through TMA tensor stores.
// Warp roles per CTA: warp 0 TMA producer (both CTAs), warp 1 TMEM allocator + MMA issuer (leader
// only), warps 2-3 idle, warps 4-7 softmax A, warps 8-11 softmax B (warp w reads TMEM lane
// quarter w % 4: thread = candidate row, all 128 key columns of its tile).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace gesr {

#ifdef GESR_TRACE
__device__ unsigned long long g_trace2[64][64][8];
#define GESR_T2(e, j)                                                                          \
  do {                                                                                         \
    const int _b = blockIdx.x;                                                                 \
    if (_b < 64 && (j) < 64) g_trace2[_b][(j)][(e)] = clock64();                               \
  } while (0)
#else
#define GESR_T2(e, j) do {} while (0)
#endif

namespace {

constexpr int kD = 128;
constexpr int kKeys = 128;                       // keys per tile (S columns)
constexpr int kThreads = 384;
constexpr uint32_t kQBytes = 128 * kD * 2;       // 32 KB: Q tile, [2 col blocks][128 rows][64]
constexpr uint32_t kHalfBytes = 16384;           // K half [2][64 keys][64] or V half [128][64]
constexpr int kStages = 9;
constexpr uint32_t kQOff = 0;
constexpr uint32_t kRingOff = kQBytes;
constexpr uint32_t kStgOff = kRingOff + kStages * kHalfBytes;      // 2 x 2 KB boxes per softmax warp
constexpr uint32_t kBarOff = kStgOff + 8 * 4096;
constexpr uint32_t kXchOff = kBarOff + 256;                          // [unit parity][WG][m, l][row]
constexpr uint32_t kSmemBytes = kXchOff + 2 * 2 * 2 * 128 * 4 + 1024;
static_assert(kSmemBytes <= 232448, "shared memory budget");
// register split: launch registers 168 x 384 threads; control warps 88, softmax warps 208
constexpr int kCtrlRegs = 88;
constexpr int kSoftRegs = 208;
static_assert(128 * kCtrlRegs + 256 * kSoftRegs <= 168 * kThreads, "setmaxnreg pool");
// TMEM columns
constexpr uint32_t kTS = 0;          // S_A at 0, S_B at 128 (P_x aliases the first 64 columns)
constexpr uint32_t kTO = 256;        // O_A at 256, O_B at 384

__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1,
                                      float c0, float c1) {
  asm("{\n .reg .b64 a, b, c, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n"
      " mov.b64 c, {%6, %7};\n fma.rn.f32x2 d, a, b, c;\n mov.b64 {%0, %1}, d;\n}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void fadd2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n .reg .b64 a, b, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n"
      " add.rn.f32x2 d, a, b;\n mov.b64 {%0, %1}, d;\n}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
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

struct Work {
  int h, L, rows_valid, nkv;
  int64_t s0, cbeg;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap map_q,
                     const __grid_constant__ CUtensorMap map_kh,
                     const __grid_constant__ CUtensorMap map_vh,
                     const __grid_constant__ CUtensorMap map_o, const AttnParams p) {
  const int U = __ldg(p.unit_count);
  const int W = U * p.H;
  const int pair = static_cast<int>(blockIdx.x >> 1);
  const int npairs = static_cast<int>(gridDim.x >> 1);
  if (pair >= W) return;                          // uniform for the pair
  const uint32_t rank = cluster_ctarank();

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* q_full = reinterpret_cast<uint64_t*>(smem + kBarOff);   // leader's used
  uint64_t* q_empty = q_full + 1;                 // each CTA
  uint64_t* kv_full = q_empty + 1;                // [kStages]  (leader's used)
  uint64_t* kv_empty = kv_full + kStages;         // [kStages]  (each CTA)
  uint64_t* s_full = kv_empty + kStages;          // [2]        (each CTA)
  uint64_t* p_full = s_full + 2;                  // [2]        (leader; 8 warps of the pair)
  uint64_t* o_done = p_full + 2;                  //            (each CTA)
  uint64_t* o_free = o_done + 1;                  //            (leader; 16 warps of the pair)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_q);
    tma_prefetch_desc(&map_kh);
    tma_prefetch_desc(&map_vh);
    if (p.o_tma) tma_prefetch_desc(&map_o);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
    }
    mbar_init(o_done, 1);
    mbar_init(o_free, 16);
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

  // the unit descriptor of work item w is one 16-byte load, fetched one item ahead
  auto fetch = [&](int w) { return __ldg(p.units + (w % U)); };
  auto decode = [&](int w, int4 d) {
    Work x;
    x.h = w / U;
    x.s0 = d.x;
    x.L = d.y;
    x.cbeg = d.z;
    x.rows_valid = d.w;
    x.nkv = (x.L + kKeys - 1) / kKeys;
    return x;
  };

  if (warp < 4) {
    setmaxnreg_dec<kCtrlRegs>();
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer (both CTAs)
      if (elect_one()) {
        int stage = 0;
        uint32_t phase = 0;
        int m = 0;                                 // units with key tiles so far
        auto load_k = [&](int32_t krow, int jj) {
          mbar_wait_sleep(&kv_empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&kv_full[stage], 2 * kHalfBytes);
          uint8_t* dst = smem + kRingOff + stage * kHalfBytes;
          const int32_t row = krow + kKeys * jj + static_cast<int32_t>(rank) * 64;
          tma_load_2d_pair(dst, &map_kh, &kv_full[stage], 0, row);
          tma_load_2d_pair(dst + 8192, &map_kh, &kv_full[stage], 64, row);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        };
        auto load_v = [&](int32_t krow, int jj) {
          mbar_wait_sleep(&kv_empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&kv_full[stage], 2 * kHalfBytes);
          uint8_t* dst = smem + kRingOff + stage * kHalfBytes;
          tma_load_2d_pair(dst, &map_vh, &kv_full[stage], static_cast<int32_t>(rank) * 64,
                           krow + kKeys * jj);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        };
        int4 nx = fetch(pair);
        for (int w = pair; w < W; w += npairs) {
          const Work x = decode(w, nx);
          if (w + npairs < W) nx = fetch(w + npairs);
          if (x.nkv == 0) continue;
          if (m > 0) mbar_wait_sleep(q_empty, (m - 1) & 1);   // previous unit's S MMAs done with Q
          const int32_t qrow = static_cast<int32_t>(static_cast<int64_t>(x.h) * p.total_C + x.cbeg) +
                               static_cast<int32_t>(rank) * 128;
          if (rank == 0) mbar_arrive_expect_tx(q_full, 2 * kQBytes);
          tma_load_2d_pair(smem + kQOff, &map_q, q_full, 0, qrow);
          tma_load_2d_pair(smem + kQOff + kQBytes / 2, &map_q, q_full, 64, qrow);
          const int32_t krow = static_cast<int32_t>(static_cast<int64_t>(x.h) * p.total_L + x.s0);
          // consumption order of the MMA issuer: K0, K1, then per j: V_j, K_{j+2}
          load_k(krow, 0);
          if (x.nkv > 1) load_k(krow, 1);
          for (int j = 0; j < x.nkv; ++j) {
            load_v(krow, j);
            if (j + 2 < x.nkv) load_k(krow, j + 2);
          }
          ++m;
        }
      }
    } else if (warp == 1 && rank == 0) {
      // ---------------------------------------------------------- MMA issuer (leader only)
      const uint32_t idesc_s = make_idesc_bf16(256, kKeys, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16(256, kD, 0, 1);
      int stage = 0;
      uint32_t phase = 0;
      int m = 0;                                   // units with key tiles so far
      uint32_t pc0 = 0, pc1 = 0;                   // p_full phases of A / B
      auto take = [&]() {
        const int s = stage;
        mbar_wait_sleep(&kv_full[s], phase);
        if (++stage == kStages) { stage = 0; phase ^= 1; }
        return s;
      };
      auto issue_s = [&](int buf, int slot, bool last) {
        const uint32_t kb = sRing + slot * kHalfBytes;
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < kD / 16; ++ks)
            mma_ss_pair(tmem + kTS + buf * kKeys, kdesc(sQ, kQBytes / 2, ks), kdesc(kb, 8192, ks),
                        idesc_s, ks > 0 ? 1u : 0u);
          mma_commit_pair_mc(&s_full[buf], 0x3);
          mma_commit_pair_mc(&kv_empty[slot], 0x3);
          if (last) mma_commit_pair_mc(q_empty, 0x3);   // the unit's last S: Q may be reloaded
        }
        __syncwarp();
      };
      int4 nx = fetch(pair);
      for (int w = pair; w < W; w += npairs) {
        const Work x = decode(w, nx);
        if (w + npairs < W) nx = fetch(w + npairs);
        const int nkv = x.nkv;
        if (nkv == 0) continue;
        mbar_wait_sleep(q_full, m & 1);
        issue_s(0, take(), nkv == 1);
        if (nkv > 1) issue_s(1, take(), nkv == 2);
        for (int j = 0; j < nkv; ++j) {
          const int xb = j & 1;
          const int vslot = take();
          // the unit's first PV overwrites O_A: the previous unit's epilogue must be done
          if (j == 0 && m > 0) mbar_wait_sleep(o_free, (m - 1) & 1);
          mbar_wait_sleep(&p_full[xb], (xb ? pc1 : pc0) & 1);
          if (xb) ++pc1; else ++pc0;
          if (lane == 0) GESR_T2(4 + xb, m * 16 + j);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t vb = sRing + vslot * kHalfBytes;
#pragma unroll
            for (int ks = 0; ks < kKeys / 16; ++ks)
              mma_ts_pair(tmem + kTO + xb * kD, tmem + kTS + xb * kKeys + ks * 8, vdesc(vb, ks),
                          idesc_o, (j >= 2 || ks > 0) ? 1u : 0u);
            mma_commit_pair_mc(&kv_empty[vslot], 0x3);
            if (j == nkv - 1) mma_commit_pair_mc(o_done, 0x3);
          }
          __syncwarp();
          // S(j+2) reuses S(j)'s buffer: P(j) is read by the PV just issued (in order)
          if (j + 2 < nkv) issue_s(xb, take(), j + 2 == nkv - 1);
        }
        ++m;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    setmaxnreg_inc<kSoftRegs>();
    const int g = (static_cast<int>(warp) - 4) >> 2;   // warpgroup: 0 = A (even tiles), 1 = B
    const uint32_t sub = warp & 3;                       // TMEM lane quarter
    const int rloc = static_cast<int>(sub) * 32 + static_cast<int>(lane);
    const int row_in_unit = static_cast<int>(rank) * 128 + rloc;
    const uint32_t lane_addr = (sub * 32) << 16;
    const uint32_t tS = tmem + lane_addr + kTS + g * kKeys;
    const uint32_t tO = tmem + lane_addr + kTO;          // O_A; O_B at + kD
    const uint32_t tOg = tO + g * kD;
    const uint32_t p_full_leader = mapa_shared(smem_u32(&p_full[g]), 0);
    const uint32_t o_free_leader = mapa_shared(smem_u32(o_free), 0);
    const uint32_t xch = smem_u32(smem + kXchOff);
    uint8_t* stg = smem + kStgOff + (warp - 4) * 4096;
    const float sl2 = p.scale_log2;
    const int64_t HD = static_cast<int64_t>(p.H) * kD;
    int sc = 0;                                          // S tiles consumed by this warpgroup
    int m = 0;                                           // units with key tiles so far
    int4 nx = fetch(pair);
    for (int w = pair; w < W; w += npairs) {
      const Work x = decode(w, nx);
      if (w + npairs < W) nx = fetch(w + npairs);
      const int L = x.L, nkv = x.nkv, h = x.h;
      const bool row_ok = row_in_unit < x.rows_valid;
      const int64_t row = x.cbeg + row_in_unit;
      const int64_t col0 = static_cast<int64_t>(h) * kD + g * 64;   // my 64 output columns
      if (nkv == 0) {
        // L_b = 0: no keys, O = 0 and lse = -inf
        if (row_ok) {
          if (p.o_bf16) {
            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.O) + row * HD + col0);
#pragma unroll
            for (int v = 0; v < 8; ++v) dst[v] = make_uint4(0u, 0u, 0u, 0u);
          } else {
            float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.O) + row * HD + col0);
#pragma unroll
            for (int v = 0; v < 16; ++v) dst[v] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
          if (g == 0 && p.lse != nullptr) p.lse[row * p.H + h] = -INFINITY;
        }
        continue;
      }
      float m_run = -INFINITY;
      float l = 0.f;
      for (int j = g; j < nkv; j += 2) {
        mbar_wait_sleep(&s_full[g], sc & 1);
        ++sc;
        const bool tr = (sub == 0 && lane == 0);
        if (tr) GESR_T2(g, m * 16 + j);
        tc_fence_after();
        uint32_t r[kKeys];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, r + c * 32);
        tmem_ld_wait();
        const int valid = L - kKeys * j;
        const bool full = valid >= kKeys;
        if (!full) {
#pragma unroll
          for (int k = 0; k < kKeys; ++k)
            if (k >= valid) r[k] = __float_as_uint(-INFINITY);   // keys beyond L_b
        }
        // One fused pass per tile: p = 2^(s*scale*log2e - m) with the running max m of this
        // warpgroup's PREVIOUS tiles (speculative), the tile's own max reduced alongside.  Only
        // if the max grew by > 2^8 are p recomputed (from S, still in TMEM) and O_g rescaled;
        // the first tile reduces its max first.  P is packed in place into r[0, 64).
        uint32_t* pk = r;
        float acc[8];
        float mx[8];
        auto exp_pass = [&](float mm, bool with_max) {
          const float neg_m = -mm;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            acc[e] = 0.f;
            mx[e] = -INFINITY;
          }
#pragma unroll
          for (int k = 0; k < kKeys / 2; ++k) {
            const float s0v = __uint_as_float(r[2 * k]), s1v = __uint_as_float(r[2 * k + 1]);
            if (with_max) {
              mx[(2 * k) & 7] = fmaxf(mx[(2 * k) & 7], s0v);
              mx[(2 * k + 1) & 7] = fmaxf(mx[(2 * k + 1) & 7], s1v);
            }
            float x0, x1;
            ffma2(x0, x1, s0v, s1v, sl2, sl2, neg_m, neg_m);
            const float p0 = ex2(x0), p1 = ex2(x1);
            const int a = (k & 3) * 2;
            fadd2(acc[a], acc[a + 1], acc[a], acc[a + 1], p0, p1);
            pk[k] = pack_bf16x2(p0, p1);
          }
        };
        const bool first = j == g;
        if (first) {
#pragma unroll
          for (int e = 0; e < 8; ++e) mx[e] = -INFINITY;
#pragma unroll
          for (int k = 0; k < kKeys; ++k) mx[k & 7] = fmaxf(mx[k & 7], __uint_as_float(r[k]));
        } else {
          exp_pass(m_run, true);
        }
        const float mraw = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                 fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        const float mt = mraw * sl2;
        if (first) {
          m_run = mt;
          exp_pass(m_run, false);
        } else {
          const bool need = mt > m_run + 8.0f;
          if (__any_sync(0xffffffffu, need)) {
            // O_g holds PV(j-2): S_g(j) was issued after it and has completed
            float alpha = 1.f;
            if (need) {
              alpha = ex2(m_run - mt);
              m_run = mt;
              l *= alpha;
            }
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              uint32_t o[32];
              tmem_ld32(tOg + c * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              tmem_st32(tOg + c * 32, o);
            }
            tmem_st_wait();
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, r + c * 32);
            tmem_ld_wait();
            if (!full) {
#pragma unroll
              for (int k = 0; k < kKeys; ++k)
                if (k >= valid) r[k] = __float_as_uint(-INFINITY);
            }
            exp_pass(m_run, false);   // recompute P with the new running max
          }
        }
        l += ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        tmem_st32(tS, pk);
        tmem_st32(tS + 32, pk + 32);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (tr) GESR_T2(2 + g, m * 16 + j);
        if (lane == 0) mbar_arrive_cluster_relaxed(p_full_leader);
      }
      // ---------------- epilogue: merge the two partial softmaxes of my rows, O for my columns
      const uint32_t xb = xch + ((m & 1) * 2 * 2 * 128) * 4;      // [WG][m, l][row]
      st_shared_f32(xb + ((g * 2 + 0) * 128 + rloc) * 4, m_run);
      st_shared_f32(xb + ((g * 2 + 1) * 128 + rloc) * 4, l);
      named_bar_sync(1 + sub, 64);                        // warp sub of A and of B
      const float m_o = ld_shared_f32(xb + (((1 - g) * 2 + 0) * 128 + rloc) * 4);
      const float l_o = ld_shared_f32(xb + (((1 - g) * 2 + 1) * 128 + rloc) * 4);
      const float mA = g == 0 ? m_run : m_o, lA = g == 0 ? l : l_o;
      const float mB = g == 0 ? m_o : m_run, lB = g == 0 ? l_o : l;
      const bool hasB = nkv > 1;
      const float mm = hasB ? fmaxf(mA, mB) : mA;
      const float wA = ex2(mA - mm);
      const float wB = hasB ? ex2(mB - mm) : 0.f;
      const float lsum = lA * wA + lB * wB;
      const float inv = 1.0f / lsum;
      const float fA = wA * inv, fB = wB * inv;
      mbar_wait_sleep(o_done, m & 1);
      tc_fence_after();
      const bool use_tma = p.o_tma && static_cast<int>(rank) * 128 + static_cast<int>(sub) * 32 + 32 <= x.rows_valid;
#pragma unroll 1
      for (int cc = 0; cc < 2; ++cc) {
        const int c = g * 2 + cc;                        // 32-column chunk of O
        uint32_t oa[32], ob[32];
        tmem_ld32(tO + c * 32, oa);
        if (hasB) tmem_ld32(tO + kD + c * 32, ob);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e)
          v[e] = hasB ? __uint_as_float(oa[e]) * fA + __uint_as_float(ob[e]) * fB
                      : __uint_as_float(oa[e]) * fA;
        if (use_tma) {
          uint32_t pk2[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) pk2[e] = pack_bf16x2(v[2 * e], v[2 * e + 1]);
          if (lane == 0) bulk_wait_group_read<1>();       // box (cc) read by its previous store
          __syncwarp();
          uint8_t* box = stg + cc * 2048;
          uint8_t* rowp = box + lane * 64;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(rowp + ((q ^ ((lane >> 1) & 3)) << 4)) =
                make_uint4(pk2[4 * q], pk2[4 * q + 1], pk2[4 * q + 2], pk2[4 * q + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&map_o, box, c * 32, h,
                         static_cast<int32_t>(x.cbeg + static_cast<int>(rank) * 128 + static_cast<int>(sub) * 32));
            bulk_commit_group();
          }
        } else if (row_ok) {
          if (p.o_bf16) {
            uint32_t pk2[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) pk2[e] = pack_bf16x2(v[2 * e], v[2 * e + 1]);
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.O) + row * HD + static_cast<int64_t>(h) * kD + c * 32;
            st_global_v8(dst, pk2);
            st_global_v8(dst + 16, pk2 + 8);
          } else {
            float* dst = static_cast<float*>(p.O) + row * HD + static_cast<int64_t>(h) * kD + c * 32;
#pragma unroll
            for (int vv = 0; vv < 4; ++vv) st_global_v8(dst + 8 * vv, reinterpret_cast<const uint32_t*>(v) + 8 * vv);
          }
        }
      }
      if (g == 0 && row_ok && p.lse != nullptr)
        p.lse[row * p.H + h] = (mm + __log2f(lsum)) * 0.69314718055994530942f;
      // O_A / O_B drained: the next unit's first PV may overwrite them
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(o_free_leader);
      if (sub == 0 && lane == 0) GESR_T2(6 + g, m * 16 + nkv - 1);
      ++m;
    }
    if (lane == 0) bulk_wait_group<0>();   // staging boxes stay allocated until read
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
                             const CUtensorMap& mo, const AttnParams& p, int64_t max_units,
                             cudaStream_t stream) {
  static int max_pairs = 0;
  if (max_pairs == 0) {
    cudaError_t e = cudaFuncSetAttribute(attn_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemBytes);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.gridDim = dim3(2, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    e = cudaOccupancyMaxActiveClusters(&clusters, attn_pair_kernel, &cfg);
    if (e != cudaSuccess || clusters <= 0) {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      clusters = sms / 2;
      (void)cudaGetLastError();
    }
    max_pairs = clusters;
  }
  const int64_t work = max_units * p.H;
  const unsigned pairs = static_cast<unsigned>(work < max_pairs ? work : max_pairs);
  attn_pair_kernel<<<2 * pairs, kThreads, kSmemBytes, stream>>>(mq, mkh, mvh, mo, p);
  return cudaGetLastError();
}

}  // namespace gesr
