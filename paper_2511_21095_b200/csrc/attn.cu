// attn.cu -- K-SCHED (work list) and K-ATTN: jagged many-candidates-to-one-history attention.
//
// For request b, head h, candidate t: O[t, h*d:(h+1)*d] = softmax_i(scale q_t . K[h, r_i]) V[h, r_i]
// over the L_b history rows r_i of request b only (PAPER.md:341 mask rules (1)-(2): candidates
// never attend to one another; PAPER.md:346 T_self rows; softmax per DESIGN.md R1).
//
// B200 design (one CTA per work unit = (request b, head h, 256 candidates)):
//   warp 0      TMA producer: the two 128-row Q tiles once, then K_j, V_j tiles (128 keys x d,
//               128B swizzle) of the user's head-major cache slab through a 4-slot mbarrier ring.
//               C candidates share one L x d K/V: the cache is read once per 256 candidates.
//   warp 1      TMEM allocator + MMA issuer (one elected thread):
//                 S_i = Q_i K_j^T    tcgen05.mma kind::f16 SS, M=128 N=128, fp32 in TMEM
//                 O_i += P_i V_j     tcgen05.mma kind::f16 TS: P (bf16) read from TMEM, V MN-major
//               interleaved so that Q tile 0's softmax overlaps Q tile 1's MMAs (ping-pong).
//   warps 4-7   softmax for Q tile 0, warps 8-11 for Q tile 1: thread = candidate row;
//               tcgen05.ld the 128 scores, mask keys >= L_b, online max with lazy rescale
//               (only when the max grows by > 2^8), exp2 with log2(e) folded into the scale,
//               running row sum in fp32, P packed to bf16 and tcgen05.st back over S.
//               Epilogue: O / l from TMEM, fp32 or bf16 stores, natural-log lse.
// TMEM: S0 [0,128) S1 [128,256) O0 [256,256+d) O1 [256+d, 256+2d) of 512 columns.
// Every row's arithmetic depends only on its own q and its user's K/V (fixed 128-key tiling
// from the user's first row), so outputs are batch-composition invariant (R9).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace gesr {

#ifdef GESR_TRACE
// Debug-only timeline trace (build with -DGESR_TRACE): clock64 at pipeline events for the first
// 64 CTAs and 32 key tiles.  Not part of the product library.
__device__ unsigned long long g_trace[64][64][8];
#define GESR_T(e, j)                                                                           \
  do {                                                                                         \
    const int _b = blockIdx.x + blockIdx.y * gridDim.x;                                        \
    if (_b < 64 && (j) < 64) g_trace[_b][(j)][(e)] = clock64();                                \
  } while (0)
#else
#define GESR_T(e, j) do {} while (0)
#endif

namespace {

constexpr int kBlockKeys = 128;
#ifndef GESR_ATTN_SPLIT
#define GESR_ATTN_SPLIT 1      // softmax warps per TMEM lane quarter and Q tile (d >= 64); 2 measured slower
#endif
#ifndef GESR_POLY_EVERY
#define GESR_POLY_EVERY 1000   // one pair in N takes the FMA-pipe exp2 (off: measured slower)
#endif

template <int D>
struct AttnCfg {
  static constexpr int kBoxCols = D >= 64 ? 64 : 32;              // elements per swizzle row
  static constexpr uint32_t kLayout = D >= 64 ? kSwizzle128B : kSwizzle64B;
  static constexpr int kColBlocks = D / kBoxCols;                 // 2 for d=128, else 1
  static constexpr uint32_t kRowBytes = kBoxCols * 2;             // 128 or 64
  static constexpr uint32_t kBoxBytes = 128 * kRowBytes;          // one 128-row box
  static constexpr uint32_t kTileBytes = kColBlocks * kBoxBytes;  // 128 rows x D bf16
  static constexpr uint32_t kSBO = 8 * kRowBytes;                 // 8-row core-matrix group
  static constexpr int kStages = 4;
  // softmax warps per (Q tile, TMEM lane quarter): 2 for d >= 64 (each takes half of the 128
  // key columns of its 32 rows: more warps per sub-partition to hide latency), 1 for d = 32
  static constexpr int kSplit = D >= 64 ? GESR_ATTN_SPLIT : 1;
  static constexpr int kThreads = 128 + 2 * 128 * kSplit;
  // setmaxnreg budget: the CTA's register pool is (launch registers x threads), launch
  // registers = floor(65536 / threads / 8) * 8; the split must fit in that pool.
  static constexpr int kLaunchRegs = (65536 / kThreads) / 8 * 8;
  static constexpr int kCtrlRegs = kSplit == 2 ? 56 : 88;
  static constexpr int kSoftRegs = kSplit == 2 ? 104 : 208;
  static_assert(128 * kCtrlRegs + 256 * kSplit * kSoftRegs <= kLaunchRegs * kThreads,
                "setmaxnreg split exceeds the CTA register pool");
  static constexpr uint32_t kQOff = 0;
  static constexpr uint32_t kKVOff = 2 * kTileBytes;
  static constexpr uint32_t kBarOff = kKVOff + kStages * kTileBytes;
  static constexpr uint32_t kXchOff = kBarOff + 256;          // row-max / row-sum exchange
  static constexpr uint32_t kXchBytes = kSplit == 2 ? 2 * 2 * 2 * 128 * 4 + 2 * 2 * 128 * 4 : 0;
  // bf16 O epilogue staging (kSplit == 1): two 2 KB boxes (32 rows x 32 columns, 64B swizzle)
  // per softmax warp, drained by TMA tensor stores while the warp moves on to the next unit
  static constexpr uint32_t kStgOff = (kXchOff + kXchBytes + 1023) / 1024 * 1024;   // swizzle atom aligned
  static constexpr uint32_t kStgBytes = kSplit == 1 ? 8 * 2 * 2048 : 0;
  static constexpr uint32_t kSmemBytes = kStgOff + kStgBytes + 1024;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
};

// K-major operand (Q or K tile) descriptor for the 16-element K step `ks`.
template <int D>
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t base, int ks) {
  using C = AttnCfg<D>;
  const int e = ks * 16;
  const uint32_t addr = base + (e / C::kBoxCols) * C::kBoxBytes + (e % C::kBoxCols) * 2;
  return make_sdesc(addr, 16, C::kSBO, C::kLayout);
}

// MN-major V tile descriptor for the 16-key K step `ks` (N = d spans kColBlocks atoms).
template <int D>
__device__ __forceinline__ uint64_t v_desc(uint32_t base, int ks) {
  using C = AttnCfg<D>;
  return make_sdesc(base + ks * 16 * C::kRowBytes, C::kBoxBytes, C::kSBO, C::kLayout);
}


// 2^x for a pair on the FMA/ALU pipes (FA4-style MUFU offload): round-to-nearest split
// x = j + f (f in [-0.5, 0.5]) with the 1.5*2^23 magic-number add, degree-3 polynomial for 2^f
// (max rel. error 2.1e-4, well below the bf16 rounding of P), exponent added in the integer
// domain.  Inputs are clamped at -126 so the exponent field never underflows.
__device__ __forceinline__ void exp2_poly2(float& y0, float& y1, float x0, float x1) {
  constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23
  x0 = fmaxf(x0, -126.0f);
  x1 = fmaxf(x1, -126.0f);
  float t0, t1, r0, r1, f0, f1, p0, p1;
  fadd2(t0, t1, x0, x1, kMagic, kMagic);          // low mantissa bits hold round(x)
  fadd2(r0, r1, t0, t1, -kMagic, -kMagic);        // round(x) as float
  ffma2(f0, f1, r0, r1, -1.0f, -1.0f, x0, x1);    // f = x - round(x)
  ffma2(p0, p1, f0, f1, 0.054848f, 0.054848f, 0.24180661f, 0.24180661f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.6932482f, 0.6932482f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.99998866f, 0.99998866f);
  y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

// kCausal: history self-attention; kHstu: HSTU pointwise normalisation SiLU(s)/L_b instead of
// the softmax (GESR_TASA_HSTU_SILU; reading R20).  Separate instantiations keep the
// default kernel's code unchanged.
template <int D, bool kCausal, bool kHstu>
__global__ void __launch_bounds__(AttnCfg<D>::kThreads, 1)
    attn_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_o,
                const AttnParams p) {
  using C = AttnCfg<D>;
  // Persistent: CTA c processes work items w = c, c + G, ... of W = units x H, w -> (unit
  // w % U, head w / U): neighbouring CTAs work on the pairs of the same (request, head) at the
  // same time, so each K/V slab is fetched from HBM once and re-read from L2.  The next unit's
  // Q load and first S MMA overlap the current unit's epilogue.
  pdl_launch_dependents();
  pdl_wait();
  const int U = unit_count_of(p);
  const int W = U * p.H;
  if (static_cast<int>(blockIdx.x) >= W) return;   // uniform for the whole CTA

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* q_full = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_empty = q_full + 1;
  uint64_t* kv_full = q_empty + 1;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;   // [2]
  uint64_t* p_full = s_full + 2;              // [2]
  uint64_t* o_done = p_full + 2;              // [2]
  uint64_t* o_free = o_done + 2;              // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_q);
    tma_prefetch_desc(&map_k);
    tma_prefetch_desc(&map_v);
    if (p.o_tma) tma_prefetch_desc(&map_o);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4 * C::kSplit);    // one arrival per softmax warp
      mbar_init(&o_done[i], 1);
      mbar_init(&o_free[i], 4 * C::kSplit);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const uint32_t sQ = smem_u32(smem + C::kQOff);
  const uint32_t sKV = smem_u32(smem + C::kKVOff);

  struct Work {
    int h, L, rows_valid, nq, nkv;
    int64_t s0, cbeg;
  };
  // the unit descriptor of work item w is one 16-byte load; it is fetched one item ahead and
  // decoded only when used, so its latency overlaps the current unit
  auto fetch = [&](int w) { return unit_of(p, w % U); };
  auto decode = [&](int w, int4 d) {
    Work x;
    x.h = w / U;
    x.s0 = d.x;
    x.L = d.y;
    x.cbeg = d.z;
    x.rows_valid = d.w;
    x.nq = x.rows_valid > 128 ? 2 : 1;
    x.nkv = (x.L + kBlockKeys - 1) / kBlockKeys;
    return x;
  };

  // Register split (per SM sub-partition: one warp of each warpgroup): the control warpgroup
  // drops registers so each softmax thread can hold its scores and the packed P.
  if (warp < 4) setmaxnreg_dec<C::kCtrlRegs>();
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int m = 0;                                 // units with key tiles so far
      int4 nx = fetch(blockIdx.x);
      for (int w = blockIdx.x; w < W; w += gridDim.x) {
        const Work x = decode(w, nx);            // descriptor fetched one unit ahead
        if (w + static_cast<int>(gridDim.x) < W) nx = fetch(w + gridDim.x);
        if (x.nkv == 0) continue;
        if (m > 0) mbar_wait_sleep(q_empty, (m - 1) & 1);   // previous unit's S MMAs done with Q
        const int32_t qrow = static_cast<int32_t>(static_cast<int64_t>(x.h) * p.total_C + x.cbeg);
        mbar_arrive_expect_tx(q_full, x.nq * C::kTileBytes);
        for (int i = 0; i < x.nq; ++i)
          for (int cb = 0; cb < C::kColBlocks; ++cb)
            tma_load_2d(smem + C::kQOff + i * C::kTileBytes + cb * C::kBoxBytes, &map_q, q_full,
                        cb * C::kBoxCols, qrow + 128 * i);
        const int32_t krow = static_cast<int32_t>(static_cast<int64_t>(x.h) * p.total_L + x.s0);
        for (int j = 0; j < x.nkv; ++j) {
          for (int which = 0; which < 2; ++which) {
            mbar_wait_sleep(&kv_empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&kv_full[stage], C::kTileBytes);
            const CUtensorMap* mp = which ? &map_v : &map_k;
            for (int cb = 0; cb < C::kColBlocks; ++cb)
              tma_load_2d(smem + C::kKVOff + stage * C::kTileBytes + cb * C::kBoxBytes, mp,
                          &kv_full[stage], cb * C::kBoxCols, krow + kBlockKeys * j);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
        }
        ++m;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc_s = make_idesc_bf16(128, kBlockKeys, 0, 0);
    const uint32_t idesc_o = make_idesc_bf16(128, D, 0, 1);
    int stage = 0;
    uint32_t phase = 0;
    int m = 0;                 // units with key tiles so far (q_full / q_empty phases)
    int cnt[2] = {0, 0};       // key tiles processed per Q tile (s_full / p_full / o_done phases)
    int act[2] = {0, 0};       // units with key tiles per Q tile (o_free phases)
    int4 nx = fetch(blockIdx.x);
    for (int w = blockIdx.x; w < W; w += gridDim.x) {
      const Work x = decode(w, nx);              // descriptor fetched one unit ahead
      if (w + static_cast<int>(gridDim.x) < W) nx = fetch(w + gridDim.x);
      if (x.nkv == 0) continue;
      const int nq = x.nq, nkv = x.nkv;
      auto issue_s = [&](int i, uint32_t kbase) {
        const uint32_t qbase = sQ + i * C::kTileBytes;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          mma_ss(tmem + i * 128, kmajor_desc<D>(qbase, ks), kmajor_desc<D>(kbase, ks), idesc_s,
                 ks > 0 ? 1u : 0u);
      };
      auto issue_pv = [&](int i, uint32_t vbase, int j) {
#pragma unroll
        for (int ks = 0; ks < kBlockKeys / 16; ++ks)
          mma_ts(tmem + 256 + i * D, tmem + i * 128 + ks * 8, v_desc<D>(vbase, ks), idesc_o,
                 (j > 0 || ks > 0) ? 1u : 0u);
      };
      mbar_wait_sleep(q_full, m & 1);
      // prologue: S_i for key tile 0 (S_i / P_i of the previous unit were consumed in order)
      int kslot = stage;
      mbar_wait_sleep(&kv_full[kslot], phase);
      tc_fence_after();
      if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      if (elect_one()) {
        const uint32_t kb = sKV + kslot * C::kTileBytes;
        issue_s(0, kb);
        mma_commit(&s_full[0]);
        if (nq == 2) {
          issue_s(1, kb);
          mma_commit(&s_full[1]);
        }
        mma_commit(&kv_empty[kslot]);
        if (nkv == 1) mma_commit(q_empty);
      }
      __syncwarp();
      for (int j = 0; j < nkv; ++j) {
        const int vslot = stage;
        mbar_wait_sleep(&kv_full[vslot], phase);
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        const bool has_next = j + 1 < nkv;
        if (has_next) {
          kslot = stage;
          mbar_wait_sleep(&kv_full[kslot], phase);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        const uint32_t vb = sKV + vslot * C::kTileBytes;
        const uint32_t kb = sKV + kslot * C::kTileBytes;
        for (int i = 0; i < nq; ++i) {
          // O_i += P_i V_j (the unit's first PV overwrites O_i: wait for the last epilogue),
          // then S_i for the next key tile
          if (j == 0 && act[i] > 0) mbar_wait_sleep(&o_free[i], (act[i] - 1) & 1);
          mbar_wait_sleep(&p_full[i], (cnt[i] + j) & 1);
          if (lane == 0) GESR_T(5 + i, cnt[i] + j);
          tc_fence_after();
          if (elect_one()) {
            issue_pv(i, vb, j);
            mma_commit(&o_done[i]);
            if (has_next) {
              issue_s(i, kb);
              mma_commit(&s_full[i]);
            }
          }
          __syncwarp();
        }
        if (elect_one()) {
          mma_commit(&kv_empty[vslot]);
          if (has_next) mma_commit(&kv_empty[kslot]);
          if (j + 2 == nkv) mma_commit(q_empty);     // the unit's last S MMAs were just issued
        }
        __syncwarp();
      }
      for (int i = 0; i < nq; ++i) {
        cnt[i] += nkv;
        act[i] += 1;
      }
      ++m;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    setmaxnreg_inc<C::kSoftRegs>();
    constexpr int kSplit = C::kSplit;
    constexpr int kCols = 128 / kSplit;        // S columns (keys) of this warp
    constexpr int kOCols = D / kSplit;         // O columns of this warp
    const int sw = warp - 4;
    const int i = sw / (4 * kSplit);           // Q tile of this warp
    const int half = (sw >> 2) % kSplit;       // column half (0 when kSplit == 1)
    const uint32_t sub = warp & 3;             // TMEM lane quarter
    const int rloc = sub * 32 + lane;          // row within the Q tile
    const int row_in_unit = i * 128 + rloc;
    uint8_t* stg = smem + C::kStgOff + sw * 4096;   // used only when kSplit == 1
    // [tile][half][buffer][row] partial maxima, [tile][half][row] partial sums
    const uint32_t xmax_s = smem_u32(smem + C::kXchOff);          // shared-space addresses
    const uint32_t xsum_s = xmax_s + 2 * 2 * 2 * 128 * 4;
    const uint32_t bar_id = 1 + i * 4 + sub;   // named barrier of the kSplit warps of a row set
    const uint32_t lane_addr = (sub * 32) << 16;
    const uint32_t tS = tmem + lane_addr + i * 128 + half * kCols;
    const uint32_t tP = tmem + lane_addr + i * 128 + half * (kCols / 2);
    const uint32_t tO = tmem + lane_addr + 256 + i * D + half * kOCols;
    const float sl2 = p.scale_log2;
    int cnt = 0;                                // key tiles processed by this Q tile so far
    int4 nx = fetch(blockIdx.x);
    for (int w = blockIdx.x; w < W; w += gridDim.x) {
      const Work x = decode(w, nx);              // descriptor fetched one unit ahead
      if (w + static_cast<int>(gridDim.x) < W) nx = fetch(w + gridDim.x);
      if (i >= x.nq) continue;
      // causal: this row sees keys [0, L - rows_valid + row] only
      int L = x.L;
      if constexpr (kCausal) L = min(x.L, x.L - x.rows_valid + row_in_unit + 1);
      const int nkv = x.nkv, rows_valid = x.rows_valid, h = x.h;
      const int64_t cbeg = x.cbeg;
      float m_run = -INFINITY;
      float l = 0.f;
      for (int j = 0; j < nkv; ++j) {
        const int gj = cnt + j;                 // global key-tile index of this Q tile
        mbar_wait_sleep(&s_full[i], gj & 1);
        const bool tr = (sub == 0 && half == 0 && lane == 0);
        if (tr) GESR_T(i == 0 ? 0 : 3, gj);
        tc_fence_after();
        uint32_t r[kCols];
#pragma unroll
        for (int c = 0; c < kCols / 32; ++c) tmem_ld32(tS + c * 32, r + c * 32);
        tmem_ld_wait();
        if constexpr (kHstu) {
          // p = SiLU(scale s) (masked keys: SiLU(0) = 0), no running max; l counts the keys
          const int hv = L - kBlockKeys * j - half * kCols;
          const float sc = sl2 * 0.69314718055994530942f;
#pragma unroll
          for (int k = 0; k < kCols / 2; ++k) {
            const float x0 = 2 * k < hv ? __uint_as_float(r[2 * k]) * sc : 0.f;
            const float x1 = 2 * k + 1 < hv ? __uint_as_float(r[2 * k + 1]) * sc : 0.f;
            float y0, y1;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(1.0f + ex2(-1.4426950408889634f * x0)));
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y1) : "f"(1.0f + ex2(-1.4426950408889634f * x1)));
            r[k] = pack_bf16x2(x0 * y0, x1 * y1);
          }
          l += static_cast<float>(hv < 0 ? 0 : (hv > kCols ? kCols : hv));
#pragma unroll
          for (int c = 0; c < kCols / 64; ++c) tmem_st32(tP + c * 32, r + c * 32);
          if constexpr (kCols / 2 % 32 != 0) tmem_st16(tP, r);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[i]);
          continue;
        }
        const int valid = L - kBlockKeys * j - half * kCols;   // valid keys in my columns
        const bool full = valid >= kCols;
        if (!full) {
#pragma unroll
          for (int k = 0; k < kCols; ++k)
            if (k >= valid) r[k] = __float_as_uint(-INFINITY);   // keys beyond L_b
        }
        // One fused pass per tile: p = 2^(s*scale*log2e - m) with the running max m of the
        // PREVIOUS tiles (speculative), the tile's own max reduced alongside (FMNMX beside
        // MUFU).  Only if the max grew by > 2^8 (rare after the first tile) are p recomputed
        // and O rescaled; the first tile reduces its max first.  Masked keys give exactly 0.
        // P is packed in place into r[0 .. kCols/2): S stays intact in TMEM until P is stored
        // over it, so the (rare) recompute reloads S from TMEM
        uint32_t* pk = r;
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
          for (int k = 0; k < kCols / 2; ++k) {
            const float s0v = __uint_as_float(r[2 * k]), s1v = __uint_as_float(r[2 * k + 1]);
            if (with_max) {
              mx[(2 * k) & 7] = fmaxf(mx[(2 * k) & 7], s0v);
              mx[(2 * k + 1) & 7] = fmaxf(mx[(2 * k + 1) & 7], s1v);
            }
            float x0, x1, p0, p1;
            ffma2(x0, x1, s0v, s1v, sl2, sl2, neg_m, neg_m);
            if ((k % GESR_POLY_EVERY) == GESR_POLY_EVERY - 1 && full) {
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
        if (j == 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) mx[e] = -INFINITY;
#pragma unroll
          for (int k = 0; k < kCols; ++k) mx[k & 7] = fmaxf(mx[k & 7], __uint_as_float(r[k]));
        } else {
          exp_pass(m_run, true);
        }
        float mraw = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                           fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        if constexpr (kSplit == 2) {
          const uint32_t xb = xmax_s + (((i * 2) * 2 + (gj & 1)) * 128 + rloc) * 4;   // [i][h][buf]
          st_shared_f32(xb + half * 2 * 128 * 4, mraw);
          named_bar_sync(bar_id, 64);
          mraw = fmaxf(mraw, ld_shared_f32(xb + (1 - half) * 2 * 128 * 4));
        }
        const float mt = mraw * sl2;
        if (tr && i == 0) GESR_T(1, gj);
        if (j == 0) {
          m_run = mt;
          exp_pass(m_run, false);
        } else {
          const bool need = mt > m_run + 8.0f;
          if (__any_sync(0xffffffffu, need)) {
            // O_i must hold P_{j-1} V_{j-1} before it is rescaled
            mbar_wait_sleep(&o_done[i], (gj - 1) & 1);
            tc_fence_after();
            float alpha = 1.f;
            if (need) {
              alpha = ex2(m_run - mt);
              m_run = mt;
              l *= alpha;
            }
#pragma unroll 1
            for (int c = 0; c < kOCols / 32; ++c) {
              uint32_t o[32];
              tmem_ld32(tO + c * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              tmem_st32(tO + c * 32, o);
            }
            tmem_st_wait();
#pragma unroll
            for (int c = 0; c < kCols / 32; ++c) tmem_ld32(tS + c * 32, r + c * 32);
            tmem_ld_wait();
            if (!full) {
#pragma unroll
              for (int k = 0; k < kCols; ++k)
                if (k >= valid) r[k] = __float_as_uint(-INFINITY);
            }
            exp_pass(m_run, false);   // recompute P with the new running max
          }
        }
        l += ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
#pragma unroll
        for (int c = 0; c < kCols / 64; ++c) tmem_st32(tP + c * 32, pk + c * 32);
        if constexpr (kCols / 2 % 32 != 0) tmem_st16(tP, pk);
        tmem_st_wait();
        tc_fence_before();
        if (tr) GESR_T(i == 0 ? 2 : 4, gj);
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[i]);
      }
      // epilogue: O / l for my columns
      if constexpr (kSplit == 2) {
        st_shared_f32(xsum_s + ((i * 2 + half) * 128 + rloc) * 4, l);
        named_bar_sync(bar_id, 64);
        l += ld_shared_f32(xsum_s + ((i * 2 + (1 - half)) * 128 + rloc) * 4);
      }
      const bool row_ok = row_in_unit < rows_valid;
      const int64_t row = cbeg + row_in_unit;
      const int64_t HD = static_cast<int64_t>(p.H) * D;
      if (nkv > 0) {
        mbar_wait_sleep(&o_done[i], (cnt + nkv - 1) & 1);
        tc_fence_after();
      }
      const float inv_l = nkv > 0 ? 1.0f / l : 0.f;
      const int64_t col0 = static_cast<int64_t>(h) * D + half * kOCols;
      // bf16 rows of a fully valid 32-row warp slab leave through the staging boxes and TMA
      // tensor stores ([total_C, H, d] map, box 32 x 1 x 32); a ragged slab (the rows past it
      // belong to the next request) stores its valid rows directly
      const bool use_tma = kSplit == 1 && p.o_tma && i * 128 + static_cast<int>(sub) * 32 + 32 <= rows_valid;
#pragma unroll 1
      for (int c = 0; c < kOCols / 32; ++c) {
        uint32_t o[32];
        if (nkv > 0) {
          tmem_ld32(tO + c * 32, o);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = 0u;
        }
        if (use_tma) {
          uint32_t pk2[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            pk2[e] = pack_bf16x2(__uint_as_float(o[2 * e]) * inv_l, __uint_as_float(o[2 * e + 1]) * inv_l);
          // this box must have been read by the store issued from it two chunks ago
          if (lane == 0) bulk_wait_group_read<1>();
          __syncwarp();
          uint8_t* box = stg + (c & 1) * 2048;
          uint8_t* rowp = box + lane * 64;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(rowp + ((q ^ ((lane >> 1) & 3)) << 4)) =
                make_uint4(pk2[4 * q], pk2[4 * q + 1], pk2[4 * q + 2], pk2[4 * q + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&map_o, box, c * 32, h, static_cast<int32_t>(cbeg + i * 128 + sub * 32));
            bulk_commit_group();
          }
        } else if (row_ok) {
          if (p.o_bf16) {
            uint32_t pk2[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              pk2[e] = pack_bf16x2(__uint_as_float(o[2 * e]) * inv_l, __uint_as_float(o[2 * e + 1]) * inv_l);
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.O) + row * HD + col0 + c * 32;
            st_global_v8(dst, pk2);
            st_global_v8(dst + 16, pk2 + 8);
          } else {
            float* dst = static_cast<float*>(p.O) + row * HD + col0 + c * 32;
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * inv_l);
#pragma unroll
            for (int v = 0; v < 4; ++v) st_global_v8(dst + 8 * v, o + 8 * v);
          }
        }
      }
      if (row_ok && half == 0 && p.lse != nullptr) {
        // m_run and log2(l) are in log2 units of the scaled score
        p.lse[row * p.H + h] = nkv > 0 ? (m_run + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      }
      if (nkv > 0) {
        // O_i drained: the next unit's first PV may overwrite it
        if (i == 0 && sub == 0 && half == 0 && lane == 0) GESR_T(7, cnt + nkv - 1);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_free[i]);
      }
      cnt += nkv;
    }
    if (lane == 0) bulk_wait_group<0>();   // staging boxes stay allocated until read
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Work list: one int4 per 256-candidate unit {first history row, L_b, first candidate row,
// valid rows}, so the attention kernel decodes a unit with a single 16-byte load.
__global__ void build_units_kernel(const int64_t* __restrict__ seq_offsets,
                                   const int64_t* __restrict__ cand_offsets, int64_t B,
                                   int4* __restrict__ units, int* __restrict__ count,
                                   int causal) {
  __shared__ int warp_sums[32];
  __shared__ int running;
  pdl_launch_dependents();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  if (threadIdx.x == 0) running = 0;
  __syncthreads();
  for (int64_t base = 0; base < B; base += blockDim.x) {
    const int64_t b = base + threadIdx.x;
    int n = 0;
    int64_t c = 0, cb0 = 0, s0 = 0, L = 0;
    if (b < B) {
      cb0 = cand_offsets[b];
      c = cand_offsets[b + 1] - cb0;
      s0 = seq_offsets[b];
      L = seq_offsets[b + 1] - s0;
      n = static_cast<int>((c + kUnitRows - 1) / kUnitRows);
    }
    int x = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
      int v = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      warp_sums[lane] = v;
    }
    __syncthreads();
    const int excl = running + (x - n) + (w > 0 ? warp_sums[w - 1] : 0);
    for (int k = 0; k < n; ++k) {
      const int64_t rem = c - static_cast<int64_t>(k) * kUnitRows;
      // causal: queries [256 k, 256 k + rows) of the history see keys up to the last of them
      if (causal) L = static_cast<int64_t>(k) * kUnitRows + (rem < kUnitRows ? rem : kUnitRows);
      units[excl + k] = make_int4(static_cast<int>(s0), static_cast<int>(L),
                                  static_cast<int>(cb0 + static_cast<int64_t>(k) * kUnitRows),
                                  static_cast<int>(rem < kUnitRows ? rem : kUnitRows));
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) running = excl + n;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = running;
}

// Self key (the candidate diagonal of the [U, T] mask; R2): one
// warp per (candidate, head).  The history attention left O = sum_i p_i v_i / sum_i p_i and
// lse = log sum_i e^{s_i}; the candidate's own score s = scale q.k_self joins as one more key:
// O' = (O e^{lse - M} + v_self e^{s - M}) / (e^{lse - M} + e^{s - M}), M = max(lse, s),
// lse' = M + log(...).  L_b = 0 (lse = -inf) gives O' = v_self, lse' = s.
__global__ void __launch_bounds__(256) attn_self_merge_kernel(const AttnParams p,
                                                              const __nv_bfloat16* __restrict__ Q,
                                                              const __nv_bfloat16* __restrict__ Ks,
                                                              const __nv_bfloat16* __restrict__ Vs,
                                                              int d, float scale) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (item >= p.total_C * p.H) return;
  const int64_t row = item / p.H;
  const int h = static_cast<int>(item % p.H);
  const int64_t kv = (static_cast<int64_t>(h) * p.total_C + row) * d;   // [H, total_C, d]
  const int64_t o0 = row * p.H * d + static_cast<int64_t>(h) * d;
  float dot = 0.f;
  for (int j = lane; j < d; j += 32)
    dot += __bfloat162float(Q[kv + j]) * __bfloat162float(Ks[kv + j]);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  const float s = dot * scale;
  const float l0 = p.lse[item];
  const float M = fmaxf(l0, s);
  const float w0 = (l0 == -INFINITY) ? 0.f : expf(l0 - M);
  const float w1 = expf(s - M);
  const float inv = 1.0f / (w0 + w1);
  for (int j = lane; j < d; j += 32) {
    const float v = __bfloat162float(Vs[kv + j]);
    if (p.o_bf16) {
      __nv_bfloat16* O = static_cast<__nv_bfloat16*>(p.O);
      O[o0 + j] = __float2bfloat16_rn((__bfloat162float(O[o0 + j]) * w0 + v * w1) * inv);
    } else {
      float* O = static_cast<float*>(p.O);
      O[o0 + j] = (O[o0 + j] * w0 + v * w1) * inv;
    }
  }
  if (lane == 0) p.lse[item] = M + logf(w0 + w1);
}

// total_L == 0: every candidate has an empty history -> O = 0, lse = -inf (R6)
__global__ void attn_empty_kernel(AttnParams p, int D) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t HD = static_cast<int64_t>(p.H) * D;
  const int64_t n = p.total_C * HD;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (p.o_bf16) static_cast<__nv_bfloat16*>(p.O)[i] = __float2bfloat16(0.f);
    else static_cast<float*>(p.O)[i] = 0.f;
    if (p.lse != nullptr && i < p.total_C * p.H) p.lse[i] = -INFINITY;
  }
}

template <int D>
cudaError_t launch_d(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                     const CUtensorMap& mo, const AttnParams& p, int64_t max_units,
                     cudaStream_t stream) {
  using C = AttnCfg<D>;
  for (const void* fn : {reinterpret_cast<const void*>(attn_kernel<D, false, false>),
                         reinterpret_cast<const void*>(attn_kernel<D, true, false>),
                         reinterpret_cast<const void*>(attn_kernel<D, false, true>)}) {
    cudaError_t e = ensure_smem_attr(fn, C::kSmemBytes);
    if (e != cudaSuccess) return e;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t work = max_units * p.H;
  const unsigned grid = static_cast<unsigned>(work < sms ? work : sms);
  auto* fn = p.hstu ? attn_kernel<D, false, true>
                    : (p.causal ? attn_kernel<D, true, false> : attn_kernel<D, false, false>);
  return launch_pdl(fn, dim3(grid), dim3(C::kThreads), C::kSmemBytes, stream, mq, mk, mv, mo, p);
}

}  // namespace

#ifdef GESR_TRACE
extern "C" int gesr_debug_trace_copy(void* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace)));
}
#endif

cudaError_t launch_build_units(const int64_t* seq_offsets, const int64_t* cand_offsets, int64_t B,
                               int4* units, int* count, int causal, cudaStream_t stream) {
  return launch_pdl(build_units_kernel, dim3(1), dim3(1024), 0, stream, seq_offsets, cand_offsets,
                    B, units, count, causal);
}

cudaError_t launch_attn(int d, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                        const CUtensorMap& mo, const AttnParams& p, int64_t max_units,
                        cudaStream_t stream) {
  switch (d) {
    case 32: return launch_d<32>(mq, mk, mv, mo, p, max_units, stream);
    case 64: return launch_d<64>(mq, mk, mv, mo, p, max_units, stream);
    case 128: return launch_d<128>(mq, mk, mv, mo, p, max_units, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_attn_self_merge(const AttnParams& p, const void* Q, const void* K_self,
                                   const void* V_self, int d, float scale, cudaStream_t stream) {
  const int64_t n = p.total_C * p.H;
  if (n == 0) return cudaSuccess;
  return launch_pdl(attn_self_merge_kernel, dim3(static_cast<unsigned>((n + 7) / 8)), dim3(256), 0,
                    stream, p, static_cast<const __nv_bfloat16*>(Q),
                    static_cast<const __nv_bfloat16*>(K_self),
                    static_cast<const __nv_bfloat16*>(V_self), d, scale);
}

cudaError_t launch_attn_empty(const AttnParams& p, int d, cudaStream_t stream) {
  return launch_pdl(attn_empty_kernel, dim3(1184), dim3(256), 0, stream, p, d);
}

}  // namespace gesr
