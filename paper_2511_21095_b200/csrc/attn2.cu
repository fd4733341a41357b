// attn2.cu -- K-ATTN for d = 128 (the default for d = 128): CTA PAIR (tcgen05 cta_group::2),
// persistent, two softmax warpgroups taking alternate key tiles.
//
// Same contract as attn.cu (PAPER.md:341 mask rules (1)-(2): each candidate attends to all L_b
// history keys of its own request and to no other candidate; softmax per DESIGN.md R1).
//
// Why (profiles/): in the 1-CTA kernel the softmax of a Q tile and its MMAs form
// one dependency chain (softmax(j) -> PV(j) -> S(j+1) -> softmax(j+1)) and every unit ends in
// an epilogue bubble.  Here:
//   * a cluster of 2 CTAs works on one unit (request b, head h, 256 candidates); CTA r owns
//     candidate rows [128 r, 128 r + 128).  The leader issues M=256 MMAs for the pair: S = Q K^T
//     (SS; each CTA stages its Q tile and HALF of each K tile -- 64 keys) and O += P V (TS; P
//     from each CTA's TMEM, each CTA stages HALF of each V tile -- 64 d-columns);
//   * ONE S buffer in TMEM serves both warpgroups and P lives in its own TMEM columns, so a
//     warpgroup releases S as soon as S is in registers and S(j+1) is computed during the
//     softmax of tile j: no MMA sits between two softmax passes; PV is a TS MMA (A = P from
//     TMEM), so the tensor core reads only Q, K and V from shared memory (P in shared memory
//     cost ~6 %: its stores stalled behind the tensor core's operand reads);
//   * key tiles alternate between softmax warpgroups A (even) and B (odd); a named-barrier
//     "MUFU token" per sub-partition orders their exp passes A(0), B(1), A(2), ... so one's exp
//     pass overlaps the other's TMEM load, x pass and P hand-off.  Both accumulate into ONE O per
//     unit with ONE running max per row (m_sh in shared memory, decided tile by tile in order);
//     the row max is exact only for tile 0, later tiles test the tile's row sum and take the
//     slow path (exact max, raise m_sh, rescale O, recompute P) only when needed.  A pass starts
//     right after the token with the warpgroup's own max, the token is handed on as soon as the
//     last MUFU op is issued, and the previous tile's decision is checked after the pass (a rare
//     raise recomputes): nothing but MUFU work sits between two exp passes;
//   * TMEM per CTA (512 columns): S [0,128), P_A [128,192), P_B [192,256), O of even units
//     [256,384), O of odd units [384,512): a unit's epilogue (warps 12-15) overlaps the next
//     unit entirely;
//   * persistent: pair c takes work items c, c + G, ... (w -> unit w % U, head w / U); the key
//     tiles of all its work items form one stream, walked independently by the Q/K producer,
//     the V producer, the S-MMA issuer and the PV-MMA issuer; full 32-row output slabs leave
//     through TMA tensor stores.
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
__device__ unsigned long long g_trace3[64][16][8];   // per unit: control-warp events
__device__ unsigned long long g_trace4[64][16][16];  // per unit: epilogue chunk loads done
#define GESR_T4(e, u)                                                                          \
  do {                                                                                         \
    const int _b = blockIdx.x;                                                                 \
    if (_b < 64 && (u) < 16) g_trace4[_b][(u)][(e)] = clock64();                               \
  } while (0)
#define GESR_T3(e, u)                                                                          \
  do {                                                                                         \
    const int _b = blockIdx.x;                                                                 \
    if (_b < 64 && (u) < 16) g_trace3[_b][(u)][(e)] = clock64();                               \
  } while (0)
#else
#define GESR_T2(e, j) do {} while (0)
#define GESR_T3(e, u) do {} while (0)
#define GESR_T4(e, u) do {} while (0)
#endif

namespace {

#ifndef GESR_PAIR_L2HINT
#define GESR_PAIR_L2HINT 1        // 1: Q loads / O stores evict_first; 2: + K/V loads evict_last
#endif
#ifndef GESR_PAIR_EPI_SLEEP
#define GESR_PAIR_EPI_SLEEP 500   // ns per retry of the epilogue's unit-long waits
#endif
#ifndef GESR_PAIR_SUM_LIMIT
#define GESR_PAIR_SUM_LIMIT 4096.0f   // tile row sums above this take the exact-max path
#endif
// mbarrier waits: 1 = try_wait spin loop, 0 = try_wait with a suspend-time hint
#ifndef GESR_PAIR_SPIN
#define GESR_PAIR_SPIN 0
#endif
// A wait that exceeds ~20 s traps.  Builds with -DGESR_DEBUG_WAITS also print the call site
// (ctx = site * 2^20 + unit * 2^8 + tile) first; the default build has no call in the wait
// loops (a call site there makes ptxas keep the softmax's registers in local memory).
// The retry loop is kept to a few instructions (a try_wait that suspends the warp in hardware,
// an iteration counter instead of a clock read and 64-bit compare): waiting warps share their
// sub-partition with an exp warp, and ncu showed the epilogue warps' unit-long waits spinning
// ~370 times per unit through ~10 integer instructions each.  `sleep_ns` > 0 adds a nanosleep
// per retry for waits that are long by construction (the epilogue waits a whole unit).
__device__ __forceinline__ void pwait(uint64_t* bar, uint32_t parity, uint32_t ctx = 0,
                                      uint32_t sleep_ns = 0) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait_hint(a, parity, GESR_PAIR_SPIN ? 0u : 1000000u)) return;
  // each try_wait may suspend up to its hint: the clock is read every 64 retries and the wait
  // traps after ~2^35 cycles (~17 s at 1.965 GHz) however long the suspensions were
  uint32_t n = 0;
  long long t0 = 0;
  while (!mbar_try_wait_hint(a, parity, GESR_PAIR_SPIN ? 0u : 1000000u)) {
    if (sleep_ns) __nanosleep(sleep_ns);
    if ((++n & 63u) == 0) {
      const long long t = clock64();
      if (t0 == 0) {
        t0 = t;
      } else if (t - t0 > (1ll << 35)) {
#ifdef GESR_DEBUG_WAITS
        if ((threadIdx.x & 31) == 0)
          printf("gesr: attn_pair mbarrier timeout block %d warp %d smem 0x%x parity %u site %u unit %u tile %u\n",
                 blockIdx.x, threadIdx.x / 32, a, parity, ctx >> 20, (ctx >> 8) & 0xfff, ctx & 0xff);
#else
        (void)ctx;
#endif
        __trap();
      }
    }
  }
}
#define CTX(site, u, t) ((static_cast<uint32_t>(site) << 20) | ((static_cast<uint32_t>(u) & 0xfff) << 8) | (static_cast<uint32_t>(t) & 0xff))
constexpr int kD = 128;
constexpr int kKeys = 128;                       // keys per tile (S columns)
constexpr int kThreads = 512;
constexpr uint32_t kQBytes = 128 * kD * 2;       // 32 KB: Q tile, [2 col blocks][128 rows][64]
constexpr uint32_t kHalfBytes = 16384;           // K half [2][64 keys][64] or V half [128][64]
// Q tiles are double-buffered: unit m+1's Q is loaded while unit m's S MMAs still read unit m's
// (a single buffer made every unit wait for its Q load after the previous unit's last S MMA:
// ~2k cycles of drained pipeline per work item)
#ifndef GESR_PAIR_QBUFS
#define GESR_PAIR_QBUFS 2
#endif
// ring stages (measured with two Q buffers, base-clock ncu at 3h: K 4 / V 3 5.382 ms, K 3 / V 4
// 5.372 ms; one Q buffer with K 4 / V 5: 5.449 ms)
#ifndef GESR_PAIR_KST
#define GESR_PAIR_KST (GESR_PAIR_QBUFS == 2 ? 3 : 4)
#endif
#ifndef GESR_PAIR_VST
#define GESR_PAIR_VST (GESR_PAIR_QBUFS == 2 ? 4 : 5)
#endif
constexpr int kQBufs = GESR_PAIR_QBUFS;
constexpr int kKStages = GESR_PAIR_KST;         // K-half ring
constexpr int kVStages = GESR_PAIR_VST;         // V-half ring
constexpr int kStages = kKStages + kVStages;
constexpr uint32_t kQOff = 0;
constexpr uint32_t kRingOff = kQBufs * kQBytes;
constexpr uint32_t kStgOff = kRingOff + kStages * kHalfBytes;        // 4 x 2 KB boxes per epilogue warp
constexpr uint32_t kBarOff = kStgOff + 4 * 8192;
constexpr uint32_t kXchOff = kBarOff + 512;                          // [unit % 4][WG][m, l][row]
constexpr uint32_t kMshOff = kXchOff + 4 * 2 * 2 * 128 * 4;          // [row] {running max, tile}
constexpr uint32_t kSmemBytes = kMshOff + 128 * 8 + 1024;
static_assert(kSmemBytes <= 232448, "shared memory budget");
// register split (setmaxnreg per warpgroup; launch registers 128 x 512 threads): control 56,
// softmax 184, epilogue 88
constexpr int kCtrlRegs = 56;
constexpr int kSoftRegs = 184;
constexpr int kEpiRegs = 88;
static_assert(128 * kCtrlRegs + 256 * kSoftRegs + 128 * kEpiRegs <= 128 * kThreads, "setmaxnreg pool");
// TMEM columns
constexpr uint32_t kTS = 0;          // S: one buffer, alternately A's and B's tiles
constexpr uint32_t kTP = 128;        // P_A at 128, P_B at 192 (bf16 pairs, 64 columns each)
constexpr uint32_t kTO = 256;        // O of even units at 256, of odd units at 384
// unit m's m / l hand-off from the softmax to the epilogue warps: named barrier 1 + m % 4 (ids
// 5-12 are the MUFU tokens), 8 softmax + 4 epilogue warps
constexpr uint32_t kMlBarBase = 1;
constexpr uint32_t kMlBarThreads = 12 * 32;

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
  int h, L, rows_valid, nkv;      // nkv: key tiles of this work item (its split's range)
  int t0, split;                  // first key tile of the range, split index
  int64_t s0, cbeg;
};

// kCausal: history self-attention (gesr_history_attention); a separate instantiation keeps the
// target-aware kernel's code unchanged
template <bool kCausal>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap map_q,
                     const __grid_constant__ CUtensorMap map_kh,
                     const __grid_constant__ CUtensorMap map_vh,
                     const __grid_constant__ CUtensorMap map_o, const AttnParams p) {
  pdl_launch_dependents();
  pdl_wait();
  const int U = unit_count_of(p);
  const int S = p.splits;
  const int W = U * p.H * S;
  const int pair = static_cast<int>(blockIdx.x >> 1);
  const int npairs = static_cast<int>(gridDim.x >> 1);
  if (pair >= W) return;                          // uniform for the pair
  const uint32_t rank = cluster_ctarank();

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* q_full = reinterpret_cast<uint64_t*>(smem + kBarOff);   // [2] leader's used
  uint64_t* q_empty = q_full + 2;                 // [2] each CTA
  uint64_t* kv_full = q_empty + 2;                // [kStages]  K ring, then V ring (leader's used)
  uint64_t* kv_empty = kv_full + kStages;         // [kStages]  (each CTA)
  uint64_t* s_full = kv_empty + kStages;          // [2]        (each CTA)
  uint64_t* s_free = s_full + 2;                  //            (leader; 4 warps x 2 CTAs per S)
  uint64_t* p_full = s_free + 2;                  // [2]        (leader; 8 warps of the pair)
  uint64_t* p_free = p_full + 2;                  // [2]        (each CTA)
  uint64_t* o_done = p_free + 2;                  // [2]        (each CTA; per O buffer)
  uint64_t* o_free = o_done + 2;                  // [2]        (leader; 8 epilogue warps of the pair)
  // per unit % 4: the softmax may publish units m+1 and m+2 (short units need no PV of their
  // own before their last tile) while an epilogue warp still waits for unit m; four barriers
  // (and four m / l slots) keep every waiter within one phase of its barrier
  uint64_t* ml_full = o_free + 2;                 // [4]        unused (named barriers 1-4)
  // slot u % 4 reused by unit u + 4 only after the epilogue read it (a warpgroup with no tile
  // in a run of 1-tile units would otherwise publish 4+ units ahead)
  uint64_t* ml_empty = ml_full + 4;               // [4]        (each CTA; its 4 epilogue warps)
  uint64_t* pv_done = ml_empty + 4;               //            (each CTA; one phase per PV)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);
  static_assert((4 + 2 * kStages + 2 * 6 + 8 + 1) * 8 + 4 <= kXchOff - kBarOff, "barrier area");

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
#if GESR_PAIR_L2HINT >= 1
  const uint64_t pol_first = policy_evict_first();   // streamed once: Q in, O out
#endif
#if GESR_PAIR_L2HINT >= 2
  const uint64_t pol_last = policy_evict_last();     // K/V: re-read by the request's other units
#endif

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_q);
    tma_prefetch_desc(&map_kh);
    tma_prefetch_desc(&map_vh);
    if (p.o_tma) tma_prefetch_desc(&map_o);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);                  // [1] unused
      mbar_init(&p_full[i], 8);
      mbar_init(&p_free[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&o_done[i], 1);
      mbar_init(&o_free[i], 8);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&ml_empty[i], 4);
    }
    mbar_init(pv_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc_pair(tmem_slot, 512);
    tmem_relinquish_pair();
  }
  if (threadIdx.x < 128) {        // running-max words: no tile decided yet
    const uint32_t w = smem_u32(smem + kMshOff) + threadIdx.x * 8;
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(w), "r"(0u), "r"(0xFFFFFFFFu) : "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sQ = smem_u32(smem + kQOff);
  const uint32_t sRing = smem_u32(smem + kRingOff);

  // the unit descriptor of work item w is one 16-byte load, fetched one item ahead
  auto fetch = [&](int w) { return unit_of(p, w % U); };
  // w -> (unit w % U, split (w / U) % S, head w / (U S)): neighbouring pairs share a head and
  // run the units of one request at the same time (K/V shared in L2; measured: a pair taking
  // a contiguous block of items, units of a request back to back, read 11% MORE from HBM)
  auto decode = [&](int w, int4 d) {
    Work x;
    const int rest = w / U;
    x.s0 = d.x;
    x.L = d.y;
    x.cbeg = d.z;
    x.rows_valid = d.w;
    const int n = (x.L + kKeys - 1) / kKeys;
    if (S == 1) {
      x.split = 0;
      x.h = rest;
      x.t0 = 0;
      x.nkv = n;
    } else {
      x.split = rest % S;
      x.h = rest / S;
      x.t0 = x.split * n / S;              // n <= 2^24, S <= 64: no int32 overflow
      x.nkv = (x.split + 1) * n / S - x.t0;
    }
    return x;
  };

  // The key tiles of all work items of this pair form one stream (units without keys skipped):
  // the producer and the MMA issuer walk it with TileStream cursors, so the next unit's first
  // S MMAs are issued while the current unit's last PVs wait for their P (no bubble at unit
  // boundaries).  Stream order of the MMA issuer: S(0), S(1), S(2), then per step S(g+3) and
  // PV(g); the producer loads K(g) / V(g) in exactly that order.
  struct Tile {
    Work x;
    int t, m;       // tile index in its unit, ordinal of its unit among units with keys
  };
  struct TileStream {
    int w, t, m;
    Work x;
    int4 nx;
  };
  auto stream_init = [&](TileStream& st) {
    st.w = pair;
    st.t = 0;
    st.m = -1;
    st.x.nkv = 0;
    st.nx = pair < W ? fetch(pair) : make_int4(0, 0, 0, 0);
  };
  auto stream_next = [&](TileStream& st, Tile& out) -> bool {
    while (st.t >= st.x.nkv) {
      if (st.w >= W) return false;
      st.x = decode(st.w, st.nx);
      st.w += npairs;
      if (st.w < W) st.nx = fetch(st.w);
      st.t = 0;
      if (st.x.nkv > 0) ++st.m;
    }
    out.x = st.x;
    out.t = st.t++;
    out.m = st.m;
    return true;
  };

  if (warp < 4) {
    setmaxnreg_dec<kCtrlRegs>();
    // Four independent control streams over the tile stream (each blocks only on its own
    // resources): warp 0 loads Q and the K halves, warp 2 the V halves (both CTAs); in the
    // leader, warp 1 issues the S MMAs and warp 3 the PV MMAs.  S(g) needs its K half, its
    // unit's Q and the s_free of its buffer's previous S; PV(g) its V half and p_full(g).
    auto krow_of = [&](const Tile& tl) {
      return static_cast<int32_t>(static_cast<int64_t>(tl.x.h) * p.total_L + tl.x.s0) +
             kKeys * (tl.x.t0 + tl.t);
    };
    TileStream st;
    stream_init(st);
    Tile tl;
    if (warp == 0) {
      // ---------------------------------------------------------- Q + K producer (both CTAs)
      if (elect_one()) {
        int kst = 0;
        uint32_t kph = 0;
        while (stream_next(st, tl)) {
          if (tl.t == 0) {
            // unit m's Q buffer (m % kQBufs) must be done with unit m - kQBufs's S MMAs
            const int qb = tl.m % kQBufs;
            if (tl.m >= kQBufs) pwait(&q_empty[qb], ((tl.m / kQBufs) - 1) & 1, CTX(1, tl.m, tl.t));
            GESR_T3(3, tl.m);
            const int32_t qrow = static_cast<int32_t>(static_cast<int64_t>(tl.x.h) * p.total_C + tl.x.cbeg) +
                                 static_cast<int32_t>(rank) * 128;
            uint8_t* qdst = smem + kQOff + qb * kQBytes;
            if (rank == 0) mbar_arrive_expect_tx(&q_full[qb], 2 * kQBytes);
#if GESR_PAIR_L2HINT >= 1
            tma_load_2d_pair_hint(qdst, &map_q, &q_full[qb], 0, qrow, pol_first);
            tma_load_2d_pair_hint(qdst + kQBytes / 2, &map_q, &q_full[qb], 64, qrow, pol_first);
#else
            tma_load_2d_pair(qdst, &map_q, &q_full[qb], 0, qrow);
            tma_load_2d_pair(qdst + kQBytes / 2, &map_q, &q_full[qb], 64, qrow);
#endif
          }
          const int slot = kst;
          pwait(&kv_empty[slot], kph ^ 1, CTX(2, tl.m, tl.t));
          if (rank == 0) mbar_arrive_expect_tx(&kv_full[slot], 2 * kHalfBytes);
          uint8_t* dst = smem + kRingOff + slot * kHalfBytes;
          const int32_t row = krow_of(tl) + static_cast<int32_t>(rank) * 64;
#if GESR_PAIR_L2HINT >= 2
          tma_load_2d_pair_hint(dst, &map_kh, &kv_full[slot], 0, row, pol_last);
          tma_load_2d_pair_hint(dst + 8192, &map_kh, &kv_full[slot], 64, row, pol_last);
#else
          tma_load_2d_pair(dst, &map_kh, &kv_full[slot], 0, row);
          tma_load_2d_pair(dst + 8192, &map_kh, &kv_full[slot], 64, row);
#endif
          if (++kst == kKStages) { kst = 0; kph ^= 1; }
        }
      }
    } else if (warp == 2) {
      // ---------------------------------------------------------- V producer (both CTAs)
      if (elect_one()) {
        int vst = 0;
        uint32_t vph = 0;
        while (stream_next(st, tl)) {
          const int slot = kKStages + vst;
          pwait(&kv_empty[slot], vph ^ 1, CTX(3, tl.m, tl.t));
          if (rank == 0) mbar_arrive_expect_tx(&kv_full[slot], 2 * kHalfBytes);
          uint8_t* dst = smem + kRingOff + slot * kHalfBytes;
#if GESR_PAIR_L2HINT >= 2
          tma_load_2d_pair_hint(dst, &map_vh, &kv_full[slot], static_cast<int32_t>(rank) * 64, krow_of(tl), pol_last);
#else
          tma_load_2d_pair(dst, &map_vh, &kv_full[slot], static_cast<int32_t>(rank) * 64, krow_of(tl));
#endif
          if (++vst == kVStages) { vst = 0; vph ^= 1; }
        }
      }
    } else if (warp == 1 && rank == 0) {
      // ---------------------------------------------------------- S MMA issuer (leader only)
      const uint32_t idesc_s = make_idesc_bf16(256, kKeys, 0, 0);
      int kst = 0;
      uint32_t kph = 0;
      uint32_t sn0 = 0;                            // S issued so far
      while (stream_next(st, tl)) {
        const int buf = tl.t & 1;
        if (tl.t == 0) {
          // the unit's Q tile (both CTAs)
          pwait(&q_full[tl.m % kQBufs], (tl.m / kQBufs) & 1, CTX(4, tl.m, tl.t));
          if (lane == 0) GESR_T3(0, tl.m);
        }
        // the single S buffer's previous S must have been loaded into registers (both CTAs)
        if (sn0 > 0) pwait(s_free, (sn0 - 1) & 1, CTX(5, tl.m, tl.t));
        ++sn0;
        const int slot = kst;
        pwait(&kv_full[slot], kph, CTX(6, tl.m, tl.t));
        if (++kst == kKStages) { kst = 0; kph ^= 1; }
        if (lane == 0) GESR_T2(7, tl.m * 16 + tl.t);
        const uint32_t kb = sRing + slot * kHalfBytes;
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < kD / 16; ++ks)
            mma_ss_pair(tmem + kTS, kdesc(sQ + (tl.m % kQBufs) * kQBytes, kQBytes / 2, ks),
                        kdesc(kb, 8192, ks), idesc_s,
                        ks > 0 ? 1u : 0u);
          mma_commit_pair_mc(&s_full[buf], 0x3);
          mma_commit_pair_mc(&kv_empty[slot], 0x3);
          // the unit's last S: its Q buffer may be reloaded
          if (tl.t == tl.x.nkv - 1) mma_commit_pair_mc(&q_empty[tl.m % kQBufs], 0x3);
        }
        __syncwarp();
      }
    } else if (warp == 3 && rank == 0) {
      // ---------------------------------------------------------- PV MMA issuer (leader only)
      const uint32_t idesc_o = make_idesc_bf16(256, kD, 0, 1);
      int vst = 0;
      uint32_t vph = 0;
      uint32_t pn0 = 0, pn1 = 0;                   // PV issued from P_A / P_B so far
      while (stream_next(st, tl)) {
        const int xb = tl.t & 1;
        const int vslot = kKStages + vst;
        pwait(&kv_full[vslot], vph, CTX(7, tl.m, tl.t));
        if (++vst == kVStages) { vst = 0; vph ^= 1; }
        const int ob = tl.m & 1;                     // O buffer of this unit
        if (tl.t == 0 && tl.m >= 2) {
          // the unit's first PV overwrites its O buffer: unit m-2's epilogue must have read it
          pwait(&o_free[ob], ((tl.m >> 1) - 1) & 1, CTX(8, tl.m, tl.t));
          if (lane == 0) GESR_T3(1, tl.m);
        }
        const uint32_t pn = xb ? pn1 : pn0;
        pwait(&p_full[xb], pn & 1, CTX(9, tl.m, tl.t));
        if (xb) ++pn1; else ++pn0;
        if (lane == 0) GESR_T2(6, tl.m * 16 + tl.t);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t vb = sRing + vslot * kHalfBytes;
#pragma unroll
          for (int ks = 0; ks < kKeys / 16; ++ks)
            mma_ts_pair(tmem + kTO + ob * kD, tmem + kTP + xb * (kKeys / 2) + ks * 8, vdesc(vb, ks),
                        idesc_o, (tl.t > 0 || ks > 0) ? 1u : 0u);
          mma_commit_pair_mc(&p_free[xb], 0x3);
          mma_commit_pair_mc(&kv_empty[vslot], 0x3);
          mma_commit_pair_mc(pv_done, 0x3);
          if (tl.t == tl.x.nkv - 1) mma_commit_pair_mc(&o_done[ob], 0x3);
        }
        __syncwarp();
        if (tl.t == tl.x.nkv - 1 && lane == 0) GESR_T3(2, tl.m);
      }
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ softmax
    // Both warpgroups accumulate into ONE O per unit (double-buffered across units in TMEM, so
    // the epilogue of unit u overlaps unit u+1) with ONE running max per row, m_sh (shared
    // memory, one {m, tile} word per row).  The MUFU token orders the tiles' exp passes A(0),
    // B(1), A(2), ...; each tile publishes its decided max in tile order, and a tile's P is
    // final only once it has been computed against the max decided by the tile before it
    // (checked after the first pass, recomputed in the rare case it was raised), so every P(j)
    // matches the max O is scaled to when PV(j) lands.  Raising m_sh (rare: a tile whose row sum
    // exceeds 2^12 and whose exact max exceeds m_sh by > 8, log2 units) waits for PV(j-1) and
    // rescales O first.  Each warpgroup keeps its own row sum l relative to the max it last
    // used (m_loc) and rescales it when it finds m_sh raised.
    setmaxnreg_inc<kSoftRegs>();
    const int g = (static_cast<int>(warp) - 4) >> 2;   // warpgroup: 0 = A (even tiles), 1 = B
    const uint32_t sub = warp & 3;                       // TMEM lane quarter
    const int rloc = static_cast<int>(sub) * 32 + static_cast<int>(lane);
    const uint32_t lane_addr = (sub * 32) << 16;
    const uint32_t tS = tmem + lane_addr + kTS;
    const uint32_t tP = tmem + lane_addr + kTP + g * (kKeys / 2);
    const uint32_t s_free_leader = mapa_shared(smem_u32(s_free), 0);
    const uint32_t p_full_leader = mapa_shared(smem_u32(&p_full[g]), 0);
    const uint32_t xch = smem_u32(smem + kXchOff);
    const uint32_t msh = smem_u32(smem + kMshOff) + rloc * 8;
    // {m, tile} of this row: the running max as decided by CTA-wide key tile `tile` (tiles
    // decide in order; one 8-byte store / load, so the pair is always consistent)
    auto publish_m = [&](float mv, int tile) {
      asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(msh), "r"(__float_as_uint(mv)),
                   "r"(static_cast<uint32_t>(tile)) : "memory");
    };
    auto wait_m = [&](int tile) {      // the running max once tile `tile` has decided
      uint32_t mv, tv;
      do {
        asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(mv), "=r"(tv) : "r"(msh) : "memory");
      } while (static_cast<int>(tv) < tile);
      return __uint_as_float(mv);
    };
    const float sl2 = p.scale_log2;
    int sc = 0;                                          // S tiles consumed by this warpgroup
    // MUFU token: the exp passes of the two warps of a sub-partition (A and B, same lane
    // quarter) alternate in tile order, so one's exp pass overlaps the other's TMEM loads, P
    // stores and waits instead of both running them at the same time.  Named barriers 5 + sub
    // ("A may exp") and 9 + sub ("B may exp"), 64 threads each (one bar.sync + one bar.arrive).
    const uint32_t tok_mine = (g == 0 ? 5u : 9u) + sub;
    const uint32_t tok_other = (g == 0 ? 9u : 5u) + sub;
    bool prev_last_b = false;                            // previous unit's last tile was B's
    int m = 0;                                           // units with key tiles so far
    int gbase = 0;                                       // stream index of the unit's tile 0
    int4 nx = fetch(pair);
    for (int w = pair; w < W; w += npairs) {
      const Work x = decode(w, nx);
      if (w + npairs < W) nx = fetch(w + npairs);
      const int nkv = x.nkv;
      // keys from this work item's first tile; causal (t0 = 0): row 128 rank + rloc of the
      // unit sees keys [0, L - rows + row] only
      int L = x.L - kKeys * x.t0;
      if constexpr (kCausal) L = min(x.L, x.L - x.rows_valid + 128 * static_cast<int>(rank) + rloc + 1);
      if (nkv == 0) continue;                          // the epilogue warps write O = 0
      const uint32_t tO = tmem + lane_addr + kTO + (m & 1) * kD;   // this unit's O
      float m_loc = -INFINITY;
      float l = 0.f;
      for (int j = g; j < nkv; j += 2) {
        pwait(&s_full[g], sc & 1, CTX(10, m, j));
        ++sc;
        const bool tr = (sub == 0 && lane == 0);
        const bool trd = tr;
        if (trd) GESR_T2(0, m * 16 + j);
        tc_fence_after();
        uint32_t r[kKeys];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, r + c * 32);
        tmem_ld_wait_regs32(r);
        tmem_ld_wait_regs32(r + 32);
        tmem_ld_wait_regs32(r + 64);
        tmem_ld_wait_regs32(r + 96);
#ifndef GESR_TRACE_LOOP
        if (trd) GESR_T2(1, m * 16 + j);
#endif
        const int valid = L - kKeys * j;
        const bool full = valid >= kKeys;
        if (!full) {
#pragma unroll
          for (int k = 0; k < kKeys; ++k)
            if (k >= valid) r[k] = __float_as_uint(-INFINITY);   // keys beyond L_b
        }
        // S is in registers: the buffer may take S(j+2)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_relaxed(s_free_leader);
#ifndef GESR_TRACE_LOOP
        if (trd) GESR_T2(2, m * 16 + j);
#endif
        // Row max.  Min/max instructions share the issue path of MUFU (scripts/micro/
        // exp_interf.cu: a max pass on the other warp of a sub-partition slows an exp pass from
        // 1.17k to 2k cycles), so only the unit's tile 0 reduces its exact max; later tiles
        // use m_sh speculatively and test the tile's row sum instead: sum <= 2^12 implies every
        // p <= 2^12 (so l <= 2^23, O far from fp32 overflow).  Only rows over it reduce their
        // exact max, and only if that exceeds m_sh by > 8 is m_sh raised.  (Each code path
        // below appears once: the softmax loop must stay small in the instruction cache.)
        auto row_max = [&]() {
          float mx[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) mx[e] = -INFINITY;
#pragma unroll
          for (int k = 0; k < kKeys; ++k) mx[k & 7] = fmaxf(mx[k & 7], __uint_as_float(r[k]));
          return fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                       fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        };
        const int gidx = gbase + j;                      // CTA-wide key tile index
        const bool first_b = j > 0 && m_loc == -INFINITY;   // B's first tile of the unit
        if (j == 0) m_loc = row_max() * sl2;
        // B's first tile takes the max tile 0 decided (published right after tile 0's pass, so
        // this wait, off the token path, is short and once per unit)
        if (first_b) m_loc = wait_m(gidx - 1);
        // the token release condition, kept out of the post-token path
        const bool pass_token = j + 1 < nkv || (g == 1 && w + npairs < W);
        // x = s*scale*log2e - m in place, before the token (FMA pipe, overlaps the other
        // warpgroup's exp pass)
        {
          const float neg_m = -m_loc;
#pragma unroll
          for (int k = 0; k < kKeys / 2; ++k) {
            float x0, x1;
            ffma2(x0, x1, __uint_as_float(r[2 * k]), __uint_as_float(r[2 * k + 1]), sl2, sl2,
                  neg_m, neg_m);
            r[2 * k] = __float_as_uint(x0);
            r[2 * k + 1] = __float_as_uint(x1);
          }
        }
        // P_g must have been read by PV(j-2) (long done, normally) before the exp pass writes it
        if (sc > 1) pwait(&p_free[g], (sc - 2) & 1, CTX(11, m, j));
        if (j > 0 || prev_last_b) named_bar_sync(tok_mine, 64);   // tile j-1's exp pass is done
        if (trd) GESR_T2(4, m * 16 + j);
        // The exp pass starts right after the token with this warpgroup's own m_loc; the previous
        // tile's decision (its sum test may raise the running max) is checked after the pass,
        // off the token's critical path, and the rare raise recomputes the tile.  The token is
        // released as soon as the first pass's MUFU work is issued.
        auto shift = [&](float d) {                      // x -= d (lanes with d = 0 unchanged)
#pragma unroll
          for (int k = 0; k < kKeys / 2; ++k) {
            float x0, x1;
            fadd2(x0, x1, __uint_as_float(r[2 * k]), __uint_as_float(r[2 * k + 1]), -d, -d);
            r[2 * k] = __float_as_uint(x0);
            r[2 * k + 1] = __float_as_uint(x1);
          }
        };
        bool checked_prev = (j == 0) || first_b;
        bool raised = false;
        float acc[8];
        float tsum;
#pragma unroll 1
        for (int pass = 0;; ++pass) {
          // p = 2^x, packed to bf16 pairs and stored to P_g (TMEM) 32 columns at a time;
          // masked keys give exactly 0
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#ifdef GESR_TRACE_LOOP
          if (trd && pass == 0) GESR_T2(1, m * 16 + j);
#endif
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
#ifdef GESR_TRACE_LOOP
            if (trd && pass == 0 && hh == 1) GESR_T2(2, m * 16 + j);
#endif
            uint32_t pk[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) {
              const int k = hh * 32 + u;
              const float p0 = ex2(__uint_as_float(r[2 * k]));
              const float p1 = ex2(__uint_as_float(r[2 * k + 1]));
              // hand the token to tile j+1's warpgroup (the next unit starts with A) as soon as
              // the first pass's last MUFU op is issued
              if (hh == 1 && u == 31 && pass == 0 && pass_token) named_bar_arrive(tok_other, 64);
              const int a = (k & 3) * 2;
              fadd2(acc[a], acc[a + 1], acc[a], acc[a + 1], p0, p1);
              pk[u] = pack_bf16x2(p0, p1);
            }
            tmem_st32(tP + hh * 32, pk);
          }
          if (trd && pass == 0) GESR_T2(3, m * 16 + j);
          tsum = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
          if (!checked_prev) {
            // the previous tile (other warpgroup) may have raised the running max after this
            // pass started: rescale l and recompute against it
            checked_prev = true;
            const float ms = wait_m(gidx - 1);
            const float d = fmaxf(ms - m_loc, 0.f);
            if (__any_sync(0xffffffffu, d != 0.f)) {
              l *= ex2(-d);
              m_loc += d;
              shift(d);
              continue;
            }
          }
          if (raised || j == 0) break;
          const bool over = !(tsum <= GESR_PAIR_SUM_LIMIT);
          if (!__any_sync(0xffffffffu, over)) break;
          const float dx = over ? row_max() : 0.f;       // exact max above m_loc (x units)
          const bool need = dx > 8.0f;
          if (!__any_sync(0xffffffffu, need)) break;
          // raise the running max: O must hold PV(j-1) (the other warpgroup's last tile) before
          // it is rescaled; no later PV can land before this warpgroup's p_full(j)
          pwait(pv_done, (gbase + j - 1) & 1, CTX(12, m, j));
          tc_fence_after();
          const float d = need ? dx : 0.f;
          const float alpha = ex2(-d);
          m_loc += d;
          l *= alpha;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait_regs32(o);
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st32(tO + c * 32, o);
          }
          tmem_st_wait();
          tc_fence_before();
          shift(d);
          raised = true;
        }
        // this tile's decision; tile 0 of a unit first lets the previous tile's decision land
        // (one word per row, written in tile order)
        if (j == 0 && gidx > 0) (void)wait_m(gidx - 1);
        publish_m(m_loc, gidx);
        l += tsum;
        tmem_st_wait();                                  // P_g in TMEM before PV(j) reads it
        tc_fence_before();
        __syncwarp();
        if (trd) GESR_T2(5, m * 16 + j);
        if (lane == 0) mbar_arrive_cluster_relaxed(p_full_leader);
      }
      prev_last_b = ((nkv - 1) & 1) == 1;
      // publish this warpgroup's max / sum of my rows for the epilogue warps
      if (m >= 4) pwait(&ml_empty[m & 3], ((m >> 2) - 1) & 1, CTX(15, m, 0));
      const uint32_t xb = xch + ((m & 3) * 2 * 2 * 128) * 4;      // [WG][m, l][row]
      st_shared_f32(xb + ((g * 2 + 0) * 128 + rloc) * 4, m_loc);
      st_shared_f32(xb + ((g * 2 + 1) * 128 + rloc) * 4, l);
      __syncwarp();
      // hardware named barrier 1 + m % 4 (8 softmax + 4 epilogue warps): the epilogue warps
      // wait for it in bar.sync, descheduled -- polling the former mbarrier spun ~390 times per
      // unit through a suspend-hint try_wait that wakes on every barrier event of the CTA (ncu:
      // 20 % of the kernel's issued instructions, on the softmax warps' sub-partitions)
      named_bar_arrive(kMlBarBase + (m & 3), kMlBarThreads);
      gbase += nkv;
      ++m;
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 12-15)
    // Normalises a unit's O (one accumulator, both warpgroups' PVs) while the softmax
    // warpgroups already work on the next unit: O / (l_A 2^(m_A-m) + l_B 2^(m_B-m)).  bf16
    // output: the warp's 32 rows x 128 columns go through four 2 KB staging boxes (32 rows x 32
    // columns, 64B swizzle), the O buffer is released as soon as it is read, then full 32-row
    // slabs leave with TMA tensor stores (a ragged slab stores its valid rows from the boxes).
    // fp32 output: direct stores.
    setmaxnreg_dec<kEpiRegs>();
    const uint32_t sub = warp & 3;
    const int rloc = static_cast<int>(sub) * 32 + static_cast<int>(lane);
    const int row_in_unit = static_cast<int>(rank) * 128 + rloc;
    const uint32_t tO0 = tmem + ((sub * 32) << 16) + kTO;   // O buffer 0; buffer 1 at + kD
    const uint32_t o_free_leader0 = mapa_shared(smem_u32(&o_free[0]), 0);
    const uint32_t o_free_leader1 = mapa_shared(smem_u32(&o_free[1]), 0);
    const uint32_t xch = smem_u32(smem + kXchOff);
    uint8_t* stg = smem + kStgOff + sub * 8192;
    const uint32_t stg_s = smem_u32(stg);
    const int64_t HD = static_cast<int64_t>(p.H) * kD;
    int m = 0;
    int4 nx = fetch(pair);
    for (int w = pair; w < W; w += npairs) {
      const Work x = decode(w, nx);
      if (w + npairs < W) nx = fetch(w + npairs);
      const int nkv = x.nkv, h = x.h;
      const bool row_ok = row_in_unit < x.rows_valid;
      const int64_t row = x.cbeg + row_in_unit;
      const bool split_out = S > 1;                     // write split-L partials, not O
      if (nkv == 0) {
        // L_b = 0 (or an empty split range): no keys, O = 0 and lse = -inf
        if (row_ok && split_out) {
          p.part_ml[(static_cast<int64_t>(x.split) * p.total_C + row) * p.H + h] =
              make_float2(-INFINITY, 0.f);
        } else if (row_ok) {
          if (p.o_bf16) {
            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.O) + row * HD + h * kD);
#pragma unroll
            for (int v = 0; v < 16; ++v) dst[v] = make_uint4(0u, 0u, 0u, 0u);
          } else {
            float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.O) + row * HD + h * kD);
#pragma unroll
            for (int v = 0; v < 32; ++v) dst[v] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
          if (p.lse != nullptr) p.lse[row * p.H + h] = -INFINITY;
        }
        continue;
      }
      named_bar_sync(kMlBarBase + (m & 3), kMlBarThreads);
      if (sub == 0 && lane == 0) GESR_T3(5, m);
      const uint32_t xb = xch + ((m & 3) * 2 * 2 * 128) * 4;
      const float mA = ld_shared_f32(xb + (0 * 128 + rloc) * 4);
      const float lA = ld_shared_f32(xb + (1 * 128 + rloc) * 4);
      const bool hasB = nkv > 1;
      const float mB = hasB ? ld_shared_f32(xb + (2 * 128 + rloc) * 4) : -INFINITY;
      const float lB = hasB ? ld_shared_f32(xb + (3 * 128 + rloc) * 4) : 0.f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&ml_empty[m & 3]);     // m / l slot read
      const float mm = hasB ? fmaxf(mA, mB) : mA;      // = the final shared max O is scaled to
      const float lsum = lA * ex2(mA - mm) + (hasB ? lB * ex2(mB - mm) : 0.f);
      const float inv = 1.0f / lsum;
      // the previous unit's TMA stores must have read the staging boxes
      if (lane == 0) bulk_wait_group_read<0>();
      __syncwarp();
      const int ob = m & 1;
      pwait(&o_done[ob], (m >> 1) & 1, CTX(14, m, 0), GESR_PAIR_EPI_SLEEP);
      if (sub == 0 && lane == 0) GESR_T3(6, m);
      tc_fence_after();
      const uint32_t tO = tO0 + ob * kD;
#pragma unroll 1
      for (int c = 0; c < kD / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + c * 32, o);
        tmem_ld_wait();
        if (sub == 0 && lane == 0) GESR_T4(c, m);
        if (c == kD / 32 - 1) {
          // O drained: unit m+2's first PV may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster_relaxed(ob ? o_free_leader1 : o_free_leader0);
          if (sub == 0 && lane == 0) GESR_T3(7, m);
        }
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float y0, y1;
          fmul2(y0, y1, __uint_as_float(o[e]), __uint_as_float(o[e + 1]), inv, inv);
          o[e] = __float_as_uint(y0);
          o[e + 1] = __float_as_uint(y1);
        }
        if (split_out) {
          if (row_ok) {
            float* dst = p.part_o + ((static_cast<int64_t>(x.split) * p.total_C + row) * p.H + h) * kD + c * 32;
#pragma unroll
            for (int vv = 0; vv < 4; ++vv) st_global_v8(dst + 8 * vv, o + 8 * vv);
          }
        } else if (p.o_bf16) {
          // box c (32 rows x 32 columns): 16-byte chunk qq of row `lane` (64B swizzle)
          const uint32_t rowp = stg_s + c * 2048 + lane * 64;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const int e = qq * 8;
            st_shared_v4(rowp + ((qq ^ ((lane >> 1) & 3)) << 4),
                         pack_bf16x2(__uint_as_float(o[e]), __uint_as_float(o[e + 1])),
                         pack_bf16x2(__uint_as_float(o[e + 2]), __uint_as_float(o[e + 3])),
                         pack_bf16x2(__uint_as_float(o[e + 4]), __uint_as_float(o[e + 5])),
                         pack_bf16x2(__uint_as_float(o[e + 6]), __uint_as_float(o[e + 7])));
          }
          if (sub == 0 && lane == 0) GESR_T4(8 + c, m);
        } else if (row_ok) {
          float* dst = static_cast<float*>(p.O) + row * HD + h * kD + c * 32;
#pragma unroll
          for (int vv = 0; vv < 4; ++vv) st_global_v8(dst + 8 * vv, o + 8 * vv);
        }
      }
      if (split_out) {
        if (row_ok)
          p.part_ml[(static_cast<int64_t>(x.split) * p.total_C + row) * p.H + h] = make_float2(mm, lsum);
      } else if (p.o_bf16) {
        const int row0 = static_cast<int>(rank) * 128 + static_cast<int>(sub) * 32;
        if (p.o_tma && row0 + 32 <= x.rows_valid) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int b = 0; b < 4; ++b)
#if GESR_PAIR_L2HINT >= 1
              tma_store_3d_hint(&map_o, stg + b * 2048, b * 32, h, static_cast<int32_t>(x.cbeg + row0), pol_first);
#else
              tma_store_3d(&map_o, stg + b * 2048, b * 32, h, static_cast<int32_t>(x.cbeg + row0));
#endif
            bulk_commit_group();
          }
        } else {
          __syncwarp();
          if (row_ok) {
            // ragged slab: copy my row out of the boxes (un-swizzle) with 16-byte stores
            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.O) + row * HD + h * kD);
#pragma unroll
            for (int b = 0; b < 4; ++b)
#pragma unroll
              for (int qq = 0; qq < 4; ++qq)
                dst[b * 4 + qq] = *reinterpret_cast<const uint4*>(
                    stg + b * 2048 + lane * 64 + ((qq ^ ((lane >> 1) & 3)) << 4));
          }
          __syncwarp();
        }
      }
      if (!split_out && row_ok && p.lse != nullptr)
        p.lse[row * p.H + h] = (mm + __log2f(lsum)) * 0.69314718055994530942f;
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

// Split-L merge, one warp per (candidate, head), lane k owning columns 4k..4k+3 (d = 128: the
// pair kernel is the only one that splits): the s-th partial holds O_s / l_s and (m_s, l_s) with
// m in log2 units of the scaled score; O = sum_s w_s (O_s / l_s) / sum_s w_s with
// w_s = l_s 2^(m_s - max_s m_s), summed in split order (deterministic).  Every split's (m, l) is
// a broadcast load and its 512-byte row one coalesced 16-byte load per lane, all independent.
constexpr int kCombineWarps = 8;
__global__ void __launch_bounds__(kCombineWarps * 32) attn_combine_kernel(const AttnParams p) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t stride = p.total_C * p.H;
  const int64_t rh = static_cast<int64_t>(blockIdx.x) * kCombineWarps + (threadIdx.x >> 5);
  if (rh >= stride) return;                        // row * H + h
  const int lane = threadIdx.x & 31;
  const int S = p.splits;                          // <= kMaxSplits = 64
  // lane k: (m, l) of splits k and k + 32, loaded at once; the max by a butterfly (exact)
  float2 ml0 = make_float2(0.f, 0.f), ml1 = make_float2(0.f, 0.f);
  if (lane < S) ml0 = __ldg(p.part_ml + lane * stride + rh);
  if (lane + 32 < S) ml1 = __ldg(p.part_ml + (lane + 32) * stride + rh);
  float mmax = fmaxf(ml0.y > 0.f ? ml0.x : -INFINITY, ml1.y > 0.f ? ml1.x : -INFINITY);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mmax = fmaxf(mmax, __shfl_xor_sync(0xffffffffu, mmax, o));
  // w_s = l_s 2^(m_s - max), negative for an empty split (skipped)
  const float w0 = ml0.y > 0.f ? ml0.y * exp2f(ml0.x - mmax) : -1.f;
  const float w1 = ml1.y > 0.f ? ml1.y * exp2f(ml1.x - mmax) : -1.f;
  float wsum = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* po = reinterpret_cast<const float4*>(p.part_o) + rh * 32 + lane;
#pragma unroll 4
  for (int s = 0; s < S; ++s) {
    const float4 o = __ldg(po + s * stride * 32);
    const float w = __shfl_sync(0xffffffffu, s < 32 ? w0 : w1, s & 31);
    if (w >= 0.f) {
      wsum += w;
      acc.x += w * o.x;
      acc.y += w * o.y;
      acc.z += w * o.z;
      acc.w += w * o.w;
    }
  }
  const float4 v = wsum > 0.f ? make_float4(acc.x / wsum, acc.y / wsum, acc.z / wsum, acc.w / wsum)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t o0 = rh * 128 + 4 * lane;          // O [total_C, H, 128] = [row][h][col]
  if (p.o_bf16) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p.O) + o0) = u;
  } else {
    *reinterpret_cast<float4*>(static_cast<float*>(p.O) + o0) = v;
  }
  if (lane == 0 && p.lse != nullptr)
    p.lse[rh] = wsum > 0.f ? (mmax + log2f(wsum)) * 0.69314718055994530942f : -INFINITY;
}

}  // namespace

cudaError_t launch_attn_combine(const AttnParams& p, int d, cudaStream_t stream) {
  const int64_t n = p.total_C * p.H;
  if (n == 0) return cudaSuccess;
  if (d != 128) return cudaErrorInvalidValue;
  return launch_pdl(attn_combine_kernel,
                    dim3(static_cast<unsigned>((n + kCombineWarps - 1) / kCombineWarps)),
                    dim3(kCombineWarps * 32), 0, stream, p);
}

#ifdef GESR_TRACE
extern "C" int gesr_debug_trace2_copy(void* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace2, sizeof(g_trace2)));
}
extern "C" int gesr_debug_trace4_copy(void* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace4, sizeof(g_trace4)));
}
extern "C" int gesr_debug_trace3_copy(void* host) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace3, sizeof(g_trace3)));
}
#endif

cudaError_t launch_attn_pair(const CUtensorMap& mq, const CUtensorMap& mkh, const CUtensorMap& mvh,
                             const CUtensorMap& mo, const AttnParams& p, int64_t max_units,
                             cudaStream_t stream) {
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(attn_pair_kernel<false>),
                                   kSmemBytes);
  if (e != cudaSuccess) return e;
  e = ensure_smem_attr(reinterpret_cast<const void*>(attn_pair_kernel<true>), kSmemBytes);
  if (e != cudaSuccess) return e;
  int max_pairs = device_cached(1);      // co-resident CTA pairs on this device
  if (max_pairs == 0) {
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
    e = cudaOccupancyMaxActiveClusters(&clusters, attn_pair_kernel<false>, &cfg);
    if (e != cudaSuccess || clusters <= 0) {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      clusters = sms / 2;
      (void)cudaGetLastError();
    }
    max_pairs = clusters;
    device_cache_store(1, max_pairs);
  }
  const int64_t work = max_units * p.H * p.splits;
  const unsigned pairs = static_cast<unsigned>(work < max_pairs ? work : max_pairs);
  return launch_pdl(p.causal ? attn_pair_kernel<true> : attn_pair_kernel<false>, dim3(2 * pairs),
                    dim3(kThreads), kSmemBytes, stream, mq, mkh, mvh, mo, p);
}

}  // namespace gesr
