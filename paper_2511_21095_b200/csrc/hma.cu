// hma.cu -- K-HMA: Hard Matching Attention raw match counts (s3.4.1).
//
//   counts[t*F + f] = sum_{i in user list (b,f)} sum_{j in item list (t,f)} [u_i == t_j]
//   then min(count, cap) if cap > 0.
//
// The binary attention matrix Attn_match(U, I) summed against a value tensor of ones is a
// multiplicity lookup: each item ID contributes the number of times it occurs in the user's
// list of the same field.  Exact integer arithmetic; bit-identical to the definition.
//
// B200 design.  The kernel streams the item-ID CSR (~8.5 int64 IDs per (candidate, field)
// segment at the headline, 1.1 GB, read once).  It is bound by instruction issue, not DRAM,
// unless a 32-ID window costs well under ~60 warp instructions (round-2 v3: ~111, 0.34 of HBM).
// v4 is built around that budget:
//   grid (B, Y): CTA (b, y) owns request b and candidate chunks y, y+Y, ... of `chunk` rows.
//   1. Tables.  The request's F user lists go into per-field hash tables in shared memory:
//      16-byte buckets of TWO 64-bit slots (one 16-byte read per lookup), >= 4 buckets per ID,
//      one slot per OCCURRENCE of a user ID (a lookup counts matching slots).  Each field's
//      table is built by one warp, which retries with a new hash seed until no bucket
//      overflows (expected < 2 tries at 64 IDs in 256 buckets); a field that never fits (a user
//      ID repeated 3+ times, or a list too long for the pool) is scanned in global memory.
//      An empty slot holds a FILLER key chosen per (field, seed) to hash into the other half of
//      the table, so no key that hashes to a bucket can equal its fillers: every int64 value,
//      INT64_MIN included, is an ordinary ID and a lookup needs no emptiness test.  The field's
//      table word is also its hash multiplier (odd by construction): h = mix(key) * tab.
//      An 8-bit-per-bucket bitmap of the user IDs' hashes is read first (one 32-bit shared
//      load); the bucket only where the bit is set (~28% of IDs: matches + false positives).
//   2. Scan: each warp takes 32 consecutive (candidate, field) segments (their IDs are one
//      contiguous range of the CSR stream) and walks the range in 32-ID windows, one coalesced
//      8-byte load per lane, 4 windows in flight, the next group's range prefetched to L2.  The segment of each ID position comes from
//      the segment starts that fall in the window: lane k contributes bit (off_k - base), one
//      redux.sync.or forms the window's start mask, and position l's segment is the running
//      start count plus popc(mask & lanemask_le) - 1 (groups with an empty segment take a
//      binary-search path).  The segment's table word comes by shuffle; a hit is a predicated
//      shared reduction on the warp's counter of that segment, and lane k stores segment k's
//      count (one coalesced 128-byte store per group).
#include <cuda_runtime.h>

#include <type_traits>

#include "kernels.h"
#include "ptx.cuh"

namespace gesr {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kChunkMax = 1024;            // candidates per CTA chunk (runtime: 1024 >> k)
constexpr int kChunkFloor = 32;
constexpr int kPoolBuckets = 4096;         // 16-byte buckets (2 slots): 64 KB of keys per CTA
constexpr int kMinBuckets = 4;             // a field owns whole 32-bit bitmap words
constexpr int kMaxSeeds = 32;              // hash seeds tried per field before going global
constexpr int kMaxFields = 256;
constexpr int kWinUnroll = 4;              // 32-ID windows in flight per warp
constexpr int kFastMaxIds = 32 * 64;       // groups up to this many IDs take the fast path
constexpr uint32_t kBitsOffset = kPoolBuckets * 16;   // byte offset of the bitmap
constexpr uint32_t kMulHi = 0x85EBCA77u;

// Table word of a field (also its hash multiplier, odd by construction):
//   bits 0-4   sh3 = 32 - log2(#buckets) - 3 (odd: tables have 4^k buckets), so
//              h >> sh3 = 8 * bucket + 3 bitmap bits; a wrapping shift by the word itself
//              uses exactly these bits (no decode)
//   bits 5-14  8 * first bucket (tables start at multiples of 4 buckets)
//   bits 15-31 hash seed (varies the multiplier between build attempts)
// Lookup: h = mix(key) * tab; fb = (tab & 0x7fe0) + (h >> (tab & 31)) is the bitmap bit and
// fb >> 3 the bucket; the top bit of h selects the table half (and so the filler).
__device__ __forceinline__ uint32_t key_mix(unsigned long long key) {
  return static_cast<uint32_t>(key) + static_cast<uint32_t>(key >> 32) * kMulHi;
}
__device__ __forceinline__ uint32_t filter_pos(uint32_t tab, uint32_t h) {
  return (tab & 0x7fe0u) + __funnelshift_r(h, 0u, tab);
}

struct HmaSmem {
  ulonglong2 bkt[kPoolBuckets];              // at byte 0: empty slots hold the half's filler
  uint32_t bits[kPoolBuckets * 8 / 32];      // at kBitsOffset: 8 bits per bucket
  uint32_t tab[kMaxFields];
  int glob[kMaxFields];                      // 1: the field's list is scanned in global memory
  long long uoff[kMaxFields + 1];            // this request's user_offsets (F+1)
  int warp_cnt[kWarps][32];
  alignas(16) uint32_t smask[kWarps][kFastMaxIds / 32];  // per warp: bit p set where a segment starts
  int slow_any;                              // some field is scanned in global memory
};
static_assert(offsetof(HmaSmem, bits) == kBitsOffset, "bitmap offset");

// Streamed item IDs (L2-prefetched, read once).  Where pos >= n the result is left undefined:
// the lookup masks those positions, so no move or zero-fill is spent on them.
__device__ __forceinline__ unsigned long long ld_ids(const int64_t* ptr, int pos, int n) {
  unsigned long long v;
  asm volatile(
      "{\n .reg .pred p;\n setp.lt.s32 p, %1, %2;\n"
      " @p ld.global.nc.L1::no_allocate.u64 %0, [%3];\n}\n"
      : "=l"(v)
      : "r"(pos), "r"(n), "l"(ptr));
  return v;
}
// One lookup of the fast path: bitmap bit, then the 16-byte bucket -- lanes whose bit is clear
// (or, in a group's tail windows, whose position is past the end) all read bucket 0 instead, a
// broadcast that costs no extra shared-memory wavefront, and their match is masked (a predicated
// bucket load would keep its registers live across loop iterations).  A pure function of its
// inputs (non-volatile asm, no memory clobber: the tables are read-only during the scan), so
// the chains of consecutive windows can overlap; returns the matching slots' count.
template <bool kCheck>
__device__ __forceinline__ uint32_t lookup_count(uint32_t bits0, uint32_t bkt0, uint32_t tab,
                                                 unsigned long long key, int lane, int lim) {
  const uint32_t h = key_mix(key) * tab;
  const uint32_t fb = filter_pos(tab, h);
  const uint32_t waddr = bits0 + ((fb >> 3) & ~3u);
  const uint32_t bkt = bkt0 + ((fb << 1) & ~15u);
  uint32_t c;
  if (kCheck) {
    asm("{\n .reg .pred p, q, r, v;\n .reg .b32 w, ad;\n .reg .b64 a, b;\n"
        " ld.shared.u32 w, [%2];\n"
        " setp.lt.s32 v, %6, %7;\n"
        " shf.r.wrap.b32 w, w, w, %3;\n"
        " and.b32 w, w, 1;\n"
        " setp.ne.and.u32 p, w, 0, v;\n"
        " selp.b32 ad, %4, %5, p;\n"
        " ld.shared.v2.u64 {a, b}, [ad];\n"
        " setp.eq.and.u64 q, a, %1, p;\n"
        " setp.eq.and.u64 r, b, %1, p;\n"
        " selp.u32 %0, 1, 0, q;\n"
        " @r add.u32 %0, %0, 1;\n}\n"
        : "=r"(c)
        : "l"(key), "r"(waddr), "r"(fb), "r"(bkt), "r"(bkt0), "r"(lane), "r"(lim));
  } else {
    asm("{\n .reg .pred p, q, r;\n .reg .b32 w, ad;\n .reg .b64 a, b;\n"
        " ld.shared.u32 w, [%2];\n"
        " shf.r.wrap.b32 w, w, w, %3;\n"
        " and.b32 w, w, 1;\n"
        " setp.ne.u32 p, w, 0;\n"
        " selp.b32 ad, %4, %5, p;\n"
        " ld.shared.v2.u64 {a, b}, [ad];\n"
        " setp.eq.and.u64 q, a, %1, p;\n"
        " setp.eq.and.u64 r, b, %1, p;\n"
        " selp.u32 %0, 1, 0, q;\n"
        " @r add.u32 %0, %0, 1;\n}\n"
        : "=r"(c)
        : "l"(key), "r"(waddr), "r"(fb), "r"(bkt), "r"(bkt0));
  }
  return c;
}

// Any field, any key (generic path): global scan for fields that did not fit, else the table.
__device__ __noinline__ int lookup_any(const HmaSmem& s, const HmaParams& p, int f,
                                       unsigned long long key) {
  if (s.glob[f]) {
    int c = 0;
    for (long long i = s.uoff[f]; i < s.uoff[f + 1]; ++i)
      c += (static_cast<unsigned long long>(__ldg(p.user_ids + i)) == key) ? 1 : 0;
    return c;
  }
  const uint32_t tab = s.tab[f];
  const uint32_t fb = filter_pos(tab, key_mix(key) * tab);
  if (((s.bits[fb >> 5] >> (fb & 31u)) & 1u) == 0u) return 0;   // (global fields: tab unused)
  const ulonglong2 b = s.bkt[fb >> 3];
  return (b.x == key) + (b.y == key);
}

__global__ void __launch_bounds__(kThreads, 2)
    hma_kernel(const HmaParams p, const int chunk) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  HmaSmem& s = *reinterpret_cast<HmaSmem*>(smem_raw);
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.x;
  const int64_t cb = p.cand_offsets[b];
  const int64_t ce = p.cand_offsets[b + 1];
  const int64_t first = cb + static_cast<int64_t>(blockIdx.y) * chunk;
  if (first >= ce) return;   // uniform
  const int F = p.F;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  // ---- 1. per-field tables of the request's user lists
  for (int f = tid; f <= F; f += kThreads) s.uoff[f] = p.user_offsets[static_cast<int64_t>(b) * F + f];
  for (int i = tid; i < kWarps * 32; i += kThreads) (&s.warp_cnt[0][0])[i] = 0;
  __syncthreads();
  // the first 64 IDs of this warp's first field are loaded now, while thread 0 lays out the
  // tables (their latency would otherwise sit between the two barriers and the build)
  unsigned long long pre0 = 0ull, pre1 = 0ull;
  if (warp < F) {
    const long long u0 = s.uoff[warp];
    const long long n = s.uoff[warp + 1] - u0;
    if (lane < n) pre0 = static_cast<unsigned long long>(__ldg(p.user_ids + u0 + lane));
    if (lane + 32 < n) pre1 = static_cast<unsigned long long>(__ldg(p.user_ids + u0 + lane + 32));
  }
  if (tid == 0) {   // bucket ranges: 4^k >= max(4, 4n) buckets, >= n if the pool is short
    int used = 0;
    s.slow_any = 0;
    for (int f = 0; f < F; ++f) {
      const long long n = s.uoff[f + 1] - s.uoff[f];
      int nb = kMinBuckets, lg = 2;
      while (nb < 4 * n && nb < kPoolBuckets) { nb <<= 2; lg += 2; }
      while (used + nb > kPoolBuckets && nb >= 4 * n && nb > kMinBuckets) { nb >>= 2; lg -= 2; }
      if (used + nb <= kPoolBuckets && nb >= n) {
        s.tab[f] = (static_cast<uint32_t>(used) << 3) | static_cast<uint32_t>(32 - lg - 3);
        s.glob[f] = 0;
        used += nb;
      } else {
        s.tab[f] = 1u;
        s.glob[f] = 1;
        s.slow_any = 1;
      }
    }
  }
  __syncthreads();
  // one warp per field: fill, insert, retry with the next seed while a bucket overflows
  for (int f = warp; f < F; f += kWarps) {
    if (s.glob[f]) continue;
    const uint32_t t0 = s.tab[f];
    const int base = static_cast<int>((t0 & 0x7fe0u) >> 3);
    const int lg = 32 - 3 - static_cast<int>(t0 & 31u);
    const int nb = 1 << lg;
    const long long u0 = s.uoff[f];
    const int n = static_cast<int>(s.uoff[f + 1] - u0);
    bool ok = false;
    for (int seed = 0; seed < kMaxSeeds && !ok; ++seed) {
      const uint32_t t = (t0 & 0x7fffu) | (static_cast<uint32_t>(seed + 1) * 0x2f5a3u) << 15;
      // fillers: the smallest values whose hash lands in the upper (fill_lo) / lower (fill_hi)
      // half; lower-half buckets hold fill_lo, upper-half buckets fill_hi
      const uint32_t top = (key_mix(static_cast<unsigned long long>(lane + 1)) * t) >> 31;
      const uint32_t up = __ballot_sync(0xffffffffu, top != 0u);
      const uint32_t lo = ~up;
      if (up == 0u || lo == 0u) continue;
      const unsigned long long fill_lo = static_cast<unsigned long long>(__ffs(up));
      const unsigned long long fill_hi = static_cast<unsigned long long>(__ffs(lo));
      for (int i = lane; i < nb; i += 32) {
        const unsigned long long e = (i < nb / 2) ? fill_lo : fill_hi;
        s.bkt[base + i] = make_ulonglong2(e, e);
      }
      for (int i = lane; i < nb / 4; i += 32) s.bits[base / 4 + i] = 0u;
      __syncwarp();
      bool over = false;
      for (int i = lane; i < n; i += 32) {
        const unsigned long long key =
            f == warp && i < 64 ? (i < 32 ? pre0 : pre1)
                                : static_cast<unsigned long long>(__ldg(p.user_ids + u0 + i));
        const uint32_t h = key_mix(key) * t;
        const uint32_t fb = filter_pos(t, h);
        const unsigned long long fill = (h >> 31) ? fill_hi : fill_lo;
        unsigned long long* slots = reinterpret_cast<unsigned long long*>(&s.bkt[fb >> 3]);
        if (atomicCAS(slots, fill, key) != fill && atomicCAS(slots + 1, fill, key) != fill)
          over = true;
        atomicOr(&s.bits[fb >> 5], 1u << (fb & 31u));
      }
      ok = !__any_sync(0xffffffffu, over);
      if (ok && lane == 0) s.tab[f] = t;
      __syncwarp();
    }
    if (!ok && lane == 0) {
      s.glob[f] = 1;
      s.slow_any = 1;
    }
  }
  __syncthreads();
  const bool slow_any = s.slow_any != 0;

  // ---- 2. the item-ID stream, 32 segments per warp step.  Positions are 32-bit offsets from
  // the chunk's first item ID (a chunk holding 2^31 IDs or more takes a 64-bit lane-per-segment
  // loop instead).
  const uint32_t cnt_base = smem_u32(&s.warp_cnt[warp][0]);
  const uint32_t le_mask = 0xffffffffu >> (31 - lane);               // lanemask_le
  for (int64_t c0 = first; c0 < ce; c0 += static_cast<int64_t>(gridDim.y) * chunk) {
    const int64_t c1 = (c0 + chunk < ce) ? c0 + chunk : ce;
    const int64_t seg_begin = c0 * F;
    const int nseg_chunk = static_cast<int>((c1 - c0) * F);
    const int64_t id0 = __ldg(p.item_offsets + seg_begin);
    if (__ldg(p.item_offsets + seg_begin + nseg_chunk) - id0 >= (1ll << 31)) {
      // a chunk of 2^31 or more item IDs: one lane per segment, 64-bit offsets (slow, exact)
      for (int q = tid; q < nseg_chunk; q += kThreads) {
        const int64_t seg = seg_begin + q;
        int c = 0;
        for (int64_t i = __ldg(p.item_offsets + seg); i < __ldg(p.item_offsets + seg + 1); ++i)
          c += lookup_any(s, p, q % F, static_cast<unsigned long long>(__ldg(p.item_ids + i)));
        if (p.cap > 0 && c > p.cap) c = p.cap;
        p.counts[seg] = c;
        if (p.E != nullptr) {
          const int64_t rowE = static_cast<int64_t>(c) + static_cast<int64_t>(q % F) * (p.cap + 1);
          for (int k = 0; k < p.dh_chunks; ++k) p.emb[seg * p.dh_chunks + k] = __ldg(p.E + rowE * p.dh_chunks + k);
        }
      }
      continue;
    }
    const bool fast_chunk = !slow_any;
    const int64_t* idp = p.item_ids + id0;
    // low 32 bits of the chunk's offsets: exact relative positions when the chunk is < 2^31 IDs
    const uint32_t* offp = reinterpret_cast<const uint32_t*>(p.item_offsets + seg_begin);
    const uint32_t id0lo = static_cast<uint32_t>(id0);
    int gl = warp * 32;                                               // group's first segment
    constexpr int kStep = kWarps * 32;
    // lane k: start of segment gg+k (lanes past the group: its end); e: the group's end.  Raw
    // low words: the chunk base is subtracted where the values are used, a group later, so no
    // instruction waits on these loads early
    auto fetch = [&](int gg, uint32_t& o, uint32_t& e) {
      if (gg + 32 <= nseg_chunk) {         // a full group (all but the chunk's last)
        const uint32_t* q = offp + 2 * gg;
        o = __ldg(q + 2 * lane);
        e = __ldg(q + 64);
      } else if (gg < nseg_chunk) {
        const int ns = nseg_chunk - gg;
        o = __ldg(offp + 2 * (gg + (lane < ns ? lane : ns)));
        e = __ldg(offp + 2 * (gg + ns));
      } else {
        o = id0lo;
        e = id0lo;
      }
    };
    int32_t* const cnt_out = p.counts + seg_begin;
    const int cap = p.cap;
    const bool emb = p.E != nullptr;
    uint32_t off_cur, end_cur, off_nxt, end_nxt;
    fetch(gl, off_cur, end_cur);
    fetch(gl + kStep, off_nxt, end_nxt);
    {
      const int s0 = static_cast<int>(__shfl_sync(0xffffffffu, off_cur, 0) - id0lo);
      const uintptr_t a0 = (reinterpret_cast<uintptr_t>(idp + s0) & ~uintptr_t(127)) + 128u * lane;
      if (gl < nseg_chunk && a0 < reinterpret_cast<uintptr_t>(idp + static_cast<int>(end_cur - id0lo)))
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a0));
    }
    int my_f = (gl + lane) % F;                                       // seg_begin % F == 0
    const int f_step = kStep % F;
    unsigned long long kk[kWinUnroll];     // IDs of the next kWinUnroll windows, in flight
    for (; gl < nseg_chunk; gl += kStep) {
      const int nseg = nseg_chunk - gl < 32 ? nseg_chunk - gl : 32;
      const int my_off = static_cast<int>(off_cur - id0lo);
      const int end = static_cast<int>(end_cur - id0lo);
      const int start = __shfl_sync(0xffffffffu, my_off, 0);
      const int nstart = static_cast<int>(__shfl_sync(0xffffffffu, off_nxt, 0) - id0lo);
      const int n_next = static_cast<int>(end_nxt - id0lo) - nstart;   // 0 past the chunk
      {   // the next group's IDs toward L2, one 128-byte line per lane (a group is ~17 lines)
        const uintptr_t a0 = (reinterpret_cast<uintptr_t>(idp + nstart) & ~uintptr_t(127)) + 128u * lane;
        if (n_next > 0 && a0 < reinterpret_cast<uintptr_t>(idp + nstart + n_next))
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a0));
      }
      off_cur = off_nxt;
      end_cur = end_nxt;
      fetch(gl + 2 * kStep, off_nxt, end_nxt);
      const int nxt = __shfl_down_sync(0xffffffffu, my_off, 1);
      const int my_end = lane + 1 < nseg ? nxt : end;
      const int n_ids = end - start;
      const uint32_t my_tab = s.tab[my_f];
      const int64_t* idl = idp + start + lane;
      const bool empty_seg = lane < nseg && my_end == my_off;
#pragma unroll
      for (int u = 0; u < kWinUnroll; ++u) kk[u] = ld_ids(idl + u * 32, u * 32 + lane, n_ids);
      if (fast_chunk && !__any_sync(0xffffffffu, empty_seg) && n_ids <= kFastMaxIds) {
        // fast path: every segment of the group non-empty (segment starts distinct), every
        // field in a shared-memory table.  The group's segment starts go into a bitmask over its
        // ID positions; a window's word of it gives each position's segment by one popc.
        uint32_t* smask = s.smask[warp];
        const int nwin = (n_ids + 31) >> 5;                            // <= 64
        if (lane < nwin) smask[lane] = 0u;
        if (lane + 32 < nwin) smask[lane + 32] = 0u;
        __syncwarp();
        if (lane < nseg) {
          const uint32_t rel = static_cast<uint32_t>(my_off - start);
          atomicOr(&smask[rel >> 5], 1u << (rel & 31u));
        }
        __syncwarp();
        int cum_m1 = -1;                                             // starts so far, minus 1
        // shared address of the start mask, passed through a volatile asm after the barrier:
        // the (non-volatile) window loads below cannot be hoisted above it
        uint32_t sm_addr;
        asm volatile("mov.u32 %0, %1;" : "=r"(sm_addr) : "r"(smem_u32(smask)));
        const uint32_t bits0 = smem_u32(&s.bits[0]), bkt0 = smem_u32(&s.bkt[0]);
        auto window = [&](unsigned long long key, int w, auto check) {
          uint32_t starts;
          asm("ld.shared.u32 %0, [%1];" : "=r"(starts) : "r"(sm_addr + 4u * w));
          const int seg = cum_m1 + __popc(starts & le_mask);
          cum_m1 += __popc(starts);
          const uint32_t t = __shfl_sync(0xffffffffu, my_tab, seg);
          const uint32_t c = lookup_count<decltype(check)::value>(bits0, bkt0, t, key, lane,
                                                                  n_ids - w * 32);
          asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n"
                       " @q red.shared.add.u32 [%0], %1;\n}\n"
                       ::"r"(cnt_base + 4u * static_cast<uint32_t>(seg)), "r"(c) : "memory");
        };
        // two full windows with every shared-memory read before either counter update, so the
        // two lookup chains overlap
        auto window2 = [&](unsigned long long k0, unsigned long long k1, int w) {
          uint32_t st0, st1;
          asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(st0), "=r"(st1) : "r"(sm_addr + 4u * w));
          const int seg0 = cum_m1 + __popc(st0 & le_mask);
          cum_m1 += __popc(st0);
          const int seg1 = cum_m1 + __popc(st1 & le_mask);
          cum_m1 += __popc(st1);
          const uint32_t t0 = __shfl_sync(0xffffffffu, my_tab, seg0);
          const uint32_t t1 = __shfl_sync(0xffffffffu, my_tab, seg1);
          const uint32_t c0 = lookup_count<false>(bits0, bkt0, t0, k0, lane, 0);
          const uint32_t c1 = lookup_count<false>(bits0, bkt0, t1, k1, lane, 0);
          asm volatile("{\n .reg .pred q, r;\n setp.ne.u32 q, %2, 0;\n setp.ne.u32 r, %3, 0;\n"
                       " @q red.shared.add.u32 [%0], %2;\n"
                       " @r red.shared.add.u32 [%1], %3;\n}\n"
                       ::"r"(cnt_base + 4u * static_cast<uint32_t>(seg0)),
                         "r"(cnt_base + 4u * static_cast<uint32_t>(seg1)), "r"(c0), "r"(c1)
                       : "memory");
        };
        // full windows, kWinUnroll at a time, each refilling its key register kWinUnroll
        // windows ahead; then the last <= kWinUnroll windows (already loaded), the partial one
        // with the position check
        const int nfull = n_ids >> 5;
        int w0 = 0;
        for (; w0 + kWinUnroll <= nfull; w0 += kWinUnroll) {
#pragma unroll
          for (int u = 0; u < kWinUnroll; u += 2) {
            window2(kk[u], kk[u + 1], w0 + u);
            const int nw = (w0 + kWinUnroll + u) * 32;
            kk[u] = ld_ids(idl + nw, nw + lane, n_ids);
            kk[u + 1] = ld_ids(idl + nw + 32, nw + 32 + lane, n_ids);
          }
        }
        // the last <= kWinUnroll windows, two at a time while two remain full
        if (w0 + 2 <= nfull) {
          window2(kk[0], kk[1], w0);
          if (w0 + 3 < nwin) {
            // (w0 + 4 > nfull here: window w0 + 2 is full, w0 + 3 the partial one)
            window(kk[2], w0 + 2, std::false_type{});
            window(kk[3], w0 + 3, std::true_type{});
          } else if (w0 + 2 < nwin) {
            window(kk[2], w0 + 2, std::true_type{});
          }
        } else {
#pragma unroll
          for (int u = 0; u < kWinUnroll; ++u) {
            if (w0 + u < nwin) window(kk[u], w0 + u, std::true_type{});
          }
        }
      } else {
        // generic path (a group with empty segments, very long lists, or a CTA with a field
        // in global memory): owning segment by binary search over the segment starts
        const int rel = my_off - start;
        const int64_t* ids = idp + start;
        for (int base = 0; base < n_ids; base += 32) {
          const int pos = base + lane;
          const bool ok = pos < n_ids;
          const unsigned long long key = ok ? static_cast<unsigned long long>(__ldg(ids + pos)) : 0ull;
          int k = 0;     // owning segment: largest k with off[k] <= pos
#pragma unroll
          for (int step = 16; step >= 1; step >>= 1) {
            const int o = __shfl_sync(0xffffffffu, rel, k + step);
            if (o <= pos) k += step;
          }
          const int f = __shfl_sync(0xffffffffu, my_f, k);
          if (ok) {
            const int c = lookup_any(s, p, f, key);
            if (c != 0) atomicAdd(&s.warp_cnt[warp][k], c);
          }
        }
      }
      __syncwarp();
      if (lane < nseg) {
        int c = s.warp_cnt[warp][lane];
        if (cap > 0 && c > cap) c = cap;
        cnt_out[gl + lane] = c;
        if (emb) {
          const int64_t seg = seg_begin + gl + lane;
          // offset embedding (stride cap + 1: DESIGN.md R14): segment
          // seg = (candidate t, field f) owns out[t][f D_h, (f + 1) D_h) -- contiguous
          const int64_t rowE = static_cast<int64_t>(c) + static_cast<int64_t>(my_f) * (cap + 1);
          const uint4* src = p.E + rowE * p.dh_chunks;
          uint4* dst = p.emb + seg * p.dh_chunks;
          for (int q = 0; q < p.dh_chunks; ++q) dst[q] = __ldg(src + q);
        }
      }
      s.warp_cnt[warp][lane] = 0;
      __syncwarp();
      my_f += f_step;
      if (my_f >= F) my_f -= F;
    }
  }
}

}  // namespace

cudaError_t launch_hma(const HmaParams& p, cudaStream_t stream) {
  const int smem = static_cast<int>(sizeof(HmaSmem));
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(hma_kernel), smem);
  if (e != cudaSuccess) return e;
  // Large chunks amortise the per-CTA table build; 256-candidate chunks when that leaves fewer
  // than 4 CTAs per SM; and with very few requests the chunk halves (down to 32 candidates)
  // while the grid is smaller than the SM count (config 4: B = 1, C = 4096 -> 128 CTAs of 32
  // candidates, 23 -> 12 us; config 2's 256 CTAs keep 256: more table builds cost more there).
  int64_t per = p.B > 0 ? (p.total_C + p.B - 1) / p.B : 1;
  int chunk = kChunkMax;
  if (p.B * ((per + kChunkMax - 1) / kChunkMax) < 4 * 148) chunk = 256;
  while (chunk > kChunkFloor && p.B * ((per + chunk - 1) / chunk) < 148) chunk >>= 1;
  int64_t y = (per + chunk - 1) / chunk;
  if (y < 1) y = 1;
  if (y > 65535) y = 65535;
  dim3 grid(static_cast<unsigned>(p.B), static_cast<unsigned>(y));
  return launch_pdl(hma_kernel, grid, dim3(kThreads), smem, stream, p, chunk);
}

}  // namespace gesr
