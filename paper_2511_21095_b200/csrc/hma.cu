// hma.cu -- K-HMA: Hard Matching Attention raw match counts (s3.4.1).
//
//   counts[t*F + f] = sum_{i in user list (b,f)} sum_{j in item list (t,f)} [u_i == t_j]
//   then min(count, cap) if cap > 0.
//
// The binary attention matrix Attn_match(U, I) summed against a value tensor of ones is a
// multiplicity lookup: each item ID contributes the number of times it occurs in the user's
// list of the same field.  Exact integer arithmetic; bit-identical to the definition.
//
// B200 design.  The kernel is bound by the item-ID stream (~8.5 int64 IDs per (candidate,
// field) segment, read once); round 1's version spent ~114 instructions per ID (owner-map
// writes, 64-bit window probes with continuation tests) and ran at 0.31 of HBM.  This one is
// built around a per-ID instruction budget of ~40:
//   grid (B, Y): CTA (b, y) owns request b and candidate chunks y, y+Y, ... of `chunk` rows.
//   1. Table build: the request's F user lists go into per-field BUCKETED hash tables in shared
//      memory -- 2^k buckets of 4 64-bit slots (32 bytes, two 16-byte reads), one slot per
//      OCCURRENCE of a user ID (so a lookup counts matching slots; no count array), >= 2 buckets
//      per ID (mean bucket load <= 1/2).  A bucket that overflows spills into a small per-CTA
//      stash; a field whose list does not fit the pool is looked up in global memory.  An empty
//      slot holds a FILLER key that hashes into the other half of the table (bucket index top
//      bit flipped), so no key that hashes to this bucket can equal it: every int64 value,
//      INT64_MIN included, is an ordinary ID and a lookup needs no emptiness test.  A 16-bit-
//      per-bucket bitmap of the user IDs' hashes is read first (one 32-bit shared load); the
//      bucket (two 16-byte loads, predicated) only for the ~28% of IDs whose bit is set.
//   2. Scan: each warp takes 32 consecutive (candidate, field) segments (their IDs are one
//      contiguous range of the CSR stream) and walks the range in 32-ID windows, one coalesced
//      8-byte load per lane, 4 windows in flight.  The segment of each ID position comes from
//      the segment starts that fall in the window: lane k contributes bit (off_k - base), one
//      redux.sync.or forms the window's start mask, and position l's segment is the running
//      start count plus popc(mask & lanemask_le) - 1 (no owner map in shared memory; groups
//      with an empty segment take a binary-search path).  The segment's table word comes by
//      shuffle from its lane; the lookup is hash -> bucket -> two 16-byte reads -> four 64-bit
//      compares; hits go to a per-warp shared counter (predicated shared atomics), and lane k
//      stores segment k's count (one coalesced 128-byte store per group).
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace gesr {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kChunkMin = 256;             // candidates per CTA chunk (runtime: 256 or 1024)
constexpr int kChunkMax = 1024;
constexpr int kPoolBuckets = 2048;         // 4 slots each: 64 KB of keys per CTA
constexpr int kStash = 256;                // overflowing user IDs (key, field)
constexpr int kMaxFields = 256;
constexpr int kWinUnroll = 4;              // 32-ID windows in flight per warp
constexpr int kFastMaxIds = 32 * 64;       // groups up to this many IDs take the fast path
constexpr uint32_t kMulLo = 0x9E3779B1u;
constexpr uint32_t kMulHi = 0x85EBCA77u;
__host__ __device__ constexpr uint32_t key_hash_c(unsigned long long key) {
  return (static_cast<uint32_t>(key) * kMulLo) ^ (static_cast<uint32_t>(key >> 32) * kMulHi);
}
// empty-slot fillers: kFill[0] fills buckets whose index has top bit 0 (its own hash has top bit
// 1), kFill[1] the others; tables have >= 2 buckets, so the top hash bit is the bucket's
constexpr unsigned long long kFill0 = 1ull, kFill1 = 2ull;
static_assert((key_hash_c(kFill0) >> 31) == 1u && (key_hash_c(kFill1) >> 31) == 0u, "fillers");

// table word of a field: first bucket (bits 0-11), hash shift (12-17), flags
constexpr uint32_t kFlagStash = 1u << 18;    // some of the field's IDs are in the stash
constexpr uint32_t kFlagGlobal = 1u << 19;   // the field's list is scanned in global memory

struct HmaSmem {
  ulonglong2 bkt[kPoolBuckets][2];           // empty slots hold the bucket half's filler
  // prefilter: 16 bits per bucket (a field's bits follow its buckets' order), bit h >> (shift-4)
  // set for every user ID of the field; a lookup reads one 32-bit word (few bank conflicts) and
  // touches its bucket only if the bit is set -- ~28% of IDs (matches + ~3% false positives)
  uint32_t bits[kPoolBuckets / 2];
  unsigned long long stash_key[kStash];
  int stash_field[kStash];
  uint32_t tab[kMaxFields];
  long long uoff[kMaxFields + 1];            // this request's user_offsets (F+1)
  int warp_cnt[kWarps][32];
  int stash_n;
  int slow_any;                              // some field has stash entries or goes global
};

__device__ __forceinline__ uint32_t key_hash(unsigned long long key) { return key_hash_c(key); }
// PTX shifts clamp the shift amount (>= 32 gives 0), unlike C++ shifts
__device__ __forceinline__ uint32_t shr_clamp(uint32_t a, uint32_t n) {
  uint32_t r;
  asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(n));
  return r;
}
__device__ __forceinline__ uint32_t shl_clamp(uint32_t a, uint32_t n) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(n));
  return r;
}
// Bulk L2 prefetch of the byte range [lo, hi) (rounded out to 16-byte boundaries): one
// instruction brings a whole group's IDs toward L2 while the warp works on the group before it.
__device__ __forceinline__ void prefetch_l2_range(const void* lo, const void* hi) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(lo) & ~uintptr_t(15);
  const uintptr_t b = (reinterpret_cast<uintptr_t>(hi) + 15) & ~uintptr_t(15);
  if (b > a)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a),
                 "r"(static_cast<uint32_t>(b - a))
                 : "memory");
}
__device__ __forceinline__ uint32_t bucket_of(uint32_t tab, unsigned long long key) {
  return (tab & 4095u) + shr_clamp(key_hash(key), (tab >> 12) & 63u);
}

__device__ __forceinline__ uint32_t filter_bit(uint32_t tab, uint32_t h) {
  return (tab & 4095u) * 16u + shr_clamp(h, ((tab >> 12) & 63u) - 4u);
}
__device__ __forceinline__ int bucket_count(const HmaSmem& s, uint32_t tab,
                                            unsigned long long key) {
  const uint32_t b = bucket_of(tab, key);
  const ulonglong2 a = s.bkt[b][0];
  const ulonglong2 c = s.bkt[b][1];
  return (a.x == key) + (a.y == key) + (c.x == key) + (c.y == key);
}

// The fast path's lookup with raw shared addresses (no generic-to-shared conversion per access)
// and the bucket read predicated on the filter bit: lanes whose bit is clear issue no bucket
// traffic (their compare registers are undefined and the count is masked to 0).
__device__ __forceinline__ int fast_count(uint32_t s_bkt, uint32_t s_bits, uint32_t tab,
                                          unsigned long long key) {
  const uint32_t h = key_hash(key);
  const uint32_t base = tab & 4095u, sh = (tab >> 12) & 63u;
  const uint32_t fb = base * 16u + shr_clamp(h, sh - 4u);
  uint32_t word;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(word) : "r"(s_bits + ((fb >> 5) << 2)));
  const uint32_t maybe = (word >> (fb & 31u)) & 1u;
  const uint32_t addr = s_bkt + ((base + shr_clamp(h, sh)) << 5);
  unsigned long long k0, k1, k2, k3;     // undefined where the bit is clear: masked below
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.u32 p, %4, 0;\n"
      " @p ld.shared.v2.u64 {%0, %1}, [%5];\n"
      " @p ld.shared.v2.u64 {%2, %3}, [%5+16];\n}\n"
      : "=l"(k0), "=l"(k1), "=l"(k2), "=l"(k3)
      : "r"(maybe), "r"(addr));
  const int c = (k0 == key) + (k1 == key) + (k2 == key) + (k3 == key);
  return maybe ? c : 0;
}

// Everything the bucket lookup does not cover: stash entries, global-memory fields.
__device__ __noinline__ int slow_count(const HmaSmem& s, const HmaParams& p, int f, uint32_t tab,
                                       unsigned long long key) {
  if (tab & kFlagGlobal) {     // (INT64_MIN included: the scan compares raw values)
    int c = 0;
    for (long long i = s.uoff[f]; i < s.uoff[f + 1]; ++i)
      c += (static_cast<unsigned long long>(__ldg(p.user_ids + i)) == key) ? 1 : 0;
    return c;
  }
  const uint32_t fb = filter_bit(tab, key_hash(key));
  int c = ((s.bits[fb >> 5] >> (fb & 31u)) & 1u) ? bucket_count(s, tab, key) : 0;
  if (tab & kFlagStash) {
    const int n = s.stash_n < kStash ? s.stash_n : kStash;
    for (int i = 0; i < n; ++i) c += (s.stash_field[i] == f && s.stash_key[i] == key) ? 1 : 0;
  }
  return c;
}

__device__ __forceinline__ int lookup_any(const HmaSmem& s, const HmaParams& p, int f,
                                          uint32_t tab, unsigned long long key) {
  if (tab & (kFlagStash | kFlagGlobal)) return slow_count(s, p, f, tab, key);
  const uint32_t fb = filter_bit(tab, key_hash(key));
  return ((s.bits[fb >> 5] >> (fb & 31u)) & 1u) ? bucket_count(s, tab, key) : 0;
}

__global__ void __launch_bounds__(kThreads, 2)
    hma_kernel(const HmaParams p, const int chunk) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  HmaSmem& s = *reinterpret_cast<HmaSmem*>(smem_raw);
  const int b = blockIdx.x;
  const int64_t cb = p.cand_offsets[b];
  const int64_t ce = p.cand_offsets[b + 1];
  const int64_t first = cb + static_cast<int64_t>(blockIdx.y) * chunk;
  if (first >= ce) return;   // uniform
  const int F = p.F;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  // ---- 1. per-field bucketed tables of the request's user lists
  for (int f = tid; f <= F; f += kThreads) s.uoff[f] = p.user_offsets[static_cast<int64_t>(b) * F + f];
  __syncthreads();
  if (tid == 0) {
    int used = 0;
    s.slow_any = 0;
    s.stash_n = 0;
    for (int f = 0; f < F; ++f) {
      const long long n = s.uoff[f + 1] - s.uoff[f];
      // 2^k >= 2 buckets, >= 2 per ID (mean load <= 2 of 4 slots) when the pool allows, else
      // >= 1 per ID
      int nb = 2, shift = 31;
      while (nb < 2 * n && nb < kPoolBuckets) { nb <<= 1; --shift; }
      if (used + nb > kPoolBuckets && nb > n && nb > 2) { nb >>= 1; ++shift; }
      if (nb >= n && used + nb <= kPoolBuckets) {
        s.tab[f] = static_cast<uint32_t>(used) | (static_cast<uint32_t>(shift & 63) << 12);
        used += nb;
      } else {
        s.tab[f] = kFlagGlobal;
        s.slow_any = 1;
      }
    }
  }
  for (int i = tid; i < kPoolBuckets / 2; i += kThreads) s.bits[i] = 0u;
  for (int i = tid; i < kWarps * 32; i += kThreads) (&s.warp_cnt[0][0])[i] = 0;
  __syncthreads();
  // empty slots: each field's lower half of buckets gets kFill0, the upper half kFill1
  for (int f = 0; f < F; ++f) {
    const uint32_t t = s.tab[f];
    if (t & kFlagGlobal) continue;
    const int base = static_cast<int>(t & 4095u);
    const int nb = 1 << (32 - static_cast<int>((t >> 12) & 63u));
    for (int i = tid; i < nb; i += kThreads) {
      const unsigned long long e = (i < nb / 2) ? kFill0 : kFill1;
      s.bkt[base + i][0] = make_ulonglong2(e, e);
      s.bkt[base + i][1] = make_ulonglong2(e, e);
    }
  }
  __syncthreads();
  {
    const long long u0 = s.uoff[0];
    const long long un = s.uoff[F] - u0;
    for (long long i = tid; i < un; i += kThreads) {
      const long long pos = u0 + i;
      int lo = 0, hi = F - 1;                 // owning field: last f with uoff[f] <= pos
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s.uoff[mid] <= pos) lo = mid; else hi = mid - 1;
      }
      const int f = lo;
      const uint32_t t = s.tab[f];
      if (t & kFlagGlobal) continue;
      const unsigned long long key = static_cast<unsigned long long>(__ldg(p.user_ids + pos));
      const uint32_t fb = filter_bit(t, key_hash(key));
      atomicOr(&s.bits[fb >> 5], 1u << (fb & 31u));
      const uint32_t bk = bucket_of(t, key);
      unsigned long long* slots = reinterpret_cast<unsigned long long*>(&s.bkt[bk][0]);
      const unsigned long long fill = (bk - (t & 4095u)) < (1u << (31 - ((t >> 12) & 63u))) ? kFill0 : kFill1;
      bool placed = false;
      for (int q = 0; q < 4 && !placed; ++q)
        placed = atomicCAS(slots + q, fill, key) == fill;
      if (!placed) {
        const int at = atomicAdd(&s.stash_n, 1);
        if (at < kStash) {
          s.stash_key[at] = key;
          s.stash_field[at] = f;
          atomicOr(&s.tab[f], kFlagStash);
        } else {
          atomicOr(&s.tab[f], kFlagGlobal);    // stash full: this field scans global memory
        }
        s.slow_any = 1;
      }
    }
  }
  __syncthreads();
  const bool slow_any = s.slow_any != 0;
  const uint32_t s_bkt = smem_u32(&s.bkt[0][0]);
  const uint32_t s_bits = smem_u32(&s.bits[0]);

  // ---- 2. the item-ID stream, 32 segments per warp step
  for (int64_t c0 = first; c0 < ce; c0 += static_cast<int64_t>(gridDim.y) * chunk) {
    const int64_t c1 = (c0 + chunk < ce) ? c0 + chunk : ce;
    const int64_t seg_begin = c0 * F, seg_end = c1 * F;
    int64_t g = seg_begin + static_cast<int64_t>(warp) * 32;
    constexpr int64_t kStep = static_cast<int64_t>(kWarps) * 32;
    int64_t off_cur = 0, end_cur = 0, off_nxt = 0, end_nxt = 0;
    auto fetch_offsets = [&](int64_t gg, int64_t& o, int64_t& e) {
      if (gg < seg_end) {
        const int ns = (seg_end - gg) < 32 ? static_cast<int>(seg_end - gg) : 32;
        o = __ldg(p.item_offsets + gg + (lane < ns ? lane : ns));
        e = __ldg(p.item_offsets + gg + ns);
      }
    };
    fetch_offsets(g, off_cur, end_cur);
    fetch_offsets(g + kStep, off_nxt, end_nxt);
    {
      const int64_t s0 = __shfl_sync(0xffffffffu, off_cur, 0);
      if (lane == 0 && g < seg_end) prefetch_l2_range(p.item_ids + s0, p.item_ids + end_cur);
    }
    int my_f = static_cast<int>((g - seg_begin + lane) % F);   // seg_begin % F == 0
    const int f_step = (kWarps * 32) % F;
    for (; g < seg_end; g += kStep) {
      const int nseg = (seg_end - g) < 32 ? static_cast<int>(seg_end - g) : 32;
      // lane k holds the start offset of segment g+k; lanes nseg..31 hold the end offset
      const int64_t my_off = off_cur;
      const int64_t end = end_cur;
      // the next group's IDs toward L2 (its offsets arrived during this group's predecessor),
      // then the offsets two groups ahead into registers
      {
        const int64_t s1 = __shfl_sync(0xffffffffu, off_nxt, 0);
        if (lane == 0 && g + kStep < seg_end) prefetch_l2_range(p.item_ids + s1, p.item_ids + end_nxt);
      }
      off_cur = off_nxt;
      end_cur = end_nxt;
      fetch_offsets(g + 2 * kStep, off_nxt, end_nxt);
      const int64_t start = __shfl_sync(0xffffffffu, my_off, 0);
      const int64_t nxt = __shfl_down_sync(0xffffffffu, my_off, 1);
      const int64_t my_end = lane + 1 < nseg ? nxt : end;
      const int n_ids = static_cast<int>(end - start);
      const uint32_t my_tab = s.tab[my_f];
      const int64_t* ids = p.item_ids + start;
      const bool empty_seg = lane < nseg && my_end == my_off;
      if (!__any_sync(0xffffffffu, empty_seg) && n_ids <= kFastMaxIds) {
        // fast path: every segment of the group non-empty, so segment starts are distinct
        const uint32_t rel = static_cast<uint32_t>(my_off - start);   // lanes >= nseg: n_ids
        const uint32_t le_mask = 0xffffffffu >> (31 - lane);         // lanemask_le
        int cum = 0;
        for (int base = 0; base < n_ids; base += kWinUnroll * 32) {
          unsigned long long kk[kWinUnroll];
#pragma unroll
          for (int u = 0; u < kWinUnroll; ++u) {
            const int pos = base + u * 32 + lane;
            kk[u] = pos < n_ids ? static_cast<unsigned long long>(__ldg(ids + pos)) : 0ull;
          }
#pragma unroll
          for (int u = 0; u < kWinUnroll; ++u) {
            const int wbase = base + u * 32;
            if (wbase >= n_ids) break;                                  // warp-uniform
            // shl by >= 32 gives 0: only starts inside the window set a bit
            const uint32_t bit = lane < nseg ? shl_clamp(1u, rel - static_cast<uint32_t>(wbase)) : 0u;
            const uint32_t starts = __reduce_or_sync(0xffffffffu, bit);
            const int seg = cum + __popc(starts & le_mask) - 1;
            cum += __popc(starts);
            const unsigned long long key = kk[u];
            const bool valid = wbase + lane < n_ids;
            const uint32_t t = __shfl_sync(0xffffffffu, my_tab, seg & 31);
            int c;
            if (!slow_any) {
              c = fast_count(s_bkt, s_bits, t, key);
            } else {
              const int f = __shfl_sync(0xffffffffu, my_f, seg & 31);
              c = valid ? lookup_any(s, p, f, t, key) : 0;
            }
            if (valid && c != 0) atomicAdd(&s.warp_cnt[warp][seg], c);
          }
        }
      } else {
        // a group with empty segments (or very long lists): owning segment by binary search
        const int rel = static_cast<int>(my_off - start);
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
          const uint32_t t = __shfl_sync(0xffffffffu, my_tab, k);
          if (ok) {
            const int c = lookup_any(s, p, f, t, key);
            if (c != 0) atomicAdd(&s.warp_cnt[warp][k], c);
          }
        }
      }
      __syncwarp();
      if (lane < nseg) {
        int c = s.warp_cnt[warp][lane];
        if (p.cap > 0 && c > p.cap) c = p.cap;
        p.counts[g + lane] = c;
        if (p.E != nullptr) {
          // offset embedding (stride cap + 1: DESIGN.md R14): segment
          // g + lane = (candidate t, field f) owns out[t][f D_h, (f + 1) D_h) -- contiguous
          const int64_t rowE = static_cast<int64_t>(c) + static_cast<int64_t>(my_f) * (p.cap + 1);
          const uint4* src = p.E + rowE * p.dh_chunks;
          uint4* dst = p.emb + (g + lane) * p.dh_chunks;
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
  // Large chunks amortise the per-CTA table build; small ones keep the grid >= 4 CTAs per SM
  // when there are few requests (config 4: B = 1, C = 4096).
  int64_t per = p.B > 0 ? (p.total_C + p.B - 1) / p.B : 1;
  int chunk = kChunkMax;
  if (p.B * ((per + kChunkMax - 1) / kChunkMax) < 4 * 148) chunk = kChunkMin;
  int64_t y = (per + chunk - 1) / chunk;
  if (y < 1) y = 1;
  if (y > 65535) y = 65535;
  dim3 grid(static_cast<unsigned>(p.B), static_cast<unsigned>(y));
  hma_kernel<<<grid, kThreads, smem, stream>>>(p, chunk);
  count_launch();
  return cudaGetLastError();
}

}  // namespace gesr
