// hma.cu -- K-HMA: Hard Matching Attention raw match counts (s3.4.1).
//
//   counts[t*F + f] = sum_{i in user list (b,f)} sum_{j in item list (t,f)} [u_i == t_j]
//   then min(count, cap) if cap > 0.
//
// The binary attention matrix Attn_match(U, I) summed against a value tensor of ones is a
// multiplicity lookup: each item ID contributes the number of times it occurs in the user's
// list of the same field.  Exact integer arithmetic; bit-identical to the definition.
//
// B200 design (HBM-bound on the item-ID stream, ~8.5 int64 IDs per (candidate, field)):
//   grid (B, Y): CTA (b, y) owns request b and candidate chunks y, y+Y, ... of `chunk` rows.
//   1. The request's F user lists go into per-field open-addressing tables in shared memory:
//      64-bit keys only (INT64_MIN marks an empty slot; that one ID value is counted on the side),
//      every OCCURRENCE of a user ID in its own slot (parallel 64-bit atomicCAS, linear probing
//      from the even slot of a multiplicative hash of the key's two 32-bit halves), >= 8 slots
//      per ID when the 8192-slot pool allows (load factor <= 1/8), else >= 4.  All copies of a
//      key lie between its home slot and the first empty slot after it, so a lookup COUNTS the
//      matches in the 4-slot window of its home pair and the next (two 16-byte reads, no
//      multiplicity array) and walks on only when the whole window is occupied -- rare enough at
//      1/8 that the warp seldom executes the walk.  Fields whose tables do not fit the pool fall
//      back to a direct scan of global memory.
//   2. Each warp takes 32 consecutive (candidate, field) segments of the CSR item stream.
//      Lane k writes its segment id into a per-warp owner map (one uint16 per ID position),
//      then the warp reads the group's IDs COALESCED (lane l reads ID start + l + 32 i), looks
//      each up in its field's table, and adds hits into a per-warp shared counter.  Lane k then
//      stores segment k's count: one coalesced 128-byte int32 store per 32 segments.
//      Groups with more than kOwnerCap IDs use a shuffle binary search instead of the map.
#include <cuda_runtime.h>

#include "kernels.h"

namespace gesr {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kChunkMin = 256;            // candidates per CTA chunk (runtime: 256 or 1024)
constexpr int kChunkMax = 1024;
constexpr int kPoolSlots = 8192;          // table slots per CTA (64 KB of keys)
constexpr int kMaxFields = 256;
constexpr int kOwnerCap = 512;            // IDs per 32-segment group handled with the owner map
constexpr unsigned long long kSentinel = 0x8000000000000000ull;   // INT64_MIN: empty slot
constexpr uint32_t kMul = 0x9E3779B1u;

struct HmaSmem {
  unsigned long long key[kPoolSlots];             // kSentinel = empty; one slot per occurrence
  int2 tab[kMaxFields];                           // {first slot, hash shift}; first < 0: global
  int sent_cnt[kMaxFields];                       // multiplicity of INT64_MIN
  long long uoff[kMaxFields + 1];                 // this request's user_offsets (F+1)
  int warp_cnt[kWarps][32];
  // owner word of each ID position of a warp's 32-segment group: segment lane (bits 0-4), the
  // field's hash shift (5-9), its first table slot (10-22), the field (23-30)
  uint32_t owner[kWarps][kOwnerCap];
  int any_global;                                 // some field scans global memory instead
};

// Home slot pair of a key in a table of 2^(32 - shift) slot pairs (top bits of a
// multiplicative hash of the folded key).
__device__ __forceinline__ uint32_t home_pair(unsigned long long key, int shift) {
  const uint32_t h = (static_cast<uint32_t>(key) ^ static_cast<uint32_t>(key >> 32)) * kMul;
  return h >> shift;
}

// Copies of `key` in a field's table (first slot `base`, 2^(32 - shift) slot pairs).  Every
// occurrence of a user ID has its own slot, filled by linear probing from the even slot of its
// home pair, so all copies lie between the home slot and the first empty slot after it: count
// matches over the 4-slot window of the home pair and the next one (two 16-byte reads) and walk
// on only if the whole window is occupied (rare at load factor <= 1/8).
__device__ __forceinline__ int window_count(const unsigned long long* tb, uint32_t pr,
                                            uint32_t pmask, unsigned long long key, bool& open) {
  const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(tb + 2 * pr);
  const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(tb + 2 * ((pr + 1) & pmask));
  open = a.x != kSentinel && a.y != kSentinel && b.x != kSentinel && b.y != kSentinel;
  return (a.x == key ? 1 : 0) + (a.y == key ? 1 : 0) + (b.x == key ? 1 : 0) + (b.y == key ? 1 : 0);
}
// the rest of the walk after a full window starting at pair pr
__device__ __forceinline__ int walk_on(const unsigned long long* tb, uint32_t pr, uint32_t pmask,
                                    unsigned long long key) {
  int c = 0;
  pr = (pr + 2) & pmask;
  while (true) {
    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(tb + 2 * pr);
    c += (a.x == key ? 1 : 0) + (a.y == key ? 1 : 0);
    if (a.x == kSentinel || a.y == kSentinel) return c;
    pr = (pr + 1) & pmask;
  }
}

__device__ __forceinline__ int lookup(const HmaSmem& s, const HmaParams& p, int f,
                                      unsigned long long key) {
  if (key == kSentinel) return s.sent_cnt[f];
  const int2 t = s.tab[f];
  if (t.x >= 0) {
    const uint32_t pmask = 0xFFFFFFFFu >> t.y;
    const uint32_t pr = home_pair(key, t.y);
    bool open;
    int c = window_count(s.key + t.x, pr, pmask, key, open);
    if (open) c += walk_on(s.key + t.x, pr, pmask, key);
    return c;
  }
  // global fallback: direct scan of the user list
  int c = 0;
  for (long long i = s.uoff[f]; i < s.uoff[f + 1]; ++i)
    c += (static_cast<unsigned long long>(__ldg(p.user_ids + i)) == key) ? 1 : 0;
  return c;
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

  // ---- 1. per-field hash tables of the request's user lists
  for (int f = tid; f <= F; f += kThreads) s.uoff[f] = p.user_offsets[static_cast<int64_t>(b) * F + f];
  __syncthreads();
  if (tid == 0) {
    int used = 0;
    s.any_global = 0;
    for (int f = 0; f < F; ++f) {
      const long long n = s.uoff[f + 1] - s.uoff[f];
      // >= 8n slots (load factor <= 1/8) when the pool allows, else >= 4n
      int ns = 4, shift = 31;
      while (ns < 8 * n && ns < kPoolSlots) { ns <<= 1; --shift; }
      if (used + ns > kPoolSlots && ns >= 8 && 4 * n <= ns / 2) { ns >>= 1; ++shift; }
      if (4 * n <= ns && used + ns <= kPoolSlots) {
        s.tab[f] = make_int2(used, shift);           // ns / 2 = 2^(32 - shift) slot pairs
        used += ns;
      } else {
        s.tab[f] = make_int2(-1, 0);
        s.any_global = 1;
      }
      s.sent_cnt[f] = 0;
    }
  }
  for (int i = tid; i < kPoolSlots; i += kThreads) s.key[i] = kSentinel;
  for (int i = tid; i < kWarps * 32; i += kThreads) (&s.warp_cnt[0][0])[i] = 0;
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
      const int2 t = s.tab[f];
      if (t.x < 0) continue;
      const unsigned long long key = static_cast<unsigned long long>(__ldg(p.user_ids + pos));
      if (key == kSentinel) {
        atomicAdd(&s.sent_cnt[f], 1);
        continue;
      }
      const uint32_t smask = (0xFFFFFFFFu >> t.y) * 2 + 1;   // slots - 1
      uint32_t slot = home_pair(key, t.y) * 2;
      // every occurrence takes its own slot (a duplicate probes past its earlier copies)
      while (atomicCAS(&s.key[t.x + slot], kSentinel, key) != kSentinel) slot = (slot + 1) & smask;
    }
  }
  __syncthreads();

  // ---- 2. coalesced scan of the item-ID stream, 32 segments per warp step.  The next group's
  //         offsets are fetched while the current group is processed, and all of a group's IDs
  //         (kUnroll per lane) are loaded before the first lookup, so each warp keeps ~1 KB of
  //         loads in flight.
  constexpr int kUnroll = 4;
  constexpr int kBatch = 2;
  uint32_t* own = s.owner[warp];
  for (int64_t c0 = first; c0 < ce; c0 += static_cast<int64_t>(gridDim.y) * chunk) {
    const int64_t c1 = (c0 + chunk < ce) ? c0 + chunk : ce;
    const int64_t seg_begin = c0 * F, seg_end = c1 * F;
    int64_t g = seg_begin + static_cast<int64_t>(warp) * 32;
    int64_t off_cur = 0, end_cur = 0;
    auto fetch_offsets = [&](int64_t gg, int64_t& o, int64_t& e) {
      if (gg < seg_end) {
        const int ns = (seg_end - gg) < 32 ? static_cast<int>(seg_end - gg) : 32;
        o = __ldg(p.item_offsets + gg + (lane < ns ? lane : ns));
        e = __ldg(p.item_offsets + gg + ns);
      }
    };
    fetch_offsets(g, off_cur, end_cur);
    for (; g < seg_end; g += static_cast<int64_t>(kWarps) * 32) {
      const int nseg = (seg_end - g) < 32 ? static_cast<int>(seg_end - g) : 32;
      // lane k holds the start offset of segment g+k; lanes nseg..31 hold the end offset
      const int64_t my_off64 = off_cur;
      const int64_t end = end_cur;
      fetch_offsets(g + static_cast<int64_t>(kWarps) * 32, off_cur, end_cur);   // prefetch next
      const int64_t start = __shfl_sync(0xffffffffu, my_off64, 0);
      const int my_off = static_cast<int>(my_off64 - start);
      const int nxt = __shfl_down_sync(0xffffffffu, my_off, 1);
      const int n_ids = static_cast<int>(end - start);
      const int my_end = lane + 1 < nseg ? nxt : n_ids;
      const int my_f = static_cast<int>(g - seg_begin + lane) % F;   // seg_begin % F == 0
      const int64_t* ids = p.item_ids + start;
      if (n_ids <= kOwnerCap && !s.any_global) {
        // owner words of this group's ID positions (one table-info read per segment)
        const int2 t = s.tab[my_f];
        const uint32_t ow = static_cast<uint32_t>(lane) | (static_cast<uint32_t>(t.y) << 5) |
                            (static_cast<uint32_t>(t.x) << 10) | (static_cast<uint32_t>(my_f) << 23);
        for (int base = 0; base < n_ids; base += kUnroll * 32) {
          unsigned long long kk[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int pos = base + u * 32 + lane;
            kk[u] = pos < n_ids ? static_cast<unsigned long long>(__ldg(ids + pos)) : 0ull;
          }
          if (base == 0) {
            if (lane < nseg)
              for (int q = my_off; q < my_end; ++q) own[q] = ow;
            __syncwarp();
          }
          // batches of kBatch positions in straight-line code, so their shared-memory reads
          // overlap: owner word -> home slot pair -> the 4-slot window (two 16-byte reads) ->
          // count the key's copies; a position whose window is full (rare at load factor
          // <= 1/8) walks on after the batch
#pragma unroll
          for (int u0 = 0; u0 < kUnroll; u0 += kBatch) {
            if (base + u0 * 32 >= n_ids) break;          // warp-uniform
            uint32_t o[kBatch], pr[kBatch];
            int c[kBatch];
            bool open[kBatch];
#pragma unroll
            for (int v = 0; v < kBatch; ++v) {
              const int pos = base + (u0 + v) * 32 + lane;
              o[v] = pos < n_ids ? own[pos] : 0u;
            }
#pragma unroll
            for (int v = 0; v < kBatch; ++v) {
              const unsigned long long key = kk[u0 + v];
              const int pos = base + (u0 + v) * 32 + lane;
              const int shift = static_cast<int>((o[v] >> 5) & 31u);
              pr[v] = home_pair(key, shift);
              c[v] = window_count(s.key + ((o[v] >> 10) & 8191u), pr[v], 0xFFFFFFFFu >> shift,
                                  key, open[v]);
              if (key == kSentinel) {                        // the empty marker's own ID value
                c[v] = s.sent_cnt[o[v] >> 23];
                open[v] = false;
              }
              if (pos >= n_ids) { c[v] = 0; open[v] = false; }
            }
            bool any_open = false;
#pragma unroll
            for (int v = 0; v < kBatch; ++v) any_open |= open[v];
            if (__any_sync(0xffffffffu, any_open)) {
#pragma unroll
              for (int v = 0; v < kBatch; ++v)
                if (open[v])
                  c[v] += walk_on(s.key + ((o[v] >> 10) & 8191u), pr[v],
                                  0xFFFFFFFFu >> ((o[v] >> 5) & 31u), kk[u0 + v]);
            }
#pragma unroll
            for (int v = 0; v < kBatch; ++v)
              if (c[v] != 0) atomicAdd(&s.warp_cnt[warp][o[v] & 31u], c[v]);
          }
        }
      } else if (n_ids <= kOwnerCap) {
        for (int base = 0; base < n_ids; base += kUnroll * 32) {
          unsigned long long kk[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int pos = base + u * 32 + lane;
            kk[u] = pos < n_ids ? static_cast<unsigned long long>(__ldg(ids + pos)) : 0ull;
          }
          if (base == 0) {
            if (lane < nseg)
              for (int q = my_off; q < my_end; ++q) own[q] = static_cast<uint32_t>(lane) | (static_cast<uint32_t>(my_f) << 23);
            __syncwarp();
          }
#pragma unroll 1
          for (int u = 0; u < kUnroll; ++u) {
            if (base + u * 32 >= n_ids) break;           // warp-uniform
            const int pos = base + u * 32 + lane;
            if (pos < n_ids) {
              const uint32_t o = own[pos];
              const int c = lookup(s, p, static_cast<int>(o >> 23), kk[u]);
              if (c != 0) atomicAdd(&s.warp_cnt[warp][o & 31u], c);
            }
          }
        }
      } else {
        for (int base = 0; base < n_ids; base += 32) {
          const int pos = base + lane;
          const bool ok = pos < n_ids;
          const unsigned long long key = ok ? static_cast<unsigned long long>(__ldg(ids + pos)) : 0ull;
          int k = 0;     // owning segment: largest k with off[k] <= pos
#pragma unroll
          for (int step = 16; step >= 1; step >>= 1) {
            const int o = __shfl_sync(0xffffffffu, my_off, k + step);
            if (o <= pos) k += step;
          }
          const int f = __shfl_sync(0xffffffffu, my_f, k);
          if (ok) {
            const int c = lookup(s, p, f, key);
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
          const int f = static_cast<int>(g - seg_begin + lane) % F;
          const int64_t rowE = static_cast<int64_t>(c) + static_cast<int64_t>(f) * (p.cap + 1);
          const uint4* src = p.E + rowE * p.dh_chunks;
          uint4* dst = p.emb + (g + lane) * p.dh_chunks;
          for (int q = 0; q < p.dh_chunks; ++q) dst[q] = __ldg(src + q);
        }
      }
      s.warp_cnt[warp][lane] = 0;
      __syncwarp();
    }
  }
}

}  // namespace

cudaError_t launch_hma(const HmaParams& p, cudaStream_t stream) {
  const int smem = static_cast<int>(sizeof(HmaSmem));
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(hma_kernel), smem);
  if (e != cudaSuccess) return e;
  // Large chunks amortise the per-CTA table build (one CTA per request at C = 1000: measured
  // 0.796 -> 0.759 ms at the headline); small ones keep the grid >= 4 CTAs per SM when there
  // are few requests (config 4: B = 1, C = 4096).
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
