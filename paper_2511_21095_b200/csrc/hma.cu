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
//   grid (B, Y): CTA (b, y) owns request b and candidate chunks y, y+Y, ... of kChunk rows.
//   1. The request's F user lists go into per-field hash tables in shared memory: buckets of
//      4 slots holding a 32-bit fingerprint, the 64-bit key and its multiplicity.  Insertion is
//      parallel (64-bit atomicCAS, linear probing over bucket-aligned slots; the one sentinel
//      key value INT64_MIN is counted on the side); load factor <= 1/4, so a miss -- the common
//      case -- is one 16-byte fingerprint read and four compares, uniform across the warp.
//      Fields whose tables do not fit the pool fall back to a direct scan of global memory.
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
constexpr int kChunk = 256;               // candidates per CTA chunk
constexpr int kPoolBuckets = 1024;        // 4-slot buckets per CTA (64 KB)
constexpr int kMaxFields = 256;
constexpr int kOwnerCap = 512;            // IDs per 32-segment group handled with the owner map
constexpr unsigned long long kSentinel = 0x8000000000000000ull;   // INT64_MIN
constexpr unsigned long long kGold = 0x9E3779B97F4A7C15ull;

struct HmaSmem {
  uint4 fp[kPoolBuckets];                         // 4 fingerprints per bucket (0 = empty)
  unsigned long long key[kPoolBuckets * 4];
  int cnt[kPoolBuckets * 4];
  int tab_off[kMaxFields];                        // first bucket of field f, -1 = global scan
  int tab_mask[kMaxFields];                       // buckets - 1
  int sent_cnt[kMaxFields];                       // multiplicity of INT64_MIN
  long long uoff[kMaxFields + 1];                 // this request's user_offsets (F+1)
  int warp_cnt[kWarps][32];
  unsigned short owner[kWarps][kOwnerCap];
};

__device__ __forceinline__ int lookup(const HmaSmem& s, const HmaParams& p, int f,
                                      unsigned long long key) {
  const int off = s.tab_off[f];
  if (off >= 0) {
    if (key == kSentinel) return s.sent_cnt[f];
    const unsigned long long hk = key * kGold;
    const uint32_t mask = static_cast<uint32_t>(s.tab_mask[f]);
    uint32_t bkt = static_cast<uint32_t>(hk >> 32) & mask;
    const uint32_t fpv = static_cast<uint32_t>(hk) | 1u;
    while (true) {
      const uint4 f4 = s.fp[off + bkt];
      const int base = (off + bkt) * 4;
      if (f4.x == fpv && s.key[base + 0] == key) return s.cnt[base + 0];
      if (f4.y == fpv && s.key[base + 1] == key) return s.cnt[base + 1];
      if (f4.z == fpv && s.key[base + 2] == key) return s.cnt[base + 2];
      if (f4.w == fpv && s.key[base + 3] == key) return s.cnt[base + 3];
      if (f4.w == 0u) return 0;        // slots fill in probe order: an empty slot ends it
      bkt = (bkt + 1) & mask;
    }
  }
  // global fallback: direct scan of the user list
  int c = 0;
  for (long long i = s.uoff[f]; i < s.uoff[f + 1]; ++i)
    c += (static_cast<unsigned long long>(__ldg(p.user_ids + i)) == key) ? 1 : 0;
  return c;
}

__global__ void __launch_bounds__(kThreads, 2)
    hma_kernel(const HmaParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  HmaSmem& s = *reinterpret_cast<HmaSmem*>(smem_raw);
  const int b = blockIdx.x;
  const int64_t cb = p.cand_offsets[b];
  const int64_t ce = p.cand_offsets[b + 1];
  const int64_t first = cb + static_cast<int64_t>(blockIdx.y) * kChunk;
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
    for (int f = 0; f < F; ++f) {
      const long long n = s.uoff[f + 1] - s.uoff[f];
      int nb = 2;
      while (nb < n && nb < kPoolBuckets) nb <<= 1;     // >= n buckets: load factor <= 1/4
      if (n <= nb && used + nb <= kPoolBuckets) {
        s.tab_off[f] = used;
        s.tab_mask[f] = nb - 1;
        used += nb;
      } else {
        s.tab_off[f] = -1;
        s.tab_mask[f] = 0;
      }
      s.sent_cnt[f] = 0;
    }
  }
  for (int i = tid; i < kPoolBuckets * 4; i += kThreads) {
    s.key[i] = kSentinel;
    s.cnt[i] = 0;
  }
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
      const int off = s.tab_off[f];
      if (off < 0) continue;
      const unsigned long long key = static_cast<unsigned long long>(__ldg(p.user_ids + pos));
      if (key == kSentinel) {
        atomicAdd(&s.sent_cnt[f], 1);
        continue;
      }
      const uint32_t nslots = static_cast<uint32_t>(s.tab_mask[f] + 1) * 4;
      uint32_t slot = (static_cast<uint32_t>((key * kGold) >> 32) &
                       static_cast<uint32_t>(s.tab_mask[f])) * 4;
      while (true) {
        const unsigned long long prev = atomicCAS(&s.key[off * 4 + slot], kSentinel, key);
        if (prev == kSentinel || prev == key) {
          atomicAdd(&s.cnt[off * 4 + slot], 1);
          break;
        }
        slot = (slot + 1 == nslots) ? 0 : slot + 1;
      }
    }
  }
  __syncthreads();
  // fingerprints of the occupied slots
  for (int bk = tid; bk < kPoolBuckets; bk += kThreads) {
    uint32_t v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const unsigned long long k = s.key[bk * 4 + e];
      v[e] = (k == kSentinel) ? 0u : (static_cast<uint32_t>(k * kGold) | 1u);
    }
    s.fp[bk] = make_uint4(v[0], v[1], v[2], v[3]);
  }
  __syncthreads();

  // ---- 2. coalesced scan of the item-ID stream, 32 segments per warp step.  The next group's
  //         offsets are fetched while the current group is processed, and all of a group's IDs
  //         (up to kUnroll per lane) are loaded before the first lookup, so each warp keeps
  //         ~2 KB of loads in flight.
  constexpr int kUnroll = 16;
  unsigned short* own = s.owner[warp];
  for (int64_t c0 = first; c0 < ce; c0 += static_cast<int64_t>(gridDim.y) * kChunk) {
    const int64_t c1 = (c0 + kChunk < ce) ? c0 + kChunk : ce;
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
      if (n_ids <= kOwnerCap) {
        for (int base = 0; base < n_ids; base += kUnroll * 32) {
          unsigned long long kk[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int pos = base + u * 32 + lane;
            kk[u] = pos < n_ids ? static_cast<unsigned long long>(__ldg(ids + pos)) : 0ull;
          }
          if (base == 0) {
            if (lane < nseg)
              for (int q = my_off; q < my_end; ++q) own[q] = static_cast<unsigned short>(lane | (my_f << 5));
            __syncwarp();
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int pos = base + u * 32 + lane;
            if (pos < n_ids) {
              const int o = own[pos];
              const int c = lookup(s, p, o >> 5, kk[u]);
              if (c != 0) atomicAdd(&s.warp_cnt[warp][o & 31], c);
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
  static bool attr_done = false;
  const int smem = static_cast<int>(sizeof(HmaSmem));
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(hma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  int64_t per = p.B > 0 ? (p.total_C + p.B - 1) / p.B : 1;
  int64_t y = (per + kChunk - 1) / kChunk;
  if (y < 1) y = 1;
  if (y > 65535) y = 65535;
  dim3 grid(static_cast<unsigned>(p.B), static_cast<unsigned>(y));
  hma_kernel<<<grid, kThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace gesr
