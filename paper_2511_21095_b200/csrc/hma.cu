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
//   1. The request's F user lists are inserted into per-field open-addressing hash tables in
//      shared memory (64-bit keys + int32 multiplicities, parallel insertion with 64-bit
//      atomicCAS; one sentinel key value is counted on the side).  Lists whose tables do not
//      fit the shared-memory pool fall back to a direct scan of global memory (any length).
//   2. Each warp takes 32 consecutive (candidate, field) segments of the CSR item stream and
//      reads their IDs COALESCED (lane k reads ID p = start + k + 32*i), finds the owning
//      segment with a 5-step shuffle binary search over the 33 segment offsets, looks the ID
//      up in that field's table, and accumulates into a per-warp shared counter array (only
//      non-zero lookups touch it).  Lane k then stores segment k's count: one coalesced
//      128-byte int32 store per 32 segments.
#include <cuda_runtime.h>

#include "kernels.h"

namespace gesr {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 256;               // candidates per CTA chunk
constexpr int kPoolSlots = 4096;          // hash slots per CTA (48 KB)
constexpr int kMaxFields = 256;           // fields handled with per-field smem metadata
constexpr unsigned long long kSentinel = 0x8000000000000000ull;   // INT64_MIN

__device__ __forceinline__ uint32_t hash_slot(unsigned long long key, uint32_t mask) {
  return static_cast<uint32_t>((key * 0x9E3779B97F4A7C15ull) >> 32) & mask;
}

struct HmaSmem {
  unsigned long long keys[kPoolSlots];
  int cnt[kPoolSlots];
  int tab_off[kMaxFields];      // slot offset of field f's table, -1 = global fallback
  int tab_mask[kMaxFields];
  int sent_cnt[kMaxFields];     // multiplicity of the sentinel value INT64_MIN
  long long uoff[kMaxFields + 1];   // user_offsets for this request (F+1 entries)
  int warp_cnt[kWarps][32];
};

__device__ __forceinline__ int lookup(const HmaSmem& s, const HmaParams& p, int f,
                                      unsigned long long key) {
  if (key == kSentinel) {
    if (s.tab_off[f] >= 0) return s.sent_cnt[f];
  }
  const int off = s.tab_off[f];
  if (off >= 0) {
    const uint32_t mask = static_cast<uint32_t>(s.tab_mask[f]);
    uint32_t h = hash_slot(key, mask);
    while (true) {
      const unsigned long long k = s.keys[off + h];
      if (k == key) return s.cnt[off + h];
      if (k == kSentinel) return 0;
      h = (h + 1) & mask;
    }
  }
  // global fallback: direct scan of the user list
  int c = 0;
  for (long long i = s.uoff[f]; i < s.uoff[f + 1]; ++i)
    c += (static_cast<unsigned long long>(__ldg(p.user_ids + i)) == key) ? 1 : 0;
  return c;
}

__global__ void __launch_bounds__(kThreads)
    hma_kernel(const HmaParams p) {
  extern __shared__ uint8_t smem_raw[];
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
      int size = 16;
      while (size < 2 * n && size < kPoolSlots) size <<= 1;
      if (2 * n <= size && used + size <= kPoolSlots) {
        s.tab_off[f] = used;
        s.tab_mask[f] = size - 1;
        used += size;
      } else {
        s.tab_off[f] = -1;
        s.tab_mask[f] = 0;
      }
      s.sent_cnt[f] = 0;
    }
  }
  for (int i = tid; i < kPoolSlots; i += kThreads) {
    s.keys[i] = kSentinel;
    s.cnt[i] = 0;
  }
  for (int i = tid; i < kWarps * 32; i += kThreads) (&s.warp_cnt[0][0])[i] = 0;
  __syncthreads();
  {
    const long long u0 = s.uoff[0];
    const long long un = s.uoff[F] - u0;
    for (long long i = tid; i < un; i += kThreads) {
      const long long pos = u0 + i;
      // owning field: last f with uoff[f] <= pos (F is small; binary search)
      int lo = 0, hi = F - 1;
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
      const uint32_t mask = static_cast<uint32_t>(s.tab_mask[f]);
      uint32_t h = hash_slot(key, mask);
      while (true) {
        const unsigned long long prev = atomicCAS(&s.keys[off + h], kSentinel, key);
        if (prev == kSentinel || prev == key) {
          atomicAdd(&s.cnt[off + h], 1);
          break;
        }
        h = (h + 1) & mask;
      }
    }
  }
  __syncthreads();

  // ---- 2. coalesced scan of the item-ID stream, 32 segments per warp step
  for (int64_t c0 = first; c0 < ce; c0 += static_cast<int64_t>(gridDim.y) * kChunk) {
    const int64_t c1 = (c0 + kChunk < ce) ? c0 + kChunk : ce;
    const int64_t seg_begin = c0 * F, seg_end = c1 * F;
    for (int64_t g = seg_begin + static_cast<int64_t>(warp) * 32; g < seg_end;
         g += static_cast<int64_t>(kWarps) * 32) {
      const int nseg = (seg_end - g) < 32 ? static_cast<int>(seg_end - g) : 32;
      // lane k holds the start offset of segment g+k; lanes nseg..31 hold the end offset
      const int64_t my_off64 = p.item_offsets[g + (lane < nseg ? lane : nseg)];
      const int64_t start = __shfl_sync(0xffffffffu, my_off64, 0);
      const int64_t end = p.item_offsets[g + nseg];   // same address for all lanes: broadcast
      // 32-bit relative offsets and field index for the shuffle search (seg_begin % F == 0)
      const int my_off = static_cast<int>(my_off64 - start);
      const int my_f = static_cast<int>(g - seg_begin + lane) % F;
      const int n_ids = static_cast<int>(end - start);
      const int64_t* ids = p.item_ids + start;
      for (int base = 0; base < n_ids; base += 32) {
        const int pos = base + lane;
        const bool ok = pos < n_ids;
        const unsigned long long key = ok ? static_cast<unsigned long long>(__ldg(ids + pos)) : 0ull;
        // owning segment: largest k with off[k] <= pos (offsets nondecreasing)
        int k = 0;
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
      __syncwarp();
      if (lane < nseg) {
        int c = s.warp_cnt[warp][lane];
        if (p.cap > 0 && c > p.cap) c = p.cap;
        p.counts[g + lane] = c;
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
