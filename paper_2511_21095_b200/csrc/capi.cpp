// capi.cpp -- the C ABI of libgesr.so (include/gesr.h): argument validation, TMA tensor-map
// encoding (cuTensorMapEncodeTiled through cudaGetDriverEntryPoint, so no -lcuda), workspace
// carving, and kernel launches on the caller's stream.  No host synchronisation, no device
// allocation, no copies.
#include "../../include/gesr.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <set>
#include <utility>

#include "kernels.h"

namespace gesr {

namespace {
std::mutex g_attr_mu;
std::set<std::pair<int, const void*>> g_attr_done;
constexpr int kMaxDev = 64;
std::atomic<int> g_dev_cache[kMaxDev][8];
std::atomic<unsigned long long> g_launches{0};
}  // namespace

cudaError_t ensure_smem_attr(const void* fn, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_attr_mu);
  if (g_attr_done.count({dev, fn})) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) g_attr_done.insert({dev, fn});
  return e;
}

int device_cached(int slot) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return 0;
  return g_dev_cache[dev][slot].load(std::memory_order_acquire);
}

void device_cache_store(int slot, int value) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return;
  g_dev_cache[dev][slot].store(value, std::memory_order_release);
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace gesr

namespace {

thread_local char g_err[512] = "";

gesr_status fail(gesr_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

gesr_status cuda_fail(cudaError_t e, const char* where) {
  return fail(GESR_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

// error reporting for the other host translation units (hostpath.cu): the same thread-local
// message gesr_last_error() returns
gesr_status gesr_internal_fail(gesr_status s, const char* msg) { return fail(s, "%s", msg); }

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int num_sms() {
  int n = gesr::device_cached(0);
  if (n > 0) return n;
  int dev = 0;
  n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  gesr::device_cache_store(0, n);
  return n;
}

// 2D bf16 tensor map over a row-major [rows, cols] array with box [box_rows, box_cols].
gesr_status make_map_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                        uint32_t box_rows, uint32_t box_cols, CUtensorMapSwizzle swz,
                        const char* what) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(GESR_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(GESR_ERR_CUDA, "cuTensorMapEncodeTiled(%s) failed: %d", what, static_cast<int>(r));
  return GESR_OK;
}

// 3D bf16 tensor map over a head-major [H, M, d] output with a {32 cols, 32 rows, 1} box and
// 64B swizzle (the projection epilogue's TMA store).
gesr_status make_out_map(CUtensorMap* map, void* base, uint64_t H, uint64_t M, uint64_t d,
                         const char* what) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(GESR_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[3] = {d, M, H};
  cuuint64_t strides[2] = {d * 2, M * d * 2};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(GESR_ERR_CUDA, "cuTensorMapEncodeTiled(%s) failed: %d", what, static_cast<int>(r));
  return GESR_OK;
}

// d = 128 runs the CTA-pair attention kernel (attn2.cu); GESR_ATTN_PAIR=0 selects the 1-CTA
// kernel instead (equal at the headline, slower on jagged / chunked workloads: DESIGN.md s10).
bool pair_attention_enabled() {
  static int cached = -1;
  if (cached < 0) {
    const char* v = getenv("GESR_ATTN_PAIR");
    cached = (v != nullptr && v[0] == '0') ? 0 : 1;
  }
  return cached == 1;
}

// bf16 attention output O [total_C, H*d] viewed as [total_C, H, d] for the epilogue's TMA
// tensor stores: box {32 columns, 1 head, 32 rows}, 64B swizzle (the staging box layout)
gesr_status make_o_map(CUtensorMap* map, void* base, uint64_t rows, uint64_t H, uint64_t d) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(GESR_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[3] = {d, H, rows};
  cuuint64_t strides[2] = {d * 2, H * d * 2};
  cuuint32_t box[3] = {32, 1, 32};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(GESR_ERR_CUDA, "cuTensorMapEncodeTiled(O) failed: %d", static_cast<int>(r));
  return GESR_OK;
}

// GESR_DEBUG=1 (read once per process): device validation of the jagged offsets before the
// kernels that index with them (debug.cu).
bool debug_enabled() {
  static const int on = [] {
    const char* v = getenv("GESR_DEBUG");
    return (v != nullptr && v[0] == '1') ? 1 : 0;
  }();
  return on == 1;
}

gesr_status debug_check(const int64_t* offsets, int64_t n, int64_t total, int tag,
                        cudaStream_t st) {
  if (!debug_enabled()) return GESR_OK;
  cudaError_t e = gesr::launch_check_offsets(offsets, n, total, tag, st);
  return e == cudaSuccess ? GESR_OK : cuda_fail(e, "check_offsets launch");
}

bool valid_d(int32_t d) { return d == 32 || d == 64 || d == 128; }

gesr_status check_common(int32_t D_in, int32_t H, int32_t d, int32_t act) {
  if (D_in < 8 || D_in > 16384 || (D_in % 8) != 0)
    return fail(GESR_ERR_INVALID_ARG, "D_in=%d must be a multiple of 8 in [8, 16384]", D_in);
  if (H < 1 || H > 4096) return fail(GESR_ERR_INVALID_ARG, "H=%d must be in [1, 4096]", H);
  if (!valid_d(d)) return fail(GESR_ERR_INVALID_ARG, "d=%d must be 32, 64 or 128", d);
  if (act != GESR_ACT_IDENTITY && act != GESR_ACT_SILU)
    return fail(GESR_ERR_INVALID_ARG, "act=%d is not a gesr_act", act);
  return GESR_OK;
}

// Workspace layout for gesr_tasa_score: [0,256) header {int unit_count}; [256, ...) units;
// then (1024-aligned) Q [H, total_C, d] bf16.
int64_t max_units(int64_t B, int64_t total_C) {
  return B + (total_C + gesr::kUnitRows - 1) / gesr::kUnitRows;
}
size_t units_end(int64_t B, int64_t total_C) {
  size_t e = 256 + static_cast<size_t>(max_units(B, total_C)) * sizeof(int4);
  return (e + 1023) & ~static_cast<size_t>(1023);
}

// Projection launch shared by K/V and Q: X [M, K] -> out0/out1 [H, M, d] head-major.
// gather != NULL: X row m is row gather[m] of the [table_rows, K] table X (TMA gather4, box
// {64 cols, 1 row}).
gesr_status run_projection(const void* X, int64_t M, int32_t K, const void* W0, const void* W1,
                           const float* b0, const float* b1, int32_t H, int32_t d, int32_t act,
                           void* out0, void* out1, cudaStream_t stream,
                           const int32_t* gather = nullptr, int64_t table_rows = 0) {
  const int HD = H * d;
  // gather mode on a large row count: 512-wide tiles (two N = 256 MMAs per K step, one TMEM
  // accumulator), so each gathered A tile feeds twice the MMA work -- the gathered projections
  // are bound by issuing the gather4 loads
#ifndef GESR_GATHER_BN512
#define GESR_GATHER_BN512 1
#endif
  const int bn = (GESR_GATHER_BN512 && gather != nullptr && HD % 512 == 0 &&
                  (M + 255) / 256 >= num_sms() / 2)
                     ? 512
                     : gesr::proj_pick_bn(M, HD, W1 ? 2 : 1, num_sms());
  const uint32_t b_box = bn >= 512 ? 128 : static_cast<uint32_t>(bn / 2);
  CUtensorMap ma, mb0, mb1;
  gesr_status s = gather != nullptr
                      ? make_map_2d(&ma, X, static_cast<uint64_t>(table_rows),
                                    static_cast<uint64_t>(K), 1, 64, CU_TENSOR_MAP_SWIZZLE_128B,
                                    "E (gather)")
                      : make_map_2d(&ma, X, static_cast<uint64_t>(M), static_cast<uint64_t>(K),
                                    128, 64, CU_TENSOR_MAP_SWIZZLE_128B, "X");
  if (s != GESR_OK) return s;
  // a CTA pair computes 256 x bn; each CTA stages its 128 rows of X and bn/2 weight rows
  s = make_map_2d(&mb0, W0, HD, K, b_box, 64, CU_TENSOR_MAP_SWIZZLE_128B, "W0");
  if (s != GESR_OK) return s;
  s = make_map_2d(&mb1, W1 ? W1 : W0, HD, K, b_box, 64, CU_TENSOR_MAP_SWIZZLE_128B, "W1");
  if (s != GESR_OK) return s;
  CUtensorMap mo0, mo1;
  s = make_out_map(&mo0, out0, H, M, d, "out0");
  if (s != GESR_OK) return s;
  s = make_out_map(&mo1, out1 ? out1 : out0, H, M, d, "out1");
  if (s != GESR_OK) return s;
  gesr::ProjParams p{};
  p.M = M;
  p.K = K;
  p.n_split = HD;
  p.d = d;
  p.act = act;
  p.num_m_blocks = static_cast<int>((M + 255) / 256);
  p.num_n_blocks = (W1 ? 2 * HD : HD) / bn;
  p.bias0 = b0;
  p.bias1 = b1;
  p.out0 = static_cast<__nv_bfloat16*>(out0);
  p.out1 = static_cast<__nv_bfloat16*>(out1);
  p.gather = gather;
  cudaError_t e = gesr::launch_proj(ma, mb0, mb1, mo0, mo1, p, bn, num_sms(), stream);
  if (e != cudaSuccess) return cuda_fail(e, "proj_kernel launch");
  return GESR_OK;
}

// Row-major projection (STU gating branch and output projection): X [M, K] -> out [M, N]
// = act(X W^T + b) (+ residual [M, N]), through a {N, M, 1} output map (one "head").
gesr_status run_projection_rm(const void* X, int64_t M, int32_t K, const void* W, const float* b,
                              int32_t N, int32_t act, const void* residual, void* out,
                              cudaStream_t stream) {
  const int bn = gesr::proj_pick_bn(M, N, 1, num_sms());
  CUtensorMap ma, mb, mo;
  gesr_status s = make_map_2d(&ma, X, static_cast<uint64_t>(M), static_cast<uint64_t>(K), 128, 64,
                              CU_TENSOR_MAP_SWIZZLE_128B, "X");
  if (s != GESR_OK) return s;
  s = make_map_2d(&mb, W, N, K, bn / 2, 64, CU_TENSOR_MAP_SWIZZLE_128B, "W");
  if (s != GESR_OK) return s;
  s = make_out_map(&mo, out, 1, M, N, "out");
  if (s != GESR_OK) return s;
  gesr::ProjParams p{};
  p.M = M;
  p.K = K;
  p.n_split = N;
  p.d = 32;                      // unused: row-major output has no head split
  p.act = act;
  p.num_m_blocks = static_cast<int>((M + 255) / 256);
  p.num_n_blocks = N / bn;
  p.bias0 = b;
  p.bias1 = b;
  p.out0 = static_cast<__nv_bfloat16*>(out);
  p.out1 = nullptr;
  p.rowmajor = 1;
  p.residual = static_cast<const __nv_bfloat16*>(residual);
  p.res_ld = N;
  cudaError_t e = gesr::launch_proj(ma, mb, mb, mo, mo, p, bn, num_sms(), stream);
  if (e != cudaSuccess) return cuda_fail(e, "proj_kernel launch (row-major)");
  return GESR_OK;
}

size_t stu_buffer_bytes(int64_t total_C, int64_t D) {
  return (static_cast<size_t>(total_C) * D * 2 + 1023) & ~static_cast<size_t>(1023);
}

}  // namespace

extern "C" {

int gesr_version(void) { return 200; }

unsigned long long gesr_launch_count(void) {
  return gesr::g_launches.load(std::memory_order_relaxed);
}

const char* gesr_status_string(int s) {
  switch (s) {
    case GESR_OK: return "GESR_OK";
    case GESR_ERR_INVALID_ARG: return "GESR_ERR_INVALID_ARG";
    case GESR_ERR_UNSUPPORTED: return "GESR_ERR_UNSUPPORTED";
    case GESR_ERR_CUDA: return "GESR_ERR_CUDA";
    case GESR_ERR_WORKSPACE: return "GESR_ERR_WORKSPACE";
    default: return "GESR_ERR_UNKNOWN";
  }
}

const char* gesr_last_error(void) { return g_err; }

gesr_status gesr_kv_project(const void* U, int64_t total_L, int32_t D_in, const void* W_k,
                            const void* W_v, const float* b_k, const float* b_v, int32_t H,
                            int32_t d, int32_t act, void* K_cache, void* V_cache, void* stream) {
  gesr_status s = check_common(D_in, H, d, act);
  if (s != GESR_OK) return s;
  if (total_L < 0) return fail(GESR_ERR_INVALID_ARG, "total_L=%lld < 0", (long long)total_L);
  if (total_L >= (int64_t(1) << 31) / H)
    return fail(GESR_ERR_INVALID_ARG, "H*total_L exceeds the 2^31 TMA coordinate range");
  if (total_L == 0) return GESR_OK;
  if (!U || !W_k || !W_v || !K_cache || !V_cache)
    return fail(GESR_ERR_INVALID_ARG, "null required pointer");
  if (!aligned16(U) || !aligned16(W_k) || !aligned16(W_v) || !aligned16(K_cache) ||
      !aligned16(V_cache) || !aligned16(b_k) || !aligned16(b_v))
    return fail(GESR_ERR_INVALID_ARG, "pointers must be 16-byte aligned");
  return run_projection(U, total_L, D_in, W_k, W_v, b_k, b_v, H, d, act, K_cache, V_cache,
                        static_cast<cudaStream_t>(stream));
}

gesr_status gesr_kv_project_gather(const void* E, int64_t n_E, int32_t D_in, const int32_t* rows,
                                   int64_t total_L, const void* W_k, const void* W_v,
                                   const float* b_k, const float* b_v, int32_t H, int32_t d,
                                   int32_t act, void* K_cache, void* V_cache, void* stream) {
  gesr_status s = check_common(D_in, H, d, act);
  if (s != GESR_OK) return s;
  if (total_L < 0) return fail(GESR_ERR_INVALID_ARG, "total_L=%lld < 0", (long long)total_L);
  if (total_L >= (int64_t(1) << 31) / H)
    return fail(GESR_ERR_INVALID_ARG, "H*total_L exceeds the 2^31 TMA coordinate range");
  if (n_E < 1 || n_E >= (int64_t(1) << 31))
    return fail(GESR_ERR_INVALID_ARG, "n_E=%lld must be in [1, 2^31)", (long long)n_E);
  if (total_L == 0) return GESR_OK;
  if (!E || !rows || !W_k || !W_v || !K_cache || !V_cache)
    return fail(GESR_ERR_INVALID_ARG, "null required pointer");
  if (!aligned16(E) || !aligned16(W_k) || !aligned16(W_v) || !aligned16(K_cache) ||
      !aligned16(V_cache) || !aligned16(b_k) || !aligned16(b_v))
    return fail(GESR_ERR_INVALID_ARG, "pointers must be 16-byte aligned");
  if ((reinterpret_cast<uintptr_t>(rows) & 3u) != 0)
    return fail(GESR_ERR_INVALID_ARG, "rows must be 4-byte aligned");
  return run_projection(E, total_L, D_in, W_k, W_v, b_k, b_v, H, d, act, K_cache, V_cache,
                        static_cast<cudaStream_t>(stream), rows, n_E);
}

// Split-L (d = 128, pair kernel): a forced kv_splits = s > 1 cuts every (unit, head) into s
// ranges of key tiles; auto (0) splits only when there are fewer (unit, head) work items than
// CTA pairs (kAutoSplitItems), into enough ranges to cover them, by up to kMaxAutoSplits and
// keeping >= 2 key tiles per split on average.
constexpr int64_t kAutoSplitItems = 74;
constexpr int kMaxAutoSplits = 16;
constexpr int kMaxSplits = 64;

int pick_splits(int64_t B, int64_t total_C, int64_t total_L, int32_t H, int32_t d,
                int32_t kv_splits) {
  if (d != 128 || !pair_attention_enabled()) return 1;
  if (kv_splits >= 1) return kv_splits;
  const int64_t items = max_units(B, total_C) * H;
  if (items >= kAutoSplitItems || B == 0) return 1;
  const int64_t tiles = (total_L / B + 127) / 128;             // mean key tiles per request
  int64_t s = (kAutoSplitItems + items - 1) / items;
  if (s > tiles / 2) s = tiles / 2;
  if (s > kMaxAutoSplits) s = kMaxAutoSplits;
  return s < 1 ? 1 : static_cast<int>(s);
}

// [splits, total_C, H] float2 (m, l), then (256-aligned) [splits, total_C, H, d] fp32
size_t split_ml_bytes(int64_t total_C, int32_t H, int splits) {
  return (static_cast<size_t>(splits) * total_C * H * 8 + 255) & ~static_cast<size_t>(255);
}
size_t split_bytes(int64_t total_C, int32_t H, int32_t d, int splits) {
  if (splits <= 1) return 0;
  return split_ml_bytes(total_C, H, splits) + static_cast<size_t>(splits) * total_C * H * d * 4;
}

size_t gesr_tasa_workspace_bytes(int64_t B, int64_t total_C, int32_t H, int32_t d,
                                 int32_t kv_splits) {
  if (B < 0 || total_C < 0 || H < 1 || !valid_d(d) || kv_splits < 0 || kv_splits > kMaxSplits)
    return 0;
  size_t part = 0;
  if (d == 128) {
    if (kv_splits > 1) {
      part = split_bytes(total_C, H, d, kv_splits);
    } else if (kv_splits == 0 && max_units(B, total_C) * H < kAutoSplitItems) {
      part = split_bytes(total_C, H, d, kMaxAutoSplits);      // bound for any auto choice
    }
  }
  const size_t q_end = units_end(B, total_C) + static_cast<size_t>(total_C) * H * d * 2;
  const size_t lse_scratch = (static_cast<size_t>(total_C) * H * 4 + 255) & ~static_cast<size_t>(255);
  return ((q_end + 255) & ~static_cast<size_t>(255)) + part + lse_scratch;
}

// Shared body of gesr_tasa_score and gesr_tasa_score_self (K_self / V_self non-null: the
// candidate's own key/value is merged into each row after the history attention).
static gesr_status tasa_impl(const void* T, int64_t total_C, int32_t D_in, const int64_t* cand_offsets,
                      const void* W_q, const float* b_q, int32_t act, const void* K_cache,
                      const void* V_cache, const int64_t* seq_offsets, int64_t B, int64_t total_L,
                      int32_t H, int32_t d, float scale, int32_t kv_splits, uint32_t flags,
                      const void* K_self, const void* V_self, void* O, int32_t o_dtype,
                      float* lse, void* workspace, size_t workspace_bytes, void* stream,
                      int causal = 0, bool validate_only = false,
                      const int32_t* t_rows = nullptr, int64_t n_E = 0) {
  // t_rows != NULL (gesr_tasa_score_gather): T is an [n_E, D_in] table and candidate row t is
  // its row t_rows[t], gathered by the Q projection
  const bool self = K_self != nullptr || V_self != nullptr;
  gesr_status s = check_common(D_in, H, d, act);
  if (s != GESR_OK) return s;
  if (B < 0 || total_C < 0 || total_L < 0)
    return fail(GESR_ERR_INVALID_ARG, "B, total_C, total_L must be >= 0");
  if (B > (int64_t(1) << 31) - 1) return fail(GESR_ERR_INVALID_ARG, "B too large");
  if (total_C >= (int64_t(1) << 31) / H || total_L >= (int64_t(1) << 31) / H)
    return fail(GESR_ERR_INVALID_ARG, "H*total rows exceed the 2^31 TMA coordinate range");
  if (o_dtype != GESR_OUT_F32 && o_dtype != GESR_OUT_BF16)
    return fail(GESR_ERR_INVALID_ARG, "o_dtype=%d is not a gesr_out_dtype", o_dtype);
  if (kv_splits < 0 || kv_splits > kMaxSplits)
    return fail(GESR_ERR_INVALID_ARG, "kv_splits=%d outside [0, %d]", kv_splits, kMaxSplits);
  if (causal && kv_splits > 1)
    return fail(GESR_ERR_UNSUPPORTED, "kv_splits > 1 is not supported for causal attention");
  if (kv_splits > 1 && (d != 128 || !pair_attention_enabled()))
    return fail(GESR_ERR_UNSUPPORTED, "kv_splits > 1 needs d = 128 (CTA-pair attention kernel)");
  if ((flags & GESR_TASA_SELF_KEY) && !self)
    return fail(GESR_ERR_UNSUPPORTED,
                "GESR_TASA_SELF_KEY needs the candidates' own K/V: use gesr_tasa_score_self");
  if (flags & ~(GESR_TASA_SELF_KEY | GESR_TASA_HSTU_SILU))
    return fail(GESR_ERR_INVALID_ARG, "unknown flags 0x%x", flags);
  const bool hstu = (flags & GESR_TASA_HSTU_SILU) != 0;
  if (hstu && (self || causal))
    return fail(GESR_ERR_UNSUPPORTED, "GESR_TASA_HSTU_SILU is not combined with a self key or "
                "causal attention");
  if (hstu && kv_splits > 1)
    return fail(GESR_ERR_UNSUPPORTED, "GESR_TASA_HSTU_SILU runs one key split");
  if (hstu && lse != nullptr)
    return fail(GESR_ERR_INVALID_ARG, "lse is undefined for GESR_TASA_HSTU_SILU (pass NULL)");
  if (total_C == 0 || B == 0) return GESR_OK;
  if (!T || !cand_offsets || !W_q || !seq_offsets || !O || !workspace)
    return fail(GESR_ERR_INVALID_ARG, "null required pointer");
  if (t_rows != nullptr && (reinterpret_cast<uintptr_t>(t_rows) & 3u) != 0)
    return fail(GESR_ERR_INVALID_ARG, "rows must be 4-byte aligned");
  if (total_L > 0 && (!K_cache || !V_cache))
    return fail(GESR_ERR_INVALID_ARG, "null K/V cache with total_L > 0");
  if (self && (!K_self || !V_self || !aligned16(K_self) || !aligned16(V_self)))
    return fail(GESR_ERR_INVALID_ARG, "K_self and V_self must both be given and 16-byte aligned");
  if (!aligned16(T) || !aligned16(W_q) || !aligned16(K_cache) || !aligned16(V_cache) ||
      !aligned16(O) || !aligned16(b_q) || !aligned16(lse) ||
      (reinterpret_cast<uintptr_t>(workspace) & 255u) != 0 ||
      (reinterpret_cast<uintptr_t>(cand_offsets) & 7u) != 0 ||
      (reinterpret_cast<uintptr_t>(seq_offsets) & 7u) != 0)
    return fail(GESR_ERR_INVALID_ARG, "misaligned pointer");
  const size_t need = gesr_tasa_workspace_bytes(B, total_C, H, d, kv_splits);
  if (workspace_bytes < need)
    return fail(GESR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);
  // the attention kernels count work items (unit, head, split) in 32 bits
  const int64_t items = max_units(B, total_C) * H;
  if (items * (kv_splits >= 1 ? kv_splits : (items < kAutoSplitItems ? kMaxAutoSplits : 1)) >=
      (int64_t(1) << 31))
    return fail(GESR_ERR_INVALID_ARG, "(units x heads x splits) exceeds 2^31 work items");
  if (validate_only) return GESR_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  s = debug_check(seq_offsets, B, total_L, 0, st);
  if (s != GESR_OK) return s;
  s = debug_check(cand_offsets, B, total_C, 1, st);
  if (s != GESR_OK) return s;

  gesr::AttnParams p{};
  p.seq_offsets = seq_offsets;
  p.cand_offsets = cand_offsets;
  p.total_C = total_C;
  p.total_L = total_L;
  p.H = H;
  const float sc = scale > 0.f ? scale : 1.0f / std::sqrt(static_cast<float>(d));
  p.scale_log2 = sc * 1.4426950408889634f;
  p.O = O;
  p.o_bf16 = o_dtype == GESR_OUT_BF16;
  p.splits = 1;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  int* count = reinterpret_cast<int*>(ws);
  int4* units = reinterpret_cast<int4*>(ws + 256);
  void* Q = ws + units_end(B, total_C);
  const size_t q_end = units_end(B, total_C) + static_cast<size_t>(total_C) * H * d * 2;
  uint8_t* part = ws + ((q_end + 255) & ~static_cast<size_t>(255));
  // the self-key merge needs the history lse: a scratch row set when the caller wants none
  float* lse_scratch = reinterpret_cast<float*>(
      part + split_bytes(total_C, H, d,
                         d == 128 ? (kv_splits > 1 ? kv_splits
                                     : (kv_splits == 0 && max_units(B, total_C) * H < kAutoSplitItems
                                            ? kMaxAutoSplits : 1))
                                  : 1));
  p.lse = (self && lse == nullptr) ? lse_scratch : lse;
  auto self_merge = [&]() -> gesr_status {
    if (!self) return GESR_OK;
    cudaError_t e2 = gesr::launch_attn_self_merge(p, Q, K_self, V_self, d, sc, st);
    return e2 == cudaSuccess ? GESR_OK : cuda_fail(e2, "attn_self_merge launch");
  };
  if (total_L == 0) {
    cudaError_t e = gesr::launch_attn_empty(p, d, st);
    if (e != cudaSuccess) return cuda_fail(e, "attn_empty launch");
    if (!self) return GESR_OK;
    s = run_projection(T, total_C, D_in, W_q, nullptr, b_q, nullptr, H, d, act, Q, nullptr, st,
                       t_rows, n_E);
    if (s != GESR_OK) return s;
    return self_merge();
  }

  // B = 1: the kernels derive the single request's units (kernels.h unit_of), no work-list launch
  p.units = B == 1 ? nullptr : units;
  p.unit_count = B == 1 ? nullptr : count;
  p.splits = (causal || hstu) ? 1 : pick_splits(B, total_C, total_L, H, d, kv_splits);
  p.causal = causal;
  p.hstu = hstu ? 1 : 0;

  if (p.splits > 1) {
    p.part_ml = reinterpret_cast<float2*>(part);
    p.part_o = reinterpret_cast<float*>(part + split_ml_bytes(total_C, H, p.splits));
  }
  const bool pair = d == 128 && pair_attention_enabled() && !hstu;
  cudaError_t e = cudaSuccess;
  if (B != 1) {
    e = gesr::launch_build_units(seq_offsets, cand_offsets, B, units, count, causal, st);
    if (e != cudaSuccess) return cuda_fail(e, "build_units launch");
  }
  s = run_projection(T, total_C, D_in, W_q, nullptr, b_q, nullptr, H, d, act, Q, nullptr, st,
                       t_rows, n_E);
  if (s != GESR_OK) return s;

  CUtensorMap mq, mk, mv;
  const uint32_t box_cols = d >= 64 ? 64 : 32;
  const CUtensorMapSwizzle swz = d >= 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  s = make_map_2d(&mq, Q, static_cast<uint64_t>(H) * total_C, d, 128, box_cols, swz, "Q");
  if (s != GESR_OK) return s;
  s = make_map_2d(&mk, K_cache, static_cast<uint64_t>(H) * total_L, d, 128, box_cols, swz, "K");
  if (s != GESR_OK) return s;
  s = make_map_2d(&mv, V_cache, static_cast<uint64_t>(H) * total_L, d, 128, box_cols, swz, "V");
  if (s != GESR_OK) return s;
  CUtensorMap mo;
  std::memset(&mo, 0, sizeof(mo));
  if (p.o_bf16 && total_C > 0 && total_C < (int64_t{1} << 31)) {
    s = make_o_map(&mo, O, static_cast<uint64_t>(total_C), H, d);
    if (s != GESR_OK) return s;
    p.o_tma = 1;
  }
  if (pair) {
    CUtensorMap mkh;
    s = make_map_2d(&mkh, K_cache, static_cast<uint64_t>(H) * total_L, d, 64, 64, swz, "K half");
    if (s != GESR_OK) return s;
    e = gesr::launch_attn_pair(mq, mkh, mv, mo, p, max_units(B, total_C), st);
    if (e != cudaSuccess) return cuda_fail(e, "attn_pair_kernel launch");
    if (p.splits > 1) {
      e = gesr::launch_attn_combine(p, d, st);
      if (e != cudaSuccess) return cuda_fail(e, "attn_combine_kernel launch");
    }
    return self_merge();
  }
  e = gesr::launch_attn(d, mq, mk, mv, mo, p, max_units(B, total_C), st);
  if (e != cudaSuccess) return cuda_fail(e, "attn_kernel launch");
  return self_merge();
}

gesr_status gesr_tasa_score(const void* T, int64_t total_C, int32_t D_in,
                            const int64_t* cand_offsets, const void* W_q, const float* b_q,
                            int32_t act, const void* K_cache, const void* V_cache,
                            const int64_t* seq_offsets, int64_t B, int64_t total_L, int32_t H,
                            int32_t d, float scale, int32_t kv_splits, uint32_t flags, void* O,
                            int32_t o_dtype, float* lse, void* workspace,
                            size_t workspace_bytes, void* stream) {
  return tasa_impl(T, total_C, D_in, cand_offsets, W_q, b_q, act, K_cache, V_cache, seq_offsets,
                   B, total_L, H, d, scale, kv_splits, flags, nullptr, nullptr, O, o_dtype, lse,
                   workspace, workspace_bytes, stream);
}

gesr_status gesr_tasa_score_gather(const void* E, int64_t n_E, int32_t D_in, const int32_t* rows,
                                   int64_t total_C, const int64_t* cand_offsets, const void* W_q,
                                   const float* b_q, int32_t act, const void* K_cache,
                                   const void* V_cache, const int64_t* seq_offsets, int64_t B,
                                   int64_t total_L, int32_t H, int32_t d, float scale,
                                   int32_t kv_splits, uint32_t flags, void* O, int32_t o_dtype,
                                   float* lse, void* workspace, size_t workspace_bytes,
                                   void* stream) {
  if (n_E < 1 || n_E >= (int64_t(1) << 31))
    return fail(GESR_ERR_INVALID_ARG, "n_E=%lld must be in [1, 2^31)", (long long)n_E);
  if (total_C > 0 && B > 0 && !rows) return fail(GESR_ERR_INVALID_ARG, "null required pointer");
  if (flags & GESR_TASA_SELF_KEY)
    return fail(GESR_ERR_UNSUPPORTED, "GESR_TASA_SELF_KEY is not offered with the gather");
  return tasa_impl(E, total_C, D_in, cand_offsets, W_q, b_q, act, K_cache, V_cache, seq_offsets,
                   B, total_L, H, d, scale, kv_splits, flags, nullptr, nullptr, O, o_dtype, lse,
                   workspace, workspace_bytes, stream, 0, false, rows, n_E);
}

gesr_status gesr_tasa_score_self(const void* T, int64_t total_C, int32_t D_in,
                                 const int64_t* cand_offsets, const void* W_q, const float* b_q,
                                 int32_t act, const void* K_cache, const void* V_cache,
                                 const int64_t* seq_offsets, int64_t B, int64_t total_L,
                                 int32_t H, int32_t d, float scale, int32_t kv_splits,
                                 const void* K_self, const void* V_self, void* O,
                                 int32_t o_dtype, float* lse, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  if (!K_self || !V_self)
    return fail(GESR_ERR_INVALID_ARG, "gesr_tasa_score_self needs K_self and V_self");
  return tasa_impl(T, total_C, D_in, cand_offsets, W_q, b_q, act, K_cache, V_cache, seq_offsets,
                   B, total_L, H, d, scale, kv_splits, GESR_TASA_SELF_KEY, K_self, V_self, O,
                   o_dtype, lse, workspace, workspace_bytes, stream);
}

static gesr_status hma_impl(const int64_t* user_ids, const int64_t* user_offsets,
                           const int64_t* item_ids, const int64_t* item_offsets,
                           const int64_t* cand_offsets, int64_t B, int64_t total_C, int32_t F,
                           int32_t cap, int32_t* counts, const void* E, int32_t D_h, void* emb,
                           void* stream) {
  if (B < 0 || total_C < 0 || F < 0)
    return fail(GESR_ERR_INVALID_ARG, "B, total_C, F must be >= 0");
  if (F > 256) return fail(GESR_ERR_INVALID_ARG, "F=%d > 256 fields", F);
  if (B > 2147483647LL) return fail(GESR_ERR_INVALID_ARG, "B too large");
  if (E != nullptr) {
    if (cap < 1) return fail(GESR_ERR_INVALID_ARG, "the offset embedding needs cap M >= 1");
    if (D_h < 8 || D_h % 8 != 0 || D_h > 4096)
      return fail(GESR_ERR_INVALID_ARG, "D_h=%d must be a multiple of 8 in [8, 4096]", D_h);
    if (!emb) return fail(GESR_ERR_INVALID_ARG, "null embedding output");
    if (!aligned16(E) || !aligned16(emb)) return fail(GESR_ERR_INVALID_ARG, "misaligned pointer");
  }
  if (B == 0 || total_C == 0 || F == 0) return GESR_OK;
  if (!user_offsets || !item_offsets || !cand_offsets || !counts)
    return fail(GESR_ERR_INVALID_ARG, "null required pointer");
  if (((reinterpret_cast<uintptr_t>(user_ids) | reinterpret_cast<uintptr_t>(user_offsets) |
        reinterpret_cast<uintptr_t>(item_ids) | reinterpret_cast<uintptr_t>(item_offsets) |
        reinterpret_cast<uintptr_t>(cand_offsets)) & 7u) != 0 ||
      (reinterpret_cast<uintptr_t>(counts) & 3u) != 0)
    return fail(GESR_ERR_INVALID_ARG, "misaligned pointer");
  gesr::HmaParams p{};
  p.user_ids = user_ids;
  p.user_offsets = user_offsets;
  p.item_ids = item_ids;
  p.item_offsets = item_offsets;
  p.cand_offsets = cand_offsets;
  p.B = B;
  p.total_C = total_C;
  p.F = F;
  p.cap = cap;
  p.counts = counts;
  p.E = static_cast<const uint4*>(E);
  p.dh_chunks = E ? D_h / 8 : 0;
  p.emb = static_cast<uint4*>(emb);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  gesr_status s = debug_check(cand_offsets, B, total_C, 1, st);
  if (s == GESR_OK) s = debug_check(user_offsets, B * F, -1, 2, st);
  if (s == GESR_OK) s = debug_check(item_offsets, total_C * F, -1, 3, st);
  if (s != GESR_OK) return s;
  cudaError_t e = gesr::launch_hma(p, st);
  return e == cudaSuccess ? GESR_OK : cuda_fail(e, "hma_kernel launch");
}

gesr_status gesr_hma_count(const int64_t* user_ids, const int64_t* user_offsets,
                           const int64_t* item_ids, const int64_t* item_offsets,
                           const int64_t* cand_offsets, int64_t B, int64_t total_C, int32_t F,
                           int32_t cap, int32_t* counts, void* stream) {
  return hma_impl(user_ids, user_offsets, item_ids, item_offsets, cand_offsets, B, total_C, F,
                  cap, counts, nullptr, 0, nullptr, stream);
}

gesr_status gesr_hma_count_embed(const int64_t* user_ids, const int64_t* user_offsets,
                                 const int64_t* item_ids, const int64_t* item_offsets,
                                 const int64_t* cand_offsets, int64_t B, int64_t total_C,
                                 int32_t F, int32_t M, int32_t* counts, const void* E,
                                 int32_t D_h, void* emb, void* stream) {
  if (!E) return fail(GESR_ERR_INVALID_ARG, "null embedding table");
  return hma_impl(user_ids, user_offsets, item_ids, item_offsets, cand_offsets, B, total_C, F, M,
                  counts, E, D_h, emb, stream);
}

size_t gesr_stu_workspace_bytes(int64_t total_C, int32_t H, int32_t d) {
  if (total_C < 0 || H < 1 || !valid_d(d)) return 0;
  return stu_buffer_bytes(total_C, static_cast<int64_t>(H) * d);
}

gesr_status gesr_stu_output(const void* T, int64_t total_C, int32_t D_in, const void* O,
                            int32_t o_dtype, const void* W_g, const float* b_g,
                            const float* ln_gamma, const float* ln_beta, float ln_eps,
                            const void* W_o, const float* b_o, const void* X_res, int32_t H,
                            int32_t d, int32_t D_out, void* Y, void* workspace,
                            size_t workspace_bytes, void* stream) {
  gesr_status s = check_common(D_in, H, d, GESR_ACT_SILU);
  if (s != GESR_OK) return s;
  const int64_t D = static_cast<int64_t>(H) * d;
  if (total_C < 0) return fail(GESR_ERR_INVALID_ARG, "total_C=%lld < 0", (long long)total_C);
  if (D_out < 32 || D_out > 16384 || (D_out % 32) != 0)
    return fail(GESR_ERR_INVALID_ARG, "D_out=%d must be a multiple of 32 in [32, 16384]", D_out);
  if (D % 32 != 0 || D > 16384)
    return fail(GESR_ERR_INVALID_ARG, "H*d=%lld must be a multiple of 32 and <= 16384", (long long)D);
  if (o_dtype != GESR_OUT_F32 && o_dtype != GESR_OUT_BF16)
    return fail(GESR_ERR_INVALID_ARG, "o_dtype=%d is not a gesr_out_dtype", o_dtype);
  if (!(ln_eps >= 0.0f) || !std::isfinite(ln_eps))
    return fail(GESR_ERR_INVALID_ARG, "ln_eps must be finite and >= 0");
  if (total_C >= (int64_t(1) << 31))
    return fail(GESR_ERR_INVALID_ARG, "total_C exceeds the 2^31 TMA coordinate range");
  if (total_C == 0) return GESR_OK;
  if (!T || !O || !W_g || !ln_gamma || !ln_beta || !W_o || !Y)
    return fail(GESR_ERR_INVALID_ARG, "null required pointer");
  if (!aligned16(T) || !aligned16(O) || !aligned16(W_g) || !aligned16(b_g) ||
      !aligned16(ln_gamma) || !aligned16(ln_beta) || !aligned16(W_o) || !aligned16(b_o) ||
      !aligned16(X_res) || !aligned16(Y) || !aligned16(workspace))
    return fail(GESR_ERR_INVALID_ARG, "pointers must be 16-byte aligned");
  const size_t need = stu_buffer_bytes(total_C, D);
  if (!workspace || workspace_bytes < need)
    return fail(GESR_ERR_WORKSPACE, "workspace of %zu bytes < %zu needed", workspace_bytes, need);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  // 1. gating branch G = SiLU(T W_g^T + b_g), row-major [total_C, D] bf16 in the workspace
  s = run_projection_rm(T, total_C, D_in, W_g, b_g, static_cast<int32_t>(D), GESR_ACT_SILU,
                        nullptr, workspace, st);
  if (s != GESR_OK) return s;
  // 2. Z = (LayerNorm(O) gamma + beta) * G, in place over G
  cudaError_t e = gesr::launch_ln_gate(O, o_dtype == GESR_OUT_BF16 ? 1 : 0,
                                       static_cast<__nv_bfloat16*>(workspace), ln_gamma, ln_beta,
                                       ln_eps, total_C, static_cast<int>(D), st);
  if (e != cudaSuccess) return cuda_fail(e, "ln_gate_kernel launch");
  // 3. Y = Z W_o^T + b_o + X_res
  return run_projection_rm(workspace, total_C, static_cast<int32_t>(D), W_o, b_o, D_out,
                           GESR_ACT_IDENTITY, X_res, Y, st);
}

static size_t nro_weight_offset(int64_t B, int64_t total_C, int32_t j, int32_t d,
                                int32_t kv_splits) {
  return (gesr_tasa_workspace_bytes(B, total_C, j, d, kv_splits) + 255) & ~static_cast<size_t>(255);
}

size_t gesr_nro_workspace_bytes(int64_t B, int64_t total_C, int32_t j, int32_t d, int32_t D_in,
                                int32_t kv_splits) {
  if (gesr_tasa_workspace_bytes(B, total_C, j, d, kv_splits) == 0 || D_in < 8) return 0;
  return nro_weight_offset(B, total_C, j, d, kv_splits) +
         static_cast<size_t>(j) * d * D_in * 2;
}

gesr_status gesr_nro_cross_score(const void* T, int64_t total_C, int32_t D_in,
                                 const int64_t* cand_offsets, const void* W_q,
                                 const float* q_gate, const float* b_q, int32_t act,
                                 const void* K_cache, const void* V_cache,
                                 const int64_t* seq_offsets, int64_t B, int64_t total_L,
                                 int32_t j, int32_t d, float scale, int32_t kv_splits, void* O,
                                 int32_t o_dtype, float* lse, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  gesr_status s = check_common(D_in, j, d, act);
  if (s != GESR_OK) return s;
  if (B < 0 || total_C < 0 || total_L < 0)
    return fail(GESR_ERR_INVALID_ARG, "B, total_C, total_L must be >= 0");
  if (kv_splits < 0 || kv_splits > kMaxSplits)
    return fail(GESR_ERR_INVALID_ARG, "kv_splits=%d outside [0, %d]", kv_splits, kMaxSplits);
  if (total_C == 0 || B == 0) return GESR_OK;
  if (!W_q || !q_gate || !workspace) return fail(GESR_ERR_INVALID_ARG, "null required pointer");
  if (!aligned16(W_q) || !aligned16(q_gate) || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return fail(GESR_ERR_INVALID_ARG, "misaligned pointer");
  const size_t need = gesr_nro_workspace_bytes(B, total_C, j, d, D_in, kv_splits);
  if (workspace_bytes < need)
    return fail(GESR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);
  const size_t off = nro_weight_offset(B, total_C, j, d, kv_splits);
  void* W_fold = static_cast<uint8_t*>(workspace) + off;
  // every host-side check of the attention call runs before the first launch (fold_gate)
  s = tasa_impl(T, total_C, D_in, cand_offsets, W_fold, b_q, act, K_cache, V_cache, seq_offsets,
                B, total_L, j, d, scale, kv_splits, 0, nullptr, nullptr, O, o_dtype, lse,
                workspace, off, stream, 0, /*validate_only=*/true);
  if (s != GESR_OK) return s;
  cudaError_t e = gesr::launch_fold_gate(W_q, q_gate, W_fold, j, d, D_in,
                                         static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fold_gate launch");
  return tasa_impl(T, total_C, D_in, cand_offsets, W_fold, b_q, act, K_cache, V_cache,
                   seq_offsets, B, total_L, j, d, scale, kv_splits, 0, nullptr, nullptr, O,
                   o_dtype, lse, workspace, off, stream);
}

gesr_status gesr_history_attention(const void* U, int64_t total_L, int32_t D_in,
                                   const int64_t* seq_offsets, int64_t B, const void* W_q,
                                   const float* b_q, int32_t act, const void* K_cache,
                                   const void* V_cache, int32_t H, int32_t d, float scale,
                                   void* O, int32_t o_dtype, float* lse, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  // the history rows are the queries: candidate offsets := sequence offsets, one split
  return tasa_impl(U, total_L, D_in, seq_offsets, W_q, b_q, act, K_cache, V_cache, seq_offsets,
                   B, total_L, H, d, scale, 1, 0, nullptr, nullptr, O, o_dtype, lse, workspace,
                   workspace_bytes, stream, 1);
}

gesr_status gesr_layer_norm(const void* X, int64_t rows, int32_t D, const float* gamma,
                            const float* beta, float eps, void* Y, void* stream) {
  if (rows < 0) return fail(GESR_ERR_INVALID_ARG, "rows=%lld < 0", (long long)rows);
  if (D < 8 || D > 16384 || (D % 8) != 0)
    return fail(GESR_ERR_INVALID_ARG, "D=%d must be a multiple of 8 in [8, 16384]", D);
  if (!(eps >= 0.0f) || !std::isfinite(eps))
    return fail(GESR_ERR_INVALID_ARG, "eps must be finite and >= 0");
  if (rows == 0) return GESR_OK;
  if (!X || !gamma || !beta || !Y) return fail(GESR_ERR_INVALID_ARG, "null required pointer");
  if (!aligned16(X) || !aligned16(gamma) || !aligned16(beta) || !aligned16(Y))
    return fail(GESR_ERR_INVALID_ARG, "pointers must be 16-byte aligned");
  cudaError_t e = gesr::launch_layer_norm(X, Y, gamma, beta, eps, rows, D,
                                          static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GESR_OK : cuda_fail(e, "layer_norm_kernel launch");
}

// RO cross attention workspace: [query rows X bf16 | offsets int64 | O_full fp32 | tasa ws]
static size_t ro_layout(int64_t B, int32_t i, int32_t d, int32_t D_in, size_t* off_offs,
                        size_t* off_o, size_t* off_ws) {
  auto up = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
  const size_t x_bytes = up(static_cast<size_t>(B) * i * D_in * 2);
  const size_t offs_bytes = up(static_cast<size_t>(B + 1) * 8);
  const size_t o_bytes = up(static_cast<size_t>(B) * i * i * d * 4);
  *off_offs = x_bytes;
  *off_o = x_bytes + offs_bytes;
  *off_ws = *off_o + o_bytes;
  return *off_ws + gesr_tasa_workspace_bytes(B, B * i, i, d, 1);
}

size_t gesr_ro_workspace_bytes(int64_t B, int32_t i, int32_t d, int32_t D_in) {
  if (B < 0 || i < 1 || !valid_d(d) || D_in < 8) return 0;
  size_t a, b, c;
  return ro_layout(B, i, d, D_in, &a, &b, &c);
}

gesr_status gesr_ro_cross_score(const void* seeds, const void* ctx, int32_t i, int32_t D_in,
                                const void* W_q, const float* b_q, int32_t act,
                                const void* K_cache, const void* V_cache,
                                const int64_t* seq_offsets, int64_t B, int64_t total_L,
                                int32_t d, float scale, void* U_cross, int32_t o_dtype,
                                void* workspace, size_t workspace_bytes, void* stream) {
  gesr_status s = check_common(D_in, i, d, act);
  if (s != GESR_OK) return s;
  if (B < 0 || total_L < 0) return fail(GESR_ERR_INVALID_ARG, "B, total_L must be >= 0");
  if (o_dtype != GESR_OUT_F32 && o_dtype != GESR_OUT_BF16)
    return fail(GESR_ERR_INVALID_ARG, "o_dtype=%d is not a gesr_out_dtype", o_dtype);
  if (B == 0) return GESR_OK;
  if (!seeds || !W_q || !seq_offsets || !U_cross || !workspace)
    return fail(GESR_ERR_INVALID_ARG, "null required pointer");
  if (!aligned16(seeds) || !aligned16(ctx) || !aligned16(W_q) || !aligned16(U_cross) ||
      (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return fail(GESR_ERR_INVALID_ARG, "misaligned pointer");
  size_t off_offs, off_o, off_ws;
  const size_t need = ro_layout(B, i, d, D_in, &off_offs, &off_o, &off_ws);
  if (workspace_bytes < need)
    return fail(GESR_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t* offs = reinterpret_cast<int64_t*>(ws + off_offs);
  float* O_full = reinterpret_cast<float*>(ws + off_o);
  cudaError_t e = gesr::launch_ro_queries(seeds, ctx, ws, offs, B, i, D_in, st);
  if (e != cudaSuccess) return cuda_fail(e, "ro_queries launch");
  // the i query rows of every request through the target-aware path with the slots as heads
  // (all slots for every row: the i x i products are tiny next to the history), one split
  s = tasa_impl(ws, B * i, D_in, offs, W_q, b_q, act, K_cache, V_cache, seq_offsets, B, total_L,
                i, d, scale, 1, 0, nullptr, nullptr, O_full, GESR_OUT_F32, nullptr, ws + off_ws,
                need - off_ws, stream);
  if (s != GESR_OK) return s;
  e = gesr::launch_ro_gather(O_full, U_cross, o_dtype == GESR_OUT_BF16 ? 1 : 0, B, i, d, st);
  return e == cudaSuccess ? GESR_OK : cuda_fail(e, "ro_gather launch");
}

}  // extern "C"
