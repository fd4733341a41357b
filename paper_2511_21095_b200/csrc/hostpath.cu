// hostpath.cu -- the end-to-end path from HOST memory (include/gesr.h: gesr_host_chunk_maxima,
// gesr_host_plan_create / _destroy, gesr_score_host): a small native runtime around the three
// device calls of a scoring step.  The batch's requests are cut into contiguous chunks; per
// chunk the inputs are copied host->device on a copy-in stream, gesr_kv_project ->
// gesr_tasa_score -> gesr_hma_count run on the caller's stream, and O / counts are copied
// device->host on a copy-out stream, with two device buffer sets alternating, so the copy
// engines of both directions and the SMs work at the same time (PCIe, not the GPU, bounds this
// path: DESIGN.md s8b).  Each chunk's offset arrays are rebased on the device by one small
// kernel (the caller's host buffers are never written).
#include "../../include/gesr.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>

#include "kernels.h"

gesr_status gesr_internal_fail(gesr_status s, const char* msg);

namespace {

constexpr int kSets = 2;

gesr_status hfail(gesr_status s, const char* msg) { return gesr_internal_fail(s, msg); }
gesr_status hcuda(cudaError_t e, const char* where) {
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
  return gesr_internal_fail(GESR_ERR_CUDA, buf);
}

// offsets[i] -= base for the chunk's four offset arrays (one launch)
__global__ void rebase_kernel(int64_t* a, int64_t na, int64_t ba, int64_t* b, int64_t nb,
                              int64_t bb, int64_t* c, int64_t nc, int64_t bc, int64_t* d,
                              int64_t nd, int64_t bd) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
       i < na + nb + nc + nd; i += stride) {
    if (i < na) a[i] -= ba;
    else if (i < na + nb) b[i - na] -= bb;
    else if (i < na + nb + nc) c[i - na - nb] -= bc;
    else d[i - na - nb - nc] -= bd;
  }
}

struct Chunk {
  int64_t b0, b1, r0, r1, c0, c1, u0, u1, i0, i1;
};

Chunk chunk_of(const int64_t* so, const int64_t* co, const int64_t* uo, const int64_t* io,
               int64_t B, int32_t F, int32_t n, int32_t k) {
  Chunk c;
  c.b0 = B * k / n;
  c.b1 = B * (k + 1) / n;
  c.r0 = so[c.b0];
  c.r1 = so[c.b1];
  c.c0 = co[c.b0];
  c.c1 = co[c.b1];
  c.u0 = uo[c.b0 * F];
  c.u1 = uo[c.b1 * F];
  c.i0 = io[c.c0 * F];
  c.i1 = io[c.c1 * F];
  return c;
}

int32_t clamp_chunks(int64_t B, int32_t n) {
  if (n < 1) n = 1;
  if (B > 0 && n > B) n = static_cast<int32_t>(B);
  return n;
}

}  // namespace

struct gesr_host_plan {
  int dev;
  int64_t mB, mL, mC, mU, mI;
  int32_t D_in, H, d, F, o_dtype;
  struct Set {
    int64_t *so, *co, *uo, *io, *ui, *ii;
    void *U, *T, *K, *V, *O, *ws;
    int32_t* counts;
    size_t ws_bytes;
    cudaEvent_t h2d, done, free_;
  } set[kSets];
  cudaStream_t s_in, s_out;
  cudaEvent_t start, end;
};

extern "C" {

gesr_status gesr_host_chunk_maxima(const int64_t* seq_offsets, const int64_t* cand_offsets,
                                   const int64_t* user_offsets, const int64_t* item_offsets,
                                   int64_t B, int32_t F, int32_t n_chunks, int64_t* maxima) {
  if (!seq_offsets || !cand_offsets || !user_offsets || !item_offsets || !maxima)
    return hfail(GESR_ERR_INVALID_ARG, "gesr_host_chunk_maxima: null pointer");
  if (B < 0 || F < 1) return hfail(GESR_ERR_INVALID_ARG, "gesr_host_chunk_maxima: B < 0 or F < 1");
  const int32_t n = clamp_chunks(B, n_chunks);
  for (int i = 0; i < 5; ++i) maxima[i] = 0;
  for (int32_t k = 0; k < n && B > 0; ++k) {
    const Chunk c = chunk_of(seq_offsets, cand_offsets, user_offsets, item_offsets, B, F, n, k);
    const int64_t v[5] = {c.b1 - c.b0, c.r1 - c.r0, c.c1 - c.c0, c.u1 - c.u0, c.i1 - c.i0};
    for (int i = 0; i < 5; ++i) maxima[i] = v[i] > maxima[i] ? v[i] : maxima[i];
  }
  return GESR_OK;
}

gesr_status gesr_host_plan_destroy(gesr_host_plan* plan) {
  if (!plan) return GESR_OK;
  for (auto& s : plan->set) {
    void* bufs[] = {s.so, s.co, s.uo, s.io, s.ui, s.ii, s.U, s.T, s.K, s.V, s.O, s.ws, s.counts};
    for (void* b : bufs)
      if (b) cudaFree(b);
    if (s.h2d) cudaEventDestroy(s.h2d);
    if (s.done) cudaEventDestroy(s.done);
    if (s.free_) cudaEventDestroy(s.free_);
  }
  if (plan->s_in) cudaStreamDestroy(plan->s_in);
  if (plan->s_out) cudaStreamDestroy(plan->s_out);
  if (plan->start) cudaEventDestroy(plan->start);
  if (plan->end) cudaEventDestroy(plan->end);
  delete plan;
  return GESR_OK;
}

gesr_status gesr_host_plan_create(const int64_t* maxima, int32_t D_in, int32_t H, int32_t d,
                                  int32_t F, int32_t o_dtype, gesr_host_plan** out) {
  if (!maxima || !out) return hfail(GESR_ERR_INVALID_ARG, "gesr_host_plan_create: null pointer");
  *out = nullptr;
  for (int i = 0; i < 5; ++i)
    if (maxima[i] < 0) return hfail(GESR_ERR_INVALID_ARG, "gesr_host_plan_create: negative maximum");
  if (D_in < 1 || H < 1 || d < 1 || F < 1 || (o_dtype != GESR_OUT_F32 && o_dtype != GESR_OUT_BF16))
    return hfail(GESR_ERR_INVALID_ARG, "gesr_host_plan_create: bad D_in / H / d / F / o_dtype");
  gesr_host_plan* p = new gesr_host_plan();
  std::memset(p, 0, sizeof(*p));
  cudaGetDevice(&p->dev);
  p->mB = maxima[0];
  p->mL = maxima[1];
  p->mC = maxima[2];
  p->mU = maxima[3];
  p->mI = maxima[4];
  p->D_in = D_in;
  p->H = H;
  p->d = d;
  p->F = F;
  p->o_dtype = o_dtype;
  const size_t HD = static_cast<size_t>(H) * d;
  const size_t osz = o_dtype == GESR_OUT_BF16 ? 2 : 4;
  auto alloc = [&](void** ptr, size_t bytes) -> bool {
    return cudaMalloc(ptr, bytes > 0 ? bytes : 256) == cudaSuccess;
  };
  bool ok = true;
  for (auto& s : p->set) {
    ok = ok && alloc(reinterpret_cast<void**>(&s.so), (p->mB + 1) * 8);
    ok = ok && alloc(reinterpret_cast<void**>(&s.co), (p->mB + 1) * 8);
    ok = ok && alloc(reinterpret_cast<void**>(&s.uo), (p->mB * F + 1) * 8);
    ok = ok && alloc(reinterpret_cast<void**>(&s.io), (p->mC * F + 1) * 8);
    ok = ok && alloc(reinterpret_cast<void**>(&s.ui), p->mU * 8);
    ok = ok && alloc(reinterpret_cast<void**>(&s.ii), p->mI * 8);
    ok = ok && alloc(&s.U, p->mL * D_in * 2);
    ok = ok && alloc(&s.T, p->mC * D_in * 2);
    ok = ok && alloc(&s.K, p->mL * HD * 2);
    ok = ok && alloc(&s.V, p->mL * HD * 2);
    ok = ok && alloc(&s.O, p->mC * HD * osz);
    ok = ok && alloc(reinterpret_cast<void**>(&s.counts), p->mC * F * 4);
    s.ws_bytes = gesr_tasa_workspace_bytes(p->mB, p->mC, H, d, 0);
    ok = ok && alloc(&s.ws, s.ws_bytes);
    ok = ok && cudaEventCreateWithFlags(&s.h2d, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&s.free_, cudaEventDisableTiming) == cudaSuccess;
  }
  ok = ok && cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaEventCreateWithFlags(&p->start, cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaEventCreateWithFlags(&p->end, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    cudaError_t e = cudaGetLastError();
    gesr_host_plan_destroy(p);
    return hcuda(e, "gesr_host_plan_create");
  }
  *out = p;
  return GESR_OK;
}

}  // extern "C"

namespace {

// The chunk pipeline of gesr_score_host (E == NULL: U / T are host bf16 rows) and
// gesr_score_host_ids (E != NULL: U / T are host int32 row ids into the device table E, and
// the projections gather the rows themselves).
gesr_status score_host_impl(gesr_host_plan* plan, int32_t n_chunks, const void* E, int64_t n_E,
                            const void* U, const int64_t* seq_offsets,
                            const void* T, const int64_t* cand_offsets, int64_t B,
                            const void* W_q, const void* W_k, const void* W_v, int32_t act,
                            const int64_t* user_ids, const int64_t* user_offsets,
                            const int64_t* item_ids, const int64_t* item_offsets, int32_t cap,
                            void* O, int32_t* counts, void* stream) {
  if (!plan) return hfail(GESR_ERR_INVALID_ARG, "gesr_score_host: null plan");
  if (!seq_offsets || !cand_offsets || !user_offsets || !item_offsets || !W_q || !W_k || !W_v ||
      !O || !counts)
    return hfail(GESR_ERR_INVALID_ARG, "gesr_score_host: null required pointer");
  if (B < 0) return hfail(GESR_ERR_INVALID_ARG, "gesr_score_host: B < 0");
  int dev = -1;
  cudaGetDevice(&dev);
  if (dev != plan->dev)
    return hfail(GESR_ERR_INVALID_ARG, "gesr_score_host: the plan belongs to another device");
  const int32_t F = plan->F, H = plan->H, d = plan->d, D_in = plan->D_in;
  const int32_t n = clamp_chunks(B, n_chunks);
  // every chunk must fit the plan (checked before anything is enqueued)
  for (int32_t k = 0; k < n && B > 0; ++k) {
    const Chunk c = chunk_of(seq_offsets, cand_offsets, user_offsets, item_offsets, B, F, n, k);
    if (c.b1 - c.b0 > plan->mB || c.r1 - c.r0 > plan->mL || c.c1 - c.c0 > plan->mC ||
        c.u1 - c.u0 > plan->mU || c.i1 - c.i0 > plan->mI)
      return hfail(GESR_ERR_WORKSPACE, "gesr_score_host: a chunk exceeds the plan's maxima");
  }
  if (B == 0) return GESR_OK;
  if ((seq_offsets[B] > 0 && !U) || (cand_offsets[B] > 0 && !T) ||
      (user_offsets[B * F] > 0 && !user_ids) || (item_offsets[cand_offsets[B] * F] > 0 && !item_ids))
    return hfail(GESR_ERR_INVALID_ARG, "gesr_score_host: null input rows / ids");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t HD = static_cast<size_t>(H) * d;
  const size_t osz = plan->o_dtype == GESR_OUT_BF16 ? 2 : 4;
  const float scale = 1.0f / std::sqrt(static_cast<float>(d));
  const bool ids = E != nullptr;
  const size_t row_bytes = ids ? 4 : static_cast<size_t>(D_in) * 2;   // per U / T row
  const char* Uh = static_cast<const char*>(U);
  const char* Th = static_cast<const char*>(T);
  char* Oh = static_cast<char*>(O);
  cudaError_t e = cudaEventRecord(plan->start, st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(plan->s_in, plan->start, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(plan->s_out, plan->start, 0);
  if (e != cudaSuccess) return hcuda(e, "gesr_score_host: stream setup");
  for (int32_t k = 0; k < n; ++k) {
    const Chunk c = chunk_of(seq_offsets, cand_offsets, user_offsets, item_offsets, B, F, n, k);
    auto& s = plan->set[k % kSets];
    const int64_t nB = c.b1 - c.b0, nL = c.r1 - c.r0, nC = c.c1 - c.c0;
    const int64_t nU = c.u1 - c.u0, nI = c.i1 - c.i0;
    // ---- host -> device (copy-in stream); a buffer set is reused once its outputs are out
    if (k >= kSets) e = cudaStreamWaitEvent(plan->s_in, s.free_, 0);
    auto h2d = [&](void* dst, const void* src, size_t bytes) {
      if (e == cudaSuccess && bytes > 0)
        e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, plan->s_in);
    };
    h2d(s.so, seq_offsets + c.b0, (nB + 1) * 8);
    h2d(s.co, cand_offsets + c.b0, (nB + 1) * 8);
    h2d(s.uo, user_offsets + c.b0 * F, (nB * F + 1) * 8);
    h2d(s.io, item_offsets + c.c0 * F, (nC * F + 1) * 8);
    h2d(s.U, Uh + c.r0 * row_bytes, nL * row_bytes);
    h2d(s.T, Th + c.c0 * row_bytes, nC * row_bytes);
    h2d(s.ui, user_ids + c.u0, nU * 8);
    h2d(s.ii, item_ids + c.i0, nI * 8);
    if (e == cudaSuccess) e = cudaEventRecord(s.h2d, plan->s_in);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, s.h2d, 0);
    if (e != cudaSuccess) return hcuda(e, "gesr_score_host: host->device copies");
    // ---- the step on the caller's stream
    const int64_t nr = (nB + 1) * 2 + nB * F + 1 + nC * F + 1;
    rebase_kernel<<<static_cast<unsigned>((nr + 255) / 256 < 148 ? (nr + 255) / 256 : 148), 256, 0, st>>>(
        s.so, nB + 1, c.r0, s.co, nB + 1, c.c0, s.uo, nB * F + 1, c.u0, s.io, nC * F + 1, c.i0);
    gesr::count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return hcuda(e, "gesr_score_host: rebase_kernel launch");
    gesr_status r = GESR_OK;
    if (nL > 0)
      r = ids ? gesr_kv_project_gather(E, n_E, D_in, static_cast<const int32_t*>(s.U), nL, W_k,
                                       W_v, nullptr, nullptr, H, d, act, s.K, s.V, st)
              : gesr_kv_project(s.U, nL, D_in, W_k, W_v, nullptr, nullptr, H, d, act, s.K, s.V,
                                st);
    if (r == GESR_OK)
      r = ids ? gesr_tasa_score_gather(E, n_E, D_in, static_cast<const int32_t*>(s.T), nC, s.co,
                                       W_q, nullptr, act, s.K, s.V, s.so, nB, nL, H, d, scale, 0,
                                       0u, s.O, plan->o_dtype, nullptr, s.ws, s.ws_bytes, st)
              : gesr_tasa_score(s.T, nC, D_in, s.co, W_q, nullptr, act, s.K, s.V, s.so, nB, nL,
                                H, d, scale, 0, 0u, s.O, plan->o_dtype, nullptr, s.ws,
                                s.ws_bytes, st);
    if (r == GESR_OK)
      r = gesr_hma_count(s.ui, s.uo, s.ii, s.io, s.co, nB, nC, F, cap, s.counts, st);
    if (r != GESR_OK) return r;
    e = cudaEventRecord(s.done, st);
    // ---- device -> host (copy-out stream)
    if (e == cudaSuccess) e = cudaStreamWaitEvent(plan->s_out, s.done, 0);
    if (e == cudaSuccess && nC > 0)
      e = cudaMemcpyAsync(Oh + c.c0 * HD * osz, s.O, nC * HD * osz, cudaMemcpyDeviceToHost, plan->s_out);
    if (e == cudaSuccess && nC > 0)
      e = cudaMemcpyAsync(counts + c.c0 * F, s.counts, nC * F * 4, cudaMemcpyDeviceToHost, plan->s_out);
    if (e == cudaSuccess) e = cudaEventRecord(s.free_, plan->s_out);
    if (e != cudaSuccess) return hcuda(e, "gesr_score_host: device->host copies");
  }
  e = cudaEventRecord(plan->end, plan->s_out);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, plan->end, 0);
  return e == cudaSuccess ? GESR_OK : hcuda(e, "gesr_score_host: join");
}

}  // namespace

extern "C" {

gesr_status gesr_score_host(gesr_host_plan* plan, int32_t n_chunks,
                            const void* U, const int64_t* seq_offsets,
                            const void* T, const int64_t* cand_offsets, int64_t B,
                            const void* W_q, const void* W_k, const void* W_v, int32_t act,
                            const int64_t* user_ids, const int64_t* user_offsets,
                            const int64_t* item_ids, const int64_t* item_offsets, int32_t cap,
                            void* O, int32_t* counts, void* stream) {
  return score_host_impl(plan, n_chunks, nullptr, 0, U, seq_offsets, T, cand_offsets, B, W_q,
                         W_k, W_v, act, user_ids, user_offsets, item_ids, item_offsets, cap, O,
                         counts, stream);
}

gesr_status gesr_score_host_ids(gesr_host_plan* plan, int32_t n_chunks, const void* E,
                                int64_t n_E, const int32_t* hist_rows,
                                const int64_t* seq_offsets, const int32_t* cand_rows,
                                const int64_t* cand_offsets, int64_t B, const void* W_q,
                                const void* W_k, const void* W_v, int32_t act,
                                const int64_t* user_ids, const int64_t* user_offsets,
                                const int64_t* item_ids, const int64_t* item_offsets, int32_t cap,
                                void* O, int32_t* counts, void* stream) {
  if (!E) return hfail(GESR_ERR_INVALID_ARG, "gesr_score_host_ids: null table");
  if (n_E < 1 || n_E >= (int64_t(1) << 31))
    return hfail(GESR_ERR_INVALID_ARG, "gesr_score_host_ids: n_E must be in [1, 2^31)");
  cudaPointerAttributes pa;
  if (plan && (cudaPointerGetAttributes(&pa, E) != cudaSuccess || pa.type != cudaMemoryTypeDevice ||
               pa.device != plan->dev)) {
    (void)cudaGetLastError();
    return hfail(GESR_ERR_INVALID_ARG,
                 "gesr_score_host_ids: E must be device memory on the plan's device");
  }
  return score_host_impl(plan, n_chunks, E, n_E, hist_rows, seq_offsets, cand_rows, cand_offsets,
                         B, W_q, W_k, W_v, act, user_ids, user_offsets, item_ids, item_offsets,
                         cap, O, counts, stream);
}

}  // extern "C"
