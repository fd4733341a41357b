/* include/gesr.h -- C ABI of libgesr.so: the GESR Mixture-of-Attention candidate-scoring hot
 * path (arxiv 2511.21095) on B200 (sm_100a).
 *
 * Three calls make one scoring step over a batch of B ranking requests:
 *
 *   gesr_kv_project   K/V projection of every user's jagged history, computed once per user and
 *                     cached for all of that user's candidates.
 *                     PAPER.md:335-341 (s3.4.2 Target-Aware Self Attention: U in R^{N x D},
 *                     D = embedding dim flattened over heads; [U, T] through self-attention),
 *                     caching PAPER.md:203, 215 (s1 "improved caching mechanisms").
 *   gesr_tasa_score   target-aware attention: every candidate's query attends over its own
 *                     user's cached K/V and over no other candidate (mask rules (1)-(2),
 *                     PAPER.md:341; output rows I_NRO), softmax normalisation
 *                     (reading R1).
 *   gesr_hma_count    Hard Matching Attention raw match counts between each (candidate, field)
 *                     item ID list and the request's user ID list of the same field:
 *                     c = sum_i sum_j [u_i == t_j], optionally min(c, M)  (PAPER.md:308-312,
 *                     s3.4.1).
 *
 * One more entry point runs the same step for a batch in HOST memory (the serving host's end to
 * end path): gesr_score_host with its plan (gesr_host_plan_create / _destroy,
 * gesr_host_chunk_maxima) -- see the end of this header; the conventions below apply to the
 * device calls, and that section states where the host path differs (host pointers, device
 * allocation in the plan, host<->device copies).
 *
 * Serving from IDs (history and candidate IDs looked up in the shared embedding
 * table to obtain U and T): gesr_kv_project_gather and gesr_tasa_score_gather fuse the lookup
 * into the projections (the rows are never written to memory), and gesr_score_host_ids runs
 * the host path from row IDs with the table resident on the device.
 *
 * Conventions (all device calls):
 *   - Every array pointer is a DEVICE pointer owned by the caller; the library never frees or
 *     retains a pointer after the call returns.  bf16 arrays are IEEE bfloat16 bit patterns.
 *   - `stream` is a cudaStream_t (passed as void*; NULL = legacy default stream).  Calls are
 *     asynchronous on that stream: no host synchronisation, no device allocation, no
 *     host<->device copies; they are CUDA-graph capturable.  Safe to call concurrently from
 *     several threads on different streams.
 *   - The hot-path kernels are launched with programmatic stream serialisation (programmatic
 *     dependent launch): each may be scheduled while the previous kernel on `stream` still runs
 *     and waits for its completion before touching memory, so stream order holds for the
 *     caller's work before and after a call exactly as with plain launches.  The kernels allow
 *     their successor to be scheduled early; a caller's own PDL-launched kernel that follows a
 *     call must execute griddepcontrol.wait (cudaGridDependencySynchronize) before reading the
 *     call's outputs, as PDL requires of any such kernel.
 *   - Host-checkable argument errors return GESR_ERR_INVALID_ARG BEFORE any launch and write
 *     nothing; unsupported options return GESR_ERR_UNSUPPORTED; a too-small workspace returns
 *     GESR_ERR_WORKSPACE; a failed launch returns GESR_ERR_CUDA.  gesr_last_error() gives a
 *     thread-local message for the last non-OK return.
 *   - Offsets are NOT validated on the device by default: offsets[0] must be 0, offsets
 *     nondecreasing and offsets[B] equal to the stated total.  Malformed offsets are undefined
 *     behaviour.  With the environment variable GESR_DEBUG=1 (read once per process) every call
 *     that takes offsets first launches a checking kernel that traps (the stream then reports
 *     cudaErrorLaunchFailure / an illegal instruction) when seq_offsets, cand_offsets,
 *     user_offsets or item_offsets break these rules.
 *   - Empty problems (B = 0, total_C = 0, F = 0) are valid no-ops.
 */
#ifndef GESR_H_
#define GESR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GESR_OK = 0,
  GESR_ERR_INVALID_ARG = 1,
  GESR_ERR_UNSUPPORTED = 2,
  GESR_ERR_CUDA = 3,
  GESR_ERR_WORKSPACE = 4
} gesr_status;

/* Projection activation act(x) (reading R3; SPEC.md:343 uses SiLU). */
typedef enum { GESR_ACT_IDENTITY = 0, GESR_ACT_SILU = 1 } gesr_act;

/* Element type of the attention output O. */
typedef enum { GESR_OUT_F32 = 0, GESR_OUT_BF16 = 1 } gesr_out_dtype;

/* gesr_tasa_score flag, reserved: the candidate also attends to its own key (SPEC.md:277's
 * diagonal, reading R2).  Returns GESR_ERR_UNSUPPORTED in this version. */
#define GESR_TASA_SELF_KEY 0x1u
/* HSTU pointwise normalisation instead of the softmax (reading R20: the paper defers
 * to HSTU, whose attention is SiLU(scale q.k)/N, N = the number of keys):
 *   O[t][h] = sum_i SiLU(scale q_h . K[h][r_i]) V[h][r_i] / L_b   (L_b = 0 -> zeros)
 * gesr_tasa_score only; lse must be NULL; one key split (kv_splits 0 or 1). */
#define GESR_TASA_HSTU_SILU 0x2u

/* Library version (major*10000 + minor*100 + patch). */
int gesr_version(void);
const char* gesr_status_string(int status);
const char* gesr_last_error(void);
/* Number of kernels this library has launched in the process so far (all devices, all
 * threads).  Diagnostic: bench.py reports its difference over the timed region. */
unsigned long long gesr_launch_count(void);

/* gesr_kv_project -- K = act(U W_k^T + b_k), V = act(U W_v^T + b_v), split into heads.
 *   U        bf16 [total_L, D_in] row-major: all requests' history rows, request b owning rows
 *            [seq_offsets[b], seq_offsets[b+1]).  Rows are projected independently, so the
 *            offsets are not needed here; the cache keeps the same row order.
 *   D_in     multiple of 8, 8 <= D_in <= 16384.
 *   W_k, W_v bf16 [H*d, D_in] row-major (nn.Linear weight layout); head h = rows [h*d,(h+1)*d).
 *   b_k, b_v fp32 [H*d] or NULL (no bias).
 *   H, d     H >= 1, d in {32, 64, 128}.
 *   act      gesr_act.
 *   K_cache, V_cache  bf16 [H, total_L, d] (written): head-major, so each (request, head)
 *            owns one contiguous L_b x d slab -- the layout gesr_tasa_score's TMA loads read.
 *   Values are rounded to bf16 round-to-nearest-even from fp32 accumulation.
 *   Pointers must be 16-byte aligned.  total_L = 0 is a no-op. */
gesr_status gesr_kv_project(const void* U, int64_t total_L, int32_t D_in,
                            const void* W_k, const void* W_v,
                            const float* b_k, const float* b_v,
                            int32_t H, int32_t d, int32_t act,
                            void* K_cache, void* V_cache,
                            void* stream);

/* gesr_kv_project_gather -- gesr_kv_project with the history rows looked up in an embedding
 * table inside the projection: U[m] = E[rows[m]], K = act(U W_k^T + b_k), V = act(U W_v^T + b_v).
 * PAPER.md:407 (s4 serving): "MoA serving combines the item POST ID with the user history
 * sequence IDs ... looked up in the shared embedding table that was learnt during training to
 * obtain the input embeddings for the MoA module (U, T)"; the shared table.  The
 * looked-up rows are never written to memory: the projection's TMA producer gathers them
 * (tile::gather4, four table rows per load) straight into its 128B-swizzled operand tiles.
 *   E        bf16 [n_E, D_in] row-major embedding table, 1 <= n_E < 2^31.
 *   rows     int32 [total_L], 4-byte aligned: table row of each history row; repeats allowed.
 *            0 <= rows[m] < n_E is required and not checked (an out-of-range row is undefined
 *            behaviour).
 *   Everything else as gesr_kv_project; the result is bit-identical to gesr_kv_project on the
 *   materialised U = E[rows]. */
gesr_status gesr_kv_project_gather(const void* E, int64_t n_E, int32_t D_in, const int32_t* rows,
                                   int64_t total_L, const void* W_k, const void* W_v,
                                   const float* b_k, const float* b_v,
                                   int32_t H, int32_t d, int32_t act,
                                   void* K_cache, void* V_cache,
                                   void* stream);

/* Workspace bytes gesr_tasa_score needs for this problem (an upper bound that depends only on
 * the arguments, never on device data).  Returns 0 for invalid arguments. */
size_t gesr_tasa_workspace_bytes(int64_t B, int64_t total_C, int32_t H, int32_t d,
                                 int32_t kv_splits);

/* gesr_tasa_score -- candidate rows of target-aware self-attention over the cached history.
 *   T          bf16 [total_C, D_in]: candidate embeddings, request b owning rows
 *              [cand_offsets[b], cand_offsets[b+1]).
 *   cand_offsets int64 [B+1] (device).
 *   W_q, b_q, act  as in gesr_kv_project: q = act(T W_q^T + b_q), head h = cols [h*d,(h+1)*d).
 *   K_cache, V_cache  bf16 [H, total_L, d] from gesr_kv_project (any number of calls may reuse
 *              one cache, e.g. candidate chunks of the same users).
 *   seq_offsets int64 [B+1] (device) into the cache rows.
 *   scale      score scale; <= 0 selects 1/sqrt(d) (reading R4).
 *   kv_splits  split-L: each (256-candidate unit, head) is cut into kv_splits ranges of key
 *              tiles computed independently and merged (weights l_s 2^(m_s - max m), summed in
 *              split order) -- occupancy for few-request calls such as one user's candidate
 *              chunks (BASELINE config 4).  0 = auto (splits only when there are fewer than 74
 *              (unit, head) items; the choice depends on B, total_C, total_L, H, so results
 *              are NOT batch-invariant), 1 = unsplit, 2..64 forced.  Splits need d = 128 (the
 *              CTA-pair kernel): d < 128 with kv_splits > 1 returns GESR_ERR_UNSUPPORTED, auto
 *              runs unsplit.  For a fixed kv_splits >= 1 each output row depends only on its
 *              own candidate and its user's K/V: results are bit-identical across chunking,
 *              batch composition and GPU count (reading R9).  kv_splits > 64 is invalid.
 *   flags      0 or GESR_TASA_HSTU_SILU (above).  GESR_TASA_SELF_KEY needs the candidates'
 *              own keys / values: it returns
 *              GESR_ERR_UNSUPPORTED here; use gesr_tasa_score_self.
 *   O          [total_C, H*d] fp32 or bf16 (o_dtype): O[t][h*d+j] = sum_i p_i V[h][r_i][j] with
 *              p = softmax_i(scale * q_h . K[h][r_i]) over the request's L_b history rows.
 *              L_b = 0 gives an all-zero row (reading R6).
 *   lse        fp32 [total_C, H] natural-log log-sum-exp of the scaled scores, or NULL.
 *              L_b = 0 gives -inf.
 *   workspace  device scratch of at least gesr_tasa_workspace_bytes(...) bytes, 256-byte
 *              aligned; contents need not be initialised and are clobbered.
 *   Same alignment / D_in / H / d constraints as gesr_kv_project. */
gesr_status gesr_tasa_score(const void* T, int64_t total_C, int32_t D_in,
                            const int64_t* cand_offsets,
                            const void* W_q, const float* b_q, int32_t act,
                            const void* K_cache, const void* V_cache,
                            const int64_t* seq_offsets, int64_t B, int64_t total_L,
                            int32_t H, int32_t d, float scale,
                            int32_t kv_splits, uint32_t flags,
                            void* O, int32_t o_dtype,
                            float* lse,
                            void* workspace, size_t workspace_bytes,
                            void* stream);

/* gesr_tasa_score_gather -- gesr_tasa_score with the candidate rows looked up in the shared
 * embedding table inside the Q projection: T[t] = E[rows[t]] (the candidate POST
 * IDs looked up in the shared table to obtain T), as gesr_kv_project_gather does
 * for the history.  The looked-up rows are never written to memory (TMA tile::gather4 loads).
 *   E        bf16 [n_E, D_in] row-major table, 1 <= n_E < 2^31, 16-byte aligned.
 *   rows     int32 [total_C], 4-byte aligned; 0 <= rows[t] < n_E is required and not checked.
 * All other arguments, the workspace size and the error behaviour are those of
 * gesr_tasa_score (flag GESR_TASA_SELF_KEY -> GESR_ERR_UNSUPPORTED); the result is bit-identical
 * to gesr_tasa_score on the materialised T = E[rows]. */
gesr_status gesr_tasa_score_gather(const void* E, int64_t n_E, int32_t D_in, const int32_t* rows,
                                   int64_t total_C, const int64_t* cand_offsets,
                                   const void* W_q, const float* b_q, int32_t act,
                                   const void* K_cache, const void* V_cache,
                                   const int64_t* seq_offsets, int64_t B, int64_t total_L,
                                   int32_t H, int32_t d, float scale, int32_t kv_splits,
                                   uint32_t flags, void* O, int32_t o_dtype, float* lse,
                                   void* workspace, size_t workspace_bytes,
                                   void* stream);

/* gesr_tasa_score_self -- gesr_tasa_score with the candidate SELF KEY: each candidate also
 * attends to its own key (the diagonal SPEC.md's mask keeps; DESIGN.md
 * reading R2 -- SURVEY s8(f) f1, the first piece of the full STU candidate row):
 *   O[t][h] = (sum_i e^{s_i} V[h][r_i] + e^{s_t} V_self[h][t]) / (sum_i e^{s_i} + e^{s_t}),
 *   s_i = scale q_h . K[h][r_i],  s_t = scale q_h . K_self[h][t]
 * over the request's history rows r_i; lse includes s_t.  L_b = 0 gives O = V_self, lse = s_t.
 *   K_self, V_self  bf16 [H, total_C, d]: the candidates' own keys / values, i.e.
 *              gesr_kv_project applied to T (U := T, total_L := total_C) with W_k, W_v.
 * All other arguments, the workspace size and the error behaviour are those of
 * gesr_tasa_score; the merge runs after the history attention on the same stream. */
gesr_status gesr_tasa_score_self(const void* T, int64_t total_C, int32_t D_in,
                                 const int64_t* cand_offsets,
                                 const void* W_q, const float* b_q, int32_t act,
                                 const void* K_cache, const void* V_cache,
                                 const int64_t* seq_offsets, int64_t B, int64_t total_L,
                                 int32_t H, int32_t d, float scale, int32_t kv_splits,
                                 const void* K_self, const void* V_self,
                                 void* O, int32_t o_dtype, float* lse,
                                 void* workspace, size_t workspace_bytes,
                                 void* stream);

/* gesr_stu_output -- the rest of the STU layer's candidate row after the attention (SURVEY
 * s8(f) f1; "layer output = output-projection(normalize(attention.value) (.)
 * gating-branch) + residual", the paper deferring STU internals to HSTU, PAPER.md:229;
 * DESIGN.md reading R15).  For every candidate row t (D = H*d):
 *   G[t]  = SiLU(T[t] W_g^T + b_g)                                  gating branch, [D]
 *   N[t]  = (O[t] - mean(O[t])) / sqrt(var(O[t]) + ln_eps) * ln_gamma + ln_beta
 *           (mean and population variance over the D features of the concatenated heads)
 *   Y[t]  = (N[t] (.) G[t]) W_o^T + b_o + X_res[t]
 *   T          bf16 [total_C, D_in]: the candidate rows the gating branch projects (the same
 *              normalised rows gesr_tasa_score projects to queries).
 *   O          [total_C, D] fp32 or bf16 (o_dtype): attention.value from gesr_tasa_score.
 *   W_g        bf16 [D, D_in] (nn.Linear layout); b_g fp32 [D] or NULL.
 *   ln_gamma, ln_beta  fp32 [D]; ln_eps >= 0 and finite.
 *   W_o        bf16 [D_out, D]; b_o fp32 [D_out] or NULL.
 *   X_res      bf16 [total_C, D_out] residual (the layer input), or NULL (no residual).
 *   D_out      a multiple of 32 in [32, 16384]; H*d a multiple of 32 and <= 16384.
 *   Y          bf16 [total_C, D_out] (written).
 *   workspace  device scratch of >= gesr_stu_workspace_bytes(total_C, H, d) bytes (G, then
 *              the normalised, gated rows in place); clobbered.
 * Precision: bf16 operands, fp32 accumulation and normalisation statistics, G and N(.)G rounded
 * to bf16 (RNE) before the output projection, Y rounded to bf16.  Rows are independent
 * (bit-identical for any batch composition).  Alignment: every pointer 16-byte aligned.
 * Errors as the other calls; total_C = 0 is a no-op. */
size_t gesr_stu_workspace_bytes(int64_t total_C, int32_t H, int32_t d);
gesr_status gesr_stu_output(const void* T, int64_t total_C, int32_t D_in,
                            const void* O, int32_t o_dtype,
                            const void* W_g, const float* b_g,
                            const float* ln_gamma, const float* ln_beta, float ln_eps,
                            const void* W_o, const float* b_o, const void* X_res,
                            int32_t H, int32_t d, int32_t D_out,
                            void* Y, void* workspace, size_t workspace_bytes,
                            void* stream);

/* gesr_nro_cross_score -- NRO cross attention (PAPER.md:373-380 s3.4.3 "each
 * query is paired with an independent attention mechanism, specialized via separate weight
 * matrices for query-modulation versus key-value relationships ... The resulting individual
 * outputs are concatenated to form T_cross"; reading R16).  Each of
 * the j query slots s gates the candidate query input elementwise, projects it with its own
 * query weight and attends over the request's RO (history) rows with its own key/value
 * projections:
 *   q_s = act((x (.) g_s) W_{Q,s}^T + b_{Q,s}),  O[t][s*d + i] = sum_r p_r V_s[r][i],
 *   p = softmax_r(scale q_s . K_s[r]) over the request's L_b history rows.
 *   T          bf16 [total_C, D_in]: the query inputs x (candidate embeddings, optionally
 *              enriched by the caller).
 *   W_q        bf16 [j*d, D_in]: slot s's query weight is rows [s*d, (s+1)*d).
 *   q_gate     fp32 [j, D_in]: the slots' elementwise query gates g_s.
 *   b_q        fp32 [j*d] or NULL.
 *   K_cache, V_cache  bf16 [j, total_L, d]: gesr_kv_project of the history with the slots' key
 *              / value weights stacked as heads (H := j).
 *   O          [total_C, j*d] fp32 or bf16: T_cross, the slots concatenated in slot order.
 *   workspace  >= gesr_nro_workspace_bytes(B, total_C, j, d, D_in, kv_splits) bytes,
 *              256-byte aligned.
 * The gate is folded into the query weight on the device (W'[s*d+i][k] = W_q[s*d+i][k] g_s[k],
 * rounded to bf16), then the call runs gesr_tasa_score's path with H = j; every other argument,
 * the tolerance and the error behaviour are gesr_tasa_score's (flags = 0). */
size_t gesr_nro_workspace_bytes(int64_t B, int64_t total_C, int32_t j, int32_t d, int32_t D_in,
                                int32_t kv_splits);
gesr_status gesr_nro_cross_score(const void* T, int64_t total_C, int32_t D_in,
                                 const int64_t* cand_offsets,
                                 const void* W_q, const float* q_gate, const float* b_q,
                                 int32_t act, const void* K_cache, const void* V_cache,
                                 const int64_t* seq_offsets, int64_t B, int64_t total_L,
                                 int32_t j, int32_t d, float scale, int32_t kv_splits,
                                 void* O, int32_t o_dtype, float* lse,
                                 void* workspace, size_t workspace_bytes,
                                 void* stream);

/* gesr_history_attention -- causal self-attention of every user's history over itself (SURVEY
 * s8(f) f4: the U rows of one [U, T] layer, PAPER.md:341 mask rule (1) "user embeddings in U
 * will not attend to future positions"; "user block lower-triangular", diagonal
 * included; reading R17).  For history row r = seq_offsets[b] + p of request b and head
 * h:
 *   q = act(U[r] W_q^T + b_q)[h*d:(h+1)*d],
 *   O[r][h*d + j] = sum_{i <= p} w_i V[h][seq_offsets[b] + i][j] / sum_{i <= p} w_i,
 *   w_i = exp(scale q . K[h][seq_offsets[b] + i] - max).
 *   U          bf16 [total_L, D_in]: the layer's (normalised) history rows.
 *   K_cache, V_cache  bf16 [H, total_L, d]: gesr_kv_project of the same U -- the cache the
 *              layer's candidates then attend to with gesr_tasa_score.
 *   O          [total_L, H*d] fp32 or bf16; lse fp32 [total_L, H] or NULL.
 *   workspace  >= gesr_tasa_workspace_bytes(B, total_L, H, d, 1) bytes, 256-byte aligned.
 * Arguments, tolerance and errors as gesr_tasa_score with T := U, cand_offsets := seq_offsets,
 * one key split (batch-invariant). */
gesr_status gesr_history_attention(const void* U, int64_t total_L, int32_t D_in,
                                   const int64_t* seq_offsets, int64_t B,
                                   const void* W_q, const float* b_q, int32_t act,
                                   const void* K_cache, const void* V_cache,
                                   int32_t H, int32_t d, float scale,
                                   void* O, int32_t o_dtype, float* lse,
                                   void* workspace, size_t workspace_bytes,
                                   void* stream);

/* gesr_layer_norm -- the STU layer's input normalisation ("per layer -- normalize
 * input"; reading R18): for every row r of X,
 *   Y[r] = (X[r] - mean(X[r])) / sqrt(var(X[r]) + eps) * gamma + beta
 * (population variance over the D features, fp32 statistics).
 *   X, Y       bf16 [rows, D] (Y may alias X); D a multiple of 8 in [8, 16384].
 *   gamma, beta  fp32 [D]; eps >= 0 and finite.  16-byte aligned pointers.
 * With gesr_kv_project, gesr_history_attention, gesr_tasa_score_self and gesr_stu_output it
 * composes one full target-aware STU layer over [U, T] (binding.stu_layer). */
gesr_status gesr_layer_norm(const void* X, int64_t rows, int32_t D, const float* gamma,
                            const float* beta, float eps, void* Y, void* stream);

/* gesr_ro_cross_score -- RO cross attention (PAPER.md:362-370 s3.4.3 "its query is a set of
 * learnable seeds, optionally enriched with customised RO tokens ... Each query attends
 * independently to user signals, and the results are concatenated to yield U_cross"; SPEC.md
 * 309-315; reading R19).  Per request b and seed s of the i seeds:
 *   q_s = act((seeds[s] + ctx[b][s]) W_{Q,s}^T + b_{Q,s}),
 *   U_cross[b][s*d + j] = sum_r p_r V_s[r][j],  p = softmax_r(scale q_s . K_s[r])
 * over the request's history rows (keys and values RO only, the prose reading of SPEC.md:358).
 *   seeds      bf16 [i, D_in]; ctx bf16 [B, i, D_in] context tokens or NULL.
 *   W_q        bf16 [i*d, D_in]: seed s's query weight is rows [s*d, (s+1)*d); b_q fp32 or NULL.
 *   K_cache, V_cache  bf16 [i, total_L, d]: gesr_kv_project of the history with the seeds' key
 *              / value weights stacked as heads (H := i).
 *   U_cross    [B, i*d] fp32 or bf16 (o_dtype); a request without history gives zeros.
 *   workspace  >= gesr_ro_workspace_bytes(B, i, d, D_in) bytes, 256-byte aligned.
 * U_cross is per request (RO): a caller expands it to the request's candidates by indexing
 * (SPEC.md:325 expand_ro).  Same tolerance and errors as gesr_tasa_score. */
size_t gesr_ro_workspace_bytes(int64_t B, int32_t i, int32_t d, int32_t D_in);
gesr_status gesr_ro_cross_score(const void* seeds, const void* ctx, int32_t i, int32_t D_in,
                                const void* W_q, const float* b_q, int32_t act,
                                const void* K_cache, const void* V_cache,
                                const int64_t* seq_offsets, int64_t B, int64_t total_L,
                                int32_t d, float scale, void* U_cross, int32_t o_dtype,
                                void* workspace, size_t workspace_bytes, void* stream);

/* gesr_hma_count -- HMA per-field match counts.
 *   user_ids / user_offsets  int64 CSR: segment b*F+f is request b's user-side ID list of
 *              field f; user_offsets has B*F+1 entries.
 *   item_ids / item_offsets  int64 CSR: segment t*F+f is candidate t's item-side ID list of
 *              field f (a single ID in the paper -- a length-1 list; reading R10);
 *              item_offsets has total_C*F+1 entries.
 *   cand_offsets int64 [B+1]: candidate t belongs to request b iff
 *              cand_offsets[b] <= t < cand_offsets[b+1].
 *   cap        <= 0: raw pairwise counts; > 0: min(count, cap)  (PAPER.md:310 cap M).
 *   counts     int32 [total_C, F] (written): counts[t*F+f] = sum_i sum_j [u_i == t_j]
 *              (pairwise; reading R11), IDs compared as int64 within the same field only.
 *   Exact integer arithmetic: bit-identical to any correct implementation.
 *   user lists of any length are supported (long lists take a slower global-memory path). */
gesr_status gesr_hma_count(const int64_t* user_ids, const int64_t* user_offsets,
                           const int64_t* item_ids, const int64_t* item_offsets,
                           const int64_t* cand_offsets, int64_t B, int64_t total_C, int32_t F,
                           int32_t cap, int32_t* counts,
                           void* stream);

/* gesr_hma_count_embed -- gesr_hma_count fused with the HMA offset-embedding lookup
 * (PAPER.md:314-318 s3.4.1 "e = E(c + o*M)"): for candidate t and field
 * (feature pair) f, with c = min(count, M),
 *   emb[t][f*D_h .. (f+1)*D_h) = E[c + f*(M+1)][0 .. D_h)
 * i.e. Concat(e_1, ..., e_F), the input of T_match = MLP(Concat(...)) (the MLP is
 * a dense layer outside this call).  The row stride is M+1, not the paper's literal M: c takes
 * M+1 values 0..M, so stride M would make c = M of pair f collide with c = 0 of pair f+1
 * (reading R14).
 *   M          cap, >= 1 (the offset needs a bounded count).
 *   counts     int32 [total_C, F] capped counts (written, as gesr_hma_count with cap = M).
 *   E          bf16 [F*(M+1), D_h] embedding table; D_h a multiple of 8 in [8, 4096].
 *   emb        bf16 [total_C, F*D_h] (written).  E and emb 16-byte aligned.
 * Bit-exact (a gather of table rows).  Other arguments and errors as gesr_hma_count. */
gesr_status gesr_hma_count_embed(const int64_t* user_ids, const int64_t* user_offsets,
                                 const int64_t* item_ids, const int64_t* item_offsets,
                                 const int64_t* cand_offsets, int64_t B, int64_t total_C,
                                 int32_t F, int32_t M, int32_t* counts,
                                 const void* E, int32_t D_h, void* emb,
                                 void* stream);

/* ---------------------------------------------------------------- end to end from HOST memory
 * One whole scoring step -- gesr_kv_project -> gesr_tasa_score -> gesr_hma_count, exactly the
 * device-resident step -- for a batch whose inputs are in HOST memory, with the results written
 * to HOST memory (the e2e path of a serving host).  The requests are cut into n_chunks
 * contiguous ranges (chunk k = requests [B*k/n_chunks, B*(k+1)/n_chunks)); per chunk the inputs
 * are copied host->device, the three calls run on `stream`, and O / counts are copied
 * device->host, pipelined over two device buffer sets and two internal copy streams (while the
 * kernels of chunk k run, chunk k+1 is copied in and chunk k-1 out).  Each chunk's offsets are
 * rebased on the device (the caller's host buffers are never written).  Results are
 * bit-identical to the device-resident step (rows depend only on their own request: reading R9;
 * split-L auto as in gesr_tasa_score).
 *
 * gesr_host_chunk_maxima -- per-chunk maxima {requests, history rows, candidate rows, user IDs,
 *   item IDs} of that cut (host offsets; the sizes gesr_host_plan_create needs).
 * gesr_host_plan_create -- allocates the two device buffer sets (sized by `maxima`), their
 *   workspaces, events and the copy streams on the current device; *plan is owned by the caller
 *   and released with gesr_host_plan_destroy (after all work using it has completed).
 * gesr_score_host -- enqueues one step:
 *   U [total_L, D_in] / T [total_C, D_in] bf16, HOST (pinned for asynchronous DMA; pageable
 *   memory works but the copies then serialise with the host); seq_offsets / cand_offsets
 *   [B+1], user_offsets [B*F+1], item_offsets [total_C*F+1], user_ids, item_ids: int64 HOST;
 *   W_q [H*d, D_in], W_k / W_v [H*d, D_in] bf16 DEVICE (model weights, resident); act as
 *   gesr_kv_project; scale 1/sqrt(d); cap as gesr_hma_count; O [total_C, H*d] (o_dtype of the
 *   plan) and counts int32 [total_C, F]: HOST (written).  Asynchronous: ordered after prior work
 *   on `stream`; O / counts are complete when `stream` reaches the point after this call.
 *   GESR_ERR_WORKSPACE if a chunk exceeds the plan's maxima (checked before anything is
 *   enqueued).  A plan serves one call at a time (not thread-safe) on the device it was created
 *   on; after an error returned mid-way (GESR_ERR_CUDA), synchronise the device before reusing or
 *   destroying the plan. */
typedef struct gesr_host_plan gesr_host_plan;
gesr_status gesr_host_chunk_maxima(const int64_t* seq_offsets, const int64_t* cand_offsets,
                                   const int64_t* user_offsets, const int64_t* item_offsets,
                                   int64_t B, int32_t F, int32_t n_chunks, int64_t* maxima);
gesr_status gesr_host_plan_create(const int64_t* maxima, int32_t D_in, int32_t H, int32_t d,
                                  int32_t F, int32_t o_dtype, gesr_host_plan** plan);
gesr_status gesr_host_plan_destroy(gesr_host_plan* plan);
gesr_status gesr_score_host(gesr_host_plan* plan, int32_t n_chunks,
                            const void* U, const int64_t* seq_offsets,
                            const void* T, const int64_t* cand_offsets, int64_t B,
                            const void* W_q, const void* W_k, const void* W_v, int32_t act,
                            const int64_t* user_ids, const int64_t* user_offsets,
                            const int64_t* item_ids, const int64_t* item_offsets, int32_t cap,
                            void* O, int32_t* counts, void* stream);

/* gesr_score_host_ids -- gesr_score_host for the serving form PAPER.md:407 describes: the host
 * holds IDs, not embeddings ("MoA serving combines the item POST ID with the user history
 * sequence IDs ... looked up in the shared embedding table ... to obtain the input embeddings
 * U, T").  The table stays resident on the device; per chunk only the int32 row ids (with the
 * HMA lists and offsets) cross PCIe, and the projections gather the rows
 * (gesr_kv_project_gather, gesr_tasa_score_gather).
 *   E          DEVICE bf16 [n_E, D_in] embedding table (plan's D_in), 1 <= n_E < 2^31.
 *   hist_rows  HOST int32 [seq_offsets[B]]: table row of each history row (replaces U).
 *   cand_rows  HOST int32 [cand_offsets[B]]: table row of each candidate (replaces T).
 * Everything else, the plan and the error behaviour as gesr_score_host; the results equal
 * gesr_score_host's on U = E[hist_rows], T = E[cand_rows] bit for bit. */
gesr_status gesr_score_host_ids(gesr_host_plan* plan, int32_t n_chunks,
                                const void* E, int64_t n_E,
                                const int32_t* hist_rows, const int64_t* seq_offsets,
                                const int32_t* cand_rows, const int64_t* cand_offsets, int64_t B,
                                const void* W_q, const void* W_k, const void* W_v, int32_t act,
                                const int64_t* user_ids, const int64_t* user_offsets,
                                const int64_t* item_ids, const int64_t* item_offsets, int32_t cap,
                                void* O, int32_t* counts, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GESR_H_ */
