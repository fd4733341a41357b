"""fp64 CPU oracle for the GESR MoA candidate-scoring hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2511_21095_b200``) never imports it, and this package never imports the product
path: the two share no code.  Inputs come from ``paper_2511_21095_b200.inputs`` (seeded
generators holding none of the method's arithmetic) or from the tests themselves.

Every function wraps one entry point of ``oracle/oracle.cpp`` (plain C++17, fp64, no
blocking/fusion), each citing the passage it follows:

* :func:`kv_project`  -- K/V = act(U W^T + b) per head. PAPER.md:335-341 (s3.4.2).
* :func:`kv_project_gather` -- the same with the history rows looked up in the shared
  embedding table first, U = E[rows].  PAPER.md:407 (s4 serving: history sequence IDs looked up
  in the shared embedding table to obtain U).
* :func:`tasa_score`  -- candidate rows of the target-aware masked softmax attention over the
  request's history.  PAPER.md:341, 346 (s3.4.2).
* :func:`full_masked_attention` -- brute force over the full (L+C)^2 mask.  SPEC.md:289-297.
* :func:`build_mask` -- the mask itself.  PAPER.md:341.
* :func:`hma_count` / :func:`hma_count_hash` -- HMA raw (optionally capped) match counts, two
  independent algorithms.  PAPER.md:308-312 (s3.4.1).
* :func:`offset_index` / :func:`hma_offset_embed` -- HMA embedding with feature-pair offsets,
  e = E(c + o(M+1)), concatenated over pairs.
  (stride M+1: DESIGN.md reading R14).  Plain numpy.
* :func:`nro_cross_attention` -- NRO cross attention: j query slots, each gating the candidate
  query input elementwise and attending over the request's RO rows with its own projections,
  concatenated.  PAPER.md:373-380 (s3.4.3); SPEC.md:316-324 (reading R16).  Numpy.
* :func:`history_attention` -- causal self-attention of each user's history over itself (the U
  rows of one [U, T] layer: mask rule (1); SPEC.md:277 user block lower-
  triangular; reading R17).  Numpy.
* :func:`ro_cross_attention` -- RO cross attention: i learnable seeds (optionally plus per-request
  context tokens) attend over the request's history with per-seed projections, concatenated.
  PAPER.md:362-370 (s3.4.3); SPEC.md:309-315 (reading R19).  Numpy.
* :func:`tasa_score_hstu` -- target-aware attention with HSTU's pointwise normalisation
  SiLU(scale q.k)/N instead of the softmax (A1's alternative reading, R20).  Numpy.
* :func:`stu_stack_forward` -- a stack of full target-aware STU layers over [U, T] per request
  (SPEC.md:298 self_attention_forward, SPEC.md:343 layer internals, mask SPEC.md:277 with the
  candidate diagonal; reading R18), brute force over the (N+n)^2 mask.  Numpy.
* :func:`stu_output` -- the rest of the STU layer's candidate row after the attention (SURVEY
  s8(f) f1): gating branch, normalisation of attention.value, output projection, residual.
  SPEC.md:343 (PAPER.md:229 defers the STU internals to HSTU); reading R15.  Plain
  numpy, fp64.

Parity pins: see tests/test_oracle_*.py.  Every function here is pinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_u16p = ctypes.POINTER(ctypes.c_uint16)
_c_f64p = ctypes.POINTER(ctypes.c_double)
_c_i32p = ctypes.POINTER(ctypes.c_int32)
_c_u8p = ctypes.POINTER(ctypes.c_uint8)


def build() -> str:
    """Compile liboracle.so (g++ -O2, no fast-math: no reassociation)."""
    src = os.path.join(_HERE, "oracle.cpp")
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-o", _LIB_PATH, src]
    subprocess.check_call(cmd)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    src = os.path.join(_HERE, "oracle.cpp")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    lib.oracle_kv_project.argtypes = [_c_u16p, ctypes.c_int64, ctypes.c_int32, _c_u16p, _c_u16p,
                                      _c_f64p, _c_f64p, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int32, _c_f64p, _c_f64p, ctypes.c_int32]
    lib.oracle_tasa_score.argtypes = [_c_u16p, ctypes.c_int64, ctypes.c_int32, _c_i64p, _c_u16p,
                                      _c_f64p, ctypes.c_int32, _c_f64p, _c_f64p, _c_i64p,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_double, ctypes.c_int32, _c_f64p,
                                      _c_f64p, ctypes.c_int32]
    lib.oracle_build_mask.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, _c_u8p]
    lib.oracle_full_masked_attention.argtypes = [
        _c_u16p, ctypes.c_int64, _c_u16p, ctypes.c_int64, ctypes.c_int32, _c_u16p, _c_u16p,
        _c_u16p, _c_f64p, _c_f64p, _c_f64p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
        ctypes.c_double, ctypes.c_int32, _c_f64p, _c_f64p]
    lib.oracle_hma_count.argtypes = [_c_i64p, _c_i64p, _c_i64p, _c_i64p, _c_i64p, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _c_i32p,
                                     ctypes.c_int32]
    lib.oracle_hma_count_hash.argtypes = [_c_i64p, _c_i64p, _c_i64p, _c_i64p, _c_i64p,
                                          ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                          ctypes.c_int32, _c_i32p]
    lib.oracle_round_to_bf16.argtypes = [_c_f64p, ctypes.c_int64]
    _lib = lib
    return lib


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


# ---------------------------------------------------------------------------------------------
# marshalling helpers (argument conversion only)

def _bits(x) -> np.ndarray:
    """bf16 tensor/array -> contiguous uint16 bit array."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            assert x.dtype == torch.bfloat16, x.dtype
            return np.ascontiguousarray(x.detach().cpu().contiguous().view(torch.int16).numpy()
                                        .view(np.uint16))
    except ImportError:  # pragma: no cover
        pass
    a = np.asarray(x)
    assert a.dtype == np.uint16, a.dtype
    return np.ascontiguousarray(a)


def _np(x, dtype) -> np.ndarray:
    try:
        import torch
        if isinstance(x, torch.Tensor):
            x = x.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(np.asarray(x, dtype=dtype))


def _p(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctype)


def _opt_f64(b):
    if b is None:
        return None, None
    a = _np(b, np.float64)
    return a, _p(a, _c_f64p)


# ---------------------------------------------------------------------------------------------

def kv_project(U, W_k, W_v, H, d, act=1, b_k=None, b_v=None, threads=None):
    """K, V fp64 [H, total_L, d] = act(U W^T + b) split into heads."""
    lib = _load()
    Ub, Wk, Wv = _bits(U), _bits(W_k), _bits(W_v)
    total_L, D_in = Ub.shape
    assert Wk.shape == (H * d, D_in) and Wv.shape == (H * d, D_in)
    K = np.zeros((H, total_L, d), np.float64)
    V = np.zeros((H, total_L, d), np.float64)
    bk, pbk = _opt_f64(b_k)
    bv, pbv = _opt_f64(b_v)
    lib.oracle_kv_project(_p(Ub, _c_u16p), total_L, D_in, _p(Wk, _c_u16p), _p(Wv, _c_u16p),
                          pbk, pbv, H, d, act, _p(K, _c_f64p), _p(V, _c_f64p),
                          threads or default_threads())
    return K, V


def kv_project_gather(E, rows, W_k, W_v, H, d, act=1, b_k=None, b_v=None, threads=None):
    """K, V fp64 [H, len(rows), d] = act(E[rows] W^T + b): the lookup of the history IDs in the
    shared embedding table, then :func:`kv_project`."""
    import torch
    E = E if isinstance(E, torch.Tensor) else torch.as_tensor(E)
    idx = torch.as_tensor(np.asarray(rows, dtype=np.int64))
    assert idx.numel() == 0 or (int(idx.min()) >= 0 and int(idx.max()) < E.shape[0])
    U = E.index_select(0, idx)          # step 1: the table lookup (a library gather)
    return kv_project(U, W_k, W_v, H, d, act=act, b_k=b_k, b_v=b_v, threads=threads)


def tasa_score(T, cand_offsets, W_q, K, V, seq_offsets, H, d, act=1, b_q=None, scale=None,
               round_q_bf16=False, threads=None):
    """O fp64 [total_C, H*d], lse fp64 [total_C, H]: each candidate's masked softmax attention
    over its request's cached history K/V.  scale None -> 1/sqrt(d)."""
    lib = _load()
    Tb, Wq = _bits(T), _bits(W_q)
    total_C, D_in = Tb.shape
    co = _np(cand_offsets, np.int64)
    so = _np(seq_offsets, np.int64)
    B = co.shape[0] - 1
    assert so.shape[0] == B + 1
    Kd = _np(K, np.float64)
    Vd = _np(V, np.float64)
    total_L = Kd.shape[1]
    assert Kd.shape == (H, total_L, d) and Vd.shape == (H, total_L, d)
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    O = np.zeros((total_C, H * d), np.float64)
    lse = np.zeros((total_C, H), np.float64)
    bq, pbq = _opt_f64(b_q)
    lib.oracle_tasa_score(_p(Tb, _c_u16p), total_C, D_in, _p(co, _c_i64p), _p(Wq, _c_u16p), pbq,
                          act, _p(Kd, _c_f64p), _p(Vd, _c_f64p), _p(so, _c_i64p), B, total_L, H,
                          d, float(scale), int(bool(round_q_bf16)), _p(O, _c_f64p),
                          _p(lse, _c_f64p), threads or default_threads())
    return O, lse


def round_to_bf16(x) -> np.ndarray:
    """Diagnostic only: round fp64 values to the nearest bf16 (RNE), returned as fp64."""
    lib = _load()
    a = np.array(x, dtype=np.float64, copy=True, order="C")
    lib.oracle_round_to_bf16(_p(a, _c_f64p), a.size)
    return a


def build_mask(N, n, self_key=False) -> np.ndarray:
    """(N+n)x(N+n) uint8 target-aware mask."""
    lib = _load()
    m = np.zeros((N + n, N + n), np.uint8)
    lib.oracle_build_mask(N, n, int(bool(self_key)), _p(m, _c_u8p))
    return m


def full_masked_attention(U, T, W_q, W_k, W_v, H, d, act=1, b_q=None, b_k=None, b_v=None,
                          scale=None, self_key=False):
    """Brute force for ONE request: candidate rows of masked attention over [U;T]."""
    lib = _load()
    Ub, Tb = _bits(U), _bits(T)
    L, D_in = Ub.shape if Ub.size else (0, _bits(T).shape[1])
    C = Tb.shape[0]
    if Ub.size == 0:
        Ub = np.zeros((1, D_in), np.uint16)
    Wq, Wk, Wv = _bits(W_q), _bits(W_k), _bits(W_v)
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    O = np.zeros((C, H * d), np.float64)
    lse = np.zeros((C, H), np.float64)
    bq, pbq = _opt_f64(b_q)
    bk, pbk = _opt_f64(b_k)
    bv, pbv = _opt_f64(b_v)
    lib.oracle_full_masked_attention(_p(Ub, _c_u16p), L, _p(Tb, _c_u16p), C, D_in,
                                     _p(Wq, _c_u16p), _p(Wk, _c_u16p), _p(Wv, _c_u16p), pbq, pbk,
                                     pbv, H, d, act, float(scale), int(bool(self_key)),
                                     _p(O, _c_f64p), _p(lse, _c_f64p))
    return O, lse


def _hma_args(user_ids, user_offsets, item_ids, item_offsets, cand_offsets):
    ui = _np(user_ids, np.int64)
    uo = _np(user_offsets, np.int64)
    ii = _np(item_ids, np.int64)
    io = _np(item_offsets, np.int64)
    co = _np(cand_offsets, np.int64)
    if ui.size == 0:
        ui = np.zeros(1, np.int64)
    if ii.size == 0:
        ii = np.zeros(1, np.int64)
    return ui, uo, ii, io, co


def hma_count(user_ids, user_offsets, item_ids, item_offsets, cand_offsets, F, cap=0,
              threads=None) -> np.ndarray:
    """int32 [total_C, F] pairwise match counts, optionally capped."""
    lib = _load()
    ui, uo, ii, io, co = _hma_args(user_ids, user_offsets, item_ids, item_offsets, cand_offsets)
    B = co.shape[0] - 1
    total_C = int(co[-1]) if B >= 0 and co.size else 0
    counts = np.zeros((max(total_C, 0), F), np.int32)
    if total_C == 0 or F == 0:
        return counts
    lib.oracle_hma_count(_p(ui, _c_i64p), _p(uo, _c_i64p), _p(ii, _c_i64p), _p(io, _c_i64p),
                         _p(co, _c_i64p), B, total_C, F, cap, _p(counts, _c_i32p),
                         threads or default_threads())
    return counts


def hma_count_hash(user_ids, user_offsets, item_ids, item_offsets, cand_offsets, F,
                   cap=0) -> np.ndarray:
    """Second, independent algorithm (multiplicity map) for the same counts."""
    lib = _load()
    ui, uo, ii, io, co = _hma_args(user_ids, user_offsets, item_ids, item_offsets, cand_offsets)
    B = co.shape[0] - 1
    total_C = int(co[-1]) if co.size else 0
    counts = np.zeros((max(total_C, 0), F), np.int32)
    if total_C == 0 or F == 0:
        return counts
    lib.oracle_hma_count_hash(_p(ui, _c_i64p), _p(uo, _c_i64p), _p(ii, _c_i64p),
                              _p(io, _c_i64p), _p(co, _c_i64p), B, total_C, F, cap,
                              _p(counts, _c_i32p))
    return counts


def offset_index(c: int, o: int, M: int) -> int:
    """Row of the offset-encoded embedding table for count c of feature pair o.

    PAPER.md:314-316 writes e = E(c + o*M); c = min(count, M) takes the M+1 values 0..M, so the
    stride is M+1 (reading R14): rows of distinct pairs never collide.
    """
    if not (0 <= c <= M):
        raise ValueError(f"count {c} outside [0, {M}]")
    return c + o * (M + 1)


def hma_offset_embed(counts, E, M: int) -> np.ndarray:
    """Concat(e_1, ..., e_F) per candidate: [total_C, F*D_h] from capped
    counts [total_C, F] and the table E [F*(M+1), D_h], one lookup per (candidate, pair)."""
    counts = np.asarray(counts)
    E = np.asarray(E)
    total_C, F = counts.shape
    D_h = E.shape[1]
    assert E.shape[0] == F * (M + 1)
    out = np.zeros((total_C, F * D_h), E.dtype)
    for t in range(total_C):
        for o in range(F):
            out[t, o * D_h:(o + 1) * D_h] = E[offset_index(int(counts[t, o]), o, M)]
    return out



def _f64(x) -> np.ndarray:
    """bf16 / fp32 / fp64 tensor or array -> fp64 numpy array (bf16 widened exactly)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().cpu().to(torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    a = np.asarray(x)
    if a.dtype == np.uint16:                       # raw bf16 bits
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def stu_output(T, O, W_g, gamma, beta, W_o, b_g=None, b_o=None, X_res=None, eps=1e-5, act=1,
               round_bf16=False, parts=False):
    """Candidate rows of one STU layer after the attention, in SPEC.md:343's order (the paper
    defers STU internals to HSTU; reading R15):

      gating branch     G = act(T W_g^T + b_g)               ("a gating branch by linear
                                                               projection with sigmoid-linear-
                                                               unit activation")
      normalisation     N = (O - mean(O)) / sqrt(var(O) + eps) * gamma + beta, per row over the
                        D = H*d features of the concatenated heads (population variance)
      layer output      Y = (N * G) W_o^T + b_o + X_res      ("output-projection(normalize(
                                                               attention.value) (.) gating-
                                                               branch) + residual")

    T [C, D_in], O [C, D] (attention.value, heads concatenated), W_g [D, D_in],
    gamma/beta [D], W_o [D_out, D], b_g [D] / b_o [D_out] / X_res [C, D_out] optional.
    Returns Y fp64 [C, D_out].  act: 1 = SiLU x/(1+e^-x), 0 = identity.
    Diagnostic only (not the parity reference): ``round_bf16`` rounds G, N*G and Y to bf16
    (RNE) where the GPU path stores them, separating kernel bugs from quantisation; ``parts``
    also returns (N, G).
    """
    T, O, W_g, W_o = _f64(T), _f64(O), _f64(W_g), _f64(W_o)
    gamma, beta = _f64(gamma), _f64(beta)
    Z = T @ W_g.T
    if b_g is not None:
        Z = Z + _f64(b_g)[None, :]
    G = Z / (1.0 + np.exp(-Z)) if act == 1 else Z
    if round_bf16:
        G = round_to_bf16(G)
    mean = O.mean(axis=1, keepdims=True)
    var = ((O - mean) ** 2).mean(axis=1, keepdims=True)
    N = (O - mean) / np.sqrt(var + eps) * gamma[None, :] + beta[None, :]
    NG = N * G
    if round_bf16:
        NG = round_to_bf16(NG)
    Y = NG @ W_o.T
    if b_o is not None:
        Y = Y + _f64(b_o)[None, :]
    if X_res is not None:
        Y = Y + _f64(X_res)
    if round_bf16:
        Y = round_to_bf16(Y)
    return (Y, N, G) if parts else Y


def nro_cross_attention(T, cand_offsets, W_q, q_gate, U, seq_offsets, W_k, W_v, j, d, act=1,
                        b_q=None, b_k=None, b_v=None, scale=None):
    """T_cross = Concat_s Attn_nro(Q_s, RO, RO) (s3.4.3; SPEC.md:316-324;
    DESIGN.md reading R16), in the paper's order, slot by slot:

      gate        x_s = x (.) g_s                   (elementwise query gate, "query-modulation")
      query       q_s = act(x_s W_{Q,s}^T + b_{Q,s})                 W_q rows [s d, (s+1) d)
      key/value   K_s = act(U W_{K,s}^T + b_{K,s}),  V_s = act(U W_{V,s}^T + b_{V,s})  (RO rows)
      attention   O_s = softmax(scale q_s K_s^T) V_s over the candidate's request's history rows
      concat      T_cross[t] = [O_0[t], ..., O_{j-1}[t]]

    T [total_C, D_in], U [total_L, D_in], W_q/W_k/W_v [j d, D_in], q_gate [j, D_in],
    offsets int64 [B+1].  Returns fp64 [total_C, j d]; a request with no history rows gives
    zero rows (reading R6).  scale defaults to 1/sqrt(d).
    """
    T, U = _f64(T), _f64(U)
    Wq, Wk, Wv, g = _f64(W_q), _f64(W_k), _f64(W_v), _f64(q_gate)
    co, so = _np(cand_offsets, np.int64), _np(seq_offsets, np.int64)
    sc = (1.0 / np.sqrt(d)) if not scale or scale <= 0 else float(scale)

    def act_(z):
        return z / (1.0 + np.exp(-z)) if act == 1 else z

    def lin(X, W, b, s):
        Z = X @ W[s * d:(s + 1) * d].T
        if b is not None:
            Z = Z + _f64(b)[s * d:(s + 1) * d][None, :]
        return act_(Z)

    out = np.zeros((T.shape[0], j * d))
    for s in range(j):
        xs = T * g[s][None, :]
        q = lin(xs, Wq, b_q, s)
        K = lin(U, Wk, b_k, s)
        V = lin(U, Wv, b_v, s)
        for b in range(len(co) - 1):
            c0, c1, r0, r1 = co[b], co[b + 1], so[b], so[b + 1]
            if c1 == c0 or r1 == r0:
                continue
            S = sc * (q[c0:c1] @ K[r0:r1].T)
            S = S - S.max(axis=1, keepdims=True)
            P = np.exp(S)
            out[c0:c1, s * d:(s + 1) * d] = (P @ V[r0:r1]) / P.sum(axis=1, keepdims=True)
    return out


def history_attention(U, seq_offsets, W_q, W_k, W_v, H, d, act=1, b_q=None, b_k=None, b_v=None,
                      scale=None):
    """U rows of one target-aware layer (PAPER.md:341 mask rule (1): "user embeddings in U will
    not attend to future positions"; the user block of the mask is lower-
    triangular, diagonal included; reading R17).  Per request b, head h and history
    position p (row r = seq_offsets[b] + p):

      q, k, v = act(U W^T + b) split into heads            (as kv_project)
      s_i = scale q_p . k_i for i <= p;  w_i = exp(s_i - max_i s_i)
      O[r][h d:(h+1) d] = sum_i w_i v_i / sum_i w_i;  lse[r][h] = max + log sum_i w_i

    U [total_L, D_in], W_* [H d, D_in].  Returns (O fp64 [total_L, H d], lse [total_L, H]).
    """
    U = _f64(U)
    Wq, Wk, Wv = _f64(W_q), _f64(W_k), _f64(W_v)
    so = _np(seq_offsets, np.int64)
    sc = (1.0 / np.sqrt(d)) if not scale or scale <= 0 else float(scale)

    def proj(W, b):
        Z = U @ W.T
        if b is not None:
            Z = Z + _f64(b)[None, :]
        return Z / (1.0 + np.exp(-Z)) if act == 1 else Z

    Q, K, V = proj(Wq, b_q), proj(Wk, b_k), proj(Wv, b_v)
    O = np.zeros((U.shape[0], H * d))
    lse = np.zeros((U.shape[0], H))
    for b in range(len(so) - 1):
        r0, r1 = so[b], so[b + 1]
        n = r1 - r0
        if n == 0:
            continue
        allowed = np.tril(np.ones((n, n), bool))           # key i <= query p
        for h in range(H):
            cs = slice(h * d, (h + 1) * d)
            S = sc * (Q[r0:r1, cs] @ K[r0:r1, cs].T)
            S = np.where(allowed, S, -np.inf)
            m = S.max(axis=1, keepdims=True)
            w = np.exp(S - m)
            l = w.sum(axis=1, keepdims=True)
            O[r0:r1, cs] = (w @ V[r0:r1, cs]) / l
            lse[r0:r1, h] = (m + np.log(l))[:, 0]
    return O, lse


def stu_stack_forward(U, T, seq_offsets, cand_offsets, layers, H, d, eps=1e-5):
    """[U_self, T_self] after len(layers) STU layers over [U, T], per request (SPEC.md:298
    self_attention_forward; reading R18), brute force, in SPEC.md:343's order per layer:

      Xn = LN_in(X)                                     "normalize input"
      Q, K, V, G = SiLU(Xn W_q^T), SiLU(Xn W_k^T), SiLU(Xn W_v^T), SiLU(Xn W_g^T)
      A = masked row-softmax(Q K^T / sqrt(d)) V per head, mask = build_mask(N, n, self_key=True)
          (user block lower-triangular, candidates see all users and themselves)
      X <- (LN_out(A) (.) G) W_o^T + X                  "output-projection(normalize(attention.
                                                          value) (.) gating-branch) + residual"

    layers: list of dicts with W_q, W_k, W_v, W_g, W_o [D, D] and ln_in / ln_out (gamma, beta)
    [D]; D = H d.  Returns (U_out fp64 [total_L, D], T_out fp64 [total_C, D]).
    """
    U, T = _f64(U), _f64(T)
    so, co = _np(seq_offsets, np.int64), _np(cand_offsets, np.int64)
    D = H * d
    Uo, To = np.zeros_like(U), np.zeros_like(T)

    def ln(X, g, b):
        mu = X.mean(axis=1, keepdims=True)
        var = ((X - mu) ** 2).mean(axis=1, keepdims=True)
        return (X - mu) / np.sqrt(var + eps) * _f64(g)[None, :] + _f64(b)[None, :]

    def silu(Z):
        return Z / (1.0 + np.exp(-Z))

    for b in range(len(so) - 1):
        N, n = int(so[b + 1] - so[b]), int(co[b + 1] - co[b])
        X = np.concatenate([U[so[b]:so[b + 1]], T[co[b]:co[b + 1]]], axis=0)
        allowed = build_mask(N, n, self_key=True).astype(bool)
        for lay in layers:
            Xn = ln(X, *lay["ln_in"])
            Q, K = silu(Xn @ _f64(lay["W_q"]).T), silu(Xn @ _f64(lay["W_k"]).T)
            V, G = silu(Xn @ _f64(lay["W_v"]).T), silu(Xn @ _f64(lay["W_g"]).T)
            A = np.zeros_like(X)
            for h in range(H):
                cs = slice(h * d, (h + 1) * d)
                S = np.where(allowed, (Q[:, cs] @ K[:, cs].T) / np.sqrt(d), -np.inf)
                w = np.exp(S - S.max(axis=1, keepdims=True))
                A[:, cs] = (w @ V[:, cs]) / w.sum(axis=1, keepdims=True)
            X = (ln(A, *lay["ln_out"]) * G) @ _f64(lay["W_o"]).T + X
        Uo[so[b]:so[b + 1]], To[co[b]:co[b + 1]] = X[:N], X[N:]
    return Uo, To


def ro_cross_attention(seeds, W_q, U, seq_offsets, W_k, W_v, i, d, ctx=None, act=1, scale=None):
    """U_cross = Concat_s Attn_ro(Q_s, RO, RO) per request (
    DESIGN.md reading R19), seed by seed:

      query       q_s = act((seed_s + ctx[b][s]) W_{Q,s}^T)           W_q rows [s d, (s+1) d)
      key/value   K_s = act(U_b W_{K,s}^T),  V_s = act(U_b W_{V,s}^T)   (the request's RO rows)
      attention   O_s = softmax(scale q_s K_s^T) V_s
      concat      U_cross[b] = [O_0, ..., O_{i-1}]

    seeds [i, D_in], ctx [B, i, D_in] or None, U [total_L, D_in], W_* [i d, D_in].
    Returns fp64 [B, i d]; a request without history rows gives zeros (reading R6).
    """
    S, U = _f64(seeds), _f64(U)
    Wq, Wk, Wv = _f64(W_q), _f64(W_k), _f64(W_v)
    so = _np(seq_offsets, np.int64)
    B = len(so) - 1
    C = None if ctx is None else _f64(ctx)
    sc = (1.0 / np.sqrt(d)) if not scale or scale <= 0 else float(scale)

    def act_(z):
        return z / (1.0 + np.exp(-z)) if act == 1 else z

    out = np.zeros((B, i * d))
    for b in range(B):
        r0, r1 = so[b], so[b + 1]
        if r1 == r0:
            continue
        for s in range(i):
            cs = slice(s * d, (s + 1) * d)
            x = S[s] + (C[b, s] if C is not None else 0.0)
            q = act_(x @ Wq[cs].T)
            K, V = act_(U[r0:r1] @ Wk[cs].T), act_(U[r0:r1] @ Wv[cs].T)
            z = sc * (K @ q)
            w = np.exp(z - z.max())
            out[b, cs] = (w @ V) / w.sum()
    return out


def tasa_score_hstu(T, cand_offsets, W_q, K, V, seq_offsets, H, d, act=1, scale=None):
    """Candidate rows of the target-aware attention with HSTU's pointwise normalisation
    (the paper defers the STU internals to HSTU; reading R20):
      q = act(T[t] W_q^T)[h d:(h+1) d];  O[t][h] = sum_i SiLU(scale q . K[h][r_i]) V[h][r_i] / L_b
    over the request's L_b history rows (L_b = 0 -> zeros).  K, V fp64 [H, total_L, d] (as
    returned by kv_project).  Returns fp64 [total_C, H d]."""
    T = _f64(T)
    Wq = _f64(W_q)
    K, V = np.asarray(K, np.float64), np.asarray(V, np.float64)
    co, so = _np(cand_offsets, np.int64), _np(seq_offsets, np.int64)
    sc = (1.0 / np.sqrt(d)) if not scale or scale <= 0 else float(scale)
    Z = T @ Wq.T
    Q = Z / (1.0 + np.exp(-Z)) if act == 1 else Z
    out = np.zeros((T.shape[0], H * d))
    for b in range(len(co) - 1):
        c0, c1, r0, r1 = co[b], co[b + 1], so[b], so[b + 1]
        if c1 == c0 or r1 == r0:
            continue
        for h in range(H):
            cs = slice(h * d, (h + 1) * d)
            s_ = sc * (Q[c0:c1, cs] @ K[h, r0:r1].T)
            w = s_ / (1.0 + np.exp(-s_))
            out[c0:c1, cs] = (w @ V[h, r0:r1]) / (r1 - r0)
    return out
