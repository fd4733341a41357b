"""Thin ctypes binding of libgesr.so (include/gesr.h) -- argument marshalling only.

Every step of the hot path runs inside the library's sm_100a kernels.  torch supplies device
memory and the current CUDA stream; there is NO CPU fallback: calling with CPU tensors, or
without the built library, raises.

  kv_project(U, W_k, W_v, H, d, ...)      -> (K_cache, V_cache)   gesr_kv_project
  kv_project_gather(E, rows, W_k, W_v, ...) -> (K_cache, V_cache)  gesr_kv_project_gather
  tasa_score(T, cand_offsets, W_q, K, V, seq_offsets, H, d, ...) -> (O, lse)   gesr_tasa_score
  hma_count(user_ids, user_offsets, item_ids, item_offsets, cand_offsets, F, cap) -> counts
  nro_cross_score(T, cand_offsets, W_q, q_gate, K, V, seq_offsets, j, d) -> T_cross
                                           gesr_nro_cross_score (NRO cross attention, f3)
  stu_output(T, O, W_g, ln_gamma, ln_beta, W_o, H, d, ...) -> Y   gesr_stu_output (f1)
  history_attention(U, seq_offsets, W_q, K, V, H, d) -> (O, lse)  gesr_history_attention (f4)
  layer_norm(X, gamma, beta) -> Y                                gesr_layer_norm
  ro_cross_score(seeds, W_q, K, V, seq_offsets, i, d, ctx) -> U_cross  gesr_ro_cross_score
  stu_layer / stu_stack(U, T, ..., layers, H, d) -> (U', T')     full STU layers (composition)
  score_step(batch)                        one full scoring step (the three calls; HMA on a
                                           second stream joined by an event)
"""
from __future__ import annotations

import ctypes
import functools
import math
import os
import re
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GESR_LIB") or os.path.join(_HERE, "libgesr.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "gesr.h")

GESR_OK, GESR_ERR_INVALID_ARG, GESR_ERR_UNSUPPORTED, GESR_ERR_CUDA, GESR_ERR_WORKSPACE = range(5)
GESR_ACT_IDENTITY, GESR_ACT_SILU = 0, 1
GESR_OUT_F32, GESR_OUT_BF16 = 0, 1
GESR_TASA_SELF_KEY = 0x1
GESR_TASA_HSTU_SILU = 0x2   # HSTU pointwise SiLU(s)/N normalisation (R20)


class GesrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{status_string(status)}: {msg}")
        self.status = status


_lib = None
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def lib():
    """Load libgesr.so (built in-tree by `make` / __graft_entry__.build()); raise if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise GesrError(GESR_ERR_CUDA, f"{LIB_PATH} is missing: build it with `make` "
                        "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.gesr_version.restype = ctypes.c_int
    L.gesr_launch_count.restype = ctypes.c_ulonglong
    L.gesr_status_string.restype = ctypes.c_char_p
    L.gesr_status_string.argtypes = [ctypes.c_int]
    L.gesr_last_error.restype = ctypes.c_char_p
    L.gesr_kv_project.restype = ctypes.c_int
    L.gesr_kv_project.argtypes = [_vp, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp,
                                  _vp]
    L.gesr_tasa_workspace_bytes.restype = ctypes.c_size_t
    L.gesr_tasa_workspace_bytes.argtypes = [_i64, _i64, _i32, _i32, _i32]
    L.gesr_tasa_score.restype = ctypes.c_int
    L.gesr_tasa_score.argtypes = [_vp, _i64, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _i64, _i64,
                                  _i32, _i32, ctypes.c_float, _i32, ctypes.c_uint32, _vp, _i32,
                                  _vp, _vp, ctypes.c_size_t, _vp]
    L.gesr_tasa_score_self.restype = ctypes.c_int
    L.gesr_tasa_score_self.argtypes = [_vp, _i64, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _i64,
                                       _i64, _i32, _i32, ctypes.c_float, _i32, _vp, _vp, _vp,
                                       _i32, _vp, _vp, ctypes.c_size_t, _vp]
    L.gesr_hma_count.restype = ctypes.c_int
    L.gesr_hma_count.argtypes = [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp]
    L.gesr_hma_count_embed.restype = ctypes.c_int
    L.gesr_hma_count_embed.argtypes = [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp,
                                       _i32, _vp, _vp]
    # entry points added after the first ABI: a GESR_LIB override (A/B of an older build) may
    # lack them; the in-tree library must export every one (tests/test_boundary.py)
    for name, res, args in (
            ("gesr_nro_workspace_bytes", ctypes.c_size_t, [_i64, _i64, _i32, _i32, _i32, _i32]),
            ("gesr_nro_cross_score", ctypes.c_int, [_vp, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _i64, _i64, _i32, _i32, ctypes.c_float, _i32, _vp, _i32, _vp, _vp, ctypes.c_size_t, _vp]),
            ("gesr_history_attention", ctypes.c_int, [_vp, _i64, _i32, _vp, _i64, _vp, _vp, _i32, _vp, _vp, _i32, _i32, ctypes.c_float, _vp, _i32, _vp, _vp, ctypes.c_size_t, _vp]),
            ("gesr_stu_workspace_bytes", ctypes.c_size_t, [_i64, _i32, _i32]),
            ("gesr_ro_workspace_bytes", ctypes.c_size_t, [_i64, _i32, _i32, _i32]),
            ("gesr_ro_cross_score", ctypes.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, _i32, _vp, _vp,
                                                   _vp, _i64, _i64, _i32, ctypes.c_float, _vp,
                                                   _i32, _vp, ctypes.c_size_t, _vp]),
            ("gesr_layer_norm", ctypes.c_int, [_vp, _i64, _i32, _vp, _vp, ctypes.c_float, _vp, _vp]),
            ("gesr_stu_output", ctypes.c_int, [_vp, _i64, _i32, _vp, _i32, _vp, _vp, _vp, _vp, ctypes.c_float, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, ctypes.c_size_t, _vp]),
            ("gesr_host_chunk_maxima", ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp]),
            ("gesr_host_plan_create", ctypes.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _vp]),
            ("gesr_host_plan_destroy", ctypes.c_int, [_vp]),
            ("gesr_score_host", ctypes.c_int, [_vp, _i32, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp,
                                               _i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp]),
            ("gesr_score_host_ids", ctypes.c_int, [_vp, _i32, _vp, _i64, _vp, _vp, _vp, _vp,
                                                   _i64, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp,
                                                   _i32, _vp, _vp, _vp]),
            ("gesr_kv_project_gather", ctypes.c_int, [_vp, _i64, _i32, _vp, _i64, _vp, _vp, _vp,
                                                      _vp, _i32, _i32, _i32, _vp, _vp, _vp]),
            ("gesr_tasa_score_gather", ctypes.c_int, [_vp, _i64, _i32, _vp, _i64, _vp, _vp, _vp,
                                                      _i32, _vp, _vp, _vp, _i64, _i64, _i32, _i32,
                                                      ctypes.c_float, _i32, ctypes.c_uint32, _vp,
                                                      _i32, _vp, _vp, ctypes.c_size_t, _vp]),
    ):
        if not hasattr(L, name) and os.environ.get("GESR_LIB"):
            continue
        getattr(L, name).restype = res
        getattr(L, name).argtypes = args
    _lib = L
    return L


def header_symbols() -> list:
    """Names of every function include/gesr.h declares."""
    with open(HEADER) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gesr_[a-z_0-9]+)\s*\(", text)))


def status_string(s: int) -> str:
    return lib().gesr_status_string(int(s)).decode()


def _check(status: int):
    if status != GESR_OK:
        raise GesrError(status, lib().gesr_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _on_stream(fn):
    """Run the wrapped call with `stream` (when given as a torch stream) as torch's current
    stream, so every tensor the call allocates -- outputs, workspaces and the temporaries
    stu_layer drops on return -- belongs to the launch stream in the caching allocator: a block
    freed here is reused only by work ordered after these kernels on that stream."""
    @functools.wraps(fn)
    def wrapper(*a, **kw):
        s = kw.get("stream")
        if isinstance(s, torch.cuda.Stream) and s != torch.cuda.current_stream(s.device):
            with torch.cuda.stream(s):
                return fn(*a, **kw)
        return fn(*a, **kw)
    return wrapper


def launch_count() -> int:
    """Kernels libgesr.so has launched in this process (gesr_launch_count)."""
    return int(lib().gesr_launch_count())


def _dev(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise GesrError(GESR_ERR_INVALID_ARG, "all tensors must be CUDA tensors "
                            "(no CPU fallback)")
        if t is not None and not t.is_contiguous():
            raise GesrError(GESR_ERR_INVALID_ARG, "all tensors must be contiguous")


def _check_cache(K_cache, V_cache, H, total_L, d):
    """The head-major cache's row stride is total_L: a cache of another shape would be written
    with one layout and read (tasa_score takes total_L from K_cache.shape[1]) with another."""
    for t in (K_cache, V_cache):
        if tuple(t.shape) != (H, total_L, d) or t.dtype != torch.bfloat16:
            raise GesrError(GESR_ERR_INVALID_ARG, f"K/V cache must be bf16 {(H, total_L, d)}, "
                            f"got {t.dtype} {tuple(t.shape)}")


@_on_stream
def kv_project(U, W_k, W_v, H: int, d: int, act: int = GESR_ACT_SILU, b_k=None, b_v=None,
               K_cache=None, V_cache=None, stream=None):
    """K_cache, V_cache bf16 [H, total_L, d] = act(U W^T + b) (gesr_kv_project)."""
    _dev(U, W_k, W_v, b_k, b_v, K_cache, V_cache)
    total_L, D_in = U.shape
    if K_cache is None:
        K_cache = torch.empty((H, total_L, d), dtype=torch.bfloat16, device=U.device)
    if V_cache is None:
        V_cache = torch.empty((H, total_L, d), dtype=torch.bfloat16, device=U.device)
    _check_cache(K_cache, V_cache, H, total_L, d)
    _check(lib().gesr_kv_project(_ptr(U), total_L, D_in, _ptr(W_k), _ptr(W_v), _ptr(b_k),
                                 _ptr(b_v), H, d, act, _ptr(K_cache), _ptr(V_cache),
                                 _stream(stream)))
    return K_cache, V_cache


@_on_stream
def kv_project_gather(E, rows, W_k, W_v, H: int, d: int, act: int = GESR_ACT_SILU, b_k=None,
                      b_v=None, K_cache=None, V_cache=None, stream=None):
    """K_cache, V_cache bf16 [H, len(rows), d] = act(E[rows] W^T + b) with the table lookup
    fused into the projection (gesr_kv_project_gather; E bf16 [n_E, D_in], rows int32)."""
    _dev(E, rows, W_k, W_v, b_k, b_v, K_cache, V_cache)
    if rows.dtype != torch.int32:
        raise GesrError(GESR_ERR_INVALID_ARG, "rows must be int32")
    n_E, D_in = E.shape
    total_L = rows.numel()
    if K_cache is None:
        K_cache = torch.empty((H, total_L, d), dtype=torch.bfloat16, device=E.device)
    if V_cache is None:
        V_cache = torch.empty((H, total_L, d), dtype=torch.bfloat16, device=E.device)
    _check_cache(K_cache, V_cache, H, total_L, d)
    _check(lib().gesr_kv_project_gather(_ptr(E), n_E, D_in, _ptr(rows), total_L, _ptr(W_k),
                                        _ptr(W_v), _ptr(b_k), _ptr(b_v), H, d, act,
                                        _ptr(K_cache), _ptr(V_cache), _stream(stream)))
    return K_cache, V_cache


def tasa_workspace_bytes(B: int, total_C: int, H: int, d: int, kv_splits: int = 0) -> int:
    return int(lib().gesr_tasa_workspace_bytes(B, total_C, H, d, kv_splits))


@_on_stream
def tasa_score(T, cand_offsets, W_q, K_cache, V_cache, seq_offsets, H: int, d: int,
               act: int = GESR_ACT_SILU, b_q=None, scale: float = 0.0, kv_splits: int = 0,
               flags: int = 0, out_dtype=torch.float32, want_lse: bool = True, O=None, lse=None,
               workspace=None, stream=None, K_self=None, V_self=None):
    """O [total_C, H*d] (fp32|bf16), lse fp32 [total_C, H] (gesr_tasa_score; with K_self /
    V_self -- the candidates' own keys / values [H, total_C, d] from kv_project(T, ...) --
    gesr_tasa_score_self: each candidate also attends to its own key)."""
    _dev(T, cand_offsets, W_q, K_cache, V_cache, seq_offsets, b_q, O, lse, workspace, K_self,
         V_self)
    total_C, D_in = T.shape
    B = cand_offsets.numel() - 1
    total_L = K_cache.shape[1]
    if O is None:
        O = torch.empty((total_C, H * d), dtype=out_dtype, device=T.device)
    o_dtype = GESR_OUT_BF16 if O.dtype == torch.bfloat16 else GESR_OUT_F32
    if lse is None and want_lse:
        lse = torch.empty((total_C, H), dtype=torch.float32, device=T.device)
    if workspace is None:
        nbytes = tasa_workspace_bytes(B, total_C, H, d, kv_splits)
        workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=T.device)
    if K_self is not None or V_self is not None:
        _check(lib().gesr_tasa_score_self(_ptr(T), total_C, D_in, _ptr(cand_offsets), _ptr(W_q),
                                          _ptr(b_q), act, _ptr(K_cache), _ptr(V_cache),
                                          _ptr(seq_offsets), B, total_L, H, d, float(scale),
                                          kv_splits, _ptr(K_self), _ptr(V_self), _ptr(O),
                                          o_dtype, _ptr(lse), _ptr(workspace), workspace.numel(),
                                          _stream(stream)))
        return O, lse
    _check(lib().gesr_tasa_score(_ptr(T), total_C, D_in, _ptr(cand_offsets), _ptr(W_q),
                                 _ptr(b_q), act, _ptr(K_cache), _ptr(V_cache), _ptr(seq_offsets),
                                 B, total_L, H, d, float(scale), kv_splits, flags, _ptr(O),
                                 o_dtype, _ptr(lse), _ptr(workspace), workspace.numel(),
                                 _stream(stream)))
    return O, lse


@_on_stream
def tasa_score_gather(E, rows, cand_offsets, W_q, K_cache, V_cache, seq_offsets, H: int, d: int,
                      act: int = GESR_ACT_SILU, b_q=None, scale: float = 0.0, kv_splits: int = 0,
                      flags: int = 0, out_dtype=torch.float32, want_lse: bool = True, O=None,
                      lse=None, workspace=None, stream=None):
    """gesr_tasa_score_gather: tasa_score with T = E[rows] looked up inside the Q projection
    (E bf16 [n_E, D_in], rows int32 [total_C])."""
    _dev(E, rows, cand_offsets, W_q, K_cache, V_cache, seq_offsets, b_q, O, lse, workspace)
    if rows.dtype != torch.int32:
        raise GesrError(GESR_ERR_INVALID_ARG, "rows must be int32")
    n_E, D_in = E.shape
    total_C = rows.numel()
    B = cand_offsets.numel() - 1
    total_L = K_cache.shape[1]
    if O is None:
        O = torch.empty((total_C, H * d), dtype=out_dtype, device=E.device)
    o_dtype = GESR_OUT_BF16 if O.dtype == torch.bfloat16 else GESR_OUT_F32
    if lse is None and want_lse:
        lse = torch.empty((total_C, H), dtype=torch.float32, device=E.device)
    if workspace is None:
        nbytes = tasa_workspace_bytes(B, total_C, H, d, kv_splits)
        workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=E.device)
    _check(lib().gesr_tasa_score_gather(_ptr(E), n_E, D_in, _ptr(rows), total_C,
                                        _ptr(cand_offsets), _ptr(W_q), _ptr(b_q), act,
                                        _ptr(K_cache), _ptr(V_cache), _ptr(seq_offsets), B,
                                        total_L, H, d, float(scale), kv_splits, flags, _ptr(O),
                                        o_dtype, _ptr(lse), _ptr(workspace), workspace.numel(),
                                        _stream(stream)))
    return O, lse


@_on_stream
def history_attention(U, seq_offsets, W_q, K_cache, V_cache, H: int, d: int,
                      act: int = GESR_ACT_SILU, b_q=None, scale: float = 0.0,
                      out_dtype=torch.float32, want_lse: bool = False, O=None, lse=None,
                      workspace=None, stream=None):
    """O [total_L, H*d]: causal self-attention of every history over itself
    (gesr_history_attention; K/V cache [H, total_L, d] from kv_project of the same U)."""
    _dev(U, seq_offsets, W_q, K_cache, V_cache, b_q, O, lse, workspace)
    total_L, D_in = U.shape
    B = seq_offsets.numel() - 1
    if O is None:
        O = torch.empty((total_L, H * d), dtype=out_dtype, device=U.device)
    o_dtype = GESR_OUT_BF16 if O.dtype == torch.bfloat16 else GESR_OUT_F32
    if lse is None and want_lse:
        lse = torch.empty((total_L, H), dtype=torch.float32, device=U.device)
    if workspace is None:
        nbytes = tasa_workspace_bytes(B, total_L, H, d, 1)
        workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=U.device)
    _check(lib().gesr_history_attention(_ptr(U), total_L, D_in, _ptr(seq_offsets), B, _ptr(W_q),
                                        _ptr(b_q), act, _ptr(K_cache), _ptr(V_cache), H, d,
                                        float(scale), _ptr(O), o_dtype, _ptr(lse),
                                        _ptr(workspace), workspace.numel(), _stream(stream)))
    return O, lse


def nro_workspace_bytes(B: int, total_C: int, j: int, d: int, D_in: int,
                        kv_splits: int = 0) -> int:
    return int(lib().gesr_nro_workspace_bytes(B, total_C, j, d, D_in, kv_splits))


@_on_stream
def nro_cross_score(T, cand_offsets, W_q, q_gate, K_cache, V_cache, seq_offsets, j: int, d: int,
                    act: int = GESR_ACT_SILU, b_q=None, scale: float = 0.0, kv_splits: int = 0,
                    out_dtype=torch.float32, want_lse: bool = False, O=None, lse=None,
                    workspace=None, stream=None):
    """T_cross [total_C, j*d] (gesr_nro_cross_score: j gated query slots over the history K/V
    cache [j, total_L, d] from kv_project with the slots' key/value weights as heads)."""
    _dev(T, cand_offsets, W_q, q_gate, K_cache, V_cache, seq_offsets, b_q, O, lse, workspace)
    total_C, D_in = T.shape
    B = cand_offsets.numel() - 1
    total_L = K_cache.shape[1]
    if O is None:
        O = torch.empty((total_C, j * d), dtype=out_dtype, device=T.device)
    o_dtype = GESR_OUT_BF16 if O.dtype == torch.bfloat16 else GESR_OUT_F32
    if lse is None and want_lse:
        lse = torch.empty((total_C, j), dtype=torch.float32, device=T.device)
    if workspace is None:
        nbytes = nro_workspace_bytes(B, total_C, j, d, D_in, kv_splits)
        workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=T.device)
    _check(lib().gesr_nro_cross_score(_ptr(T), total_C, D_in, _ptr(cand_offsets), _ptr(W_q),
                                      _ptr(q_gate), _ptr(b_q), act, _ptr(K_cache),
                                      _ptr(V_cache), _ptr(seq_offsets), B, total_L, j, d,
                                      float(scale), kv_splits, _ptr(O), o_dtype, _ptr(lse),
                                      _ptr(workspace), workspace.numel(), _stream(stream)))
    return O


def stu_workspace_bytes(total_C: int, H: int, d: int) -> int:
    return int(lib().gesr_stu_workspace_bytes(total_C, H, d))


@_on_stream
def stu_output(T, O, W_g, ln_gamma, ln_beta, W_o, H: int, d: int, b_g=None, b_o=None,
               X_res=None, ln_eps: float = 1e-5, Y=None, workspace=None, stream=None):
    """Y bf16 [total_C, D_out] = (LayerNorm(O) * SiLU(T W_g^T + b_g)) W_o^T + b_o + X_res
    (gesr_stu_output: the STU layer's candidate row after the attention)."""
    _dev(T, O, W_g, ln_gamma, ln_beta, W_o, b_g, b_o, X_res, Y, workspace)
    total_C, D_in = T.shape
    D_out = W_o.shape[0]
    if Y is None:
        Y = torch.empty((total_C, D_out), dtype=torch.bfloat16, device=T.device)
    o_dtype = GESR_OUT_BF16 if O.dtype == torch.bfloat16 else GESR_OUT_F32
    if workspace is None:
        workspace = torch.empty(max(stu_workspace_bytes(total_C, H, d), 256), dtype=torch.uint8,
                                device=T.device)
    _check(lib().gesr_stu_output(_ptr(T), total_C, D_in, _ptr(O), o_dtype, _ptr(W_g), _ptr(b_g),
                                 _ptr(ln_gamma), _ptr(ln_beta), float(ln_eps), _ptr(W_o),
                                 _ptr(b_o), _ptr(X_res), H, d, D_out, _ptr(Y), _ptr(workspace),
                                 workspace.numel(), _stream(stream)))
    return Y


@_on_stream
def ro_cross_score(seeds, W_q, K_cache, V_cache, seq_offsets, i: int, d: int, ctx=None,
                   act: int = GESR_ACT_SILU, b_q=None, scale: float = 0.0,
                   out_dtype=torch.float32, U_cross=None, workspace=None, stream=None):
    """U_cross [B, i*d] (gesr_ro_cross_score: i seeds, plus optional per-request context tokens
    ctx [B, i, D_in], over the history K/V cache [i, total_L, d] from kv_project with the seeds'
    key/value weights as heads)."""
    _dev(seeds, W_q, K_cache, V_cache, seq_offsets, ctx, b_q, U_cross, workspace)
    D_in = seeds.shape[1]
    B = seq_offsets.numel() - 1
    total_L = K_cache.shape[1]
    if U_cross is None:
        U_cross = torch.empty((B, i * d), dtype=out_dtype, device=seeds.device)
    o_dtype = GESR_OUT_BF16 if U_cross.dtype == torch.bfloat16 else GESR_OUT_F32
    if workspace is None:
        nbytes = int(lib().gesr_ro_workspace_bytes(B, i, d, D_in))
        workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=seeds.device)
    _check(lib().gesr_ro_cross_score(_ptr(seeds), _ptr(ctx), i, D_in, _ptr(W_q), _ptr(b_q), act,
                                     _ptr(K_cache), _ptr(V_cache), _ptr(seq_offsets), B, total_L,
                                     d, float(scale), _ptr(U_cross), o_dtype, _ptr(workspace),
                                     workspace.numel(), _stream(stream)))
    return U_cross


@_on_stream
def layer_norm(X, gamma, beta, eps: float = 1e-5, Y=None, stream=None):
    """Y bf16 [rows, D] = LayerNorm(X) * gamma + beta (gesr_layer_norm; Y may be X)."""
    _dev(X, gamma, beta, Y)
    rows, D = X.shape
    if Y is None:
        Y = torch.empty_like(X)
    _check(lib().gesr_layer_norm(_ptr(X), rows, D, _ptr(gamma), _ptr(beta), float(eps), _ptr(Y),
                                 _stream(stream)))
    return Y


@_on_stream
def stu_layer(U, T, seq_offsets, cand_offsets, layer: dict, H: int, d: int, eps: float = 1e-5,
              stream=None):
    """One full target-aware STU layer over [U, T] (mask SPEC.md:277 with the
    candidate diagonal; reading R18) as a sequence of C-ABI calls:
      Un, Tn = layer_norm(U), layer_norm(T)                            input normalisation
      K, V   = kv_project(Un)  (the cache), K_T, V_T = kv_project(Tn)  (candidate self keys)
      O_U    = history_attention(Un, K, V)                             causal, rule (1)
      O_T    = tasa_score_self(Tn, K, V, K_T, V_T)                     history + own key
      U', T' = stu_output(Un, O_U, ..., X_res=U), stu_output(Tn, O_T, ..., X_res=T)
    layer: W_q, W_k, W_v, W_g, W_o bf16 [D, D]; ln_in, ln_out (gamma, beta) fp32 [D].
    Returns (U', T') bf16."""
    act = GESR_ACT_SILU
    Un = layer_norm(U, *layer["ln_in"], eps=eps, stream=stream)
    Tn = layer_norm(T, *layer["ln_in"], eps=eps, stream=stream)
    K, V = kv_project(Un, layer["W_k"], layer["W_v"], H, d, act, stream=stream)
    K_T, V_T = kv_project(Tn, layer["W_k"], layer["W_v"], H, d, act, stream=stream)
    O_U, _ = history_attention(Un, seq_offsets, layer["W_q"], K, V, H, d, act, stream=stream)
    O_T, _ = tasa_score(Tn, cand_offsets, layer["W_q"], K, V, seq_offsets, H, d, act,
                        want_lse=False, stream=stream, K_self=K_T, V_self=V_T)
    U2 = stu_output(Un, O_U, layer["W_g"], *layer["ln_out"], layer["W_o"], H, d, X_res=U,
                    ln_eps=eps, stream=stream)
    T2 = stu_output(Tn, O_T, layer["W_g"], *layer["ln_out"], layer["W_o"], H, d, X_res=T,
                    ln_eps=eps, stream=stream)
    return U2, T2


@_on_stream
def stu_stack(U, T, seq_offsets, cand_offsets, layers, H: int, d: int, eps: float = 1e-5,
              stream=None):
    """[U_self, T_self] after len(layers) STU layers (SPEC.md:298 self_attention_forward)."""
    for layer in layers:
        U, T = stu_layer(U, T, seq_offsets, cand_offsets, layer, H, d, eps, stream)
    return U, T


@_on_stream
def hma_count(user_ids, user_offsets, item_ids, item_offsets, cand_offsets, F: int, cap: int = 0,
              counts=None, stream=None):
    """counts int32 [total_C, F] (gesr_hma_count)."""
    _dev(user_ids, user_offsets, item_ids, item_offsets, cand_offsets, counts)
    B = cand_offsets.numel() - 1
    total_C = (item_offsets.numel() - 1) // F if F > 0 else 0
    if counts is None:
        counts = torch.empty((total_C, F), dtype=torch.int32, device=cand_offsets.device)
    _check(lib().gesr_hma_count(_ptr(user_ids), _ptr(user_offsets), _ptr(item_ids),
                                _ptr(item_offsets), _ptr(cand_offsets), B, total_C, F, cap,
                                _ptr(counts), _stream(stream)))
    return counts


@_on_stream
def hma_count_embed(user_ids, user_offsets, item_ids, item_offsets, cand_offsets, F: int, M: int,
                    E, counts=None, emb=None, stream=None):
    """(counts int32 [total_C, F] capped at M, emb bf16 [total_C, F*D_h]) with
    emb[t][f] = E[min(c, M) + f (M+1)] (gesr_hma_count_embed; E bf16 [F (M+1), D_h])."""
    _dev(user_ids, user_offsets, item_ids, item_offsets, cand_offsets, counts, E, emb)
    B = cand_offsets.numel() - 1
    total_C = (item_offsets.numel() - 1) // F if F > 0 else 0
    D_h = E.shape[1]
    if counts is None:
        counts = torch.empty((total_C, F), dtype=torch.int32, device=cand_offsets.device)
    if emb is None:
        emb = torch.empty((total_C, F * D_h), dtype=torch.bfloat16, device=cand_offsets.device)
    _check(lib().gesr_hma_count_embed(_ptr(user_ids), _ptr(user_offsets), _ptr(item_ids),
                                      _ptr(item_offsets), _ptr(cand_offsets), B, total_C, F, M,
                                      _ptr(counts), _ptr(E), D_h, _ptr(emb), _stream(stream)))
    return counts, emb


class StepBuffers:
    """Preallocated outputs/workspace for repeated score_step calls on one batch shape."""

    def __init__(self, batch, out_dtype=torch.float32, want_lse=False):
        cfg = batch.cfg
        dev = batch.cand_offsets.device
        H, d = cfg.H, cfg.d
        self.K = torch.empty((H, batch.total_L, d), dtype=torch.bfloat16, device=dev)
        self.V = torch.empty((H, batch.total_L, d), dtype=torch.bfloat16, device=dev)
        self.O = torch.empty((batch.total_C, H * d), dtype=out_dtype, device=dev)
        self.lse = torch.empty((batch.total_C, H), dtype=torch.float32, device=dev) \
            if want_lse else None
        self.counts = torch.empty((batch.total_C, cfg.F), dtype=torch.int32, device=dev)
        nbytes = tasa_workspace_bytes(batch.B, batch.total_C, H, d, 0)
        if cfg.chunk and batch.B == 1:
            # score_step(chunk=...) reuses this workspace for every candidate chunk: the
            # split-L reserve is not monotone in total_C (auto splits only small calls)
            nbytes = max(nbytes, tasa_workspace_bytes(1, min(cfg.chunk, batch.total_C), H, d, 0))
        self.workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
        self.hma_stream = torch.cuda.Stream(device=dev)
        self.ev_fork = torch.cuda.Event()
        self.ev_join = torch.cuda.Event()


def score_step(batch, bufs: StepBuffers, act: int = GESR_ACT_SILU, cap: int = 0,
               chunk: int = 0, hma: bool = True, stream=None, hma_order=None, events=None):
    """One scoring step: gesr_kv_project -> gesr_tasa_score (optionally in candidate chunks
    reusing one K/V cache) and gesr_hma_count.
    hma_order (default "serial"): "serial" runs HMA on the main stream after the attention,
    "fork" launches it first on the side stream joined by an event, "kv" forks it after the K/V
    projection is enqueued.  The persistent projection and attention kernels leave no room for
    HMA CTAs, so HMA serialises in every order; "serial" keeps the per-call
    timing events clean.  events: optional dict of lists; timing events "kv0", "kv1", "t1" (main stream)
    and "h0", "h1" (HMA's stream) are appended to it (bench.py's per-call times)."""
    cfg = batch.cfg
    main = torch.cuda.current_stream() if stream is None else stream
    order = hma_order or "serial"

    def _ev(name, s):
        if events is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            events.setdefault(name, []).append(e)

    def _hma(s):
        _ev("h0", s)
        hma_count(batch.user_ids, batch.user_offsets, batch.item_ids, batch.item_offsets,
                  batch.cand_offsets, cfg.F, cap, counts=bufs.counts, stream=s)
        _ev("h1", s)

    def _fork():
        bufs.ev_fork.record(main)
        bufs.hma_stream.wait_event(bufs.ev_fork)
        _hma(bufs.hma_stream)
        bufs.ev_join.record(bufs.hma_stream)

    if hma and order == "fork":
        _fork()
    _ev("kv0", main)
    kv_project(batch.U, batch.W_k, batch.W_v, cfg.H, cfg.d, act, K_cache=bufs.K, V_cache=bufs.V,
               stream=main)
    _ev("kv1", main)
    if hma and order == "kv":
        _fork()
    if chunk and batch.B == 1:
        # config 4: the same user's cache reused across candidate chunks (one call per chunk)
        for c0 in range(0, batch.total_C, chunk):
            c1 = min(batch.total_C, c0 + chunk)
            key = f"_co_{c0}"            # chunk offsets built once (no copies in graph capture)
            if key not in bufs.__dict__:
                bufs.__dict__[key] = torch.tensor([0, c1 - c0], dtype=torch.int64,
                                                  device=batch.T.device)
            co = bufs.__dict__[key]
            tasa_score(batch.T[c0:c1], co, batch.W_q, bufs.K, bufs.V, batch.seq_offsets, cfg.H,
                       cfg.d, act, O=bufs.O[c0:c1],
                       lse=None if bufs.lse is None else bufs.lse[c0:c1],
                       want_lse=bufs.lse is not None, workspace=bufs.workspace, stream=main)
    else:
        tasa_score(batch.T, batch.cand_offsets, batch.W_q, bufs.K, bufs.V, batch.seq_offsets,
                   cfg.H, cfg.d, act, O=bufs.O, lse=bufs.lse, want_lse=bufs.lse is not None,
                   workspace=bufs.workspace, stream=main)
    _ev("t1", main)
    if hma and order == "serial":
        _hma(main)
    elif hma:
        main.wait_event(bufs.ev_join)
    return bufs.O, bufs.counts


def plan_chunks(hb, n_chunks: int, pin: bool = False) -> list:
    """Cut a host batch into n_chunks contiguous request ranges -- the cut gesr_score_host makes
    (a Python mirror used by the tests): per chunk the row / candidate ranges, the sliced inputs
    and the offsets rebased to the chunk (seq, cand, user [b*F], item [t*F] offsets at 0)."""
    F, B = hb.cfg.F, hb.B
    so, co = hb.seq_offsets.tolist(), hb.cand_offsets.tolist()
    uo, io = hb.user_offsets, hb.item_offsets
    n_chunks = max(1, min(n_chunks, B))
    edges = [B * k // n_chunks for k in range(n_chunks + 1)]
    fix = (lambda t: t.contiguous().pin_memory()) if pin else (lambda t: t.contiguous())
    chunks = []
    for b0, b1 in zip(edges[:-1], edges[1:]):
        r0, r1, c0, c1 = so[b0], so[b1], co[b0], co[b1]
        u0, u1 = int(uo[b0 * F]), int(uo[b1 * F])
        i0, i1 = int(io[c0 * F]), int(io[c1 * F])
        chunks.append(dict(
            B=b1 - b0, reqs=(b0, b1), rows=(r0, r1), cands=(c0, c1),
            h_so=fix(hb.seq_offsets[b0:b1 + 1] - r0), h_co=fix(hb.cand_offsets[b0:b1 + 1] - c0),
            h_uo=fix(uo[b0 * F:b1 * F + 1] - u0), h_io=fix(io[c0 * F:c1 * F + 1] - i0),
            h_U=hb.U[r0:r1], h_T=hb.T[c0:c1], h_ui=hb.user_ids[u0:u1], h_ii=hb.item_ids[i0:i1]))
    return chunks


def host_chunk_maxima(hb, n_chunks: int) -> list:
    """gesr_host_chunk_maxima: per-chunk maxima {requests, history rows, candidate rows, user
    IDs, item IDs} of the contiguous request cut gesr_score_host uses (host offsets)."""
    m = (ctypes.c_int64 * 5)()
    _check(lib().gesr_host_chunk_maxima(_ptr(hb.seq_offsets), _ptr(hb.cand_offsets),
                                        _ptr(hb.user_offsets), _ptr(hb.item_offsets), hb.B,
                                        hb.cfg.F, n_chunks, m))
    return list(m)


class HostPlan:
    """End-to-end scoring of a HOST-resident batch through the C ABI: `gesr_score_host` (the
    native runtime in csrc/hostpath.cu) cuts the requests into n_chunks, pipelines each chunk's
    host->device copies, gesr_kv_project -> gesr_tasa_score -> gesr_hma_count and the
    device->host copies of O / counts over two device buffer sets and two copy streams.  This
    class only marshals: it creates the plan (device buffers sized by gesr_host_chunk_maxima)
    and passes host pointers.

        plan = HostPlan(host_batch, n_chunks=16, out_dtype=torch.bfloat16)
        plan.run(h_O, h_counts)      # enqueued on the current stream; synchronize to read
    """

    def __init__(self, hb, n_chunks: int = 16, out_dtype=torch.bfloat16,
                 act: int = GESR_ACT_SILU, cap: int = 0, device=None):
        cfg = hb.cfg
        self.hb, self.cfg, self.act, self.cap, self.n_chunks = hb, cfg, act, cap, n_chunks
        n_cut = max(1, min(n_chunks, hb.B))     # the library's clamp (csrc/hostpath.cu)
        self.out_dtype = out_dtype
        dev = torch.device("cuda") if device is None else torch.device(device)
        self.W = tuple(w.to(dev).contiguous() for w in (hb.W_q, hb.W_k, hb.W_v))
        maxima = (ctypes.c_int64 * 5)(*host_chunk_maxima(hb, n_chunks))
        self._plan = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _check(lib().gesr_host_plan_create(
                maxima, cfg.D_in, cfg.H, cfg.d, cfg.F,
                GESR_OUT_BF16 if out_dtype == torch.bfloat16 else GESR_OUT_F32,
                ctypes.byref(self._plan)))
        self.h2d_bytes = sum(t.numel() * t.element_size() for t in (
            hb.U, hb.T, hb.user_ids, hb.item_ids)) + 8 * (
            2 * (hb.B + n_cut) + hb.B * cfg.F + n_cut + hb.total_C * cfg.F + n_cut)

    def run(self, h_O, h_counts, stream=None):
        """Enqueue one end-to-end step; h_O [total_C, H*d] and h_counts [total_C, F] on the host
        (pinned for asynchronous copies); inputs from the host batch given at construction."""
        hb = self.hb
        W_q, W_k, W_v = self.W
        _check(lib().gesr_score_host(
            self._plan, self.n_chunks, _ptr(hb.U), _ptr(hb.seq_offsets), _ptr(hb.T),
            _ptr(hb.cand_offsets), hb.B, _ptr(W_q), _ptr(W_k), _ptr(W_v), self.act,
            _ptr(hb.user_ids), _ptr(hb.user_offsets), _ptr(hb.item_ids), _ptr(hb.item_offsets),
            self.cap, _ptr(h_O), _ptr(h_counts), _stream(stream)))

    def run_ids(self, E, hist_rows, cand_rows, h_O, h_counts, stream=None):
        """gesr_score_host_ids: the same step with the host holding int32 table row ids
        (hist_rows [total_L], cand_rows [total_C]) instead of U / T; E is the device-resident
        bf16 [n_E, D_in] shared embedding table."""
        hb = self.hb
        W_q, W_k, W_v = self.W
        for t in (hist_rows, cand_rows):
            if t.dtype != torch.int32 or t.is_cuda:
                raise GesrError(GESR_ERR_INVALID_ARG, "row ids must be int32 host tensors")
        if E.dim() != 2 or E.shape[1] != self.cfg.D_in or E.dtype != torch.bfloat16:
            raise GesrError(GESR_ERR_INVALID_ARG, "E must be bf16 [n_E, D_in] with the plan's D_in")
        _check(lib().gesr_score_host_ids(
            self._plan, self.n_chunks, _ptr(E), E.shape[0], _ptr(hist_rows),
            _ptr(hb.seq_offsets), _ptr(cand_rows), _ptr(hb.cand_offsets), hb.B, _ptr(W_q),
            _ptr(W_k), _ptr(W_v), self.act, _ptr(hb.user_ids), _ptr(hb.user_offsets),
            _ptr(hb.item_ids), _ptr(hb.item_offsets), self.cap, _ptr(h_O), _ptr(h_counts),
            _stream(stream)))

    def h2d_bytes_ids(self, hist_rows, cand_rows):
        """Host->device bytes per run_ids: the row ids replace U and T."""
        hb = self.hb
        return self.h2d_bytes - sum(t.numel() * t.element_size() for t in (hb.U, hb.T)) + \
            4 * (hist_rows.numel() + cand_rows.numel())

    def close(self):
        if getattr(self, "_plan", None) and self._plan.value:
            lib().gesr_host_plan_destroy(self._plan)
            self._plan = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
