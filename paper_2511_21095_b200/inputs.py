"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

This module holds NONE of the method's arithmetic (no projection, attention or matching);
it only draws numbers.  The generator is counter-based: every value is a pure function of
(config seed, stream, request index, element index), so request b's data are identical at
any batch split, request subset or GPU count.  It runs with torch integer ops
on any device (CPU for the oracle tests, the GPU for large bench batches).

Recipe:
  * U, T ~ N(0, 1) (Box-Muller on two counter-hashed uniforms), rounded RNE to bf16.
  * W_q, W_k, W_v ~ Uniform(+-sqrt(6/(D_in + H*d))) (SPEC.md:91 Xavier), rounded to bf16.
  * L_b, C_b per the config's distribution.
  * HMA: per (request, field) user list of n ~ U{user_len} IDs and per (candidate, field) item
    list of m ~ U{item_len} IDs, each a duplicate-free arithmetic progression (odd stride) over
    the field's vocabulary of size V (power of two), mapped to full-range int64 IDs by a
    bijective 64-bit mix of (field, vocab index).  Overlaps arise with probability ~ n*m/V.
    ``hma_duplicates=True`` draws vocab indices with replacement instead (pins pairwise counts).
"""
from __future__ import annotations

import functools
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from .configs import Config

_M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    """uint64 constant -> int64 two's complement (torch has no uint64 arithmetic)."""
    x &= _M64
    return x - (1 << 64) if x >= (1 << 63) else x


_GOLDEN = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)

# stream ids
S_LEN_L, S_LEN_C, S_U, S_T, S_W, S_UL, S_IL, S_UID, S_IID, S_IDMAP = range(1, 11)


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    return (z >> k) & ((1 << (64 - k)) - 1)


def mix64(z: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (wrapping arithmetic = uint64 bits)."""
    z = z + _GOLDEN
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    return z ^ _lsr(z, 31)


def _seed(cfg: Config, stream: int) -> int:
    x = (0x25112109500 + cfg.cfg_id) * 0x100 + stream
    t = mix64(torch.tensor([_s64(x)], dtype=torch.int64))
    return int(t.item())


def _uniform(keys: torch.Tensor) -> torch.Tensor:
    """float64 in (0, 1) from int64 keys."""
    z = mix64(keys)
    return (_lsr(z, 11).to(torch.float64) + 0.5) * (2.0 ** -53)


def _request_keys(cfg: Config, stream: int, req: torch.Tensor) -> torch.Tensor:
    return mix64(torch.full_like(req, _seed(cfg, stream)) ^ (req * _GOLDEN))


def _normal_bf16(keys: torch.Tensor) -> torch.Tensor:
    u1 = _uniform(keys)
    u2 = _uniform(keys ^ _s64(0xD1B54A32D192ED03))
    n = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)
    return n.to(torch.float32).to(torch.bfloat16)


def _lengths(cfg: Config, spec: tuple, stream: int, req: torch.Tensor) -> torch.Tensor:
    kind = spec[0]
    if kind == "fixed":
        return torch.full_like(req, int(spec[1]))
    u = _uniform(_request_keys(cfg, stream, req))
    lo, hi = int(spec[1]), int(spec[2])
    if kind == "uniform":
        return (lo + torch.floor(u * (hi - lo + 1))).to(torch.int64).clamp(lo, hi)
    if kind == "loguniform":
        v = torch.exp(math.log(lo) + u * (math.log(hi) - math.log(lo)))
        return torch.round(v).to(torch.int64).clamp(lo, hi)
    raise ValueError(kind)


def _offsets(lens: torch.Tensor) -> torch.Tensor:
    off = torch.zeros(lens.numel() + 1, dtype=torch.int64, device=lens.device)
    if lens.numel():
        off[1:] = torch.cumsum(lens, 0)
    return off


def _rows_normal(cfg: Config, stream: int, req: torch.Tensor, lens: torch.Tensor, width: int,
                 chunk_rows: int = 1 << 20) -> torch.Tensor:
    """bf16 [sum(lens), width]; element (b, i, k) keyed by (request key b, i*width + k)."""
    dev = req.device
    total = int(lens.sum().item()) if lens.numel() else 0
    out = torch.empty((total, width), dtype=torch.bfloat16, device=dev)
    if total == 0:
        return out
    rkeys = _request_keys(cfg, stream, req)
    owner = torch.repeat_interleave(torch.arange(req.numel(), device=dev), lens)
    starts = _offsets(lens)
    col = torch.arange(width, device=dev, dtype=torch.int64)
    for r0 in range(0, total, chunk_rows):
        r1 = min(total, r0 + chunk_rows)
        rows = torch.arange(r0, r1, device=dev, dtype=torch.int64)
        o = owner[r0:r1]
        local = rows - starts[o]
        keys = rkeys[o].unsqueeze(1) ^ mix64(local.unsqueeze(1) * width + col.unsqueeze(0))
        out[r0:r1] = _normal_bf16(keys)
    return out


def weights(cfg: Config, device="cpu"):
    """W_q, W_k, W_v bf16 [H*d, D_in], Xavier-uniform; shared by all requests."""
    HD, D = cfg.H * cfg.d, cfg.D_in
    a = math.sqrt(6.0 / (D + HD))
    idx = torch.arange(HD * D, device=device, dtype=torch.int64)
    out = []
    for which in range(3):
        base = _seed(cfg, S_W) ^ _s64((which + 1) * 0x9E3779B97F4A7C15)
        u = _uniform(mix64(idx + base))
        w = ((2.0 * u - 1.0) * a).to(torch.float32).to(torch.bfloat16).reshape(HD, D)
        out.append(w)
    return tuple(out)


def _id_of(cfg: Config, f: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
    """Full-range int64 ID of vocab index v in field f: a bijection of (f, v)."""
    return mix64((f * cfg.vocab + v) ^ _seed(cfg, S_IDMAP))


def _progression(cfg: Config, stream: int, seg_keys: torch.Tensor, lens: torch.Tensor,
                 fields: torch.Tensor, duplicates: bool):
    """IDs for segments: duplicate-free arithmetic progression over the field vocab."""
    dev = seg_keys.device
    V = cfg.vocab
    total = int(lens.sum().item()) if lens.numel() else 0
    if total == 0:
        return torch.zeros(0, dtype=torch.int64, device=dev)
    owner = torch.repeat_interleave(torch.arange(lens.numel(), device=dev), lens)
    starts = _offsets(lens)
    k = torch.arange(total, device=dev, dtype=torch.int64) - starts[owner]
    sk = seg_keys[owner]
    if duplicates:
        v = (_uniform(mix64(sk ^ mix64(k))) * V).to(torch.int64).clamp(0, V - 1)
    else:
        start = (_uniform(mix64(sk + 1)) * V).to(torch.int64).clamp(0, V - 1)
        stride = 2 * (_uniform(mix64(sk + 2)) * (V // 2)).to(torch.int64).clamp(0, V // 2 - 1) + 1
        v = (start + k * stride) % V
    return _id_of(cfg, fields[owner], v)


@dataclass
class Batch:
    cfg: Config
    requests: torch.Tensor          # int64 [B] global request indices
    seq_offsets: torch.Tensor       # int64 [B+1]
    cand_offsets: torch.Tensor      # int64 [B+1]
    U: Optional[torch.Tensor]       # bf16 [sum L, D_in]
    T: Optional[torch.Tensor]       # bf16 [sum C, D_in]
    W_q: torch.Tensor
    W_k: torch.Tensor
    W_v: torch.Tensor
    user_ids: Optional[torch.Tensor]
    user_offsets: Optional[torch.Tensor]   # [B*F + 1]
    item_ids: Optional[torch.Tensor]
    item_offsets: Optional[torch.Tensor]   # [sum C * F + 1]

    @property
    def B(self) -> int:
        return int(self.requests.numel())

    # cached on first use (a device read): later uses, e.g. inside CUDA-graph capture, do not sync
    @functools.cached_property
    def total_L(self) -> int:
        return int(self.seq_offsets[-1].item())

    @functools.cached_property
    def total_C(self) -> int:
        return int(self.cand_offsets[-1].item())

    def to(self, device) -> "Batch":
        def mv(x):
            return None if x is None else x.to(device)
        return Batch(self.cfg, mv(self.requests), mv(self.seq_offsets), mv(self.cand_offsets),
                     mv(self.U), mv(self.T), mv(self.W_q), mv(self.W_k), mv(self.W_v),
                     mv(self.user_ids), mv(self.user_offsets), mv(self.item_ids),
                     mv(self.item_offsets))


def request_lengths(cfg: Config, requests: Optional[Sequence[int]] = None, device="cpu"):
    """(L_b, C_b) int64 tensors for the given global request indices (all by default)."""
    req = torch.arange(cfg.B, dtype=torch.int64, device=device) if requests is None else \
        torch.as_tensor(list(requests), dtype=torch.int64, device=device)
    return _lengths(cfg, cfg.L, S_LEN_L, req), _lengths(cfg, cfg.C, S_LEN_C, req)


def make_batch(cfg: Config, requests: Optional[Sequence[int]] = None, device="cpu",
               attention: bool = True, hma: bool = True, hma_duplicates: bool = False) -> Batch:
    """Generate the inputs of the given requests (default: all cfg.B), offsets rebased."""
    if requests is None:
        req = torch.arange(cfg.B, dtype=torch.int64, device=device)
    elif isinstance(requests, torch.Tensor):
        req = requests.to(device=device, dtype=torch.int64)
    else:
        req = torch.as_tensor(list(requests), dtype=torch.int64, device=device)
    Ls = _lengths(cfg, cfg.L, S_LEN_L, req)
    Cs = _lengths(cfg, cfg.C, S_LEN_C, req)
    so, co = _offsets(Ls), _offsets(Cs)
    W_q, W_k, W_v = weights(cfg, device)
    U = T = None
    if attention:
        U = _rows_normal(cfg, S_U, req, Ls, cfg.D_in)
        T = _rows_normal(cfg, S_T, req, Cs, cfg.D_in)
    ui = uo = ii = io = None
    if hma:
        F = cfg.F
        Bn = req.numel()
        fields_u = torch.arange(F, device=device, dtype=torch.int64).repeat(Bn)
        ureq = torch.repeat_interleave(req, F)
        useg = mix64(_request_keys(cfg, S_UL, ureq) ^ fields_u)
        lo, hi = cfg.user_len
        ulen = (lo + torch.floor(_uniform(useg) * (hi - lo + 1))).to(torch.int64).clamp(lo, hi)
        ulen = ulen.clamp(max=cfg.vocab)
        uo = _offsets(ulen)
        ui = _progression(cfg, S_UID, mix64(useg ^ S_UID), ulen, fields_u, hma_duplicates)
        # item side: candidate t of request b, local index j, field f
        nC = int(co[-1].item())
        cowner = torch.repeat_interleave(torch.arange(Bn, device=device), Cs)
        clocal = torch.arange(nC, device=device, dtype=torch.int64) - co[cowner]
        ckey = mix64(_request_keys(cfg, S_IL, req)[cowner] ^ mix64(clocal))
        iseg = mix64(torch.repeat_interleave(ckey, F) ^
                     torch.arange(F, device=device, dtype=torch.int64).repeat(nC))
        fields_i = torch.arange(F, device=device, dtype=torch.int64).repeat(nC)
        lo, hi = cfg.item_len
        ilen = (lo + torch.floor(_uniform(iseg) * (hi - lo + 1))).to(torch.int64).clamp(lo, hi)
        ilen = ilen.clamp(max=cfg.vocab)
        io = _offsets(ilen)
        ii = _progression(cfg, S_IID, mix64(iseg ^ S_IID), ilen, fields_i, hma_duplicates)
    return Batch(cfg, req, so, co, U, T, W_q, W_k, W_v, ui, uo, ii, io)


def _seg_index(offsets: torch.Tensor, segs: torch.Tensor) -> torch.Tensor:
    """Element indices of the given CSR segments, concatenated in the order given."""
    lo, hi = offsets[segs], offsets[segs + 1]
    n = hi - lo
    if int(n.sum().item()) == 0:
        return torch.zeros(0, dtype=torch.int64, device=offsets.device)
    start = torch.repeat_interleave(lo, n)
    first = torch.repeat_interleave(_offsets(n)[:-1], n)
    return start + torch.arange(int(n.sum().item()), device=offsets.device) - first


def select_requests(batch: Batch, idx: Sequence[int], device="cpu") -> Batch:
    """The sub-batch of the given LOCAL request positions (in the order given), moved to
    `device`, offsets rebased: the same rows / IDs the full batch holds for those requests (so
    a test can feed the oracle exactly the inputs the device batch was scored on).  Index
    bookkeeping only."""
    dev = batch.seq_offsets.device
    idx = torch.as_tensor(list(idx), dtype=torch.int64, device=dev)
    so, co = batch.seq_offsets, batch.cand_offsets
    Ls, Cs = (so[idx + 1] - so[idx]), (co[idx + 1] - co[idx])
    rows = _seg_index(so, idx)
    cands = _seg_index(co, idx)
    mv = lambda x: None if x is None else x.to(device)    # noqa: E731
    U = None if batch.U is None else batch.U[rows]
    T = None if batch.T is None else batch.T[cands]
    ui = uo = ii = io = None
    if batch.user_ids is not None:
        F = batch.cfg.F
        useg = (idx[:, None] * F + torch.arange(F, device=dev)).reshape(-1)
        iseg = (cands[:, None] * F + torch.arange(F, device=dev)).reshape(-1)
        uo = _offsets(batch.user_offsets[useg + 1] - batch.user_offsets[useg])
        io = _offsets(batch.item_offsets[iseg + 1] - batch.item_offsets[iseg])
        ui = batch.user_ids[_seg_index(batch.user_offsets, useg)]
        ii = batch.item_ids[_seg_index(batch.item_offsets, iseg)]
    return Batch(batch.cfg, mv(batch.requests[idx]), mv(_offsets(Ls)), mv(_offsets(Cs)), mv(U),
                 mv(T), mv(batch.W_q), mv(batch.W_k), mv(batch.W_v), mv(ui), mv(uo), mv(ii),
                 mv(io))
