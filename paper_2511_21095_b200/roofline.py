"""Algorithmic FLOP and byte counts per call.

Only the work the method defines is counted -- never the avoided naive forms (per-candidate
copies of the history, re-projecting K/V per candidate).

  kv_project : FLOP 4*sum(L)*D_in*H*d        bytes 2*sum(L)*D_in + 2*2*sum(L)*H*d + 2*2*H*d*D_in
  q projection: FLOP 2*sum(C)*D_in*H*d
  attention   : FLOP 4*sum_b(C_b*L_b)*H*d    (QK^T and PV, 2 flop per MAC)
  tasa_score  : q projection + attention;   bytes 2*sum(C)*D_in (T) + 2*2*sum(L)*H*d (K,V once)
                + out_bytes*sum(C)*H*d (O) + 2*H*d*D_in (W_q)
  hma_count   : bytes 8*(#item ids) + 8*(sum(C)*F + 1) + 4*sum(C)*F + 8*(#user ids) + 8*(B*F+1)
"""
from __future__ import annotations

import numpy as np


def counts(cfg, L: np.ndarray, C: np.ndarray, n_item_ids: int = 0, n_user_ids: int = 0,
           out_bytes: int = 4) -> dict:
    L = np.asarray(L, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    H, d, D = cfg.H, cfg.d, cfg.D_in
    HD = H * d
    sL, sC = L.sum(), C.sum()
    kv_flop = 4.0 * sL * D * HD
    q_flop = 2.0 * sC * D * HD
    attn_flop = 4.0 * float((C * L).sum()) * HD
    kv_bytes = 2.0 * sL * D + 4.0 * sL * HD + 4.0 * HD * D
    tasa_bytes = 2.0 * sC * D + 4.0 * sL * HD + out_bytes * sC * HD + 2.0 * HD * D
    hma_bytes = 8.0 * n_item_ids + 8.0 * (sC * cfg.F + 1) + 4.0 * sC * cfg.F + \
        8.0 * n_user_ids + 8.0 * (len(L) * cfg.F + 1)
    return {
        "kv_flop": kv_flop, "q_flop": q_flop, "attn_flop": attn_flop,
        "tasa_flop": q_flop + attn_flop, "total_flop": kv_flop + q_flop + attn_flop,
        "kv_bytes": kv_bytes, "tasa_bytes": tasa_bytes, "hma_bytes": hma_bytes,
        "exps": float((C * L).sum()) * H,
        "candidates": sC,
    }


def roof_time(flop: float, nbytes: float, peak_tflops: float, hbm_gbs: float) -> float:
    """Roofline time in seconds: max(flop / P, bytes / BW)."""
    return max(flop / (peak_tflops * 1e12), nbytes / (hbm_gbs * 1e9))
