"""Request sharding across GPUs -- host-side logic only.

Requests are independent (each has its own history K/V, candidates and HMA lists: candidate
isolation / RO sharing), so the hot path shards by request with NO data-path
collective.  Every rank computes the same deterministic partition from the request metadata,
generates only its own requests (the input generator is counter-based per request), and the
only collectives are the setup weight broadcast and an optional post-step gather of scores.

  request_cost(cfg, L, C)      per-request cost model (FLOP-equivalent)
  lpt_partition(cost, world)   longest-processing-time-first bin packing -> per-rank indices
  contiguous_partition(B, world)
  gather_rows(local, counts, group, dst=0)   variable-size gather with point-to-point ops
"""
from __future__ import annotations

import heapq
from typing import List, Sequence

import numpy as np


def request_cost(cfg, L: Sequence[int], C: Sequence[int]) -> np.ndarray:
    """w_b = 4 L D_in H d + 2 C D_in H d + 4 C L H d (kv + q projection + attention FLOPs)."""
    L = np.asarray(L, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    HD = cfg.H * cfg.d
    return 4.0 * L * cfg.D_in * HD + 2.0 * C * cfg.D_in * HD + 4.0 * C * L * HD


def lpt_partition(cost: Sequence[float], world: int) -> List[np.ndarray]:
    """Deterministic LPT: requests sorted by (-cost, index) go to the least-loaded rank
    (ties -> lowest rank).  Each rank's list is returned in ascending request order."""
    cost = np.asarray(cost, dtype=np.float64)
    order = np.lexsort((np.arange(cost.size), -cost))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    owner = np.empty(cost.size, dtype=np.int64)
    for i in order:
        load, r = heapq.heappop(heap)
        owner[i] = r
        heapq.heappush(heap, (load + float(cost[i]), r))
    return [np.flatnonzero(owner == r) for r in range(world)]


def contiguous_partition(B: int, world: int) -> List[np.ndarray]:
    edges = [(B * r) // world for r in range(world + 1)]
    return [np.arange(edges[r], edges[r + 1], dtype=np.int64) for r in range(world)]


def imbalance(cost: Sequence[float], parts: List[np.ndarray]) -> float:
    cost = np.asarray(cost, dtype=np.float64)
    loads = np.array([cost[p].sum() for p in parts])
    return float(loads.max() / loads.mean() - 1.0) if loads.mean() > 0 else 0.0


def gather_rows(local, counts: Sequence[int], group=None, dst: int = 0):
    """Gather each rank's [n_r, ...] tensor to `dst` (rank order) with send/recv; shards have
    variable size so all_gather does not apply.  Returns the concatenation on dst, None else."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if rank != dst:
        if local.shape[0] > 0:
            dist.send(local.contiguous(), dst=dist.get_global_rank(group, dst) if group else dst,
                      group=group)
        return None
    parts = []
    for r in range(world):
        if r == dst:
            parts.append(local)
            continue
        n = int(counts[r])
        buf = torch.empty((n,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        if n > 0:
            dist.recv(buf, src=dist.get_global_rank(group, r) if group else r, group=group)
        parts.append(buf)
    return torch.cat(parts, dim=0)
