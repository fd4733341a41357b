"""K-HMA v4 table paths (csrc/hma.cu), bit-exact against the oracle's pairwise count
(reading R11):

* a user ID repeated 3+ times in a field cannot fit a two-slot bucket under any hash seed: the
  field falls back to the global-memory scan (and its CTA to the generic scan path);
* an ID repeated exactly twice fills one bucket (a match counts 2);
* lists long enough that the 4096-bucket pool is short (tables shrink to >= 1 bucket per ID,
  seeds are retried, some fields go global);
* many distinct IDs per field (seed retries are frequent at 64 IDs in 256 buckets);
* several candidate chunks per request (C > 1024) and groups with empty item lists.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_21095_b200 import binding as gb

pytestmark = pytest.mark.gpu


def _run(users, items, co, F, cap=0):
    dev = torch.device("cuda:0")
    uo = np.concatenate([[0], np.cumsum([len(x) for x in users])]).astype(np.int64)
    io = np.concatenate([[0], np.cumsum([len(x) for x in items])]).astype(np.int64)
    ui = (np.concatenate(users) if sum(map(len, users)) else np.zeros(0)).astype(np.int64)
    ii = (np.concatenate(items) if sum(map(len, items)) else np.zeros(0)).astype(np.int64)
    co = np.asarray(co, np.int64)
    want = oracle.hma_count(ui, uo, ii, io, co, F, cap=cap)
    got = gb.hma_count(torch.tensor(ui, device=dev), torch.tensor(uo, device=dev),
                       torch.tensor(ii, device=dev), torch.tensor(io, device=dev),
                       torch.tensor(co, device=dev), F, cap)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy(), want)
    return want


def _items_from(users, B, C, F, rng, lo=1, hi=17, p_hit=0.5):
    """Item lists that hit the request's user IDs about p_hit of the time."""
    items = []
    for b in range(B):
        for _ in range(C[b]):
            for f in range(F):
                u = users[b * F + f]
                n = int(rng.integers(lo, hi))
                hit = rng.random(n) < p_hit
                pick = rng.choice(u, size=n) if len(u) else np.zeros(n, np.int64)
                miss = rng.integers(-(1 << 62), 1 << 62, size=n)
                items.append(np.where(hit & (len(u) > 0), pick, miss).astype(np.int64))
    return items


def test_hma_triplicate_ids_go_global():
    rng = np.random.default_rng(31)
    F, B = 4, 3
    C = [50, 70, 40]
    users = []
    for b in range(B):
        for f in range(F):
            u = rng.integers(-(1 << 62), 1 << 62, size=int(rng.integers(5, 40))).astype(np.int64)
            if (b + f) % 3 == 0:
                u[:3] = u[0]                 # one ID three times: no seed can place it
            if (b + f) % 3 == 1:
                u[:2] = u[0]                 # one ID twice: one full bucket
            users.append(u)
    items = _items_from(users, B, C, F, rng)
    want = _run(users, items, np.concatenate([[0], np.cumsum(C)]), F)
    assert want.max() >= 3                   # the triplicate counted three times
    _run(users, items, np.concatenate([[0], np.cumsum(C)]), F, cap=2)


def test_hma_pool_pressure_and_seed_retries():
    rng = np.random.default_rng(32)
    F, B = 16, 4
    C = [30, 30, 30, 30]
    users = []
    for b in range(B):
        for f in range(F):
            # request 0: 64 IDs per field (exactly fills the pool at 4 buckets per ID);
            # request 1: 200 per field (tables shrink, seeds retried, some fields global);
            # requests 2-3: mixed
            n = [64, 200, int(rng.integers(0, 300)), int(rng.integers(0, 65))][b]
            users.append(rng.integers(-(1 << 62), 1 << 62, size=n).astype(np.int64))
    items = _items_from(users, B, C, F, rng)
    want = _run(users, items, np.concatenate([[0], np.cumsum(C)]), F)
    assert want.sum() > 0


def test_hma_multi_chunk_requests_and_empty_item_lists():
    rng = np.random.default_rng(33)
    F, B = 3, 2
    C = [2500, 1100]                         # > 1024 candidates: several CTA chunks per request
    users = [rng.integers(0, 200, size=int(rng.integers(10, 60))).astype(np.int64) for _ in range(B * F)]
    users = [np.unique(u) for u in users]
    items = _items_from(users, B, C, F, rng, lo=0, hi=9)   # some empty item lists
    want = _run(users, items, np.concatenate([[0], np.cumsum(C)]), F)
    assert (want == 0).any() and want.sum() > 0


@pytest.mark.parametrize("F,ulen,B,C", [(1, 64, 40, 300), (33, 16, 6, 200), (256, 4, 2, 40),
                                        (64, 64, 3, 50)])
def test_hma_field_count_extremes(F, ulen, B, C):
    """F from 1 to kMaxFields = 256 (a segment group then spans many candidates or one
    candidate spans many groups; the shared-memory pool is split F ways, so at F = 64 with 64 IDs
    per list some fields must shrink their tables or go global)."""
    rng = np.random.default_rng(F * 1000 + ulen)
    users = [rng.integers(-(1 << 40), 1 << 40, size=int(rng.integers(0, ulen + 1)))
             for _ in range(B * F)]
    Cs = [int(rng.integers(1, C + 1)) for _ in range(B)]
    items = _items_from(users, B, Cs, F, rng, lo=0, hi=12)
    co = np.concatenate([[0], np.cumsum(Cs)])
    want = _run(users, items, co, F)
    assert want.sum() > 0
    _run(users, items, co, F, cap=1)
