"""Randomised GPU parity sweep: many small jagged batches with random shapes (heads, head dim,
input width, requests, history / candidate lengths including 0, HMA fields and list lengths
including empty lists) through gesr_kv_project -> gesr_tasa_score -> gesr_hma_count and
gesr_history_attention, each against the fp64 oracle.  Gates as tests/test_gpu_parity.py:
attention max-abs 2e-2 / mean-abs 2e-3, HMA bit-exact."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_21095_b200 import binding as gb
from paper_2511_21095_b200 import configs, inputs

pytestmark = pytest.mark.gpu

CASES = []
_rng = np.random.default_rng(2025)
for _i in range(12):
    d = int(_rng.choice([32, 64, 128]))
    H = int(_rng.integers(1, 4))
    D_in = int(_rng.choice([32, 64, 96, 128, 256]))
    B = int(_rng.integers(1, 7))
    CASES.append(configs.Config(
        f"sweep{_i}", 500 + _i, B=B, L=("uniform", 0, int(_rng.integers(1, 700))),
        C=("uniform", 0, int(_rng.integers(1, 600))), H=H, d=d, D_in=D_in,
        F=int(_rng.integers(1, 6)), user_len=(0, 40), item_len=(0, 12), vocab=64))
# tiny lengths: many empty histories / candidate lists and single rows in one batch
CASES.append(configs.Config("sweep_tiny", 520, B=24, L=("uniform", 0, 3), C=("uniform", 0, 3),
                            H=2, d=64, D_in=128, F=3, user_len=(0, 3), item_len=(0, 3), vocab=8))
CASES.append(configs.Config("sweep_tiny128", 521, B=24, L=("uniform", 0, 2), C=("uniform", 0, 300),
                            H=1, d=128, D_in=128, F=2, user_len=(0, 2), item_len=(0, 2), vocab=4))


def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200 (run through gpurun)"
    return torch.device("cuda:0")


def _tol(got, want, what):
    if want.size == 0:
        return
    diff = np.abs(got - want)
    assert np.isfinite(got).all(), what
    assert diff.max() <= 2e-2 and diff.mean() <= 2e-3, \
        f"{what}: max-abs {diff.max():.3e} mean-abs {diff.mean():.3e}"


@pytest.mark.parametrize("cfg", CASES, ids=[c.name for c in CASES])
def test_random_shapes(cfg):
    dev = _cuda()
    bt = inputs.make_batch(cfg)
    g = bt.to(dev)
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, cfg.H, cfg.d, cfg.act)
    O, lse = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, cfg.H, cfg.d,
                           cfg.act)
    counts = gb.hma_count(g.user_ids, g.user_offsets, g.item_ids, g.item_offsets,
                          g.cand_offsets, cfg.F)
    Oh, _ = gb.history_attention(g.U, g.seq_offsets, g.W_q, K, V, cfg.H, cfg.d, cfg.act)
    torch.cuda.synchronize()
    Ko, Vo = oracle.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, act=cfg.act)
    O_or, _ = oracle.tasa_score(bt.T, bt.cand_offsets, bt.W_q, Ko, Vo, bt.seq_offsets, cfg.H,
                                cfg.d, act=cfg.act)
    _tol(O.cpu().double().numpy(), O_or, f"{cfg.name} tasa")
    Oh_or, _ = oracle.history_attention(bt.U, bt.seq_offsets, bt.W_q, bt.W_k, bt.W_v, cfg.H,
                                        cfg.d, act=cfg.act)
    _tol(Oh.cpu().double().numpy(), Oh_or, f"{cfg.name} history")
    c_or = oracle.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                            bt.cand_offsets, cfg.F)
    assert np.array_equal(counts.cpu().numpy(), c_or), cfg.name
