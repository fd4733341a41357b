"""GPU parity of gesr_nro_cross_score (NRO cross attention; PAPER.md:373-380,
SPEC.md:316-324, reading R16) against the fp64 oracle (oracle.nro_cross_attention) on
the same seeded inputs.  Gate: the attention tolerance of BASELINE.json north_star (max-abs 2e-2,
mean-abs 2e-3 vs pure fp64), the folded gate weight being one more bf16 rounding of the query
operand, like the bf16 query itself.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_21095_b200 import binding as gb
from paper_2511_21095_b200 import configs, inputs

pytestmark = pytest.mark.gpu

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200 (run through gpurun)"
    return torch.device("cuda:0")


def _case(name, j, B=None, seed=5):
    cfg = configs.get(name)
    if B is not None:
        cfg = cfg.with_(B=B)
    cfg = cfg.with_(H=j)                      # the slots are heads of the K/V cache
    bt = inputs.make_batch(cfg, hma=False)
    g = torch.Generator().manual_seed(seed)
    gate = torch.rand(j, cfg.D_in, generator=g) * 2.0          # elementwise gates in [0, 2)
    return cfg, bt, gate


def _gpu(cfg, bt, gate, j, out_dtype=torch.float32, kv_splits=0):
    dev = _cuda()
    g = bt.to(dev)
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, j, cfg.d, cfg.act)
    O = gb.nro_cross_score(g.T, g.cand_offsets, g.W_q, gate.to(dev), K, V, g.seq_offsets, j,
                           cfg.d, cfg.act, out_dtype=out_dtype, kv_splits=kv_splits)
    torch.cuda.synchronize()
    return O.float().cpu().double().numpy()


def _oracle(cfg, bt, gate, j):
    return oracle.nro_cross_attention(bt.T, bt.cand_offsets, bt.W_q, gate, bt.U, bt.seq_offsets,
                                      bt.W_k, bt.W_v, j, cfg.d, act=cfg.act)


def _tol(got, want, what):
    diff = np.abs(got - want)
    assert np.isfinite(got).all(), what
    assert diff.max() <= MAX_ABS and diff.mean() <= MEAN_ABS, \
        f"{what}: max-abs {diff.max():.3e} mean-abs {diff.mean():.3e}"


@pytest.mark.parametrize("name,j,B", [("1", 1, None), ("1", 3, None), ("2", 2, 24), ("2", 4, 12),
                                      ("3", 2, 3)])
def test_nro_parity(name, j, B):
    cfg, bt, gate = _case(name, j, B)
    _tol(_gpu(cfg, bt, gate, j), _oracle(cfg, bt, gate, j), f"config {name} j={j}")


def test_nro_bf16_out_and_forced_splits():
    cfg, bt, gate = _case("3", 2, B=2, seed=8)
    want = _oracle(cfg, bt, gate, 2)
    _tol(_gpu(cfg, bt, gate, 2, out_dtype=torch.bfloat16), want, "bf16 out")
    _tol(_gpu(cfg, bt, gate, 2, kv_splits=3), want, "kv_splits=3")


def test_nro_unit_gate_equals_tasa_score_exactly():
    # gate of ones: the folded weight is W_q itself (x * 1.0 is exact), so the call must be
    # bit-identical to gesr_tasa_score with H = j on the same cache
    cfg, bt, _ = _case("2", 2, B=16)
    dev = _cuda()
    g = bt.to(dev)
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, 2, cfg.d, cfg.act)
    ones = torch.ones(2, cfg.D_in, device=dev)
    O1 = gb.nro_cross_score(g.T, g.cand_offsets, g.W_q, ones, K, V, g.seq_offsets, 2, cfg.d,
                            cfg.act, kv_splits=1)
    O2, _ = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, 2, cfg.d, cfg.act,
                          kv_splits=1)
    torch.cuda.synchronize()
    assert torch.equal(O1, O2)
