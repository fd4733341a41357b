"""GPU parity of gesr_tasa_score with GESR_TASA_HSTU_SILU (HSTU pointwise normalisation
SiLU(scale q.k)/L_b; reading R20) against the fp64 oracle (oracle.tasa_score_hstu):
north_star's attention tolerance (max-abs 2e-2, mean-abs 2e-3); the flag's argument rules."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_21095_b200 import binding as gb
from paper_2511_21095_b200 import configs, inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,B,out", [("1", None, torch.float32), ("2", 32, torch.float32),
                                        ("2", 16, torch.bfloat16), ("3", 3, torch.float32)])
def test_hstu_parity(name, B, out):
    cfg = configs.get(name)
    if B is not None:
        cfg = cfg.with_(B=B)
    bt = inputs.make_batch(cfg, hma=False)
    dev = torch.device("cuda:0")
    g = bt.to(dev)
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, cfg.H, cfg.d, cfg.act)
    O, _ = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, cfg.H, cfg.d, cfg.act,
                         flags=gb.GESR_TASA_HSTU_SILU, want_lse=False, out_dtype=out)
    torch.cuda.synchronize()
    Ko, Vo = oracle.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, act=cfg.act)
    want = oracle.tasa_score_hstu(bt.T, bt.cand_offsets, bt.W_q, Ko, Vo, bt.seq_offsets, cfg.H,
                                  cfg.d, act=cfg.act)
    diff = np.abs(O.float().cpu().double().numpy() - want)
    assert diff.max() <= 2e-2 and diff.mean() <= 2e-3, (diff.max(), diff.mean())


def test_hstu_argument_rules():
    cfg = configs.get("1")
    bt = inputs.make_batch(cfg, hma=False)
    dev = torch.device("cuda:0")
    g = bt.to(dev)
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, cfg.H, cfg.d, cfg.act)
    with pytest.raises(gb.GesrError) as e:                     # lse is undefined here
        gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, cfg.H, cfg.d, cfg.act,
                      flags=gb.GESR_TASA_HSTU_SILU, want_lse=True)
    assert e.value.status == gb.GESR_ERR_INVALID_ARG
