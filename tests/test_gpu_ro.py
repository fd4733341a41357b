"""GPU parity of gesr_ro_cross_score (RO cross attention: PAPER.md:362-370; SPEC.md:309-315;
DESIGN.md reading R19) against the fp64 oracle (oracle.ro_cross_attention) -- attention
tolerance of north_star (max-abs 2e-2, mean-abs 2e-3)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_21095_b200 import binding as gb
from paper_2511_21095_b200 import configs, inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,i,B,with_ctx,out", [("1", 2, None, True, torch.float32),
                                                   ("2", 4, 16, True, torch.bfloat16),
                                                   ("2", 3, 8, False, torch.float32),
                                                   ("3", 4, 3, True, torch.float32)])
def test_ro_parity(name, i, B, with_ctx, out):
    cfg = configs.get(name)
    cfg = cfg.with_(H=i, **({} if B is None else {"B": B}))
    bt = inputs.make_batch(cfg, hma=False)
    g = torch.Generator().manual_seed(17)
    seeds = torch.randn(i, cfg.D_in, generator=g).to(torch.bfloat16)
    ctx = ((torch.randn(cfg.B, i, cfg.D_in, generator=g) * 0.5).to(torch.bfloat16)
           if with_ctx else None)
    dev = torch.device("cuda:0")
    G = bt.to(dev)
    K, V = gb.kv_project(G.U, G.W_k, G.W_v, i, cfg.d, cfg.act)
    Uc = gb.ro_cross_score(seeds.to(dev), G.W_q, K, V, G.seq_offsets, i, cfg.d,
                           ctx=None if ctx is None else ctx.to(dev), act=cfg.act, out_dtype=out)
    torch.cuda.synchronize()
    # the query rows are seeds + context rounded to bf16 on the device (one more bf16 rounding
    # of the query input): the oracle gets the same rounded rows
    q_in = (seeds.float()[None].expand(cfg.B, i, cfg.D_in) +
            (ctx.float() if ctx is not None else 0.0)).to(torch.bfloat16)
    # per request b: its own rounded query rows as the "seeds", no context
    want = np.stack([oracle.ro_cross_attention(q_in[b].double().numpy(), bt.W_q, bt.U,
                                               bt.seq_offsets, bt.W_k, bt.W_v, i, cfg.d,
                                               act=cfg.act)[b] for b in range(cfg.B)])
    got = Uc.float().cpu().double().numpy()
    diff = np.abs(got - want)
    assert diff.max() <= 2e-2 and diff.mean() <= 2e-3, (diff.max(), diff.mean())
