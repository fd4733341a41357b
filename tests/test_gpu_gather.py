"""GPU parity of gesr_kv_project_gather (the shared-embedding-table lookup fused into the K/V
projection): bit-identical to gesr_kv_project on the materialised U = E[rows]
(the same MMAs over the same operand bytes), and within the K/V tolerance of the fp64 oracle
(oracle.kv_project_gather).  Shapes cover ragged row counts, D_in not a multiple of the 64-column
TMA box, a one-row table, repeated and extreme row ids, and enough rows for the m-major walk."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_21095_b200 import binding as gb
from paper_2511_21095_b200 import configs, inputs

from test_gpu_parity import _check_kv, _cuda

pytestmark = pytest.mark.gpu


def _problem(M, D_in, H, d, n_E, seed):
    cfg = configs.Config("gather", 91, B=1, L=("fixed", 1), C=("fixed", 1), H=H, d=d,
                         D_in=D_in, F=1)
    W = inputs.make_batch(cfg, hma=False)
    g = torch.Generator().manual_seed(seed)
    E = torch.randn(n_E, D_in, generator=g).to(torch.bfloat16)
    rows = torch.randint(0, n_E, (M,), generator=g, dtype=torch.int64)
    if M >= 2:
        rows[0], rows[-1] = 0, n_E - 1          # both ends of the table
    if M >= 8:
        rows[3:7] = rows[2]                     # repeats inside one gather4 group and across
    return E, rows.to(torch.int32), W.W_k, W.W_v


@pytest.mark.parametrize("M,D_in,H,d,n_E", [(300, 512, 4, 128, 1000), (129, 64, 1, 32, 50),
                                             (1, 40, 2, 64, 3), (1000, 256, 3, 64, 1),
                                             (4097, 128, 2, 64, 7), (70000, 512, 4, 128, 5000)])
@pytest.mark.parametrize("act", [0, 1])
def test_kv_project_gather_bit_identical_to_materialised(M, D_in, H, d, n_E, act):
    dev = _cuda()
    E, rows, Wk, Wv = _problem(M, D_in, H, d, n_E, seed=M + D_in)
    Eg, rg, Wkg, Wvg = E.to(dev), rows.to(dev), Wk.to(dev), Wv.to(dev)
    bk = torch.linspace(-0.3, 0.3, H * d, device=dev)
    K, V = gb.kv_project_gather(Eg, rg, Wkg, Wvg, H, d, act, b_k=bk)
    U = Eg.index_select(0, rg.long())
    K0, V0 = gb.kv_project(U, Wkg, Wvg, H, d, act, b_k=bk)
    torch.cuda.synchronize()
    assert torch.equal(K, K0) and torch.equal(V, V0)


@pytest.mark.parametrize("M,D_in,H,d,n_E", [(300, 512, 4, 128, 1000), (129, 64, 1, 32, 50)])
def test_kv_project_gather_oracle_parity(M, D_in, H, d, n_E):
    dev = _cuda()
    E, rows, Wk, Wv = _problem(M, D_in, H, d, n_E, seed=5)
    K_or, V_or = oracle.kv_project_gather(E, rows.numpy(), Wk, Wv, H, d, act=1)
    K, V = gb.kv_project_gather(E.to(dev), rows.to(dev), Wk.to(dev), Wv.to(dev), H, d, 1)
    torch.cuda.synchronize()
    U = E.index_select(0, rows.long())
    _check_kv(U, Wk, K.cpu(), K_or, H, d)
    _check_kv(U, Wv, V.cpu(), V_or, H, d)


def test_kv_project_gather_feeds_attention_like_dense():
    """The gathered cache drives gesr_tasa_score exactly like the dense one (config-2 shapes)."""
    dev = _cuda()
    cfg = configs.get("2").with_(B=16)
    bt = inputs.make_batch(cfg, hma=False, device=dev)
    n_E = 3000
    g = torch.Generator().manual_seed(3)
    E = torch.randn(n_E, cfg.D_in, generator=g).to(torch.bfloat16).to(dev)
    rows = torch.randint(0, n_E, (bt.U.shape[0],), generator=g, dtype=torch.int32).to(dev)
    K, V = gb.kv_project_gather(E, rows, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act)
    K0, V0 = gb.kv_project(E.index_select(0, rows.long()), bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act)
    O, _ = gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H, cfg.d,
                         cfg.act, kv_splits=1)
    O0, _ = gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K0, V0, bt.seq_offsets, cfg.H, cfg.d,
                          cfg.act, kv_splits=1)
    torch.cuda.synchronize()
    assert torch.equal(O, O0)


@pytest.mark.parametrize("name,B,kv_splits", [("2", 16, 1), ("3", 6, 0), ("4", 1, 0)])
def test_tasa_score_gather_bit_identical_to_materialised(name, B, kv_splits):
    """gesr_tasa_score_gather (T = E[rows] inside the Q projection) equals gesr_tasa_score on the
    materialised T, for the 1-CTA (d = 64) and CTA-pair (d = 128, split-L at B = 1) kernels."""
    dev = _cuda()
    cfg = configs.get(name).with_(B=B)
    bt = inputs.make_batch(cfg, hma=False, device=dev)
    n_E = 2000
    g = torch.Generator().manual_seed(11)
    E = torch.randn(n_E, cfg.D_in, generator=g).to(torch.bfloat16).to(dev)
    rows = torch.randint(0, n_E, (bt.total_C,), generator=g, dtype=torch.int32).to(dev)
    K, V = gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act)
    O, lse = gb.tasa_score_gather(E, rows, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H,
                                  cfg.d, cfg.act, kv_splits=kv_splits)
    O0, lse0 = gb.tasa_score(E.index_select(0, rows.long()), bt.cand_offsets, bt.W_q, K, V,
                             bt.seq_offsets, cfg.H, cfg.d, cfg.act, kv_splits=kv_splits)
    torch.cuda.synchronize()
    assert torch.equal(O, O0) and torch.equal(lse, lse0)


def test_fused_lookup_step_matches_oracle():
    """The serving step with both lookups fused (history and candidate IDs looked
    up in ONE shared table, then the MoA attention): gesr_kv_project_gather +
    gesr_tasa_score_gather against the fp64 oracle on the looked-up rows, within the attention
    tolerance of tests/test_gpu_parity.py."""
    from test_gpu_parity import MAX_ABS, MEAN_ABS
    dev = _cuda()
    cfg = configs.get("3").with_(B=3, L=("uniform", 1, 300), C=("uniform", 1, 300))
    bt = inputs.make_batch(cfg, hma=False)
    n_E = 5000
    g = torch.Generator().manual_seed(13)
    E = torch.randn(n_E, cfg.D_in, generator=g).to(torch.bfloat16)
    hist = torch.randint(0, n_E, (bt.U.shape[0],), generator=g, dtype=torch.int32)
    cand = torch.randint(0, n_E, (bt.total_C,), generator=g, dtype=torch.int32)
    Eg = E.to(dev)
    K, V = gb.kv_project_gather(Eg, hist.to(dev), bt.W_k.to(dev), bt.W_v.to(dev), cfg.H, cfg.d,
                                cfg.act)
    O, _ = gb.tasa_score_gather(Eg, cand.to(dev), bt.cand_offsets.to(dev), bt.W_q.to(dev), K, V,
                                bt.seq_offsets.to(dev), cfg.H, cfg.d, cfg.act)
    torch.cuda.synchronize()
    K_or, V_or = oracle.kv_project_gather(E, hist.numpy(), bt.W_k, bt.W_v, cfg.H, cfg.d,
                                          act=cfg.act)
    T = E.index_select(0, cand.long())
    O_or, _ = oracle.tasa_score(T, bt.cand_offsets, bt.W_q, K_or, V_or, bt.seq_offsets, cfg.H,
                                cfg.d, act=cfg.act)
    err = np.abs(O.cpu().numpy().astype(np.float64) - O_or)
    assert err.max() < MAX_ABS and err.mean() < MEAN_ABS, (err.max(), err.mean())


def test_tasa_score_gather_hstu_flag_and_bias():
    """The gather feeds the same Q projection for the HSTU-normalisation flag and a query bias."""
    dev = _cuda()
    cfg = configs.get("2").with_(B=8)
    bt = inputs.make_batch(cfg, hma=False, device=dev)
    n_E = 700
    g = torch.Generator().manual_seed(17)
    E = torch.randn(n_E, cfg.D_in, generator=g).to(torch.bfloat16).to(dev)
    rows = torch.randint(0, n_E, (bt.total_C,), generator=g, dtype=torch.int32).to(dev)
    bq = torch.linspace(-0.2, 0.2, cfg.H * cfg.d, device=dev)
    K, V = gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act)
    T = E.index_select(0, rows.long())
    for flags in (0, gb.GESR_TASA_HSTU_SILU):
        O, _ = gb.tasa_score_gather(E, rows, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H,
                                    cfg.d, cfg.act, b_q=bq, flags=flags, want_lse=False)
        O0, _ = gb.tasa_score(T, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H, cfg.d,
                              cfg.act, b_q=bq, flags=flags, want_lse=False)
        torch.cuda.synchronize()
        assert torch.equal(O, O0), flags


@pytest.mark.parametrize("kv_splits,out_dtype", [(3, torch.float32), (1, torch.bfloat16)])
def test_tasa_score_gather_splits_lse_and_dtypes(kv_splits, out_dtype):
    """Forced key splits (combine kernel) with the lse output, fp32 and bf16 O, both biases on
    the gathered K/V projection: every output equals the materialised path's."""
    dev = _cuda()
    cfg = configs.get("3").with_(B=5, L=("uniform", 1, 700), C=("uniform", 1, 600))
    bt = inputs.make_batch(cfg, hma=False, device=dev)
    n_E = 4000
    g = torch.Generator().manual_seed(23)
    E = torch.randn(n_E, cfg.D_in, generator=g).to(torch.bfloat16).to(dev)
    hist = torch.randint(0, n_E, (bt.U.shape[0],), generator=g, dtype=torch.int32).to(dev)
    cand = torch.randint(0, n_E, (bt.total_C,), generator=g, dtype=torch.int32).to(dev)
    bk = torch.linspace(-0.1, 0.2, cfg.H * cfg.d, device=dev)
    bv = torch.linspace(0.3, -0.3, cfg.H * cfg.d, device=dev)
    K, V = gb.kv_project_gather(E, hist, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act, b_k=bk, b_v=bv)
    K0, V0 = gb.kv_project(E.index_select(0, hist.long()), bt.W_k, bt.W_v, cfg.H, cfg.d,
                           cfg.act, b_k=bk, b_v=bv)
    O, lse = gb.tasa_score_gather(E, cand, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H,
                                  cfg.d, cfg.act, kv_splits=kv_splits, out_dtype=out_dtype)
    O0, lse0 = gb.tasa_score(E.index_select(0, cand.long()), bt.cand_offsets, bt.W_q, K0, V0,
                             bt.seq_offsets, cfg.H, cfg.d, cfg.act, kv_splits=kv_splits,
                             out_dtype=out_dtype)
    torch.cuda.synchronize()
    assert torch.equal(K, K0) and torch.equal(V, V0)
    assert torch.equal(O, O0) and torch.equal(lse, lse0)
