"""CPU pins of the roofline numerators (paper_2511_21095_b200/roofline.py): the
algorithmic FLOPs and bytes bench.py divides by measured time, recounted by brute force on a
small jagged batch -- one multiply-add (2 FLOP) per term of each definition, one element per
array entry -- so `roofline.achieved` can never include work the method does not define."""
import numpy as np

from paper_2511_21095_b200 import configs, inputs, roofline


def test_counts_match_brute_force():
    cfg = configs.get("2").with_(B=7)
    bt = inputs.make_batch(cfg)
    L = (bt.seq_offsets[1:] - bt.seq_offsets[:-1]).numpy()
    C = (bt.cand_offsets[1:] - bt.cand_offsets[:-1]).numpy()
    H, d, D = cfg.H, cfg.d, cfg.D_in
    kv = q = attn = exps = 0
    for b in range(cfg.B):
        # K and V: every history row x every output column (H*d) x D_in multiply-adds, twice
        kv += 2 * (L[b] * (H * d) * D) * 2
        # Q: every candidate row x H*d x D_in multiply-adds
        q += (C[b] * (H * d) * D) * 2
        for _t in range(C[b]):
            for _h in range(H):
                # s_i = q.k_i (d MACs) and o += p_i v_i (d MACs) for each of the L_b keys
                attn += L[b] * (2 * d + 2 * d)
                exps += L[b]
    got = roofline.counts(cfg, L, C, n_item_ids=bt.item_ids.numel(),
                          n_user_ids=bt.user_ids.numel(), out_bytes=2)
    assert got["kv_flop"] == kv and got["q_flop"] == q and got["attn_flop"] == attn
    assert got["tasa_flop"] == q + attn and got["exps"] == exps
    assert got["candidates"] == C.sum()
    # bytes: each input element read once, each output element written once (bf16 = 2 B)
    sL, sC, HD = L.sum(), C.sum(), H * d
    assert got["kv_bytes"] == 2 * sL * D + 2 * (2 * sL * HD) + 2 * (2 * HD * D)
    assert got["tasa_bytes"] == 2 * sC * D + 2 * (2 * sL * HD) + 2 * sC * HD + 2 * HD * D
    n_seg_t, n_seg_u = sC * cfg.F, cfg.B * cfg.F
    assert got["hma_bytes"] == (8 * bt.item_ids.numel() + 8 * (n_seg_t + 1) + 4 * n_seg_t +
                                8 * bt.user_ids.numel() + 8 * (n_seg_u + 1))


def test_roof_time_is_the_binding_bound():
    assert roofline.roof_time(2e12, 1e9, 1000.0, 5000.0) == 2e-3          # compute-bound
    assert roofline.roof_time(1e9, 5e9, 1000.0, 5000.0) == 1e-3           # memory-bound
