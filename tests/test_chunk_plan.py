"""CPU tests of the end-to-end pipeline's host logic (binding.plan_chunks): the request chunks
partition the batch, every chunk's inputs are the right slices, and its rebased offsets
reproduce the original CSR structure (so each chunk is a valid batch of its own)."""
import numpy as np
import pytest
import torch

from paper_2511_21095_b200 import binding as gb
from paper_2511_21095_b200 import configs, inputs


@pytest.mark.parametrize("n", [1, 3, 7, 64])
def test_chunks_partition_and_rebase(n):
    cfg = configs.get("2").with_(B=23)
    hb = inputs.make_batch(cfg)
    F = cfg.F
    ch = gb.plan_chunks(hb, n)
    assert len(ch) == min(n, hb.B)
    assert ch[0]["reqs"][0] == 0 and ch[-1]["reqs"][1] == hb.B
    for a, b in zip(ch[:-1], ch[1:]):
        assert a["reqs"][1] == b["reqs"][0]
    for c in ch:
        b0, b1 = c["reqs"]
        for k in ("h_so", "h_co", "h_uo", "h_io"):
            assert int(c[k][0]) == 0 and bool((c[k][1:] >= c[k][:-1]).all())
        assert torch.equal(c["h_so"] + hb.seq_offsets[b0], hb.seq_offsets[b0:b1 + 1])
        assert torch.equal(c["h_co"] + hb.cand_offsets[b0], hb.cand_offsets[b0:b1 + 1])
        assert c["h_so"][-1] == c["h_U"].shape[0] and c["h_co"][-1] == c["h_T"].shape[0]
        assert c["h_uo"].numel() == c["B"] * F + 1 and c["h_uo"][-1] == c["h_ui"].numel()
        assert c["h_io"].numel() == c["h_T"].shape[0] * F + 1
        assert c["h_io"][-1] == c["h_ii"].numel()
        r0, r1 = c["rows"]
        assert torch.equal(c["h_U"], hb.U[r0:r1])
        # every (candidate, field) segment of the chunk holds the original IDs
        c0, _ = c["cands"]
        io = hb.item_offsets.numpy()
        for t in range(0, c["h_T"].shape[0], 17):
            for f in range(F):
                s0, s1 = int(c["h_io"][t * F + f]), int(c["h_io"][t * F + f + 1])
                g0, g1 = io[(c0 + t) * F + f], io[(c0 + t) * F + f + 1]
                assert np.array_equal(c["h_ii"][s0:s1].numpy(), hb.item_ids[g0:g1].numpy())


@pytest.mark.parametrize("n", [1, 3, 7, 64])
def test_native_chunk_maxima_match_the_cut(n):
    """gesr_host_chunk_maxima (host code in libgesr.so, no GPU needed) reports the maxima of
    exactly the cut plan_chunks mirrors: {requests, history rows, candidate rows, user IDs,
    item IDs} per chunk."""
    cfg = configs.get("2").with_(B=23)
    hb = inputs.make_batch(cfg)
    ch = gb.plan_chunks(hb, n)
    want = [max(c["B"] for c in ch), max(c["h_U"].shape[0] for c in ch),
            max(c["h_T"].shape[0] for c in ch), max(c["h_ui"].numel() for c in ch),
            max(c["h_ii"].numel() for c in ch)]
    assert gb.host_chunk_maxima(hb, n) == want


def test_score_host_argument_errors():
    """gesr_score_host / gesr_host_plan_create reject bad arguments before touching a device."""
    import ctypes
    L = gb.lib()
    m = (ctypes.c_int64 * 5)(1, 1, 1, 1, 1)
    plan = ctypes.c_void_p()
    assert L.gesr_host_plan_create(m, 0, 1, 32, 1, 1, ctypes.byref(plan)) == gb.GESR_ERR_INVALID_ARG
    bad = (ctypes.c_int64 * 5)(1, -1, 1, 1, 1)
    assert L.gesr_host_plan_create(bad, 32, 1, 32, 1, 1, ctypes.byref(plan)) == gb.GESR_ERR_INVALID_ARG
    assert L.gesr_score_host(None, 1, None, None, None, None, 1, None, None, None, 1, None, None,
                             None, None, 0, None, None, None) == gb.GESR_ERR_INVALID_ARG
    assert "null plan" in L.gesr_last_error().decode()
    assert L.gesr_host_plan_destroy(None) == gb.GESR_OK
