"""Host-side input bookkeeping: request sub-batches and the s8(c) subset rule (CPU)."""
import numpy as np
import torch

from paper_2511_21095_b200 import configs, inputs
from subsets import survey_subset


def test_select_requests_equals_regeneration():
    """select_requests(full batch, idx) holds exactly the data make_batch generates for those
    requests (the generator is counter-based per request), in the order given."""
    cfg = configs.get("2").with_(B=20)
    full = inputs.make_batch(cfg)
    order = [3, 7, 0, 19, 11]
    sub = inputs.select_requests(full, order)
    ref = inputs.make_batch(cfg, requests=order)
    for k in ("requests", "seq_offsets", "cand_offsets", "U", "T", "user_ids", "user_offsets",
              "item_ids", "item_offsets"):
        assert torch.equal(getattr(sub, k), getattr(ref, k)), k


def test_select_requests_empty_segments():
    cfg = configs.get("3").with_(B=9, L=("uniform", 0, 3), C=("uniform", 0, 2), user_len=(0, 2),
                                 item_len=(0, 2), F=3)
    full = inputs.make_batch(cfg)
    idx = list(range(9))[::-1]
    sub = inputs.select_requests(full, idx)
    ref = inputs.make_batch(cfg, requests=idx)
    for k in ("seq_offsets", "cand_offsets", "U", "T", "user_ids", "item_ids", "item_offsets"):
        assert torch.equal(getattr(sub, k), getattr(ref, k)), k


def test_survey_subset_rule():
    Ls = np.array([5, 1, 9, 9, 3, 7, 2, 8, 6, 4] * 10)
    Cs = np.arange(100)[::-1].copy()
    s = survey_subset(Ls, Cs)
    assert len(s) == 64 and len(set(s)) == 64
    assert set(np.argsort(-Cs, kind="stable")[:8]) <= set(s)
    assert set(np.argsort(Cs, kind="stable")[:8]) <= set(s)


