"""Pins for oracle.nro_cross_attention (
DESIGN.md reading R16), each against something other than the function itself:
  * gate all ones, j = 1: plain single-head cross attention = the C++ oracle's tasa_score
    (itself pinned by tests/test_oracle_attention.py) -- SPEC.md:322;
  * j = 2 random case: every slot equals tasa_score run on the gated input x (.) g_s with that
    slot's weights (per-slot recomputation), and the slots concatenate in order;
  * torch fp64 scaled_dot_product_attention per request and slot (library);
  * two candidates with identical queries give identical rows;
  * a zero gate without query bias gives q = act(0) = 0: uniform weights, O = mean of V rows;
  * a request with no history rows gives zero rows (reading R6).
"""
import numpy as np
import pytest
import torch

import oracle


def _case(j=2, d=8, D_in=16, Ls=(5, 0, 9), Cs=(3, 2, 4), seed=0):
    rng = np.random.default_rng(seed)
    so = np.concatenate([[0], np.cumsum(Ls)]).astype(np.int64)
    co = np.concatenate([[0], np.cumsum(Cs)]).astype(np.int64)
    return dict(
        T=rng.standard_normal((co[-1], D_in)), U=rng.standard_normal((so[-1], D_in)),
        W_q=rng.standard_normal((j * d, D_in)) * 0.4, W_k=rng.standard_normal((j * d, D_in)) * 0.4,
        W_v=rng.standard_normal((j * d, D_in)) * 0.4, q_gate=rng.uniform(0, 2, (j, D_in)),
        cand_offsets=co, seq_offsets=so), j, d


def _run(c, j, d, **kw):
    return oracle.nro_cross_attention(c["T"], c["cand_offsets"], c["W_q"], c["q_gate"], c["U"],
                                      c["seq_offsets"], c["W_k"], c["W_v"], j, d, **kw)


def _bf(x):
    return torch.tensor(x).to(torch.bfloat16)


def test_unit_gate_single_slot_is_plain_cross_attention():
    c, j, d = _case(j=1)
    c["q_gate"] = np.ones_like(c["q_gate"])
    # bf16-representable inputs so the C++ oracle (bf16 bit inputs) sees the same values
    for k in ("T", "U", "W_q", "W_k", "W_v"):
        c[k] = _bf(c[k]).double().numpy()
    got = _run(c, j, d)
    K, V = oracle.kv_project(_bf(c["U"]), _bf(c["W_k"]), _bf(c["W_v"]), 1, d, act=1)
    want, _ = oracle.tasa_score(_bf(c["T"]), c["cand_offsets"], _bf(c["W_q"]), K, V,
                                c["seq_offsets"], 1, d, act=1)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)


def test_each_slot_is_attention_on_its_gated_input():
    c, j, d = _case(j=2, seed=1)
    for k in ("T", "U", "W_q", "W_k", "W_v"):
        c[k] = _bf(c[k]).double().numpy()
    c["q_gate"] = np.array([[0.5] * 16, [2.0] * 16])          # gated inputs stay bf16-exact
    got = _run(c, j, d)
    for s in range(j):
        sl = slice(s * d, (s + 1) * d)
        K, V = oracle.kv_project(_bf(c["U"]), _bf(c["W_k"][sl]), _bf(c["W_v"][sl]), 1, d, act=1)
        want, _ = oracle.tasa_score(_bf(c["T"] * c["q_gate"][s]), c["cand_offsets"],
                                    _bf(c["W_q"][sl]), K, V, c["seq_offsets"], 1, d, act=1)
        np.testing.assert_allclose(got[:, sl], want, rtol=0, atol=1e-12)


def test_matches_torch_sdpa_per_request_and_slot():
    c, j, d = _case(j=3, d=4, D_in=8, seed=2)
    got = _run(c, j, d, act=0)
    t = {k: torch.tensor(v, dtype=torch.float64) for k, v in c.items()}
    co, so = c["cand_offsets"], c["seq_offsets"]
    for s in range(j):
        sl = slice(s * d, (s + 1) * d)
        q = (t["T"] * t["q_gate"][s]) @ t["W_q"][sl].T
        K, V = t["U"] @ t["W_k"][sl].T, t["U"] @ t["W_v"][sl].T
        for b in range(len(co) - 1):
            if so[b + 1] == so[b]:
                continue
            o = torch.nn.functional.scaled_dot_product_attention(
                q[co[b]:co[b + 1]][None], K[so[b]:so[b + 1]][None], V[so[b]:so[b + 1]][None])
            np.testing.assert_allclose(got[co[b]:co[b + 1], sl], o[0].numpy(), rtol=0, atol=1e-12)


def test_identical_queries_identical_rows_and_empty_history():
    c, j, d = _case(seed=3)
    c["T"][1] = c["T"][0]
    got = _run(c, j, d)
    assert np.array_equal(got[0], got[1])
    co = c["cand_offsets"]
    assert np.array_equal(got[co[1]:co[2]], np.zeros((co[2] - co[1], j * d)))  # L_b = 0


def test_zero_gate_gives_mean_pooling():
    c, j, d = _case(seed=4)
    c["q_gate"] = np.zeros_like(c["q_gate"])
    got = _run(c, j, d)
    co, so = c["cand_offsets"], c["seq_offsets"]
    for s in range(j):
        V = c["U"] @ c["W_v"][s * d:(s + 1) * d].T
        V = V / (1 + np.exp(-V))
        for b in range(len(co) - 1):
            if so[b + 1] > so[b]:
                np.testing.assert_allclose(got[co[b]:co[b + 1], s * d:(s + 1) * d],
                                           np.broadcast_to(V[so[b]:so[b + 1]].mean(0),
                                                           (co[b + 1] - co[b], d)),
                                           rtol=0, atol=1e-12)
