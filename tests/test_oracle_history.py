"""Pins for oracle.history_attention (PAPER.md:341 mask rule (1); SPEC.md:277;
DESIGN.md reading R17), each against something other than the function itself:
  * torch fp64 scaled_dot_product_attention(is_causal=True) per request and head (library);
  * the LAST history row equals the C++ oracle's tasa_score of a candidate with that row's
    embedding over the whole history (a pinned, independent implementation);
  * the first row of every request returns its own value row exactly (one key);
  * a zero query weight gives the prefix means of the value rows (numpy cumsum);
  * causality: editing history row p leaves rows < p bit-identical.
"""
import numpy as np
import torch

import oracle


def _case(Ls=(7, 1, 12, 0, 5), H=2, d=8, D_in=16, seed=0, bf16=True):
    rng = np.random.default_rng(seed)
    so = np.concatenate([[0], np.cumsum(Ls)]).astype(np.int64)
    c = dict(U=rng.standard_normal((so[-1], D_in)), W_q=rng.standard_normal((H * d, D_in)) * 0.4,
             W_k=rng.standard_normal((H * d, D_in)) * 0.4,
             W_v=rng.standard_normal((H * d, D_in)) * 0.4)
    if bf16:
        c = {k: torch.tensor(v).to(torch.bfloat16) for k, v in c.items()}
    return c, so, H, d


def _run(c, so, H, d, **kw):
    return oracle.history_attention(c["U"], so, c["W_q"], c["W_k"], c["W_v"], H, d, **kw)


def test_matches_torch_causal_sdpa():
    c, so, H, d = _case(bf16=False)
    O, _ = _run(c, so, H, d, act=0)
    t = {k: torch.tensor(v, dtype=torch.float64) for k, v in c.items()}
    for b in range(len(so) - 1):
        r0, r1 = so[b], so[b + 1]
        if r1 == r0:
            continue
        for h in range(H):
            cs = slice(h * d, (h + 1) * d)
            q = t["U"][r0:r1] @ t["W_q"][cs].T
            k = t["U"][r0:r1] @ t["W_k"][cs].T
            v = t["U"][r0:r1] @ t["W_v"][cs].T
            o = torch.nn.functional.scaled_dot_product_attention(q[None], k[None], v[None],
                                                                 is_causal=True)
            np.testing.assert_allclose(O[r0:r1, cs], o[0].numpy(), rtol=0, atol=1e-12)


def test_last_row_is_candidate_attention_over_the_whole_history():
    c, so, H, d = _case(seed=1)
    O, lse = _run(c, so, H, d)
    K, V = oracle.kv_project(c["U"], c["W_k"], c["W_v"], H, d, act=1)
    for b in range(len(so) - 1):
        r0, r1 = so[b], so[b + 1]
        if r1 == r0:
            continue
        co = np.array([0, 1], np.int64)
        sub = np.array([0, r1 - r0], np.int64)
        Ob, lb = oracle.tasa_score(c["U"][r1 - 1:r1], co, c["W_q"], K[:, r0:r1].copy(),
                                   V[:, r0:r1].copy(), sub, H, d, act=1)
        np.testing.assert_allclose(O[r1 - 1], Ob[0], rtol=0, atol=1e-12)
        np.testing.assert_allclose(lse[r1 - 1], lb[0], rtol=0, atol=1e-12)


def test_first_row_returns_its_value_and_zero_query_gives_prefix_means():
    c, so, H, d = _case(seed=2, bf16=False)
    O, _ = _run(c, so, H, d, act=0)
    V = c["U"] @ c["W_v"].T
    for b in range(len(so) - 1):
        if so[b + 1] > so[b]:
            assert np.array_equal(O[so[b]], V[so[b]])
    c["W_q"] = np.zeros_like(c["W_q"])
    O0, _ = _run(c, so, H, d, act=0)
    for b in range(len(so) - 1):
        r0, r1 = so[b], so[b + 1]
        want = np.cumsum(V[r0:r1], axis=0) / np.arange(1, r1 - r0 + 1)[:, None]
        np.testing.assert_allclose(O0[r0:r1], want, rtol=0, atol=1e-12)


def test_causality_future_edit_leaves_past_rows_identical():
    c, so, H, d = _case(seed=3, bf16=False)
    O, _ = _run(c, so, H, d)
    p = so[2] + 6                       # request 2, position 6
    c["U"][p] += 1.0
    O2, _ = _run(c, so, H, d)
    assert np.array_equal(O[:p], O2[:p])
    assert not np.array_equal(O[p], O2[p])
