"""Pins for oracle.ro_cross_attention (R19):
  * i = 1, a single history row, identity activation and W_V = I: the output is that row
    whatever the seed;
  * permuting the history rows leaves U_cross unchanged (set attention);
  * every seed equals the C++ oracle's tasa_score of a one-row "candidate" (the seed plus its
    context token) with that seed's weights (per-seed recomputation);
  * torch fp64 SDPA per request and seed (library); empty history -> zeros.
"""
import numpy as np
import torch

import oracle


def _case(i=3, d=8, D_in=16, Ls=(6, 0, 11), seed=0):
    rng = np.random.default_rng(seed)
    so = np.concatenate([[0], np.cumsum(Ls)]).astype(np.int64)
    bf = lambda x: torch.tensor(x).to(torch.bfloat16).double().numpy()   # noqa: E731
    return dict(seeds=bf(rng.standard_normal((i, D_in))), U=bf(rng.standard_normal((so[-1], D_in))),
                W_q=bf(rng.standard_normal((i * d, D_in)) * 0.4),
                W_k=bf(rng.standard_normal((i * d, D_in)) * 0.4),
                W_v=bf(rng.standard_normal((i * d, D_in)) * 0.4),
                ctx=bf(rng.standard_normal((len(Ls), i, D_in)) * 0.5), so=so), i, d


def _run(c, i, d, **kw):
    return oracle.ro_cross_attention(c["seeds"], c["W_q"], c["U"], c["so"], c["W_k"], c["W_v"],
                                     i, d, **kw)


def test_single_row_identity_value_returns_the_row():
    rng = np.random.default_rng(1)
    D = 8
    U = rng.standard_normal((1, D))
    for seed in (rng.standard_normal((1, D)), np.zeros((1, D))):
        out = oracle.ro_cross_attention(seed, rng.standard_normal((D, D)), U, np.array([0, 1]),
                                        rng.standard_normal((D, D)), np.eye(D), 1, D, act=0)
        np.testing.assert_allclose(out[0], U[0], rtol=0, atol=1e-14)


def test_history_permutation_invariance():
    c, i, d = _case(seed=2)
    a = _run(c, i, d, ctx=c["ctx"])
    perm = np.concatenate([np.random.default_rng(3).permutation(np.arange(c["so"][b], c["so"][b + 1]))
                           for b in range(len(c["so"]) - 1)]).astype(int)
    c2 = dict(c, U=c["U"][perm])
    np.testing.assert_allclose(_run(c2, i, d, ctx=c["ctx"]), a, rtol=0, atol=1e-12)


def test_each_seed_is_one_row_candidate_attention():
    # no context tokens: request b's query row for seed s is the (bf16-exact) seed itself, so
    # seed s of every request equals the C++ tasa_score of one candidate row = seed s
    c, i, d = _case(seed=4)
    got = _run(c, i, d)
    so = c["so"]
    B = len(so) - 1
    bf = lambda x: torch.tensor(x).to(torch.bfloat16)   # noqa: E731
    for s in range(i):
        sl = slice(s * d, (s + 1) * d)
        K, V = oracle.kv_project(bf(c["U"]), bf(c["W_k"][sl]), bf(c["W_v"][sl]), 1, d, act=1)
        T = bf(np.repeat(c["seeds"][s][None], B, axis=0))
        want, _ = oracle.tasa_score(T, np.arange(B + 1, dtype=np.int64), bf(c["W_q"][sl]), K, V,
                                    so, 1, d, act=1)
        np.testing.assert_allclose(got[:, sl], want, rtol=0, atol=1e-12)
    assert np.array_equal(got[1], np.zeros(i * d))          # request 1 has no history


def test_matches_torch_sdpa():
    c, i, d = _case(seed=5)
    got = _run(c, i, d, act=0, ctx=c["ctx"])
    t = {k: torch.tensor(v, dtype=torch.float64) for k, v in c.items() if k != "so"}
    so = c["so"]
    for b in range(len(so) - 1):
        if so[b + 1] == so[b]:
            continue
        for s in range(i):
            sl = slice(s * d, (s + 1) * d)
            q = ((t["seeds"][s] + t["ctx"][b, s]) @ t["W_q"][sl].T)[None, None]
            K = (t["U"][so[b]:so[b + 1]] @ t["W_k"][sl].T)[None]
            V = (t["U"][so[b]:so[b + 1]] @ t["W_v"][sl].T)[None]
            o = torch.nn.functional.scaled_dot_product_attention(q, K, V)
            np.testing.assert_allclose(got[b, sl], o[0, 0].numpy(), rtol=0, atol=1e-12)
