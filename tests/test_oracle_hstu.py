"""Pins for oracle.tasa_score_hstu (HSTU pointwise normalisation, reading R20):
  * torch fp64 composition silu(scale q K^T) @ V / L per request and head (library);
  * a zero query weight gives SiLU(0) = 0 weights: O = 0 exactly (unlike the softmax's mean);
  * a single history row gives O = SiLU(scale q.k) v exactly;
  * O is linear in V (doubling V doubles O) -- no normalisation by the weights' sum.
"""
import numpy as np
import torch

import oracle


def _case(seed=0, H=2, d=8, D_in=16, Ls=(5, 1, 0, 9), Cs=(3, 2, 2, 4)):
    rng = np.random.default_rng(seed)
    so = np.concatenate([[0], np.cumsum(Ls)]).astype(np.int64)
    co = np.concatenate([[0], np.cumsum(Cs)]).astype(np.int64)
    return (rng.standard_normal((co[-1], D_in)), rng.standard_normal((H * d, D_in)) * 0.5,
            rng.standard_normal((H, so[-1], d)), rng.standard_normal((H, so[-1], d)), so, co, H, d)


def test_matches_torch_composition():
    T, Wq, K, V, so, co, H, d = _case()
    got = oracle.tasa_score_hstu(T, co, Wq, K, V, so, H, d, act=1)
    Q = torch.nn.functional.silu(torch.tensor(T) @ torch.tensor(Wq).T)
    for b in range(len(co) - 1):
        if so[b + 1] == so[b]:
            assert np.array_equal(got[co[b]:co[b + 1]], np.zeros((co[b + 1] - co[b], H * d)))
            continue
        for h in range(H):
            cs = slice(h * d, (h + 1) * d)
            s = Q[co[b]:co[b + 1], cs] @ torch.tensor(K[h, so[b]:so[b + 1]]).T / np.sqrt(d)
            want = torch.nn.functional.silu(s) @ torch.tensor(V[h, so[b]:so[b + 1]]) / (so[b + 1] - so[b])
            np.testing.assert_allclose(got[co[b]:co[b + 1], cs], want.numpy(), rtol=0, atol=1e-12)


def test_closed_forms():
    T, Wq, K, V, so, co, H, d = _case(seed=1)
    assert np.array_equal(oracle.tasa_score_hstu(T, co, np.zeros_like(Wq), K, V, so, H, d),
                          np.zeros((co[-1], H * d)))
    a = oracle.tasa_score_hstu(T, co, Wq, K, V, so, H, d)
    b = oracle.tasa_score_hstu(T, co, Wq, K, 2 * V, so, H, d)
    np.testing.assert_allclose(b, 2 * a, rtol=1e-15, atol=0)
    # request 1 has a single history row r: O = SiLU(scale q.k_r) v_r
    r = so[1]
    q = T[co[1]] @ Wq.T
    q = q / (1 + np.exp(-q))
    for h in range(H):
        s = q[h * d:(h + 1) * d] @ K[h, r] / np.sqrt(d)
        np.testing.assert_allclose(a[co[1], h * d:(h + 1) * d], s / (1 + np.exp(-s)) * V[h, r],
                                   rtol=1e-13, atol=1e-15)
