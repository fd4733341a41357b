"""Pins for the oracle's bias, scale and activation arguments.

Every projection of the method is `act(X W^T + b)` (reading R3; "linear
projection with sigmoid-linear-unit activation"), the score scale is `scale` (reading R4,
SPEC.md:343 "scaled dot products"), and the normalisation is a row softmax (reading R1).  The
checks below compare each oracle with a different implementation -- torch's fp64
`nn.functional.linear(x, W, b)` followed by `silu`, and `scaled_dot_product_attention(scale=...)`
-- with DISTINCT b_q / b_k / b_v vectors, so a plausible slip fails one of them:

  * b_k added to V (or b_v to K), b_q dropped            -> the per-operand bias checks
  * bias applied after the activation instead of before  -> silu(xW + b) != silu(xW) + b
  * scale ignored / applied twice / 1/sqrt(d) hard-coded  -> the scale sweep {0.05, 1/sqrt d, 0.5}
"""
import math

import numpy as np
import pytest
import torch

import oracle

H, D = 2, 16


def _bf16(x):
    return torch.as_tensor(x, dtype=torch.float32).to(torch.bfloat16)


def _problem(seed, Ls=(6, 3, 1, 0), Cs=(4, 0, 3, 2), D_in=24):
    g = torch.Generator().manual_seed(seed)
    so = torch.tensor(np.concatenate([[0], np.cumsum(Ls)]), dtype=torch.int64)
    co = torch.tensor(np.concatenate([[0], np.cumsum(Cs)]), dtype=torch.int64)
    U = _bf16(torch.randn(int(so[-1]), D_in, generator=g))
    T = _bf16(torch.randn(int(co[-1]), D_in, generator=g))
    a = math.sqrt(6.0 / (D_in + H * D))
    W = [_bf16((torch.rand(H * D, D_in, generator=g) * 2 - 1) * a) for _ in range(3)]
    # three different bias vectors: a bias landing on the wrong operand changes the result
    b = [torch.linspace(-0.7, 0.9, H * D, dtype=torch.float64) * (k + 1) * (-1) ** k
         for k in range(3)]
    return so, co, U, T, W, b


def _lin(X, W, b, act):
    y = torch.nn.functional.linear(X.to(torch.float64), W.to(torch.float64),
                                   None if b is None else b.to(torch.float64))
    return torch.nn.functional.silu(y) if act == 1 else y


def _heads(Z):
    return Z.reshape(Z.shape[0], H, D).transpose(0, 1)      # [H, rows, d]


@pytest.mark.parametrize("act", [0, 1])
def test_kv_project_bias_per_operand(act):
    so, co, U, T, (Wq, Wk, Wv), (bq, bk, bv) = _problem(11)
    K, V = oracle.kv_project(U, Wk, Wv, H, D, act=act, b_k=bk.numpy(), b_v=bv.numpy())
    np.testing.assert_allclose(K, _heads(_lin(U, Wk, bk, act)).numpy(), rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(V, _heads(_lin(U, Wv, bv, act)).numpy(), rtol=1e-13, atol=1e-13)
    # b_v only: K must not move
    K0, V1 = oracle.kv_project(U, Wk, Wv, H, D, act=act, b_v=bv.numpy())
    np.testing.assert_allclose(K0, _heads(_lin(U, Wk, None, act)).numpy(), rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(V1, V, rtol=0, atol=0)


def _sdpa_ref(so, co, U, T, W, b, act, scale):
    (Wq, Wk, Wv), (bq, bk, bv) = W, b
    Q, K, V = _lin(T, Wq, bq, act), _lin(U, Wk, bk, act), _lin(U, Wv, bv, act)
    out = np.zeros((T.shape[0], H * D))
    for i in range(len(so) - 1):
        r0, r1, c0, c1 = int(so[i]), int(so[i + 1]), int(co[i]), int(co[i + 1])
        if c1 == c0 or r1 == r0:
            continue
        o = torch.nn.functional.scaled_dot_product_attention(
            _heads(Q[c0:c1]), _heads(K[r0:r1]), _heads(V[r0:r1]), scale=scale)
        out[c0:c1] = o.transpose(0, 1).reshape(c1 - c0, H * D).numpy()
    return out


@pytest.mark.parametrize("act", [0, 1])
@pytest.mark.parametrize("scale", [0.05, 1.0 / math.sqrt(D), 0.5])
def test_tasa_bias_and_scale_sweep_vs_sdpa(act, scale):
    so, co, U, T, W, b = _problem(12)
    (Wq, Wk, Wv), (bq, bk, bv) = W, b
    K, V = oracle.kv_project(U, Wk, Wv, H, D, act=act, b_k=bk.numpy(), b_v=bv.numpy())
    O, lse = oracle.tasa_score(T, co, Wq, K, V, so, H, D, act=act, b_q=bq.numpy(), scale=scale)
    ref = _sdpa_ref(so, co, U, T, W, b, act, scale)
    np.testing.assert_allclose(O, ref, rtol=1e-12, atol=1e-12)
    # the default scale is 1/sqrt(d) (reading R4)
    if abs(scale - 1.0 / math.sqrt(D)) < 1e-15:
        O2, _ = oracle.tasa_score(T, co, Wq, K, V, so, H, D, act=act, b_q=bq.numpy())
        np.testing.assert_array_equal(O, O2)


@pytest.mark.parametrize("act", [0, 1])
def test_tasa_bias_before_activation(act):
    """b_q enters before the activation: with W_q = 0 the query is act(b_q) for every candidate,
    so all candidates of a request get the same row, equal to softmax(scale act(b_q) K^T) V."""
    so, co, U, T, (Wq, Wk, Wv), (bq, bk, bv) = _problem(13, Ls=(5,), Cs=(3,))
    Wz = torch.zeros_like(Wq)
    K, V = oracle.kv_project(U, Wk, Wv, H, D, act=act)
    O, _ = oracle.tasa_score(T, co, Wz, K, V, so, H, D, act=act, b_q=bq.numpy(), scale=0.3)
    q = bq.numpy() / (1 + np.exp(-bq.numpy())) if act else bq.numpy()
    for h in range(H):
        s = 0.3 * K[h] @ q[h * D:(h + 1) * D]
        w = np.exp(s - s.max())
        want = (w[:, None] * V[h]).sum(0) / w.sum()
        for t in range(3):
            np.testing.assert_allclose(O[t, h * D:(h + 1) * D], want, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("act", [0, 1])
def test_full_mask_bias_vs_sdpa(act):
    so, co, U, T, W, b = _problem(14, Ls=(5,), Cs=(3,))
    (Wq, Wk, Wv), (bq, bk, bv) = W, b
    O, _ = oracle.full_masked_attention(U, T, Wq, Wk, Wv, H, D, act=act, b_q=bq.numpy(),
                                        b_k=bk.numpy(), b_v=bv.numpy(), scale=0.21)
    np.testing.assert_allclose(O, _sdpa_ref(so, co, U, T, W, b, act, 0.21), rtol=1e-12,
                               atol=1e-12)


@pytest.mark.parametrize("act", [0, 1])
def test_nro_bias_vs_sdpa(act):
    """nro_cross_attention's b_q/b_k/b_v: slot s = a head with the gate folded into x."""
    so, co, U, T, W, b = _problem(15)
    (Wq, Wk, Wv), (bq, bk, bv) = W, b
    g = torch.linspace(0.3, 1.7, T.shape[1], dtype=torch.float64).repeat(H, 1)
    got = oracle.nro_cross_attention(T, co, Wq, g, U, so, Wk, Wv, H, D, act=act,
                                     b_q=bq.numpy(), b_k=bk.numpy(), b_v=bv.numpy(), scale=0.4)
    Tg = T.to(torch.float64)
    ref = np.zeros_like(got)
    for s in range(H):
        sl = slice(s * D, (s + 1) * D)
        q = _lin(Tg * g[s], Wq[sl], bq[sl], act)
        k, v = _lin(U, Wk[sl], bk[sl], act), _lin(U, Wv[sl], bv[sl], act)
        for i in range(len(so) - 1):
            r0, r1, c0, c1 = int(so[i]), int(so[i + 1]), int(co[i]), int(co[i + 1])
            if c1 > c0 and r1 > r0:
                ref[c0:c1, sl] = torch.nn.functional.scaled_dot_product_attention(
                    q[c0:c1][None], k[r0:r1][None], v[r0:r1][None], scale=0.4)[0].numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("act", [0, 1])
def test_history_bias_vs_causal_sdpa(act):
    so, co, U, T, W, b = _problem(16)
    (Wq, Wk, Wv), (bq, bk, bv) = W, b
    O, _ = oracle.history_attention(U, so, Wq, Wk, Wv, H, D, act=act, b_q=bq.numpy(),
                                    b_k=bk.numpy(), b_v=bv.numpy(), scale=0.35)
    Q, K, V = _lin(U, Wq, bq, act), _lin(U, Wk, bk, act), _lin(U, Wv, bv, act)
    ref = np.zeros_like(O)
    for i in range(len(so) - 1):
        r0, r1 = int(so[i]), int(so[i + 1])
        if r1 > r0:
            o = torch.nn.functional.scaled_dot_product_attention(
                _heads(Q[r0:r1]), _heads(K[r0:r1]), _heads(V[r0:r1]), is_causal=True, scale=0.35)
            ref[r0:r1] = o.transpose(0, 1).reshape(r1 - r0, H * D).numpy()
    np.testing.assert_allclose(O, ref, rtol=1e-12, atol=1e-12)
