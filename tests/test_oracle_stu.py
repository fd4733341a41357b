"""Pins for oracle.stu_output (reading R15).

The oracle is checked against things other than itself:
  * the same layer assembled from torch library routines in fp64 (layer_norm, silu, linear);
  * a pure-Python scalar evaluation on a tiny non-square case (D_out != D != D_in), so a
    transposed W_g / W_o or a swapped axis cannot pass;
  * closed forms: a zero output projection returns the residual exactly; a zero gating weight
    gives G = SiLU(b_g) and, with W_o = I, rows of mean 0 and variance SiLU(b_g)^2 var/(var+eps);
  * the layer-norm invariance under O -> a O + b (a > 0, eps = 0).
"""
import math

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.filterwarnings("ignore::DeprecationWarning")


def _case(C=5, D_in=12, D=16, D_out=8, seed=0):
    rng = np.random.default_rng(seed)
    return dict(
        T=rng.standard_normal((C, D_in)),
        O=rng.standard_normal((C, D)) * 0.7 + 0.3,
        W_g=rng.standard_normal((D, D_in)) * 0.3,
        gamma=rng.uniform(0.5, 1.5, D),
        beta=rng.standard_normal(D) * 0.1,
        W_o=rng.standard_normal((D_out, D)) * 0.3,
        b_g=rng.standard_normal(D) * 0.1,
        b_o=rng.standard_normal(D_out) * 0.1,
        X_res=rng.standard_normal((C, D_out)),
    )


def test_matches_torch_library_composition():
    c = _case()
    t = {k: torch.tensor(v, dtype=torch.float64) for k, v in c.items()}
    G = torch.nn.functional.silu(torch.nn.functional.linear(t["T"], t["W_g"], t["b_g"]))
    N = torch.nn.functional.layer_norm(t["O"], (t["O"].shape[1],), t["gamma"], t["beta"],
                                       eps=1e-5)
    want = torch.nn.functional.linear(N * G, t["W_o"], t["b_o"]) + t["X_res"]
    got = oracle.stu_output(c["T"], c["O"], c["W_g"], c["gamma"], c["beta"], c["W_o"],
                            b_g=c["b_g"], b_o=c["b_o"], X_res=c["X_res"], eps=1e-5)
    np.testing.assert_allclose(got, want.numpy(), rtol=0, atol=1e-12)


def test_matches_scalar_python_on_nonsquare_case():
    c = _case(C=3, D_in=5, D=6, D_out=4, seed=3)
    eps = 1e-3
    C, D_in = c["T"].shape
    D, D_out = c["O"].shape[1], c["W_o"].shape[0]
    want = np.zeros((C, D_out))
    for t in range(C):
        g = []
        for j in range(D):
            z = sum(c["T"][t][k] * c["W_g"][j][k] for k in range(D_in)) + c["b_g"][j]
            g.append(z / (1.0 + math.exp(-z)))
        mu = sum(c["O"][t]) / D
        var = sum((x - mu) ** 2 for x in c["O"][t]) / D
        n = [(c["O"][t][j] - mu) / math.sqrt(var + eps) * c["gamma"][j] + c["beta"][j]
             for j in range(D)]
        for i in range(D_out):
            want[t][i] = (sum(n[j] * g[j] * c["W_o"][i][j] for j in range(D)) + c["b_o"][i]
                          + c["X_res"][t][i])
    got = oracle.stu_output(c["T"], c["O"], c["W_g"], c["gamma"], c["beta"], c["W_o"],
                            b_g=c["b_g"], b_o=c["b_o"], X_res=c["X_res"], eps=eps)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)


def test_zero_output_projection_returns_residual_exactly():
    c = _case()
    got = oracle.stu_output(c["T"], c["O"], c["W_g"], c["gamma"], c["beta"],
                            np.zeros_like(c["W_o"]), b_g=c["b_g"], X_res=c["X_res"])
    assert np.array_equal(got, c["X_res"])
    got = oracle.stu_output(c["T"], c["O"], c["W_g"], c["gamma"], c["beta"],
                            np.zeros_like(c["W_o"]), b_g=c["b_g"], b_o=c["b_o"])
    assert np.array_equal(got, np.broadcast_to(c["b_o"], got.shape))


def test_constant_gate_identity_projection_normalises_rows():
    c = _case(D=16, D_out=16)
    bg = 0.8
    eps = 1e-5
    got = oracle.stu_output(c["T"], c["O"], np.zeros_like(c["W_g"]), np.ones(16), np.zeros(16),
                            np.eye(16), b_g=np.full(16, bg), eps=eps)
    s = bg / (1.0 + math.exp(-bg))
    var = c["O"].var(axis=1)
    np.testing.assert_allclose(got.mean(axis=1), 0.0, atol=1e-13)
    np.testing.assert_allclose(got.var(axis=1), s * s * var / (var + eps), rtol=1e-12)


def test_zero_gate_weight_without_bias_kills_the_attention_term():
    c = _case()
    got = oracle.stu_output(c["T"], c["O"], np.zeros_like(c["W_g"]), c["gamma"], c["beta"],
                            c["W_o"], b_o=c["b_o"], X_res=c["X_res"])
    np.testing.assert_allclose(got, c["X_res"] + c["b_o"][None, :], rtol=0, atol=0)


def test_layer_norm_affine_invariance():
    c = _case()
    kw = dict(b_g=c["b_g"], b_o=c["b_o"], X_res=c["X_res"], eps=0.0)
    a = oracle.stu_output(c["T"], c["O"], c["W_g"], c["gamma"], c["beta"], c["W_o"], **kw)
    b = oracle.stu_output(c["T"], 3.5 * c["O"] - 2.0, c["W_g"], c["gamma"], c["beta"], c["W_o"],
                          **kw)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)


def test_identity_activation_and_bf16_bits_input():
    c = _case()
    T16 = torch.tensor(c["T"], dtype=torch.bfloat16)
    a = oracle.stu_output(T16, c["O"], c["W_g"], c["gamma"], c["beta"], c["W_o"], act=0)
    # bf16 widened exactly: the same as passing the fp64 value of the rounded tensor
    b = oracle.stu_output(T16.double().numpy(), c["O"], c["W_g"], c["gamma"], c["beta"],
                          c["W_o"], act=0)
    assert np.array_equal(a, b)
    # identity gate: G = T W_g^T exactly
    N = (c["O"] - c["O"].mean(1, keepdims=True)) / np.sqrt(c["O"].var(1, keepdims=True) + 1e-5)
    want = (N * c["gamma"] + c["beta"]) * (T16.double().numpy() @ c["W_g"].T) @ c["W_o"].T
    np.testing.assert_allclose(a, want, rtol=0, atol=1e-12)


def test_rounding_aware_mode_within_the_bf16_bound():
    # diagnostic mode: G, N*G and Y rounded to bf16; differs from fp64 by at most the rounding
    # bound the GPU tolerance uses, and equals it where nothing rounds (zero gate: Y = X_res
    # with bf16-exact residual and no output bias)
    c = _case(C=40, D_in=32, D=64, D_out=48, seed=5)
    kw = dict(b_g=c["b_g"], b_o=c["b_o"], X_res=c["X_res"])
    Y, N, G = oracle.stu_output(c["T"], c["O"], c["W_g"], c["gamma"], c["beta"], c["W_o"],
                                parts=True, **kw)
    Yr = oracle.stu_output(c["T"], c["O"], c["W_g"], c["gamma"], c["beta"], c["W_o"],
                           round_bf16=True, **kw)
    assert not np.array_equal(Y, Yr)
    bound = 2.0 ** -8 * np.abs(Y) + 2.0 ** -8 * (np.abs(N * G) @ np.abs(c["W_o"]).T)
    assert (np.abs(Yr - Y) <= bound).all()
    X16 = torch.tensor(c["X_res"]).to(torch.bfloat16).double().numpy()
    Yz = oracle.stu_output(c["T"], c["O"], np.zeros_like(c["W_g"]), c["gamma"], c["beta"],
                           c["W_o"], X_res=X16, round_bf16=True)
    assert np.array_equal(Yz, X16)
