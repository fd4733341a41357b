"""GPU parity of gesr_stu_output (the STU layer's candidate row after the
attention -- gating branch, layer norm of attention.value, output projection, residual;
SPEC.md:343, reading R15) against the fp64 oracle (oracle.stu_output).

Tolerance (DESIGN.md s3 R15), derived from the arithmetic: G and the normalised, gated rows
N(.)G are rounded to bf16 (relative error <= 2^-9 each) before the output projection, and Y is
rounded to bf16, so elementwise
  |Y_gpu - Y_oracle| <= 2^-8 |Y_oracle| + 2^-8 sum_j |W_o[i][j]| |N_j G_j|
(worst case, fp32 accumulation being far below it).  The tight check is against the oracle's
diagnostic rounding-aware mode (the same three roundings in fp64): fewer than 2 % of the
elements may differ at all (rounding flips: fp32 on the GPU vs fp64 there), each by at most two
ulps of Y plus two upstream flips in G or N(.)G -- an indexing or arithmetic bug in the kernels
moves nearly every element and fails it.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_21095_b200 import binding as gb

pytestmark = pytest.mark.gpu


def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200 (run through gpurun)"
    return torch.device("cuda:0")


def _weights(C, D_in, H, d, D_out, seed, biases=True, residual=True, o_dtype=torch.float32):
    g = torch.Generator().manual_seed(seed)
    D = H * d

    def xavier(n_out, n_in):
        a = (6.0 / (n_in + n_out)) ** 0.5
        return ((torch.rand(n_out, n_in, generator=g) * 2 - 1) * a).to(torch.bfloat16)

    w = dict(
        T=torch.randn(C, D_in, generator=g).to(torch.bfloat16),
        # attention.value rows: convex combinations of SiLU'd values, mean ~0.3, spread ~0.5
        O=(torch.randn(C, D, generator=g) * 0.5 + 0.3).to(o_dtype),
        W_g=xavier(D, D_in),
        ln_gamma=torch.rand(D, generator=g) + 0.5,
        ln_beta=torch.randn(D, generator=g) * 0.1,
        W_o=xavier(D_out, D),
        b_g=torch.randn(D, generator=g) * 0.1 if biases else None,
        b_o=torch.randn(D_out, generator=g) * 0.1 if biases else None,
        X_res=torch.randn(C, D_out, generator=g).to(torch.bfloat16) if residual else None,
    )
    return w


def _oracle(w, rows=None, eps=1e-5, round_bf16=False, parts=False):
    sel = (lambda t: t) if rows is None else (lambda t: t[rows])
    return oracle.stu_output(sel(w["T"]), sel(w["O"]), w["W_g"], w["ln_gamma"], w["ln_beta"],
                             w["W_o"], b_g=w["b_g"], b_o=w["b_o"],
                             X_res=None if w["X_res"] is None else sel(w["X_res"]), eps=eps,
                             round_bf16=round_bf16, parts=parts)


def _gpu(w, H, d, eps=1e-5):
    dev = _cuda()
    g = {k: (None if v is None else v.to(dev)) for k, v in w.items()}
    Y = gb.stu_output(g["T"], g["O"], g["W_g"], g["ln_gamma"], g["ln_beta"], g["W_o"], H, d,
                      b_g=g["b_g"], b_o=g["b_o"], X_res=g["X_res"], ln_eps=eps)
    torch.cuda.synchronize()
    return Y


def _bf16_ulp(x):
    ax = np.maximum(np.abs(x), 2.0 ** -126)
    return 2.0 ** (np.floor(np.log2(ax)) - 7)


def _check(Y_gpu, w, what, rows=None):
    got = Y_gpu.float().cpu().double().numpy()
    assert np.isfinite(got).all(), what
    Y, N, G = _oracle(w, rows=rows, parts=True)
    W_o = w["W_o"].double().numpy()
    bound = 2.0 ** -8 * np.abs(Y) + 2.0 ** -8 * (np.abs(N * G) @ np.abs(W_o).T) + 1e-6
    err = np.abs(got - Y)
    bad = err > bound
    assert not bad.any(), f"{what}: {bad.sum()} elements beyond the bf16 bound, max {err.max():.3e}"
    Yr = _oracle(w, rows=rows, round_bf16=True)
    err_r = np.abs(got - Yr)
    # two ulps of Y for rounding flips of Y itself, plus two flips upstream: an element of G or
    # N*G evaluated in fp32 on the GPU (fp64 here) landing on the other side of a bf16 rounding
    # boundary moves Y[t][i] by <= |W_o[i][j]| ulp(Z[t][j]) <= 2^-7 max|Z[t]| max|W_o[i]|
    Zmax = np.abs(N * G).max(axis=1, keepdims=True)
    Wmax = np.abs(W_o).max(axis=1)[None, :]
    flips = 2 * 2.0 ** -7 * Zmax * Wmax
    bad = err_r > 2 * _bf16_ulp(Yr) + flips
    assert not bad.any(), (f"{what}: {bad.sum()} elements off the rounding-aware oracle, "
                           f"max {err_r.max():.3e}")
    assert np.mean(err_r > 0) < 0.02, f"{what}: too many rounding flips {np.mean(err_r > 0):.3f}"


@pytest.mark.parametrize("H,d,D_in", [(1, 32, 32), (2, 64, 128), (4, 128, 512)])
@pytest.mark.parametrize("o_dtype", [torch.float32, torch.bfloat16])
def test_stu_output_parity(H, d, D_in, o_dtype):
    # 600 rows: two full 256-row pair tiles and a ragged tail; D_out = D_in (residual)
    w = _weights(600, D_in, H, d, D_in, seed=H * 100 + d, o_dtype=o_dtype)
    _check(_gpu(w, H, d), w, f"H={H} d={d} {o_dtype}")


def test_stu_output_nonsquare_no_bias_no_residual():
    # D_out (96) != D (128) != D_in (64): a transposed operand cannot pass
    w = _weights(333, 64, 2, 64, 96, seed=7, biases=False, residual=False)
    _check(_gpu(w, 2, 64), w, "non-square")


def test_stu_output_zero_projection_returns_residual_exactly():
    w = _weights(300, 128, 2, 64, 128, seed=9, biases=False)
    w["W_o"] = torch.zeros_like(w["W_o"])
    Y = _gpu(w, 2, 64)
    assert torch.equal(Y.cpu(), w["X_res"])


def test_stu_output_rows_independent_exact():
    # a row's result does not depend on the batch it is computed in (bit-identical)
    w = _weights(700, 128, 2, 64, 128, seed=11)
    Y = _gpu(w, 2, 64)
    sub = {k: (v if (v is None or v.dim() == 1 or v.shape[0] != 700) else v[123:456].contiguous())
           for k, v in w.items()}
    Y2 = _gpu(sub, 2, 64)
    assert torch.equal(Y[123:456], Y2)


def test_stu_output_headline_size_sampled():
    # ESR dims at the headline row count (1024 requests x 1000 candidates, H=4, d=128,
    # D_in = D_out = 512); 2048 sampled rows against the oracle
    C = 1024 * 1000
    w = _weights(C, 512, 4, 128, 512, seed=13, o_dtype=torch.bfloat16)
    Y = _gpu(w, 4, 128)
    rows = np.sort(np.random.default_rng(0).choice(C, 2048, replace=False))
    rows = np.concatenate([rows, [0, C - 1]])
    _check(Y[torch.as_tensor(rows, device=Y.device)], w, "headline sampled",
           rows=torch.as_tensor(rows))


def test_stu_output_edges():
    dev = _cuda()
    w = _weights(8, 64, 1, 64, 64, seed=3)
    g = {k: (None if v is None else v.to(dev)) for k, v in w.items()}
    # total_C = 0: no-op
    Y0 = gb.stu_output(g["T"][:0], g["O"][:0], g["W_g"], g["ln_gamma"], g["ln_beta"], g["W_o"],
                       1, 64)
    assert Y0.shape == (0, 64)
    # too-small workspace
    with pytest.raises(gb.GesrError) as e:
        gb.stu_output(g["T"], g["O"], g["W_g"], g["ln_gamma"], g["ln_beta"], g["W_o"], 1, 64,
                      workspace=torch.empty(256, dtype=torch.uint8, device=dev))
    assert e.value.status == gb.GESR_ERR_WORKSPACE
