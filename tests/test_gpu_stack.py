"""GPU parity of a stack of full target-aware STU layers (binding.stu_stack: gesr_layer_norm,
gesr_kv_project, gesr_history_attention, gesr_tasa_score_self, gesr_stu_output per layer;
SPEC.md:298/343, reading R18) against the brute-force fp64 oracle
(oracle.stu_stack_forward over the (N+n)^2 mask of every request).

Tolerance (R18): every layer stores its normalised input, K/V, Q, P, the gate and the
output in bf16, so a layer's output carries the attention's north_star error (max-abs 2e-2,
mean-abs 2e-3 on O) through LayerNorm, the gate and W_o plus the bf16 rounding of Y (half an ulp:
|Y| 2^-9).  Gate per layer count n_l: max |Y_gpu - Y| <= n_l * (3e-2 + 2^-8 max|Y|) and
mean-abs <= n_l * 3e-3.
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


def _case(Ls, Cs, H, d, n_layers, seed):
    g = torch.Generator().manual_seed(seed)
    D = H * d
    so = torch.tensor(np.concatenate([[0], np.cumsum(Ls)]), dtype=torch.int64)
    co = torch.tensor(np.concatenate([[0], np.cumsum(Cs)]), dtype=torch.int64)
    U = torch.randn(int(so[-1]), D, generator=g).to(torch.bfloat16)
    T = torch.randn(int(co[-1]), D, generator=g).to(torch.bfloat16)
    a = (6.0 / (2 * D)) ** 0.5
    layers = []
    for _ in range(n_layers):
        w = lambda: ((torch.rand(D, D, generator=g) * 2 - 1) * a).to(torch.bfloat16)   # noqa
        layers.append(dict(W_q=w(), W_k=w(), W_v=w(), W_g=w(), W_o=w(),
                           ln_in=(torch.rand(D, generator=g) + 0.5, torch.randn(D, generator=g) * 0.1),
                           ln_out=(torch.rand(D, generator=g) + 0.5,
                                   torch.randn(D, generator=g) * 0.1)))
    return U, T, so, co, layers


def _run(U, T, so, co, layers, H, d):
    dev = _cuda()
    mv = lambda x: tuple(mv(y) for y in x) if isinstance(x, tuple) else x.to(dev)   # noqa
    lay_d = [{k: mv(v) for k, v in lay.items()} for lay in layers]
    Uo, To = gb.stu_stack(U.to(dev), T.to(dev), so.to(dev), co.to(dev), lay_d, H, d)
    torch.cuda.synchronize()
    return Uo.float().cpu().double().numpy(), To.float().cpu().double().numpy()


def _check(got, want, n_layers, what):
    err = np.abs(got - want)
    assert np.isfinite(got).all(), what
    lim = n_layers * (3e-2 + 2.0 ** -8 * np.abs(want).max())
    print(f"{what}: max-abs {err.max():.3e} (limit {lim:.3e}) mean-abs {err.mean():.3e}")
    assert err.max() <= lim and err.mean() <= n_layers * 3e-3, \
        f"{what}: max-abs {err.max():.3e} mean-abs {err.mean():.3e}"


@pytest.mark.parametrize("H,d,n_layers", [(1, 32, 1), (2, 64, 2), (4, 128, 2)])
def test_stack_parity(H, d, n_layers):
    # jagged: an empty history, a single row, tile and unit boundaries; C_b = 1 and ragged
    Ls, Cs = [0, 1, 37, 300, 700], [3, 1, 130, 257, 40]
    U, T, so, co, layers = _case(Ls, Cs, H, d, n_layers, seed=H * 10 + d)
    Uo, To = _run(U, T, so, co, layers, H, d)
    Uw, Tw = oracle.stu_stack_forward(U, T, so, co, layers, H, d)
    _check(Uo, Uw, n_layers, f"U rows H={H} d={d} layers={n_layers}")
    _check(To, Tw, n_layers, f"T rows H={H} d={d} layers={n_layers}")


def test_stack_candidate_isolation_exact():
    # editing one candidate leaves every other row of the stack bit-identical
    U, T, so, co, layers = _case([300, 64], [20, 9], 2, 64, 2, seed=7)
    Uo, To = _run(U, T, so, co, layers, 2, 64)
    T2 = T.clone()
    T2[5] = -T2[5]
    Uo2, To2 = _run(U, T2, so, co, layers, 2, 64)
    keep = np.ones(To.shape[0], bool)
    keep[5] = False
    assert np.array_equal(To2[keep], To[keep]) and np.array_equal(Uo2, Uo)
