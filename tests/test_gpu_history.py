"""GPU parity of gesr_history_attention (causal self-attention of each user's
history over itself; PAPER.md:341 rule (1); reading R17) against the fp64
oracle (oracle.history_attention) on the same seeded inputs.  Gate: the attention tolerance of
BASELINE.json north_star (max-abs 2e-2, mean-abs 2e-3 vs pure fp64).  Both kernels are covered:
the CTA-pair kernel (d = 128) and the 1-CTA kernel (d = 32 / 64, and d = 128 with
GESR_ATTN_PAIR=0 in a subprocess).
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
from paper_2511_21095_b200 import binding as gb
from paper_2511_21095_b200 import configs, inputs

pytestmark = pytest.mark.gpu

MAX_ABS, MEAN_ABS = 2e-2, 2e-3
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200 (run through gpurun)"
    return torch.device("cuda:0")


def _batch(Ls, H, d, D_in, seed=3):
    cfg = configs.Config("hist", 90 + seed, B=len(Ls), L=("fixed", 1), C=("fixed", 1), H=H, d=d,
                         D_in=D_in, F=4)
    bt = inputs.make_batch(cfg, hma=False)
    g = torch.Generator().manual_seed(seed)
    so = torch.tensor(np.concatenate([[0], np.cumsum(Ls)]), dtype=torch.int64)
    U = torch.randn(int(so[-1]), D_in, generator=g).to(torch.bfloat16)
    return cfg, U, so, bt.W_q, bt.W_k, bt.W_v


def _gpu(U, so, W_q, W_k, W_v, H, d, act=1, out_dtype=torch.float32):
    dev = _cuda()
    U, so, W_q, W_k, W_v = (t.to(dev) for t in (U, so, W_q, W_k, W_v))
    K, V = gb.kv_project(U, W_k, W_v, H, d, act)
    O, lse = gb.history_attention(U, so, W_q, K, V, H, d, act, out_dtype=out_dtype,
                                  want_lse=True)
    torch.cuda.synchronize()
    return O.float().cpu().double().numpy(), lse.cpu().double().numpy()


def _tol(got, want, what):
    diff = np.abs(got - want)
    assert np.isfinite(got).all(), what
    assert diff.max() <= MAX_ABS and diff.mean() <= MEAN_ABS, \
        f"{what}: max-abs {diff.max():.3e} mean-abs {diff.mean():.3e}"


# jagged lengths: empty, single row, < one 128-key tile, exactly 256 (one unit), ragged over
# several units (the diagonal crossing tile and unit boundaries), long
LENS = [0, 1, 37, 128, 256, 300, 513, 1100]


@pytest.mark.parametrize("H,d,D_in", [(1, 32, 32), (2, 64, 128), (2, 128, 256)])
@pytest.mark.parametrize("act", [0, 1])
def test_history_parity(H, d, D_in, act):
    cfg, U, so, W_q, W_k, W_v = _batch(LENS, H, d, D_in)
    O, lse = _gpu(U, so, W_q, W_k, W_v, H, d, act)
    O_or, lse_or = oracle.history_attention(U, so, W_q, W_k, W_v, H, d, act=act)
    _tol(O, O_or, f"H={H} d={d} act={act}")
    ok = np.isfinite(lse_or)
    np.testing.assert_allclose(lse[ok], lse_or[ok], rtol=0, atol=5e-2)


def test_history_first_rows_and_bf16_out():
    # row 0 of each request attends to itself only: O = its bf16 V row exactly (p = 1, l = 1)
    cfg, U, so, W_q, W_k, W_v = _batch([5, 130, 260], 2, 128, 256, seed=4)
    dev = _cuda()
    K, V = gb.kv_project(U.to(dev), W_k.to(dev), W_v.to(dev), 2, 128, 1)
    O, _ = gb.history_attention(U.to(dev), so.to(dev), W_q.to(dev), K, V, 2, 128, 1)
    torch.cuda.synchronize()
    for b in range(3):
        r = int(so[b])
        want = torch.cat([V[h, r] for h in range(2)]).float()
        assert torch.equal(O[r], want)
    Ob, _ = _gpu(U, so, W_q, W_k, W_v, 2, 128, 1, out_dtype=torch.bfloat16)
    O_or, _ = oracle.history_attention(U, so, W_q, W_k, W_v, 2, 128, act=1)
    _tol(Ob, O_or, "bf16 out")


def test_history_causality_exact():
    # editing a later history row leaves every earlier row's output bit-identical
    cfg, U, so, W_q, W_k, W_v = _batch([700], 2, 128, 256, seed=5)
    O1, _ = _gpu(U, so, W_q, W_k, W_v, 2, 128)
    U2 = U.clone()
    U2[400] = -U2[400]
    O2, _ = _gpu(U2, so, W_q, W_k, W_v, 2, 128)
    assert np.array_equal(O1[:400], O2[:400])
    assert not np.array_equal(O1[400], O2[400])


def test_history_one_cta_kernel_d128_subprocess():
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r);"
            "import test_gpu_history as t; t.test_history_parity(2, 128, 256, 1)"
            % (ROOT, os.path.join(ROOT, "tests")))
    env = dict(os.environ, GESR_ATTN_PAIR="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
