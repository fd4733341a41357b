"""Debug: gesr_stu_output vs the fp64 oracle and a rounding-aware emulation (G, Z, Y -> bf16)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from test_gpu_stu import _weights, _gpu, _oracle  # noqa: E402


def bf(x):
    return torch.tensor(x).to(torch.bfloat16).double().numpy()


for (H, d, D_in) in [(1, 32, 32), (2, 64, 128)]:
    w = _weights(600, D_in, H, d, D_in, seed=H * 100 + d)
    Y = _gpu(w, H, d).float().cpu().double().numpy()
    Yo = _oracle(w)
    f = {k: (None if v is None else v.double().numpy()) for k, v in w.items()}
    Gp = f["T"] @ f["W_g"].T + f["b_g"]
    G = bf(Gp / (1 + np.exp(-Gp)))
    O = f["O"]
    mu = O.mean(1, keepdims=True)
    var = ((O - mu) ** 2).mean(1, keepdims=True)
    N = (O - mu) / np.sqrt(var + 1e-5) * f["ln_gamma"] + f["ln_beta"]
    Z = bf(N * G)
    Ye = bf(Z @ f["W_o"].T + f["b_o"] + f["X_res"])
    e1 = np.abs(Y - Yo)
    e2 = np.abs(Y - Ye)
    i = np.unravel_index(e1.argmax(), e1.shape)
    print(f"H={H} d={d}: vs fp64 max {e1.max():.3e} mean {e1.mean():.3e} at {i} Y={Y[i]:.4f} "
          f"Yo={Yo[i]:.4f} Ye={Ye[i]:.4f}; vs emulation max {e2.max():.3e} mean {e2.mean():.3e} "
          f"frac>0 {np.mean(e2 > 0):.3f}; |Z| max {np.abs(Z).max():.2f} |Y| max {np.abs(Yo).max():.2f}")
    # error of the emulation itself against fp64
    e3 = np.abs(Ye - Yo)
    print(f"   emulation vs fp64: max {e3.max():.3e} mean {e3.mean():.3e}")
    rows_bad = np.where((e1 > 2 ** -8 * np.abs(Yo) + 4e-3).any(1))[0]
    cols_bad = np.where((e1 > 2 ** -8 * np.abs(Yo) + 4e-3).any(0))[0]
    print("   bad rows", rows_bad[:20], len(rows_bad), "bad cols", cols_bad[:20], len(cols_bad))
