"""Timing of gesr_stu_output at the headline row count (1024 x 1000 candidate
rows, H=4, d=128, D_in = D_out = 512, O bf16), CUDA events around the C-ABI call, inputs
resident in HBM (larger than L2).  Prints one JSON line with ms, TFLOP/s, GB/s and the
per-kernel roofline time (max(flop/P, bytes/BW) summed over the three kernels).

    python scripts/stu_bench.py [--iters 20]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_21095_b200 import binding as gb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--rows", type=int, default=1024 * 1000)
    args = ap.parse_args()
    dev = torch.device("cuda")
    C, D_in, H, d, D_out = args.rows, 512, 4, 128, 512
    D = H * d
    g = torch.Generator(device=dev).manual_seed(1)
    T = torch.randn(C, D_in, device=dev, generator=g).to(torch.bfloat16)
    O = (torch.randn(C, D, device=dev, generator=g) * 0.5 + 0.3).to(torch.bfloat16)
    W_g = ((torch.rand(D, D_in, device=dev, generator=g) * 2 - 1) * 0.077).to(torch.bfloat16)
    W_o = ((torch.rand(D_out, D, device=dev, generator=g) * 2 - 1) * 0.077).to(torch.bfloat16)
    gam = torch.rand(D, device=dev, generator=g) + 0.5
    bet = torch.randn(D, device=dev, generator=g) * 0.1
    X = torch.randn(C, D_out, device=dev, generator=g).to(torch.bfloat16)
    Y = torch.empty(C, D_out, device=dev, dtype=torch.bfloat16)
    ws = torch.empty(gb.stu_workspace_bytes(C, H, d), dtype=torch.uint8, device=dev)

    def call():
        gb.stu_output(T, O, W_g, gam, bet, W_o, H, d, X_res=X, Y=Y, workspace=ws)

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.iters):
        call()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.iters
    flop = 2.0 * C * D_in * D + 2.0 * C * D * D_out
    # algorithmic bytes per kernel: G GEMM (T in, G out), LN-gate (O, G in, Z out), W_o GEMM
    # (Z, X_res in, Y out); weights negligible
    b_g = 2.0 * C * (D_in + D)
    b_ln = 2.0 * C * (D + D + D)
    b_o = 2.0 * C * (D + D_out + D_out)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    P = float(peaks.get("bf16_tflops_sustained", 1378.5)) * 1e12
    BW = float(peaks.get("hbm_gbs", 6549.8)) * 1e9
    roof = (max(2.0 * C * D_in * D / P, b_g / BW) + b_ln / BW +
            max(2.0 * C * D * D_out / P, b_o / BW)) * 1e3
    print(json.dumps({"op": "gesr_stu_output", "rows": C, "ms": ms,
                      "tflops": flop / ms / 1e9, "gbs": (b_g + b_ln + b_o) / ms / 1e6,
                      "roof_ms": roof, "frac": roof / ms, "peaks": {"tflops": P / 1e12,
                                                                    "gbs": BW / 1e9}}))


if __name__ == "__main__":
    main()
