"""Timing of gesr_history_attention at ESR dims: B requests of L history rows
(default 1024 x 2048), H=4, d=128, D_in=512, K/V cache from gesr_kv_project (not timed), CUDA
events around the C-ABI call (Q projection + causal attention).  Prints one JSON line with ms,
the algorithmic TFLOP/s (causal: sum_p (p+1) keys per row) and the fraction of the sustained
bf16 peak.

    python scripts/history_bench.py [--B 1024] [--L 2048] [--iters 10]
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
    ap.add_argument("--B", type=int, default=1024)
    ap.add_argument("--L", type=int, default=2048)
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda")
    B, L, H, d, D_in = args.B, args.L, 4, 128, 512
    g = torch.Generator(device=dev).manual_seed(2)
    U = torch.randn(B * L, D_in, device=dev, generator=g).to(torch.bfloat16)
    a = (6.0 / (D_in + H * d)) ** 0.5
    W = [((torch.rand(H * d, D_in, device=dev, generator=g) * 2 - 1) * a).to(torch.bfloat16)
         for _ in range(3)]
    so = torch.arange(B + 1, device=dev, dtype=torch.int64) * L
    K, V = gb.kv_project(U, W[1], W[2], H, d, 1)
    O = torch.empty(B * L, H * d, device=dev, dtype=torch.bfloat16)
    ws = torch.empty(gb.tasa_workspace_bytes(B, B * L, H, d, 1), dtype=torch.uint8, device=dev)

    def call():
        gb.history_attention(U, so, W[0], K, V, H, d, 1, O=O, workspace=ws)

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.iters
    keys = B * L * (L + 1) / 2                     # sum over rows of the keys each row sees
    flop = 4.0 * keys * H * d + 2.0 * B * L * D_in * H * d
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    P = json.load(open(peaks_path)).get("bf16_tflops_sustained", 1378.5) \
        if os.path.exists(peaks_path) else 1378.5
    print(json.dumps({"op": "gesr_history_attention", "B": B, "L": L, "H": H, "d": d,
                      "ms": ms, "tflops": flop / ms / 1e9, "frac_sustained": flop / ms / 1e9 / P,
                      "rows_per_s": B * L / ms * 1e3}))


if __name__ == "__main__":
    main()
