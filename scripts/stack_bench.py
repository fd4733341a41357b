"""Timing of a stack of full STU layers (binding.stu_stack; R18) at ESR dims: B
requests of L history rows and C candidates (default 1024 x 2048 x 1000), H=4, d=128 (D=512),
n layers (default 2).  CUDA events around the whole stack; prints ms, rows/s, candidates/s and
the algorithmic TFLOP/s (projections Q/K/V/G/O over all rows, causal history attention, the
candidates' attention over the history and their own key).

    python scripts/stack_bench.py [--B 1024] [--L 2048] [--C 1000] [--layers 2] [--iters 5]
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
    ap.add_argument("--C", type=int, default=1000)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    dev = torch.device("cuda")
    B, L, C, H, d = args.B, args.L, args.C, 4, 128
    D = H * d
    g = torch.Generator(device=dev).manual_seed(3)
    U = torch.randn(B * L, D, device=dev, generator=g).to(torch.bfloat16)
    T = torch.randn(B * C, D, device=dev, generator=g).to(torch.bfloat16)
    so = torch.arange(B + 1, device=dev, dtype=torch.int64) * L
    co = torch.arange(B + 1, device=dev, dtype=torch.int64) * C
    a = (6.0 / (2 * D)) ** 0.5
    w = lambda: ((torch.rand(D, D, device=dev, generator=g) * 2 - 1) * a).to(torch.bfloat16)  # noqa
    layers = [dict(W_q=w(), W_k=w(), W_v=w(), W_g=w(), W_o=w(),
                   ln_in=(torch.ones(D, device=dev), torch.zeros(D, device=dev)),
                   ln_out=(torch.ones(D, device=dev), torch.zeros(D, device=dev)))
              for _ in range(args.layers)]

    def call():
        gb.stu_stack(U, T, so, co, layers, H, d)

    for _ in range(2):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.iters
    rows = B * (L + C)
    proj = 2.0 * rows * D * D * 5 + 2.0 * B * C * D * D      # Q, K, V, G, O (+ K/V of T rows)
    attn = 4.0 * B * (L * (L + 1) / 2 + C * (L + 1)) * D
    flop = args.layers * (proj + attn)
    print(json.dumps({"op": "stu_stack", "layers": args.layers, "B": B, "L": L, "C": C, "H": H,
                      "d": d, "ms": ms, "cand_per_s": B * C / ms * 1e3,
                      "rows_per_s": rows / ms * 1e3, "tflops": flop / ms / 1e9}))


if __name__ == "__main__":
    main()
