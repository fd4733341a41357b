"""Fused embedding lookup + K/V projection (gesr_kv_project_gather) vs lookup then projection,
at the headline's history size (ΣL = 1024 x 2048 rows, D_in = 512, H = 4, d = 128).

    python scripts/gather_bench.py [--table-rows 8000000] [--iters 20]

(a) gesr_kv_project_gather(E, rows)          -- TMA gather4 straight into the GEMM's operand tiles
(b) U = E.index_select(0, rows); kv_project  -- the lookup materialised in HBM first
(c) kv_project(U) on an already materialised U (the headline's K/V step)
Prints one JSON line of CUDA-event times (ms per call, mean over --iters back-to-back calls).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_21095_b200 import binding as gb  # noqa: E402
from paper_2511_21095_b200 import configs, inputs  # noqa: E402


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--table-rows", type=int, default=8_000_000)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = configs.get("3h")
    H, d, D_in = cfg.H, cfg.d, cfg.D_in
    M = cfg.B * 2048
    W = inputs.make_batch(cfg.with_(B=1), hma=False, device=dev)
    g = torch.Generator(device=dev).manual_seed(1)
    E = torch.randn(args.table_rows, D_in, generator=g, device=dev).to(torch.bfloat16)
    rows = torch.randint(0, args.table_rows, (M,), generator=g, device=dev, dtype=torch.int32)
    K = torch.empty((H, M, d), dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    U = torch.empty((M, D_in), dtype=torch.bfloat16, device=dev)
    rows64 = rows.long()

    def fused():
        gb.kv_project_gather(E, rows, W.W_k, W.W_v, H, d, cfg.act, K_cache=K, V_cache=V)

    def lookup_then_project():
        torch.index_select(E, 0, rows64, out=U)
        gb.kv_project(U, W.W_k, W.W_v, H, d, cfg.act, K_cache=K, V_cache=V)

    def lookup_only():
        torch.index_select(E, 0, rows64, out=U)

    def project_only():
        gb.kv_project(U, W.W_k, W.W_v, H, d, cfg.act, K_cache=K, V_cache=V)

    fused()
    K1, V1 = K.clone(), V.clone()
    lookup_then_project()
    same = bool(torch.equal(K, K1) and torch.equal(V, V1))
    out = {"rows": M, "table_rows": args.table_rows, "D_in": D_in, "H": H, "d": d,
           "fused_gather_ms": timed(fused, args.iters),
           "lookup_then_project_ms": timed(lookup_then_project, args.iters),
           "lookup_ms": timed(lookup_only, args.iters),
           "project_materialised_ms": timed(project_only, args.iters),
           "bit_identical": same}
    out["speedup_vs_lookup_then_project"] = out["lookup_then_project_ms"] / out["fused_gather_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
