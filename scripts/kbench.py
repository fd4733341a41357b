"""Per-call isolated timing (CUDA events, serialized) of the three C-ABI calls on a config.

    python scripts/kbench.py [--config 3h] [--iters 10]

Development tool: prints one JSON line with the average ms and achieved TFLOP/s or GB/s of
gesr_kv_project, gesr_tasa_score and gesr_hma_count timed separately (no stream overlap).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_21095_b200 import binding as gb  # noqa: E402
from paper_2511_21095_b200 import configs, inputs, roofline  # noqa: E402


def timeit(fn, iters):
    for _ in range(2):
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
    ap.add_argument("--config", default="3h")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out-dtype", default="f32")
    args = ap.parse_args()
    cfg = configs.get(args.config)
    dev = torch.device("cuda:0")
    bt = inputs.make_batch(cfg, device=dev)
    od = torch.bfloat16 if args.out_dtype == "bf16" else torch.float32
    bufs = gb.StepBuffers(bt, out_dtype=od)
    Ls = (bt.seq_offsets[1:] - bt.seq_offsets[:-1]).cpu().numpy()
    Cs = (bt.cand_offsets[1:] - bt.cand_offsets[:-1]).cpu().numpy()
    cnt = roofline.counts(cfg, Ls, Cs, bt.item_ids.numel(), bt.user_ids.numel(),
                          out_bytes=2 if od == torch.bfloat16 else 4)
    kv = timeit(lambda: gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act,
                                      K_cache=bufs.K, V_cache=bufs.V), args.iters)
    tasa = timeit(lambda: gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, bufs.K, bufs.V,
                                        bt.seq_offsets, cfg.H, cfg.d, cfg.act, O=bufs.O,
                                        want_lse=False, workspace=bufs.workspace), args.iters)
    hma = timeit(lambda: gb.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids,
                                      bt.item_offsets, bt.cand_offsets, cfg.F, 0,
                                      counts=bufs.counts), args.iters)
    step = timeit(lambda: gb.score_step(bt, bufs, chunk=cfg.chunk), args.iters)

    def serial():   # the three calls back to back on one stream (no overlap)
        gb.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                     bt.cand_offsets, cfg.F, 0, counts=bufs.counts)
        gb.score_step(bt, bufs, chunk=cfg.chunk, hma=False)
    step_serial = timeit(serial, args.iters)
    print(json.dumps({
        "config": args.config, "kv_ms": kv, "kv_tflops": cnt["kv_flop"] / kv / 1e9,
        "tasa_ms": tasa, "tasa_tflops": cnt["tasa_flop"] / tasa / 1e9,
        "hma_ms": hma, "hma_gbs": cnt["hma_bytes"] / hma / 1e6,
        "step_ms": step, "cand_per_s": cnt["candidates"] / step * 1e3,
        "serial_sum_ms": kv + tasa + hma, "step_serial_ms": step_serial}))


if __name__ == "__main__":
    main()
