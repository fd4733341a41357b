"""CUPTI kernel timeline of bench steps of a small (launch-bound) config: which kernels, how long
each runs and the gaps between them.

    python scripts/small_timeline.py --config 4 --tag r2u
Writes gpurun_out/timeline_<config>_<tag>.csv and prints per-kernel totals, the sum of the gaps
between consecutive kernels on the main stream and the step span, as one JSON line.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="4")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--tag", default="r2")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = configs.get(args.config)
    bt = inputs.make_batch(cfg, device=dev)
    bufs = gb.StepBuffers(bt, out_dtype=torch.bfloat16)
    stream = torch.cuda.Stream()

    def step():
        gb.score_step(bt, bufs, chunk=cfg.chunk, stream=stream)

    with torch.cuda.stream(stream):
        for _ in range(5):
            step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                step()
        torch.cuda.synchronize()
    rows = []
    for e in prof.profiler.kineto_results.events():
        if e.device_type().name != "CUDA":
            continue
        rows.append((e.name(), e.device_resource_id(), e.start_ns(), e.start_ns() + e.duration_ns()))
    rows.sort(key=lambda r: r[2])
    t0 = rows[0][2] if rows else 0
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", f"timeline_{args.config}_{args.tag}.csv")
    with open(path, "w") as fh:
        fh.write("kernel,stream,start_us,end_us,dur_us\n")
        for n, s, a, b in rows:
            fh.write(f"\"{n[:80]}\",{s},{(a - t0) / 1e3:.2f},{(b - t0) / 1e3:.2f},"
                     f"{(b - a) / 1e3:.2f}\n")
    agg = {}
    for n, s, a, b in rows:
        k = n.split("<")[0].split("(")[0].replace("void ", "").split("::")[-1][:40]
        agg[k] = agg.get(k, 0.0) + (b - a) / 1e3 / args.steps
    gaps = sum(max(0, rows[i + 1][2] - rows[i][3]) for i in range(len(rows) - 1)) / 1e3
    span = (rows[-1][3] - rows[0][2]) / 1e3 if rows else 0.0
    print(json.dumps({"config": args.config, "kernels_us_per_step": {k: round(v, 2) for k, v in agg.items()},
                      "launches_per_step": len(rows) / args.steps,
                      "gaps_us_per_step": round(gaps / args.steps, 2),
                      "span_us_per_step": round(span / args.steps, 2)}))


if __name__ == "__main__":
    main()
