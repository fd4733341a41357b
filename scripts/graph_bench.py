"""Configs 1, 2 and 4 eager vs CUDA-graph capture, and config 4's K/V-cache reuse speedup.

    python scripts/graph_bench.py [--iters 50]

SURVEY.md s8(d): configs 1 and 4 are launch-bound, so they are also reported under CUDA-graph
capture of one whole step (the C-ABI calls do no host synchronisation and no allocation).
Config 4 also reports the reuse speedup: one gesr_kv_project + 8 chunked gesr_tasa_score calls
against one cache, versus re-projecting the history for every chunk.  One JSON line per case.
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


def time_it(fn, iters):
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
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    out = []
    for name in ("1", "2", "4"):
        cfg = configs.get(name)
        bt = inputs.make_batch(cfg, device=dev)
        bufs = gb.StepBuffers(bt, out_dtype=torch.bfloat16)
        stream = torch.cuda.Stream()
        step = lambda: gb.score_step(bt, bufs, chunk=cfg.chunk, stream=stream)  # noqa: E731
        with torch.cuda.stream(stream):
            eager = time_it(step, args.iters)
            ref = bufs.O.clone()
            g = torch.cuda.CUDAGraph()
            step()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=stream):
                step()
            graph = time_it(g.replay, args.iters)
            same = bool(torch.equal(bufs.O, ref))
        rec = {"config": name, "eager_ms": eager, "graph_ms": graph,
               "graph_speedup": eager / graph, "graph_output_identical": same,
               "cand_per_s_graph": bt.total_C / (graph * 1e-3)}
        if name == "4":
            # reuse: project once, score 8 chunks; vs re-project the 4096-row history per chunk
            def reproject():
                with torch.cuda.stream(stream):
                    for c0 in range(0, bt.total_C, cfg.chunk):
                        c1 = min(bt.total_C, c0 + cfg.chunk)
                        gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act,
                                      K_cache=bufs.K, V_cache=bufs.V, stream=stream)
                        co = bufs.__dict__[f"_co_{c0}"]
                        gb.tasa_score(bt.T[c0:c1], co, bt.W_q, bufs.K, bufs.V, bt.seq_offsets,
                                      cfg.H, cfg.d, cfg.act, O=bufs.O[c0:c1], want_lse=False,
                                      workspace=bufs.workspace, stream=stream)

            def reuse():
                gb.score_step(bt, bufs, chunk=cfg.chunk, hma=False, stream=stream)
            with torch.cuda.stream(stream):     # events on the stream the work runs on
                rec["reuse_ms"] = time_it(reuse, args.iters)
                rec["reproject_ms"] = time_it(reproject, args.iters)
            rec["reuse_speedup"] = rec["reproject_ms"] / rec["reuse_ms"]
        out.append(rec)
        print(json.dumps(rec))


if __name__ == "__main__":
    main()
