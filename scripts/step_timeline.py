"""Where does the in-step time go?  (4.05 ms isolated vs 5.35 ms in-step tasa)

Runs the bench's headline step (config 3h) and variants of it, each timed with CUDA events on
the launching streams while NVML samples the SM clock:

  step_fork      kv_project -> tasa_score, hma_count forked first on a side stream (bench.py)
  step_nohma     the same without hma_count
  step_serial    hma_count on the main stream after the attention
  tasa_b2b       gesr_tasa_score alone, back to back
  tasa_cool      gesr_tasa_score alone, 100 ms idle before each call (a cool, unthrottled GPU,
                 like ncu's serialised launch list)
  kv_b2b / hma_b2b

and records a CUPTI (torch.profiler / kineto) kernel timeline of three bench steps: per kernel
name, stream, start and end (ns), written as CSV.  Output: one JSON summary on stdout and
gpurun_out/timeline_<tag>.csv.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_21095_b200 import binding as gb  # noqa: E402
from paper_2511_21095_b200 import configs, inputs  # noqa: E402


class Clocks:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.s = []
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            self.s.append((time.perf_counter(), self.nv.nvmlDeviceGetClockInfo(
                self.h, self.nv.NVML_CLOCK_SM), self.nv.nvmlDeviceGetPowerUsage(self.h) / 1e3))
            time.sleep(0.001)

    def __enter__(self):
        self.s = []
        self._stop.clear()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join()

    def summary(self):
        if not self.s:
            return {}
        mhz = np.array([x[1] for x in self.s])
        w = np.array([x[2] for x in self.s])
        return {"sm_mhz_median": float(np.median(mhz)), "sm_mhz_min": float(mhz.min()),
                "power_w_median": float(np.median(w)), "samples": len(self.s)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="3h")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--tag", default="r2")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = configs.get(args.config)
    batch = inputs.make_batch(cfg, device=dev)
    bufs = gb.StepBuffers(batch, out_dtype=torch.bfloat16)
    main_s = torch.cuda.current_stream()
    act = cfg.act

    def kv(s=None):
        gb.kv_project(batch.U, batch.W_k, batch.W_v, cfg.H, cfg.d, act, K_cache=bufs.K,
                      V_cache=bufs.V, stream=s or main_s)

    def tasa(s=None):
        gb.tasa_score(batch.T, batch.cand_offsets, batch.W_q, bufs.K, bufs.V, batch.seq_offsets,
                      cfg.H, cfg.d, act, O=bufs.O, want_lse=False, workspace=bufs.workspace,
                      stream=s or main_s)

    def hma(s=None):
        gb.hma_count(batch.user_ids, batch.user_offsets, batch.item_ids, batch.item_offsets,
                     batch.cand_offsets, cfg.F, 0, counts=bufs.counts, stream=s or main_s)

    def step(order):
        if order == "fork":
            bufs.ev_fork.record(main_s)
            bufs.hma_stream.wait_event(bufs.ev_fork)
            hma(bufs.hma_stream)
            bufs.ev_join.record(bufs.hma_stream)
        kv()
        tasa()
        if order == "serial":
            hma()
        elif order == "fork":
            main_s.wait_event(bufs.ev_join)

    variants = {
        "step_fork": lambda: step("fork"),
        "step_nohma": lambda: step("none"),
        "step_serial": lambda: step("serial"),
        "tasa_b2b": tasa,
        "kv_b2b": kv,
        "hma_b2b": hma,
    }
    out = {"config": args.config}
    for _ in range(3):
        step("fork")
    torch.cuda.synchronize()
    for name, fn in variants.items():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks() as ck:
            a.record(main_s)
            for _ in range(args.iters):
                fn()
            b.record(main_s)
            torch.cuda.synchronize()
        out[name] = {"ms": a.elapsed_time(b) / args.iters, **ck.summary()}
    # cool: 100 ms idle before each call, each call timed alone
    for name, fn in (("tasa_cool", tasa), ("kv_cool", kv), ("hma_cool", hma)):
        ts, ckl = [], []
        for _ in range(8):
            time.sleep(0.1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with Clocks() as ck:
                a.record(main_s)
                fn()
                b.record(main_s)
                torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
            ckl.append(ck.summary().get("sm_mhz_median", 0))
        out[name] = {"ms": float(np.median(ts)), "ms_min": float(min(ts)),
                     "sm_mhz_median": float(np.median(ckl))}

    # CUPTI kernel timeline of three bench steps (fork order)
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            step("fork")
        torch.cuda.synchronize()
    rows = []
    for e in prof.profiler.kineto_results.events():
        if e.device_type().name != "CUDA":
            continue
        rows.append((e.name(), e.device_resource_id(), e.start_ns(), e.start_ns() + e.duration_ns()))
    rows.sort(key=lambda r: r[2])
    t0 = rows[0][2] if rows else 0
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", f"timeline_{args.tag}.csv")
    with open(path, "w") as fh:
        fh.write("kernel,stream,start_us,end_us,dur_us\n")
        for n, s, a, b in rows:
            fh.write(f"\"{n[:80]}\",{s},{(a - t0) / 1e3:.1f},{(b - t0) / 1e3:.1f},"
                     f"{(b - a) / 1e3:.1f}\n")
    agg = {}
    for n, s, a, b in rows:
        k = n.split("<")[0].split("(")[0][:40]
        agg.setdefault(k, []).append((b - a) / 1e6)
    out["timeline_kernels_ms"] = {k: [round(x, 3) for x in v] for k, v in agg.items()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
