#!/usr/bin/env python
"""bench.py -- GESR MoA candidate scoring on B200: candidate-scores/sec at L=2048, C=1000.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 3h]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)

One step = one pass of the whole hot path over one batch: gesr_kv_project -> gesr_tasa_score,
with gesr_hma_count on a second stream joined by an event.  Workload: config
"3h" = B=1024 requests per GPU, L=2048 history rows, C=1000 candidates, H=4, d=128, D_in=512,
F=16 HMA fields (BASELINE.json metric).  Requests shard across GPUs with no data-path
collective (weak scaling: rank r scores requests [r*B, (r+1)*B)); NCCL is used only for the
setup weight broadcast and the max-over-ranks timing reduction.

Rank 0 prints ONE JSON line.  `--impl reference` times the fp64 CPU oracle (oracle/) on a
bounded sample of the same workload, on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "candidate-scores/sec at L=2048, C=1000; % of tensor-pipe/HBM roofline"
UNIT = "candidate-scores/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="3h")
    ap.add_argument("--out-dtype", default="bf16", choices=["f32", "bf16"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=16,
                    help="request chunks of the end-to-end pipeline (H2D / kernels / D2H "
                         "overlapped on three streams); 1 = copy in, score, copy out")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gather", action="store_true", help="NCCL gather of scores after timing")
    return ap.parse_args()


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d, "measured"
    # fallback figures of /opt/skills/guides/B200_PROFILING.md
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while the timed region runs."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self._nv = None
            self.error = str(e)

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(s)}


def _cpu_sample(cfg, requests, threads=None):
    """Run the fp64 oracle on the given requests (all three calls); returns (seconds, cands)."""
    import oracle
    from paper_2511_21095_b200 import inputs
    bt = inputs.make_batch(cfg, requests=requests)
    t0 = time.perf_counter()
    K, V = oracle.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, act=cfg.act, threads=threads)
    oracle.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H, cfg.d,
                      act=cfg.act, threads=threads)
    oracle.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                     bt.cand_offsets, cfg.F, threads=threads)
    return time.perf_counter() - t0, bt.total_C


def run_reference(args, rank):
    """The base contract's reference arm for this tier: the oracle as it stands, host cores."""
    if rank != 0:
        return
    import oracle
    from paper_2511_21095_b200 import configs
    cfg = configs.get(args.config)
    threads = oracle.default_threads()
    times = []
    cands = 0
    for i in range(args.warmup + args.steps):
        # each step a bounded sample: one whole request of the workload (all C_b candidates)
        dt, c = _cpu_sample(cfg, [i % cfg.B], threads)
        if i >= args.warmup:
            times.append(dt)
            cands += c
    total = sum(times)
    value = cands / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name} (config {args.config}): 1 request/step sample",
                   "L": 2048, "C": 1000, "H": cfg.H, "d": cfg.d, "D_in": cfg.D_in, "F": cfg.F},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"1 request (L={cfg.L[1]}, C={cfg.C[1]}) per step; "
                                   "kv_project+tasa_score+hma_count in fp64"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = _args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2511_21095_b200 import binding as gb
    from paper_2511_21095_b200 import configs, inputs, roofline

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = configs.get(args.config)
    B = cfg.B
    reqs = torch.arange(rank * B, (rank + 1) * B, dtype=torch.int64)
    batch = inputs.make_batch(cfg, requests=reqs, device=dev)
    if world > 1:
        for w in (batch.W_q, batch.W_k, batch.W_v):     # setup-time weight broadcast (NCCL)
            dist.broadcast(w, src=0)
    out_dtype = torch.bfloat16 if args.out_dtype == "bf16" else torch.float32
    bufs = gb.StepBuffers(batch, out_dtype=out_dtype)
    main_stream = torch.cuda.current_stream()
    act = cfg.act

    ev = {k: [] for k in ("kv0", "kv1", "t1", "h0", "h1")}
    # where gesr_hma_count runs: "fork" = first, on a side stream joined by an event;
    # "kv" = forked after the K/V projection; "serial" = on the main stream after the attention
    hma_order = os.environ.get("GESR_HMA_ORDER", "fork")

    def step(record=False):
        E = (lambda: torch.cuda.Event(enable_timing=True)) if record else None
        if record:
            e_h0, e_h1, e_kv0, e_kv1, e_t1 = E(), E(), E(), E(), E()
        def hma(stream):
            if record:
                e_h0.record(stream)
            gb.hma_count(batch.user_ids, batch.user_offsets, batch.item_ids, batch.item_offsets,
                         batch.cand_offsets, cfg.F, 0, counts=bufs.counts, stream=stream)
            if record:
                e_h1.record(stream)

        def fork():
            bufs.ev_fork.record(main_stream)
            bufs.hma_stream.wait_event(bufs.ev_fork)
            hma(bufs.hma_stream)
            bufs.ev_join.record(bufs.hma_stream)

        if hma_order == "fork":
            fork()
        if record:
            e_kv0.record(main_stream)
        gb.kv_project(batch.U, batch.W_k, batch.W_v, cfg.H, cfg.d, act, K_cache=bufs.K,
                      V_cache=bufs.V, stream=main_stream)
        if record:
            e_kv1.record(main_stream)
        if hma_order == "kv":
            fork()
        gb.tasa_score(batch.T, batch.cand_offsets, batch.W_q, bufs.K, bufs.V, batch.seq_offsets,
                      cfg.H, cfg.d, act, O=bufs.O, want_lse=False, workspace=bufs.workspace,
                      stream=main_stream)
        if record:
            e_t1.record(main_stream)
        if hma_order == "serial":
            hma(main_stream)
        else:
            main_stream.wait_event(bufs.ev_join)
        if record:
            for k, e in (("kv0", e_kv0), ("kv1", e_kv1), ("t1", e_t1), ("h0", e_h0), ("h1", e_h1)):
                ev[k].append(e)

    launches_per_step = 5  # hma + kv proj + (build_units + q proj + attention)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_start.record(main_stream)
        for _ in range(args.steps):
            step(record=True)
        t_end.record(main_stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    kv_ms = float(np.mean([a.elapsed_time(b) for a, b in zip(ev["kv0"], ev["kv1"])]))
    tasa_ms = float(np.mean([a.elapsed_time(b) for a, b in zip(ev["kv1"], ev["t1"])]))
    hma_ms = float(np.mean([a.elapsed_time(b) for a, b in zip(ev["h0"], ev["h1"])]))
    if world > 1:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())

    Ls = (batch.seq_offsets[1:] - batch.seq_offsets[:-1]).cpu().numpy()
    Cs = (batch.cand_offsets[1:] - batch.cand_offsets[:-1]).cpu().numpy()
    cnt = roofline.counts(cfg, Ls, Cs, n_item_ids=batch.item_ids.numel(),
                          n_user_ids=batch.user_ids.numel(),
                          out_bytes=2 if out_dtype == torch.bfloat16 else 4)
    cands_per_step = cnt["candidates"] * world
    value = cands_per_step * args.steps / (elapsed_ms / 1e3)
    ms_per_step = elapsed_ms / args.steps

    peaks, peak_src = _peaks()
    peak_tf = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
    hbm = float(peaks["hbm_gbs"])
    achieved = cnt["tasa_flop"] / (tasa_ms / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get(args.config, {}).get("tasa_bytes_per_launch")
    roof_step_s = roofline.roof_time(cnt["kv_flop"], cnt["kv_bytes"], peak_tf, hbm) + max(
        roofline.roof_time(cnt["tasa_flop"], cnt["tasa_bytes"], peak_tf, hbm),
        cnt["hma_bytes"] / (hbm * 1e9))

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"{cfg.name} (BASELINE config {args.config}): {B} requests per GPU,"
                               f" L={cfg.L[1]}, C={cfg.C[1]}", "requests_per_gpu": B,
                   "H": cfg.H, "d": cfg.d, "D_in": cfg.D_in, "F": cfg.F,
                   "out_dtype": args.out_dtype, "act": "silu", "parallelism": f"dp{world}",
                   "l2": "inputs larger than L2 (U 2.1 GB, item ids 1.1 GB per GPU); no flush"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved / peak_tf, "traffic": traffic,
                     "kernel": "gesr_tasa_score (q-projection + attention kernels)",
                     "peak_source": f"{peak_src} bf16_tflops_sustained (MEASURED_PEAKS.json)"},
        "step_roofline": {"roof_ms": roof_step_s * 1e3, "frac": roof_step_s * 1e3 / ms_per_step,
                          "kv_ms": kv_ms, "tasa_ms": tasa_ms, "hma_ms": hma_ms,
                          "kv_tflops": cnt["kv_flop"] / (kv_ms / 1e3) / 1e12,
                          "hma_gbs": cnt["hma_bytes"] / (hma_ms / 1e3) / 1e9},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }

    # ---------------------------------------------------------------- e2e through host buffers
    if not args.no_e2e:
        pin = lambda t: t.cpu().pin_memory()   # noqa: E731
        hb = inputs.Batch(cfg, batch.requests.cpu(), pin(batch.seq_offsets),
                          pin(batch.cand_offsets), pin(batch.U), pin(batch.T), batch.W_q.cpu(),
                          batch.W_k.cpu(), batch.W_v.cpu(), pin(batch.user_ids),
                          pin(batch.user_offsets), pin(batch.item_ids), pin(batch.item_offsets))
        scorer = gb.PipelinedHostScorer(hb, n_chunks=args.e2e_chunks, out_dtype=bufs.O.dtype,
                                        act=act, device=dev)
        h_O = torch.empty(bufs.O.shape, dtype=bufs.O.dtype).pin_memory()
        h_counts = torch.empty(bufs.counts.shape, dtype=torch.int32).pin_memory()
        h2d = scorer.h2d_bytes
        d2h = h_O.numel() * h_O.element_size() + h_counts.numel() * 4

        def e2e_step():
            scorer.run(h_O, h_counts, stream=main_stream)

        e2e_step()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        n_e2e = max(1, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        a.record(main_stream)
        for _ in range(n_e2e):
            e2e_step()
        b.record(main_stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        line["e2e"] = {"value": cands_per_step * n_e2e / (e_ms / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": n_e2e,
                       "chunks": len(scorer.chunks),
                       "pipeline": "request chunks: H2D of chunk i+1 and D2H of chunk i-1 "
                                   "overlap the kernels of chunk i (PipelinedHostScorer)"}

    # ---------------------------------------------------------------- optional score gather
    if args.gather and world > 1:
        t0 = time.perf_counter()
        if rank == 0:
            for r in range(1, world):
                buf = torch.empty_like(bufs.O)
                dist.recv(buf, src=r)
        else:
            dist.send(bufs.O, dst=0)
        torch.cuda.synchronize()
        line["gather_s"] = time.perf_counter() - t0

    # ---------------------------------------------------------------- cpu baseline (oracle)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        threads = oracle.default_threads()
        tot, c, n = 0.0, 0, 0
        while tot < 12.0 and n < 64:
            dt, cc = _cpu_sample(cfg, [n], threads)
            tot += dt
            c += cc
            n += 1
        line["cpu_baseline"] = {"value": c / tot, "unit": UNIT, "cores": threads,
                                "kind": "oracle",
                                "sample": f"{n} request(s) of config {args.config} (L=2048, "
                                          f"C=1000 each), fp64 kv_project+tasa_score+hma_count, "
                                          f"{tot:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
