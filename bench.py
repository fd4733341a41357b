#!/usr/bin/env python
"""bench.py -- GESR MoA candidate scoring on B200: candidate-scores/sec at L=2048, C=1000.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 3h]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)

`python bench.py --gpus N` with no torchrun environment re-launches itself under
`torch.distributed.run` with N local ranks (one process per GPU).

One step = one pass of the whole hot path over one batch: gesr_kv_project -> gesr_tasa_score ->
gesr_hma_count on one stream (`--hma-order fork` forks HMA on a second stream joined by an event,
SURVEY.md s8(d)'s layout: the persistent kernels leave it no SMs, so it serialises either way and
only blurs the per-call timing), exactly
`binding.score_step(batch, StepBuffers(batch, out_dtype=bf16))` (the configuration
tests/test_gpu_configs.py checks against the oracle).

Workloads (paper_2511_21095_b200/configs.py):
  3h (default)  B=1024 requests per GPU, L=2048, C=1000, H=4, d=128, D_in=512, F=16 -- the
                metric's workload; WEAK scaling: rank r scores requests [r B, (r+1) B).
  5             the fixed 8192-request serving mix (L log-uniform 32-4096, C 100-2000); STRONG
                scaling: every rank computes the same LPT partition (shard.lpt_partition) and
                generates only its own requests.
  1, 2, 3, 4    the other BASELINE configs (weak).
No collective is on the data path: NCCL carries the setup weight broadcast, the max-over-ranks
time reduction and (with --gather) the post-timing score gather.

Rank 0 prints ONE JSON line.  `--impl reference` times the fp64 CPU oracle (oracle/) on a
bounded sample of the same workload, on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "candidate-scores/sec at L=2048, C=1000; % of tensor-pipe/HBM roofline"
UNIT = "candidate-scores/s"
STRONG_CONFIGS = ("5",)


def _args(argv=None):
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
    ap.add_argument("--graph", action="store_true",
                    help="time replays of one step captured into a CUDA graph (launch-bound "
                         "configs 1, 2, 4: no per-call host overhead)")
    ap.add_argument("--gather", action="store_true", help="NCCL gather of scores after timing")
    ap.add_argument("--hma-order", default="serial", choices=["fork", "kv", "serial"],
                    help="where gesr_hma_count runs in the step: forked first on a side stream, "
                         "forked after the K/V projection, or on the main stream after the "
                         "attention (the persistent projection / attention kernels leave no room "
                         "for HMA CTAs, so it serialises in every order: DESIGN.md s6)")
    return ap.parse_args(argv)


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


# ------------------------------------------------------------------------------ orchestration

def plan_requests(cfg_name: str, rank: int, world: int):
    """This rank's global request indices, the scaling mode and the partition's model
    imbalance.  Weak: rank r takes [r B, (r+1) B) of the config's request stream.  Strong
    (config 5): the cfg.B requests LPT-packed by the cost model of shard.request_cost
    (SURVEY.md s8(e)); every rank computes the same partition."""
    import numpy as np

    from paper_2511_21095_b200 import configs, inputs, shard
    cfg = configs.get(cfg_name)
    if cfg_name in STRONG_CONFIGS:
        L, C = inputs.request_lengths(cfg)
        cost = shard.request_cost(cfg, L.numpy(), C.numpy())
        parts = shard.lpt_partition(cost, world)
        return cfg, parts[rank], "strong", shard.imbalance(cost, parts)
    return cfg, np.arange(rank * cfg.B, (rank + 1) * cfg.B, dtype=np.int64), "weak", 0.0


def orchestrate(cfg_name: str, rank: int, world: int, steps: int, warmup: int, engine,
                group=None) -> dict:
    """The bench's multi-rank protocol, independent of what a step computes (tests drive it
    with a stub engine over gloo): plan this rank's requests, engine.setup(cfg, requests) (the
    rank generates only its own requests), broadcast the weights from rank 0, W >= 3 untimed
    warm-up steps, barrier + sync, K timed steps (engine.time_steps: device time in ms), barrier,
    max over ranks.  Returns the per-job numbers rank 0 reports."""
    import torch
    import torch.distributed as dist
    cfg, reqs, scaling, model_imb = plan_requests(cfg_name, rank, world)
    engine.setup(cfg, reqs)
    if world > 1:
        engine.broadcast_weights(group)
    for _ in range(max(3, warmup)):
        engine.step()
    engine.sync()
    if world > 1:
        dist.barrier(group)
    engine.sync()
    ms = float(engine.time_steps(steps))
    if world > 1:
        dist.barrier(group)
    cands = float(engine.candidates)
    per_rank = torch.tensor([[ms, cands, float(len(reqs))]], dtype=torch.float64,
                            device=engine.reduce_device)
    if world > 1:
        allr = [torch.zeros_like(per_rank) for _ in range(world)]
        dist.all_gather(allr, per_rank, group=group)
        per_rank = torch.cat(allr)
    per_rank = per_rank.cpu()
    t_max = float(per_rank[:, 0].max())
    total_cands = float(per_rank[:, 1].sum())
    return {
        "cfg": cfg, "scaling": scaling, "requests": reqs, "elapsed_ms": t_max,
        "ms_per_step": t_max / steps, "cands_per_step": total_cands,
        "value": total_cands * steps / (t_max / 1e3),
        "per_rank_ms": [float(x) for x in per_rank[:, 0]],
        "per_rank_requests": [int(x) for x in per_rank[:, 2]],
        "imbalance_measured": float(per_rank[:, 0].max() / per_rank[:, 0].mean() - 1.0),
        "imbalance_model": model_imb,
    }


class GpuEngine:
    """One rank's device state: the batch of its requests, preallocated buffers, and the step
    (binding.score_step: kv_project -> tasa_score, hma_count forked on a side stream)."""

    L2_FLUSH_BYTES = 256 << 20          # > 2x the 126 MB L2

    def __init__(self, device, out_dtype, hma_order="serial", graph=False):
        import torch
        self.dev, self.out_dtype, self.hma_order = device, out_dtype, hma_order
        self.reduce_device = device
        self.events = {}
        # graph capture needs a non-default stream
        self.stream = torch.cuda.Stream(device) if graph else torch.cuda.current_stream(device)
        self.use_graph, self.graph = graph, None

    def setup(self, cfg, reqs):
        import torch

        from paper_2511_21095_b200 import binding as gb
        from paper_2511_21095_b200 import inputs
        self.cfg = cfg
        self.batch = inputs.make_batch(cfg, requests=torch.as_tensor(reqs), device=self.dev)
        self.bufs = gb.StepBuffers(self.batch, out_dtype=self.out_dtype)
        self.candidates = self.batch.total_C
        self.gb = gb
        b = self.batch
        self.input_bytes = sum(t.numel() * t.element_size() for t in (
            b.U, b.T, b.W_q, b.W_k, b.W_v, b.user_ids, b.item_ids, b.item_offsets))
        # inputs that fit in L2 would stay resident across steps: flush it before each step
        self.flush = (torch.empty(self.L2_FLUSH_BYTES, dtype=torch.uint8, device=self.dev)
                      if self.input_bytes < self.L2_FLUSH_BYTES else None)

    def broadcast_weights(self, group=None):
        import torch.distributed as dist
        for w in (self.batch.W_q, self.batch.W_k, self.batch.W_v):   # setup-time, NCCL
            dist.broadcast(w, src=0, group=group)

    def step(self, record=False):
        self.gb.score_step(self.batch, self.bufs, act=self.cfg.act, chunk=self.cfg.chunk,
                           stream=self.stream, hma_order=self.hma_order,
                           events=self.events if record else None)

    def sync(self):
        import torch
        torch.cuda.synchronize(self.dev)

    def capture(self):
        """--graph: one whole step captured into a CUDA graph (the C-ABI calls allocate nothing
        and never synchronise the host), replayed as the timed step."""
        import torch
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(self.stream):
            with torch.cuda.graph(self.graph, stream=self.stream):
                self.step()
        torch.cuda.synchronize(self.dev)

    def _replay(self):
        import torch
        with torch.cuda.stream(self.stream):     # replay() launches on the current stream
            self.graph.replay()

    def time_steps(self, steps):
        import torch
        if self.use_graph and self.graph is None:
            self.capture()
            n0 = self.gb.launch_count()
            self.step()                     # launches per step (a replay does not count them)
            torch.cuda.synchronize(self.dev)
            self.graph_launches = self.gb.launch_count() - n0
        self.launch0 = self.gb.launch_count()
        ev = lambda: torch.cuda.Event(enable_timing=True)   # noqa: E731
        with ClockSampler(self.dev.index) as clk:
            if self.flush is None:
                # inputs larger than L2: the K steps back to back between two events
                a, b = ev(), ev()
                a.record(self.stream)
                for _ in range(steps):
                    self._replay() if self.graph is not None else self.step(record=True)
                b.record(self.stream)
                torch.cuda.synchronize(self.dev)
                ms = a.elapsed_time(b)
            else:
                # L2 flushed (a 256 MB memset) before every step, each step timed alone
                pairs = []
                for _ in range(steps):
                    with torch.cuda.stream(self.stream):
                        self.flush.zero_()
                    a, b = ev(), ev()
                    a.record(self.stream)
                    self._replay() if self.graph is not None else self.step(record=True)
                    b.record(self.stream)
                    pairs.append((a, b))
                torch.cuda.synchronize(self.dev)
                ms = sum(a.elapsed_time(b) for a, b in pairs)
        self.launches = (self.gb.launch_count() - self.launch0 if self.graph is None
                         else self.graph_launches * steps)
        self.clocks = clk.summary()
        if self.graph is not None:
            # per-call times (roofline numerators) from a few eager steps after the timed region
            for _ in range(min(steps, 5)):
                self.step(record=True)
            torch.cuda.synchronize(self.dev)
        return ms

    def call_ms(self, a, b):
        import numpy as np
        ev = self.events
        if not ev.get(a):
            return None
        return float(np.mean([x.elapsed_time(y) for x, y in zip(ev[a], ev[b])]))


# ------------------------------------------------------------------------------ CPU baseline

def _cpu_info() -> dict:
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        aff = None
    return {"nproc": os.cpu_count(), "affinity": aff, "cpu_model": model}


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


def cpu_baseline(cfg, config_name, budget_s=10.0, budget_1t_s=4.0) -> dict:
    """The oracle as it stands on the host cores: all threads (std::thread over requests /
    rows) on requests 0, 1, ... until ~budget_s, then ONE thread on the next request(s) until
    ~budget_1t_s (both thread counts, nproc, affinity and CPU model)."""
    import oracle
    threads = oracle.default_threads()
    tot, c, n = 0.0, 0, 0
    while tot < budget_s and n < 64:
        dt, cc = _cpu_sample(cfg, [n], threads)
        tot, c, n = tot + dt, c + cc, n + 1
    tot1, c1, n1 = 0.0, 0, 0
    while tot1 < budget_1t_s and n1 < 8:
        dt, cc = _cpu_sample(cfg, [n + n1], 1)
        tot1, c1, n1 = tot1 + dt, c1 + cc, n1 + 1
    return {"value": c / tot, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{n} request(s) of config {config_name} with {threads} threads, "
                      f"fp64 kv_project+tasa_score+hma_count, {tot:.1f} s",
            "value_1thread": c1 / tot1,
            "sample_1thread": f"{n1} request(s) on 1 thread, {tot1:.1f} s",
            **_cpu_info()}


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
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "strong" if args.config in STRONG_CONFIGS else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name} (config {args.config}): 1 request/step sample",
                   "H": cfg.H, "d": cfg.d, "D_in": cfg.D_in, "F": cfg.F},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": "1 whole request of the workload per step; "
                                   "kv_project+tasa_score+hma_count in fp64", **_cpu_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ launcher

def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` (N > 1) without a torchrun environment: start N local ranks, one per GPU."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible",
              file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = _args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    import torch
    import torch.distributed as dist

    from paper_2511_21095_b200 import binding as gb
    from paper_2511_21095_b200 import inputs, roofline

    assert torch.cuda.device_count() > local, "one GPU per rank"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    out_dtype = torch.bfloat16 if args.out_dtype == "bf16" else torch.float32
    eng = GpuEngine(dev, out_dtype, args.hma_order, graph=args.graph)
    res = orchestrate(args.config, rank, world, args.steps, args.warmup, eng)
    cfg, batch, bufs = res["cfg"], eng.batch, eng.bufs
    kv_ms, tasa_ms, hma_ms = eng.call_ms("kv0", "kv1"), eng.call_ms("kv1", "t1"), \
        eng.call_ms("h0", "h1")

    Ls = (batch.seq_offsets[1:] - batch.seq_offsets[:-1]).cpu().numpy()
    Cs = (batch.cand_offsets[1:] - batch.cand_offsets[:-1]).cpu().numpy()
    cnt = roofline.counts(cfg, Ls, Cs, n_item_ids=batch.item_ids.numel(),
                          n_user_ids=batch.user_ids.numel(),
                          out_bytes=2 if out_dtype == torch.bfloat16 else 4)
    peaks, peak_src = _peaks()
    peak_sus = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
    peak_burst = float(peaks["bf16_tflops"])
    hbm = float(peaks["hbm_gbs"])
    achieved = cnt["tasa_flop"] / (tasa_ms / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get(args.config, {}).get("tasa_bytes_per_launch")

    def step_roof(P):
        return roofline.roof_time(cnt["kv_flop"], cnt["kv_bytes"], P, hbm) + max(
            roofline.roof_time(cnt["tasa_flop"], cnt["tasa_bytes"], P, hbm),
            cnt["hma_bytes"] / (hbm * 1e9))

    ms_per_step = res["ms_per_step"]
    strong = res["scaling"] == "strong"
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": res["scaling"], "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "config": {"workload": (f"{cfg.name} (BASELINE config {args.config}): "
                                + (f"{cfg.B} requests LPT-sharded over {world} GPU(s)" if strong
                                   else f"{cfg.B} requests per GPU")),
                   "requests_total": cfg.B if strong else cfg.B * world,
                   "requests_per_rank": res["per_rank_requests"],
                   "H": cfg.H, "d": cfg.d, "D_in": cfg.D_in, "F": cfg.F, "L": list(cfg.L),
                   "C": list(cfg.C), "out_dtype": args.out_dtype, "act": "silu",
                   "parallelism": f"dp{world}", "hma_order": args.hma_order,
                   "l2": ("inputs larger than L2 (per GPU: U and HMA item ids exceed 126 MB); "
                          "no flush" if eng.flush is None else
                          f"inputs {eng.input_bytes / 2**20:.1f} MiB fit in L2: a 256 MiB memset "
                          "flushes it before every step, each step timed alone (flush excluded)"),
                   "cuda_graph": bool(args.graph)},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_sus,
                     "unit": "TFLOP/s", "frac": achieved / peak_sus, "traffic": traffic,
                     "kernel": "gesr_tasa_score (q-projection + attention kernels), timed "
                               "inside the step",
                     "peak_source": f"{peak_src} bf16_tflops_sustained (MEASURED_PEAKS.json): "
                                    "the kernel runs inside back-to-back steps",
                     "peak_burst": peak_burst, "frac_burst": achieved / peak_burst,
                     "algorithmic_bytes": cnt["tasa_bytes"],
                     "traffic_source": "profiles/ncu_traffic.json (ncu --set full, DRAM read + "
                                       "write of the q-projection and attention launches); "
                                       "the excess over algorithmic_bytes is the Q round trip "
                                       "through HBM and K/V re-reads"},
        "step_roofline": {"roof_ms_sustained": step_roof(peak_sus) * 1e3,
                          "frac_sustained": step_roof(peak_sus) * 1e3 / ms_per_step,
                          "roof_ms_burst": step_roof(peak_burst) * 1e3,
                          "frac_burst": step_roof(peak_burst) * 1e3 / ms_per_step,
                          "kv_ms": kv_ms, "tasa_ms": tasa_ms, "hma_ms": hma_ms,
                          # SURVEY s8(d)'s MUFU ceiling beside the tensor roofline: the softmax's
                          # exps at 16 ex2 / clk / SM on 148 SMs at the maximum SM clock
                          "exps": cnt["exps"],
                          "mufu_ceiling_ms": cnt["exps"] / (16 * 148 * float(
                              peaks.get("sm_max_mhz", 1965.0)) * 1e6) * 1e3,
                          "attn_tensor_ms_burst": cnt["attn_flop"] / (peak_burst * 1e12) * 1e3,
                          "kv_tflops": cnt["kv_flop"] / (kv_ms / 1e3) / 1e12,
                          "hma_gbs": cnt["hma_bytes"] / (hma_ms / 1e3) / 1e9},
        "gpu_launches": eng.launches,
        "clocks": eng.clocks,
    }
    if world > 1:
        line["per_rank_ms"] = res["per_rank_ms"]
        line["imbalance"] = {"measured": res["imbalance_measured"],
                             "cost_model": res["imbalance_model"]}

    # ---------------------------------------------------------------- e2e through host buffers
    if not args.no_e2e:
        pin = lambda t: t.cpu().pin_memory()   # noqa: E731
        hb = inputs.Batch(cfg, batch.requests.cpu(), pin(batch.seq_offsets),
                          pin(batch.cand_offsets), pin(batch.U), pin(batch.T), batch.W_q.cpu(),
                          batch.W_k.cpu(), batch.W_v.cpu(), pin(batch.user_ids),
                          pin(batch.user_offsets), pin(batch.item_ids), pin(batch.item_offsets))
        scorer = gb.HostPlan(hb, n_chunks=args.e2e_chunks, out_dtype=bufs.O.dtype, act=cfg.act,
                             device=dev)
        h_O = torch.empty(bufs.O.shape, dtype=bufs.O.dtype).pin_memory()
        h_counts = torch.empty(bufs.counts.shape, dtype=torch.int32).pin_memory()
        h2d = scorer.h2d_bytes
        d2h = h_O.numel() * h_O.element_size() + h_counts.numel() * 4
        main_stream = eng.stream
        scorer.run(h_O, h_counts, stream=main_stream)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        n_e2e = max(1, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        a.record(main_stream)
        for _ in range(n_e2e):
            scorer.run(h_O, h_counts, stream=main_stream)
        b.record(main_stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        line["e2e"] = {"value": res["cands_per_step"] * n_e2e / (e_ms / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": n_e2e,
                       "chunks": min(args.e2e_chunks, batch.B),
                       "api": "gesr_score_host (C ABI, host buffers in and out)",
                       "pipeline": "request chunks: H2D of chunk i+1 and D2H of chunk i-1 "
                                   "overlap the kernels of chunk i (csrc/hostpath.cu)"}
        # the bound of this leg: one pinned host -> device copy of the same size class, timed
        # alone on the copy engine (best of 3)
        src = hb.U.reshape(-1)[: min(hb.U.numel(), 1 << 29)]
        dst = torch.empty(src.shape, dtype=src.dtype, device=dev)
        best = float("inf")
        for _ in range(3):
            a.record(main_stream)
            with torch.cuda.stream(main_stream):
                dst.copy_(src, non_blocking=True)
            b.record(main_stream)
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        copy_gbs = src.numel() * src.element_size() / (best / 1e3) / 1e9
        h2d_gbs = h2d * n_e2e / (e_ms / 1e3) / 1e9
        line["e2e"]["h2d_bound"] = {"achieved_gbs": h2d_gbs, "copy_gbs": copy_gbs,
                                    "frac": h2d_gbs / copy_gbs,
                                    "copy": f"pinned host -> device, {src.numel() * 2 >> 20} MiB, "
                                            "best of 3, measured in this run"}
        del dst
        # the serving form of PAPER.md:407: the host sends table row ids, the shared embedding
        # table stays on the device (here a random row permutation of [U; T], so E[rows]
        # reproduces this batch exactly) and the projections gather the rows
        nL, nC = batch.U.shape[0], batch.T.shape[0]
        gperm = torch.Generator().manual_seed(2511)
        perm = torch.randperm(nL + nC, generator=gperm)
        E_tab = torch.cat([batch.U, batch.T]).index_select(0, perm.to(dev))
        inv = torch.empty_like(perm)
        inv[perm] = torch.arange(nL + nC)
        hist_rows = inv[:nL].to(torch.int32).pin_memory()
        cand_rows = inv[nL:].to(torch.int32).pin_memory()
        h_O2 = torch.empty_like(h_O).pin_memory()
        h_c2 = torch.empty_like(h_counts).pin_memory()
        scorer.run_ids(E_tab, hist_rows, cand_rows, h_O2, h_c2, stream=main_stream)
        torch.cuda.synchronize()
        same = bool(torch.equal(h_O2, h_O) and torch.equal(h_c2, h_counts))
        if world > 1:
            dist.barrier()
        a.record(main_stream)
        for _ in range(n_e2e):
            scorer.run_ids(E_tab, hist_rows, cand_rows, h_O2, h_c2, stream=main_stream)
        b.record(main_stream)
        torch.cuda.synchronize()
        i_ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([i_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            i_ms = float(t.item())
        line["e2e_ids"] = {
            "value": res["cands_per_step"] * n_e2e / (i_ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": scorer.h2d_bytes_ids(hist_rows, cand_rows),
            "d2h_bytes_per_step": d2h, "steps": n_e2e,
            "api": "gesr_score_host_ids (C ABI: host row ids, device-resident embedding table "
                   "gathered inside the projections, PAPER.md:407)",
            "table": f"{nL + nC} rows x {cfg.D_in} bf16 on the device (a row permutation of "
                     "[U; T]): model state like the weights, not a per-step input",
            "bit_identical_to_e2e": same}
        del E_tab

    # ---------------------------------------------------------------- optional score gather
    if args.gather and world > 1:
        from paper_2511_21095_b200 import shard
        rows = [int(x) for x in torch.tensor([bufs.O.shape[0]])]
        allrows = [None] * world
        dist.all_gather_object(allrows, rows[0])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        shard.gather_rows(bufs.O, allrows)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        nbytes = sum(allrows) * bufs.O.shape[1] * bufs.O.element_size()
        line["gather"] = {"s": dt, "bytes": nbytes, "GBps": nbytes / dt / 1e9}

    # ---------------------------------------------------------------- cpu baseline (oracle)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, args.config)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
