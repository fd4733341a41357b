"""GPU parity on the five BASELINE configs at full size, in bench.py's exact launch configuration
(VERDICT r1 missing 2, weak 2-3), plus the ABI arguments the headline never exercises.

bench.py times `binding.score_step(batch, StepBuffers(batch, out_dtype=bf16))`: HMA after the
attention on the same stream, kv_splits = 0 (auto), bf16 O through the TMA-store epilogue.  Here the
same two calls run on the whole config batch, then:

  * HMA counts are compared with the fp64/int64 oracle for EVERY candidate of all five configs
    (1, 2, 3, 3h, 4, 5; bit-exact; the oracle runs over request chunks of the same
    device-generated inputs);
  * attention rows are compared element by element (max-abs 2e-2, mean-abs 2e-3 vs fp64) on the
    SURVEY.md s8(c) seeded subset of >= 64 requests: the 8 longest-L, 8 shortest-L, 8 largest-C,
    8 smallest-C and 32 random requests (seed 2511), topped up with random ones if these overlap
    -- and every request of configs 1 (B = 1), 2 (B = 256) and 4 (B = 1, 8 candidate chunks of
    512 against one K/V cache, as bench.py runs it): SURVEY.md s8(c)'s full parity.

The oracle is fed `inputs.select_requests(...)` of the device batch: exactly the rows and IDs
the kernels scored (generator output, never a kernel output).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2511_21095_b200 import binding as gb
from paper_2511_21095_b200 import configs, inputs
from subsets import survey_subset

pytestmark = pytest.mark.gpu

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200 (run through gpurun)"
    return torch.device("cuda:0")


def _attn_check(O_gpu, O_or, what):
    O_gpu = O_gpu.astype(np.float64)
    assert np.isfinite(O_gpu).all(), f"{what}: non-finite output"
    diff = np.abs(O_gpu - O_or)
    mx, mn = float(diff.max()), float(diff.mean())
    assert mx <= MAX_ABS and mn <= MEAN_ABS, f"{what}: max-abs {mx:.3e} mean-abs {mn:.3e}"
    return mx, mn


def _rows_of(co: np.ndarray, reqs):
    return np.concatenate([np.arange(co[b], co[b + 1]) for b in reqs])


@pytest.mark.parametrize("name", ["1", "2", "3", "3h", "4", "5"])
def test_config_bench_launch_parity(name):
    dev = _cuda()
    cfg = configs.get(name)
    bt = inputs.make_batch(cfg, device=dev)
    bufs = gb.StepBuffers(bt, out_dtype=torch.bfloat16)      # bench.py's buffers
    gb.score_step(bt, bufs, chunk=cfg.chunk)                   # bench.py's step
    torch.cuda.synchronize()
    co = bt.cand_offsets.cpu().numpy()
    so = bt.seq_offsets.cpu().numpy()

    # HMA: every candidate, bit-exact, oracle over request chunks
    chunk = 512
    checked = 0
    for b0 in range(0, cfg.B, chunk):
        reqs = list(range(b0, min(cfg.B, b0 + chunk)))
        sub = inputs.select_requests(bt, reqs)
        want = oracle.hma_count(sub.user_ids, sub.user_offsets, sub.item_ids, sub.item_offsets,
                                sub.cand_offsets, cfg.F)
        got = bufs.counts[co[b0]:co[reqs[-1] + 1]].cpu().numpy()
        assert np.array_equal(got, want), f"config {name}: HMA mismatch in requests {b0}.."
        checked += got.shape[0]
    assert checked == bt.total_C

    # attention: the s8(c) subset, elementwise
    Ls, Cs = np.diff(so), np.diff(co)
    # full oracle parity for configs 1, 2 and 4, the seeded subset for 3 and 5
    reqs = list(range(cfg.B)) if cfg.B <= 256 else survey_subset(Ls, Cs)
    assert len(reqs) >= min(64, cfg.B)
    sub = inputs.select_requests(bt, reqs)
    K, V = oracle.kv_project(sub.U, sub.W_k, sub.W_v, cfg.H, cfg.d, act=cfg.act)
    O_or, _ = oracle.tasa_score(sub.T, sub.cand_offsets, sub.W_q, K, V, sub.seq_offsets, cfg.H,
                                cfg.d, act=cfg.act)
    rows = torch.as_tensor(_rows_of(co, reqs), device=dev)
    O = bufs.O[rows].float().cpu().numpy()
    mx, mn = _attn_check(O, O_or, f"config {name} subset of {len(reqs)} requests")
    print(f"config {name}: HMA {checked} candidates exact; attention {len(reqs)} requests "
          f"({rows.numel()} rows) max-abs {mx:.2e} mean-abs {mn:.2e}")


# ----------------------------------------------------------------------------- ABI arguments

def _ragged(d, H, D_in, cfg_id):
    cfg = configs.Config("args", cfg_id, B=7, L=("uniform", 0, 300), C=("uniform", 0, 280), H=H,
                         d=d, D_in=D_in, F=2)
    return cfg, inputs.make_batch(cfg, hma=False)


@pytest.mark.parametrize("d,H,D_in", [(32, 2, 64), (64, 2, 128), (128, 2, 256)])
@pytest.mark.parametrize("act", [0, 1])
@pytest.mark.parametrize("scale", [0.05, 0.0, 0.5])
def test_tasa_bias_scale_act(d, H, D_in, act, scale):
    """gesr_tasa_score with b_q != NULL, a non-default scale (0 -> 1/sqrt(d)) and act =
    identity / SiLU at d = 32 / 64 / 128 (1-CTA and pair kernels), fp32 O and lse.

    Gates: (1) against the rounding-aware oracle -- the same fp64 algorithm with K, V and q
    rounded to bf16 where the GPU path stores them (R8; oracle.round_to_bf16 and
    round_q_bf16) -- the north_star tolerance at every scale; (2) against the pure fp64 oracle
    the north_star tolerance at scales up to the configs' 1/sqrt(d).  Above it the bf16
    quantisation of q and K alone moves a score by up to ~scale * sum_j |q_j k_j| * 2^-8
    (0.5 * ~60 * 2^-8 ~ 0.1 at d = 32, identity act), which the softmax turns into O errors past
    2e-2 whatever the kernel does; there (2) is reported only."""
    dev = _cuda()
    cfg, bt = _ragged(d, H, D_in, 300 + d + act)
    HD = H * d
    b_q = torch.linspace(-0.8, 0.6, HD, dtype=torch.float32)
    b_k = torch.linspace(0.5, -0.5, HD, dtype=torch.float32)
    b_v = torch.linspace(-0.3, 0.9, HD, dtype=torch.float32)
    sc = None if scale == 0.0 else scale
    K_or, V_or = oracle.kv_project(bt.U, bt.W_k, bt.W_v, H, d, act=act, b_k=b_k.double(),
                                   b_v=b_v.double())
    O_or, lse_or = oracle.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K_or, V_or, bt.seq_offsets,
                                     H, d, act=act, b_q=b_q.double(), scale=sc)
    O_rq, _ = oracle.tasa_score(bt.T, bt.cand_offsets, bt.W_q, oracle.round_to_bf16(K_or),
                                oracle.round_to_bf16(V_or), bt.seq_offsets, H, d, act=act,
                                b_q=b_q.double(), scale=sc, round_q_bf16=True)
    g = bt.to(dev)
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, H, d, act, b_k=b_k.to(dev), b_v=b_v.to(dev))
    O, lse = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, H, d, act,
                           b_q=b_q.to(dev), scale=scale)
    torch.cuda.synchronize()
    O = O.cpu().numpy()
    _attn_check(O, O_rq, f"d={d} act={act} scale={scale} vs rounding-aware oracle")
    if scale <= 1.0 / math.sqrt(d):
        _attn_check(O, O_or, f"d={d} act={act} scale={scale} vs fp64 oracle")
        lse = lse.cpu().numpy()
        fin = np.isfinite(lse_or)
        assert np.array_equal(fin, np.isfinite(lse))
        assert np.abs(lse[fin] - lse_or[fin]).max() < 3e-2


@pytest.mark.parametrize("d", [64, 128])
def test_tasa_identity_bf16_out_forced_splits(d):
    """act = identity with bf16 O and forced kv_splits (split-L runs on the d = 128 pair kernel
    only): every split count gives the oracle's rows within tolerance; splits = 1 is
    bit-identical run to run."""
    dev = _cuda()
    cfg, bt = _ragged(d, 2, 128, 400 + d)
    K_or, V_or = oracle.kv_project(bt.U, bt.W_k, bt.W_v, 2, d, act=0)
    O_or, _ = oracle.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K_or, V_or, bt.seq_offsets, 2, d,
                                act=0)
    g = bt.to(dev)
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, 2, d, 0)
    outs = {}
    for s in ((1, 2, 3) if d == 128 else (1,)):
        O, _ = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, 2, d, 0,
                             kv_splits=s, out_dtype=torch.bfloat16, want_lse=False)
        outs[s] = O.clone()
        _attn_check(O.float().cpu().numpy(), O_or, f"identity d={d} splits={s}")
    O1b, _ = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, 2, d, 0,
                           kv_splits=1, out_dtype=torch.bfloat16, want_lse=False)
    torch.cuda.synchronize()
    assert torch.equal(O1b, outs[1])


def test_config5_lpt_shard_rows_bit_identical_to_larger_batch():
    """SURVEY s8(e) / VERDICT r1 next 4: an LPT shard of config 5's 8192 requests (the
    partition bench.py --gpus N --config 5 uses, here into 32 shards) scored alone gives exactly
    the rows the same requests get inside a larger batch (that shard followed by another one):
    d = 128 CTA-pair attention at a fixed kv_splits = 1, K/V projection and HMA counts.  Rows
    depend only on their own request, so the multi-GPU result is the single-GPU result."""
    from paper_2511_21095_b200 import shard
    dev = torch.device("cuda", 0)
    cfg = configs.get("5")
    L, C = inputs.request_lengths(cfg)
    parts = shard.lpt_partition(shard.request_cost(cfg, L.numpy(), C.numpy()), 32)
    a, b = [int(x) for x in parts[3]], [int(x) for x in parts[17]]

    def run(reqs):
        bt = inputs.make_batch(cfg, requests=reqs, device=dev)
        K, V = gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act)
        O, lse = gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H, cfg.d,
                               cfg.act, kv_splits=1, out_dtype=torch.bfloat16)
        c = gb.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                         bt.cand_offsets, cfg.F)
        torch.cuda.synchronize()
        return bt, K, O, lse, c

    bt_a, K_a, O_a, lse_a, c_a = run(a)
    _, K_u, O_u, lse_u, c_u = run(a + b)
    nL, nC = bt_a.U.shape[0], bt_a.T.shape[0]
    assert torch.equal(K_u[:, :nL], K_a)
    assert torch.equal(O_u[:nC], O_a) and torch.equal(lse_u[:nC], lse_a)
    assert torch.equal(c_u[:nC], c_a)
