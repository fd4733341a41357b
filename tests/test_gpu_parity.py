"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same seeded inputs.

Gates (BASELINE.json north_star): HMA counts and jagged indexing bit-exact; attention within
max-abs 2e-2 and mean-abs 2e-3 of the pure fp64 oracle; K/V cache within one bf16 ulp plus the
fp32-accumulation term 2^-20 * sum_k |U_k W_k| (DESIGN.md s3 R8).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2511_21095_b200 import binding as gb
from paper_2511_21095_b200 import configs, inputs

pytestmark = pytest.mark.gpu

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200 (run through gpurun)"
    return torch.device("cuda:0")


def _bf16_ulp(x: np.ndarray) -> np.ndarray:
    ax = np.maximum(np.abs(x), 2.0 ** -126)
    return 2.0 ** (np.floor(np.log2(ax)) - 7)


def _check_kv(U, W, K_gpu, K_or, H, d):
    Uf = U.double()
    acc = (Uf.abs() @ W.double().abs().T).reshape(-1, H, d).permute(1, 0, 2).numpy()
    got = K_gpu.float().cpu().double().numpy()
    err = np.abs(got - K_or)
    tol = _bf16_ulp(K_or) + 2.0 ** -20 * acc + 1e-30
    bad = err > tol
    assert not bad.any(), f"{bad.sum()} K/V elements out of tolerance; max err {err.max()}"


def _attn_tol(O_gpu, O_or, what=""):
    diff = np.abs(O_gpu.astype(np.float64) - O_or)
    assert np.isfinite(O_gpu).all(), f"{what}: non-finite output"
    mx, mn = diff.max() if diff.size else 0.0, diff.mean() if diff.size else 0.0
    assert mx <= MAX_ABS and mn <= MEAN_ABS, f"{what}: max-abs {mx:.3e} mean-abs {mn:.3e}"
    return mx, mn


def _run_oracle_attn(bt, act=1):
    cfg = bt.cfg
    K, V = oracle.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, act=act)
    O, lse = oracle.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H,
                               cfg.d, act=act)
    return K, V, O, lse


def _run_gpu_attn(bt, act=1, out_dtype=torch.float32):
    cfg = bt.cfg
    g = bt.to(_cuda())
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, cfg.H, cfg.d, act)
    O, lse = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, cfg.H, cfg.d, act,
                           out_dtype=out_dtype)
    torch.cuda.synchronize()
    return K.cpu(), V.cpu(), O.float().cpu().numpy(), lse.cpu().numpy()


def _custom(Ls, Cs, H=2, d=64, D_in=128, cfg_id=77):
    cfg = configs.Config("custom", cfg_id, B=len(Ls), L=("fixed", 1), C=("fixed", 1), H=H, d=d,
                         D_in=D_in, F=4)
    bt = inputs.make_batch(cfg, hma=False)
    # overwrite lengths: regenerate rows for the requested jagged shape
    so = torch.tensor(np.concatenate([[0], np.cumsum(Ls)]), dtype=torch.int64)
    co = torch.tensor(np.concatenate([[0], np.cumsum(Cs)]), dtype=torch.int64)
    g = torch.Generator().manual_seed(cfg_id * 1000 + len(Ls))
    U = torch.randn(int(so[-1]), D_in, generator=g).to(torch.bfloat16)
    T = torch.randn(int(co[-1]), D_in, generator=g).to(torch.bfloat16)
    return inputs.Batch(cfg, torch.arange(len(Ls)), so, co, U, T, bt.W_q, bt.W_k, bt.W_v,
                        None, None, None, None)


# ----------------------------------------------------------------------------- K/V projection

@pytest.mark.parametrize("name", ["1", "2"])
@pytest.mark.parametrize("act", [0, 1])
def test_kv_project_parity(name, act):
    cfg = configs.get(name)
    bt = inputs.make_batch(cfg, hma=False)
    K_or, V_or = oracle.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, act=act)
    g = bt.to(_cuda())
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, cfg.H, cfg.d, act)
    torch.cuda.synchronize()
    _check_kv(bt.U, bt.W_k, K.cpu(), K_or, cfg.H, cfg.d)
    _check_kv(bt.U, bt.W_v, V.cpu(), V_or, cfg.H, cfg.d)


@pytest.mark.parametrize("M,D_in,H,d", [(300, 512, 4, 128), (129, 64, 1, 32), (1, 40, 2, 64),
                                         (1000, 256, 3, 64)])
def test_kv_project_shapes(M, D_in, H, d):
    cfg = configs.Config("kvshape", 90, B=1, L=("fixed", M), C=("fixed", 1), H=H, d=d, D_in=D_in,
                         F=1)
    bt = inputs.make_batch(cfg, hma=False)
    K_or, V_or = oracle.kv_project(bt.U, bt.W_k, bt.W_v, H, d, act=1)
    g = bt.to(_cuda())
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, H, d, 1)
    torch.cuda.synchronize()
    _check_kv(bt.U, bt.W_k, K.cpu(), K_or, H, d)
    _check_kv(bt.U, bt.W_v, V.cpu(), V_or, H, d)


def test_kv_project_bias():
    cfg = configs.get("2").with_(B=3)
    bt = inputs.make_batch(cfg, hma=False)
    HD = cfg.H * cfg.d
    bk = torch.linspace(-1, 1, HD, dtype=torch.float32)
    bv = torch.linspace(2, -2, HD, dtype=torch.float32)
    K_or, V_or = oracle.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, 1, b_k=bk.double(),
                                   b_v=bv.double())
    g = bt.to(_cuda())
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, cfg.H, cfg.d, 1, b_k=bk.cuda(), b_v=bv.cuda())
    torch.cuda.synchronize()
    # the bias adds |b| to the accumulation scale
    _check_kv(bt.U, bt.W_k, K.cpu(), K_or, cfg.H, cfg.d)
    _check_kv(bt.U, bt.W_v, V.cpu(), V_or, cfg.H, cfg.d)


# ----------------------------------------------------------------------------- attention

@pytest.mark.parametrize("name", ["1", "2"])
def test_tasa_parity_configs(name):
    cfg = configs.get(name)
    bt = inputs.make_batch(cfg, hma=False)
    _, _, O_or, lse_or = _run_oracle_attn(bt)
    _, _, O, lse = _run_gpu_attn(bt)
    _attn_tol(O, O_or, f"config {name}")
    fin = np.isfinite(lse_or)
    assert np.array_equal(fin, np.isfinite(lse))
    assert np.abs(lse[fin] - lse_or[fin]).max() < 2e-2


@pytest.mark.parametrize("d,H,D_in", [(128, 2, 256), (64, 2, 128), (32, 3, 96)])
def test_tasa_ragged_edges(d, H, D_in):
    # L in {0, 1, 127, 128, 129, 300}, C in {0, 1, 128, 129, 256, 257, 300}: empty, single,
    # exact-tile and ragged tails on both axes
    Ls = [0, 1, 127, 128, 129, 300, 5, 260]
    Cs = [3, 1, 128, 129, 256, 257, 0, 300]
    bt = _custom(Ls, Cs, H=H, d=d, D_in=D_in, cfg_id=d)
    _, _, O_or, lse_or = _run_oracle_attn(bt)
    _, _, O, lse = _run_gpu_attn(bt)
    _attn_tol(O, O_or, "ragged")
    # L_b = 0 rows are exactly zero with lse = -inf (reading R6)
    assert np.all(O[:3] == 0) and np.all(np.isneginf(lse[:3]))


def test_tasa_bf16_output():
    bt = _custom([200, 50], [130, 7], H=2, d=128, D_in=128, cfg_id=5)
    _, _, O_or, _ = _run_oracle_attn(bt)
    _, _, O, _ = _run_gpu_attn(bt, out_dtype=torch.bfloat16)
    _attn_tol(O, O_or, "bf16 out")


def test_single_token_history_returns_cached_v_exactly():
    bt = _custom([1, 1, 1], [5, 130, 2], H=2, d=64, D_in=128, cfg_id=11)
    K, V, O, _ = _run_gpu_attn(bt)
    Vf = V.float().numpy()
    co = bt.cand_offsets.numpy()
    for b in range(3):
        for h in range(2):
            want = Vf[h, b]
            got = O[co[b]:co[b + 1], h * 64:(h + 1) * 64]
            assert np.array_equal(got, np.broadcast_to(want, got.shape))


def test_uniform_scores_mean_pooling():
    bt = _custom([300, 7], [10, 140], H=2, d=64, D_in=128, cfg_id=12)
    bt.W_q.zero_()
    K, V, O, _ = _run_gpu_attn(bt)
    # closed form on the GPU's own bf16 cache: O = mean of V rows (within fp32/bf16-P rounding)
    Vf = V.double().numpy()
    so, co = bt.seq_offsets.numpy(), bt.cand_offsets.numpy()
    for b in range(2):
        mean = Vf[:, so[b]:so[b + 1]].mean(axis=1).reshape(-1)     # [H*d] in head order
        got = O[co[b]:co[b + 1]]
        assert np.abs(got - mean).max() < 1e-5


def test_request_boundary_canary():
    """K = 0, V = +1 for even b and 1000 for odd b: any key leaked from a neighbour request
    (or head) shifts O by >= 999/(L_b+1)."""
    dev = _cuda()
    Ls = [130, 1, 257, 128, 3, 700]
    Cs = [260, 2, 1, 129, 300, 5]
    H, d, D_in = 2, 128, 128
    so = torch.tensor(np.concatenate([[0], np.cumsum(Ls)]), dtype=torch.int64, device=dev)
    co = torch.tensor(np.concatenate([[0], np.cumsum(Cs)]), dtype=torch.int64, device=dev)
    tl, tc = int(so[-1]), int(co[-1])
    K = torch.zeros((H, tl, d), dtype=torch.bfloat16, device=dev)
    V = torch.empty((H, tl, d), dtype=torch.bfloat16, device=dev)
    for b in range(len(Ls)):
        for h in range(H):
            V[h, so[b]:so[b + 1]] = (1.0 if b % 2 == 0 else 1000.0) + 10 * h
    T = torch.randn(tc, D_in, device=dev).to(torch.bfloat16)
    Wq = (torch.randn(H * d, D_in, device=dev) * 0.05).to(torch.bfloat16)
    O, _ = gb.tasa_score(T, co, Wq, K, V, so, H, d)
    torch.cuda.synchronize()
    O = O.cpu().numpy()
    coc = co.cpu().numpy()
    Vc = V.float().cpu().numpy()
    soc = so.cpu().numpy()
    for b in range(len(Ls)):
        for h in range(H):
            want = float(Vc[h, soc[b], 0])      # the bf16 value actually stored
            got = O[coc[b]:coc[b + 1], h * d:(h + 1) * d]
            assert np.abs(got - want).max() <= 1e-2 * max(1.0, want / 100), (b, h)


def test_output_canary_tail_untouched():
    bt = _custom([100, 200], [3, 130], H=2, d=64, D_in=64, cfg_id=13)
    g = bt.to(_cuda())
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, 2, 64, 1)
    big = torch.full((bt.total_C + 37, 128), 12345.0, device="cuda")
    lse_big = torch.full((bt.total_C + 37, 2), 777.0, device="cuda")
    gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, 2, 64, O=big[:bt.total_C],
                  lse=lse_big[:bt.total_C])
    torch.cuda.synchronize()
    assert torch.all(big[bt.total_C:] == 12345.0) and torch.all(lse_big[bt.total_C:] == 777.0)
    assert not torch.any(big[:bt.total_C] == 12345.0)


def test_chunk_invariance_and_determinism_exact():
    """Config 4 style: one cache, candidates scored in chunks of 512 vs one call: bit-exact."""
    cfg = configs.get("4").with_(L=("fixed", 1000), C=("fixed", 1100))
    bt = inputs.make_batch(cfg, hma=False)
    g = bt.to(_cuda())
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, cfg.H, cfg.d, 1)
    O1, l1 = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, cfg.H, cfg.d, kv_splits=1)
    parts = []
    for c0 in range(0, 1100, 512):
        c1 = min(1100, c0 + 512)
        co = torch.tensor([0, c1 - c0], dtype=torch.int64, device="cuda")
        parts.append(gb.tasa_score(g.T[c0:c1].contiguous(), co, g.W_q, K, V, g.seq_offsets,
                                   cfg.H, cfg.d, kv_splits=1)[0])
    O2 = torch.cat(parts)
    O3, l3 = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, cfg.H, cfg.d, kv_splits=1)
    torch.cuda.synchronize()
    assert torch.equal(O1, O2)
    assert torch.equal(O1, O3) and torch.equal(l1, l3)


def test_batch_composition_invariance_exact():
    """A request's rows are bit-identical whether scored alone or inside a batch (R9)."""
    cfg = configs.get("2").with_(B=12)
    full = inputs.make_batch(cfg, hma=False)
    _, _, O_full, _ = _run_gpu_attn(full)
    sub = [3, 7, 8]
    part = inputs.make_batch(cfg, requests=sub, hma=False)
    _, _, O_part, _ = _run_gpu_attn(part)
    co = full.cand_offsets.numpy()
    rows = np.concatenate([np.arange(co[b], co[b + 1]) for b in sub])
    assert np.array_equal(O_full[rows], O_part)


def test_large_scores_no_overflow():
    bt = _custom([300, 129], [140, 20], H=2, d=64, D_in=128, cfg_id=14)
    g = bt.to(_cuda())
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, 2, 64, 1)
    O, lse = gb.tasa_score(g.T, g.cand_offsets, g.W_q * 40, K * 40, V, g.seq_offsets, 2, 64)
    torch.cuda.synchronize()
    assert torch.isfinite(O).all() and torch.isfinite(lse).all()
    Vmax = V.float().abs().max()
    assert O.abs().max() <= Vmax * 1.01


@pytest.mark.parametrize("d", [128, 64])
def test_growing_scores_raise_running_max(d):
    # Key tiles whose scores grow tile by tile (x(1 + 3t)) and, at the end of request 0, jump by
    # far more than 128 (log2 units) over everything before: exercises the lazy-rescale slow
    # paths (running max raised, O rescaled, P recomputed after an overflowing speculative exp)
    H, D_in = 2, 128
    Ls, Cs = [1024, 700, 129], [150, 37, 260]
    bt = _custom(Ls, Cs, H=H, d=d, D_in=D_in, cfg_id=300 + d)
    K, V = oracle.kv_project(bt.U, bt.W_k, bt.W_v, H, d, act=1)
    so = bt.seq_offsets.numpy()
    f = np.ones(K.shape[1])
    for b in range(len(Ls)):
        t = np.arange(Ls[b]) // 128
        f[so[b]:so[b + 1]] = 1.0 + 3.0 * t
    f[so[0] + 1000:so[0] + 1024] = 60.0
    f[so[2] + 128] = 80.0                       # a lone huge key in a 1-key tail tile
    Kb = torch.from_numpy(K * f[None, :, None]).to(torch.bfloat16)
    Vb = torch.from_numpy(V).to(torch.bfloat16)
    # Q rounded to bf16 as the kernel's Q is (R8): with keys scaled x60-80 the
    # 2^-9 rounding of Q alone moves scores by ~0.3
    O_or, lse_or = oracle.tasa_score(bt.T, bt.cand_offsets, bt.W_q, Kb.double().numpy(),
                                     Vb.double().numpy(), bt.seq_offsets, H, d, round_q_bf16=True)
    g = bt.to(_cuda())
    O, lse = gb.tasa_score(g.T, g.cand_offsets, g.W_q, Kb.to(_cuda()), Vb.to(_cuda()),
                           g.seq_offsets, H, d, 1)
    torch.cuda.synchronize()
    _attn_tol(O.float().cpu().numpy(), O_or, f"growing scores d={d}")
    assert np.abs(lse.cpu().numpy() - lse_or).max() < 5e-2


@pytest.mark.parametrize("splits", [2, 3, 8])
def test_split_l_parity(splits):
    # forced split-L (d = 128): ranges of key tiles computed apart and merged; L < 128 * splits
    # leaves empty splits, L = 0 gives O = 0 / lse = -inf
    Ls = [0, 1, 127, 129, 300, 700, 1030, 5]
    Cs = [3, 40, 128, 129, 256, 257, 130, 2]
    bt = _custom(Ls, Cs, H=2, d=128, D_in=256, cfg_id=400 + splits)
    K, V, O_or, lse_or = _run_oracle_attn(bt)
    g = bt.to(_cuda())
    Kg, Vg = gb.kv_project(g.U, g.W_k, g.W_v, 2, 128, 1)
    O, lse = gb.tasa_score(g.T, g.cand_offsets, g.W_q, Kg, Vg, g.seq_offsets, 2, 128, 1,
                           kv_splits=splits)
    torch.cuda.synchronize()
    _attn_tol(O.cpu().numpy(), O_or, f"split-L {splits}")
    lse = lse.cpu().numpy()
    fin = np.isfinite(lse_or)
    assert np.array_equal(fin, np.isfinite(lse))
    assert np.abs(lse[fin] - lse_or[fin]).max() < 2e-2
    assert np.all(O.cpu().numpy()[:3] == 0)


def test_split_l_batch_invariance_exact():
    # a fixed kv_splits is batch-invariant: config 4 style chunks of one cache == one call
    cfg = configs.get("4").with_(L=("fixed", 1500), C=("fixed", 700))
    bt = inputs.make_batch(cfg, hma=False)
    g = bt.to(_cuda())
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, cfg.H, cfg.d, 1)
    O1, l1 = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, cfg.H, cfg.d,
                           kv_splits=6)
    parts = []
    for c0 in range(0, 700, 256):
        c1 = min(700, c0 + 256)
        co = torch.tensor([0, c1 - c0], dtype=torch.int64, device="cuda")
        parts.append(gb.tasa_score(g.T[c0:c1].contiguous(), co, g.W_q, K, V, g.seq_offsets,
                                   cfg.H, cfg.d, kv_splits=6)[0])
    torch.cuda.synchronize()
    assert torch.equal(O1, torch.cat(parts))


@pytest.mark.parametrize("name", ["1", "4"])
def test_cuda_graph_capture_identical(name):
    # the C-ABI calls are capturable (no host sync, no allocation): a captured step replays to
    # the eager step's exact outputs (configs 1 and 4 are measured under graphs)
    cfg = configs.get(name)
    bt = inputs.make_batch(cfg, device=_cuda())
    bufs = gb.StepBuffers(bt, out_dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        gb.score_step(bt, bufs, chunk=cfg.chunk, stream=s)
        torch.cuda.synchronize()
        O_ref, c_ref = bufs.O.clone(), bufs.counts.clone()
        bufs.O.zero_()
        bufs.counts.zero_()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            gb.score_step(bt, bufs, chunk=cfg.chunk, stream=s)
        g.replay()
        torch.cuda.synchronize()
    assert torch.equal(bufs.O, O_ref) and torch.equal(bufs.counts, c_ref)


@pytest.mark.parametrize("d,H,D_in", [(128, 2, 256), (64, 2, 128), (32, 1, 64)])
def test_self_key_parity(d, H, D_in):
    # gesr_tasa_score_self: the candidate also attends to its own key (SPEC.md's mask diagonal)
    # vs the brute-force oracle over the full [U; T] mask with self_key=True; L_b = 0 included
    Ls, Cs = [0, 1, 130, 300, 7], [3, 5, 140, 129, 2]
    bt = _custom(Ls, Cs, H=H, d=d, D_in=D_in, cfg_id=500 + d)
    g = bt.to(_cuda())
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, H, d, 1)
    Ks, Vs = gb.kv_project(g.T, g.W_k, g.W_v, H, d, 1)
    for odt in (torch.float32, torch.bfloat16):
        O, lse = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, H, d, 1,
                               out_dtype=odt, K_self=Ks, V_self=Vs)
        torch.cuda.synchronize()
        O, lse = O.float().cpu().numpy(), lse.cpu().numpy()
        so, co = bt.seq_offsets.numpy(), bt.cand_offsets.numpy()
        for b in range(len(Ls)):
            O_or, lse_or = oracle.full_masked_attention(bt.U[so[b]:so[b + 1]], bt.T[co[b]:co[b + 1]],
                                                        bt.W_q, bt.W_k, bt.W_v, H, d,
                                                        self_key=True)
            _attn_tol(O[co[b]:co[b + 1]], O_or, f"self key d={d} request {b}")
            assert np.abs(lse[co[b]:co[b + 1]] - lse_or).max() < 2e-2


def test_one_cta_kernel_d128_subprocess():
    # d = 128 runs the CTA-pair kernel by default; the 1-CTA kernel (GESR_ATTN_PAIR=0, read once
    # per process) keeps its own parity check on ragged shapes and bf16 output
    import os
    import subprocess
    import sys
    code = (
        "import importlib.util, sys; sys.path.insert(0, '.'); "
        "spec = importlib.util.spec_from_file_location('tgp', 'tests/test_gpu_parity.py'); "
        "t = importlib.util.module_from_spec(spec); spec.loader.exec_module(t); "
        "t.test_tasa_ragged_edges(128, 2, 256); t.test_tasa_bf16_output(); "
        "t.test_growing_scores_raise_running_max(128); print('one-cta ok')")
    env = dict(os.environ, GESR_ATTN_PAIR="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "one-cta ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


# ----------------------------------------------------------------------------- HMA

def _hma_gpu(bt, F, cap=0):
    g = bt.to(_cuda())
    c = gb.hma_count(g.user_ids, g.user_offsets, g.item_ids, g.item_offsets, g.cand_offsets, F,
                     cap)
    torch.cuda.synchronize()
    return c.cpu().numpy()


@pytest.mark.parametrize("name", ["1", "2"])
@pytest.mark.parametrize("cap", [0, 16])
def test_hma_bit_exact_configs(name, cap):
    cfg = configs.get(name)
    bt = inputs.make_batch(cfg, attention=False)
    want = oracle.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                            bt.cand_offsets, cfg.F, cap=cap)
    assert np.array_equal(_hma_gpu(bt, cfg.F, cap), want)


def test_hma_duplicates_and_long_lists():
    # duplicates (pairwise reading R11), user lists longer than the smem pool (global fallback)
    cfg = configs.get("2").with_(B=9, user_len=(0, 3000), vocab=4096, F=3)
    bt = inputs.make_batch(cfg, attention=False, hma_duplicates=True)
    for cap in (0, 5):
        want = oracle.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                                bt.cand_offsets, cfg.F, cap=cap)
        assert np.array_equal(_hma_gpu(bt, cfg.F, cap), want)


def test_hma_oversized_groups_and_empty_item_lists():
    # item lists of 0..32 IDs: some 32-segment groups exceed the per-warp staging buffer
    # (512 IDs) and read their IDs from global memory; empty item lists count 0
    cfg = configs.get("2").with_(B=6, item_len=(0, 32), vocab=256, F=5)
    bt = inputs.make_batch(cfg, attention=False, hma_duplicates=True)
    for cap in (0, 3):
        want = oracle.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                                bt.cand_offsets, cfg.F, cap=cap)
        assert np.array_equal(_hma_gpu(bt, cfg.F, cap), want)


def test_hma_edge_ids_and_empty():
    dev = _cuda()
    F = 2
    # request 0: 3 candidates; request 1: 0 candidates; request 2: 2 candidates
    co = torch.tensor([0, 3, 3, 5], dtype=torch.int64)
    imin, imax = -(1 << 63), (1 << 63) - 1
    users = [[imin, imin, 5], [], [], [imax, 0], [7], [7, 7, 7]]
    items = [[imin], [5, 5], [], [imax], [1, 2, 3], [imin, 0], [], [7, 7], [imin], [9]]
    uo = np.concatenate([[0], np.cumsum([len(x) for x in users])])
    io = np.concatenate([[0], np.cumsum([len(x) for x in items])])
    ui = np.array([v for x in users for v in x], np.int64)
    ii = np.array([v for x in items for v in x], np.int64)
    want = oracle.hma_count(ui, uo, ii, io, co, F)
    c = gb.hma_count(torch.tensor(ui, device=dev), torch.tensor(uo, device=dev),
                     torch.tensor(ii, device=dev), torch.tensor(io, device=dev), co.to(dev), F)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy(), want)
    assert want[0, 0] == 2   # sentinel-valued ID counted


@pytest.mark.parametrize("name,M,D_h", [("2", 16, 8), ("3", 4, 64), ("1", 1, 16)])
def test_hma_offset_embed_exact(name, M, D_h):
    # fused counting + offset-embedding gather: counts and the concatenated rows
    # bit-exact against the oracle's counts (cap M) and its plain-numpy gather
    cfg = configs.get(name)
    if cfg.B > 64:
        cfg = cfg.with_(B=64)
    bt = inputs.make_batch(cfg, attention=False)
    g = torch.Generator().manual_seed(11)
    E = torch.randn(cfg.F * (M + 1), D_h, generator=g).to(torch.bfloat16)
    dev = _cuda()
    c, e = gb.hma_count_embed(bt.user_ids.to(dev), bt.user_offsets.to(dev), bt.item_ids.to(dev),
                              bt.item_offsets.to(dev), bt.cand_offsets.to(dev), cfg.F, M,
                              E.to(dev))
    torch.cuda.synchronize()
    want_c = oracle.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                              bt.cand_offsets, cfg.F, M)
    assert np.array_equal(c.cpu().numpy(), want_c)
    want_e = oracle.hma_offset_embed(want_c, E.view(torch.int16).numpy(), M)
    assert np.array_equal(e.view(torch.int16).cpu().numpy(), want_e)


def test_hma_headline_subset():
    cfg = configs.get("3h")
    sub = list(range(0, 1024, 97))
    bt = inputs.make_batch(cfg, requests=sub, attention=False)
    want = oracle.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                            bt.cand_offsets, cfg.F)
    assert np.array_equal(_hma_gpu(bt, cfg.F), want)


# ----------------------------------------------------------------------------- full size, sampled

def test_headline_full_size_sampled():
    """Config 3h (L=2048, C=1000, B=1024) run in full on the GPU exactly as bench.py launches
    it; sampled requests checked against the oracle (attention tolerance, HMA bit-exact)."""
    dev = _cuda()
    cfg = configs.get("3h")
    bt = inputs.make_batch(cfg, device=dev)
    bufs = gb.StepBuffers(bt, want_lse=True)
    O, counts = gb.score_step(bt, bufs)
    torch.cuda.synchronize()
    sample = [0, 1, 511, 1023]
    sub = inputs.make_batch(cfg, requests=sample)
    _, _, O_or, _ = _run_oracle_attn(sub)
    co = bt.cand_offsets.cpu().numpy()
    rows = np.concatenate([np.arange(co[b], co[b + 1]) for b in sample])
    _attn_tol(O[torch.as_tensor(rows, device=dev)].cpu().numpy(), O_or, "3h sampled")
    want = oracle.hma_count(sub.user_ids, sub.user_offsets, sub.item_ids, sub.item_offsets,
                            sub.cand_offsets, cfg.F)
    assert np.array_equal(counts[torch.as_tensor(rows, device=dev)].cpu().numpy(), want)


@pytest.mark.parametrize("name", ["3", "4", "5"])
def test_config_full_size_sampled(name):
    """BASELINE configs 3 (jagged L <= 2048), 4 (L=4096 cache reused over 8 candidate chunks of
    512) and 5 (8192 requests, L log-uniform 32-4096, C 100-2000) run in full through
    score_step; sampled requests checked against the oracle (attention tolerance, HMA exact)."""
    dev = _cuda()
    cfg = configs.get(name)
    bt = inputs.make_batch(cfg, device=dev)
    bufs = gb.StepBuffers(bt, want_lse=True)
    O, counts = gb.score_step(bt, bufs, chunk=cfg.chunk)
    torch.cuda.synchronize()
    sample = sorted({0, cfg.B // 3, cfg.B // 2, cfg.B - 1})
    sub = inputs.make_batch(cfg, requests=sample)
    _, _, O_or, _ = _run_oracle_attn(sub)
    co = bt.cand_offsets.cpu().numpy()
    rows = np.concatenate([np.arange(co[b], co[b + 1]) for b in sample])
    _attn_tol(O[torch.as_tensor(rows, device=dev)].cpu().numpy(), O_or, f"config {name} sampled")
    want = oracle.hma_count(sub.user_ids, sub.user_offsets, sub.item_ids, sub.item_offsets,
                            sub.cand_offsets, cfg.F)
    assert np.array_equal(counts[torch.as_tensor(rows, device=dev)].cpu().numpy(), want)



@pytest.mark.parametrize("pattern", ["hi_bits", "sequential", "same_fold"])
def test_hma_structured_ids(pattern):
    # IDs built to collide under the table hash (low halves zero / consecutive values / equal
    # lo^hi folds): long probe chains, results must stay exact
    dev = _cuda()
    rng = np.random.default_rng(5)
    F, B, C = 3, 4, 50
    def ids(n, f):
        v = rng.integers(0, 96, size=n).astype(np.int64)
        if pattern == "hi_bits":
            return (v + 1000 * f) << 32
        if pattern == "sequential":
            return v + 1000 * f
        return ((v + 7 * f) << 32) | (v + 7 * f)        # lo ^ hi = 0 for every ID
    ulen = rng.integers(0, 65, size=B * F)
    users = [ids(int(n), k % F) for k, n in enumerate(ulen)]
    ilen = rng.integers(1, 17, size=B * C * F)
    items = [ids(int(n), k % F) for k, n in enumerate(ilen)]
    uo = np.concatenate([[0], np.cumsum([len(x) for x in users])]).astype(np.int64)
    io = np.concatenate([[0], np.cumsum([len(x) for x in items])]).astype(np.int64)
    co = np.arange(B + 1, dtype=np.int64) * C
    ui = np.concatenate(users).astype(np.int64)
    ii = np.concatenate(items).astype(np.int64)
    want = oracle.hma_count(ui, uo, ii, io, co, F)
    c = gb.hma_count(torch.tensor(ui, device=dev), torch.tensor(uo, device=dev),
                     torch.tensor(ii, device=dev), torch.tensor(io, device=dev),
                     torch.tensor(co, device=dev), F)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy(), want)
    assert want.sum() > 0


def test_score_host_matches_score_step_exactly():
    """End-to-end path through the C ABI (gesr_score_host: host-resident pinned inputs, request
    chunks pipelined over H2D / kernels / D2H inside the library) gives the same O and counts as
    score_step on device-resident inputs: rows are independent of batch composition (reading
    R9; no split-L at these sizes).  Also pageable host buffers and a single chunk."""
    dev = _cuda()
    cfg = configs.get("2")
    bt = inputs.make_batch(cfg)
    g = bt.to(dev)
    bufs = gb.StepBuffers(g, out_dtype=torch.bfloat16)
    O, counts = gb.score_step(g, bufs)
    pin = lambda t: t.contiguous().pin_memory()   # noqa: E731
    hb = inputs.Batch(cfg, bt.requests, pin(bt.seq_offsets), pin(bt.cand_offsets), pin(bt.U),
                      pin(bt.T), bt.W_q, bt.W_k, bt.W_v, pin(bt.user_ids), pin(bt.user_offsets),
                      pin(bt.item_ids), pin(bt.item_offsets))
    for batch, chunks in ((hb, 1), (hb, 3), (hb, 5), (bt, 4)):
        plan = gb.HostPlan(batch, n_chunks=chunks, out_dtype=torch.bfloat16, device=dev)
        h_O = torch.zeros(O.shape, dtype=O.dtype).pin_memory()
        h_c = torch.zeros(counts.shape, dtype=torch.int32).pin_memory()
        plan.run(h_O, h_c)
        plan.run(h_O, h_c)         # twice: buffer sets reused across passes
        torch.cuda.synchronize()
        assert torch.equal(h_O, O.cpu()), chunks
        assert torch.equal(h_c, counts.cpu()), chunks
        plan.close()


@pytest.mark.parametrize("B,L,C", [(20, ("uniform", 0, 5), ("uniform", 0, 300)),
                                   (16, ("uniform", 0, 400), ("uniform", 0, 4))])
def test_score_host_jagged_d128_fp32_cap(B, L, C):
    """gesr_score_host on a jagged d=128 batch (the CTA-pair kernel) with empty histories (first
    case: 3 of 20) or empty candidate lists (second: 2 of 16), fp32 output and an HMA cap:
    bit-identical to the device-resident calls with the same options."""
    dev = _cuda()
    cfg = configs.get("3").with_(B=B, L=L, C=C, F=4)
    bt = inputs.make_batch(cfg)
    g = bt.to(dev)
    K, V = gb.kv_project(g.U, g.W_k, g.W_v, cfg.H, cfg.d, cfg.act)
    O, _ = gb.tasa_score(g.T, g.cand_offsets, g.W_q, K, V, g.seq_offsets, cfg.H, cfg.d, cfg.act,
                         want_lse=False)
    counts = gb.hma_count(g.user_ids, g.user_offsets, g.item_ids, g.item_offsets,
                          g.cand_offsets, cfg.F, 3)
    torch.cuda.synchronize()
    pin = lambda t: t.contiguous().pin_memory()   # noqa: E731
    hb = inputs.Batch(cfg, bt.requests, pin(bt.seq_offsets), pin(bt.cand_offsets), pin(bt.U),
                      pin(bt.T), bt.W_q, bt.W_k, bt.W_v, pin(bt.user_ids), pin(bt.user_offsets),
                      pin(bt.item_ids), pin(bt.item_offsets))
    for chunks in (2, 4):
        plan = gb.HostPlan(hb, n_chunks=chunks, out_dtype=torch.float32, cap=3, device=dev)
        h_O = torch.full(O.shape, float("nan"), dtype=torch.float32).pin_memory()
        h_c = torch.full(counts.shape, -1, dtype=torch.int32).pin_memory()
        plan.run(h_O, h_c)
        torch.cuda.synchronize()
        assert torch.equal(h_O, O.cpu()), chunks
        assert torch.equal(h_c, counts.cpu()), chunks
        plan.close()


def test_hma_int64_min_in_long_and_short_lists():
    """INT64_MIN inside a user list too long for the shared-memory tables (the
    global-memory path) and inside short lists (the bucket path: an ordinary key there), plus
    the two empty-slot filler values (1 and 2) as user and item IDs."""
    dev = _cuda()
    rng = np.random.default_rng(17)
    imin = -(1 << 63)
    F = 3
    # request 0: field 0 has a 3000-long list with INT64_MIN twice; request 1: short lists
    long_list = rng.integers(-(1 << 62), 1 << 62, size=3000).astype(np.int64)
    long_list[[7, 2999]] = imin
    users = [long_list, np.array([imin, 1, 2], np.int64), np.array([2, 2, 5], np.int64),
             np.array([imin], np.int64), np.array([1, imin, 9], np.int64), np.array([], np.int64)]
    C = [40, 30]
    co = np.array([0, C[0], C[0] + C[1]], np.int64)
    items = []
    for b in range(2):
        for t in range(C[b]):
            for f in range(F):
                u = users[b * F + f]
                pick = rng.choice(np.concatenate([u, [imin, 1, 2, 3]]).astype(np.int64),
                                  size=int(rng.integers(1, 9)))
                items.append(pick.astype(np.int64))
    uo = np.concatenate([[0], np.cumsum([len(x) for x in users])]).astype(np.int64)
    io = np.concatenate([[0], np.cumsum([len(x) for x in items])]).astype(np.int64)
    ui = np.concatenate(users).astype(np.int64)
    ii = np.concatenate(items).astype(np.int64)
    want = oracle.hma_count(ui, uo, ii, io, co, F)
    c = gb.hma_count(torch.tensor(ui, device=dev), torch.tensor(uo, device=dev),
                     torch.tensor(ii, device=dev), torch.tensor(io, device=dev),
                     torch.tensor(co, device=dev), F)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy(), want)
    assert want[:, 0].max() >= 2          # INT64_MIN matched twice in the long list


def test_chunked_score_step_workspace_large_chunked_request():
    """score_step(chunk=...) on one request with C >= 4608 (the split-L reserve of a
    512-row chunk exceeds the full batch's): StepBuffers sizes the workspace for both."""
    dev = _cuda()
    cfg = configs.get("4").with_(C=("fixed", 5120), L=("fixed", 1024))
    bt = inputs.make_batch(cfg, device=dev)
    bufs = gb.StepBuffers(bt, out_dtype=torch.bfloat16)
    O, counts = gb.score_step(bt, bufs, chunk=cfg.chunk)
    torch.cuda.synchronize()
    sub = inputs.select_requests(bt, [0])
    reqs = [0]
    K, V = oracle.kv_project(sub.U, sub.W_k, sub.W_v, cfg.H, cfg.d, act=cfg.act)
    rows = np.arange(0, 5120, 7)           # a strided sample of the 5120 rows
    T = sub.T[torch.as_tensor(rows)]
    co = torch.tensor([0, len(rows)], dtype=torch.int64)
    O_or, _ = oracle.tasa_score(T, co, sub.W_q, K, V, sub.seq_offsets, cfg.H, cfg.d, act=cfg.act)
    _attn_tol(O[torch.as_tensor(rows, device=dev)].float().cpu().numpy(), O_or, "chunked C=5120")
    assert reqs == [0]


@pytest.mark.parametrize("B,chunks", [(3, 8), (1, 4), (2, 2)])
def test_score_host_more_chunks_than_requests(B, chunks):
    """gesr_score_host with n_chunks >= B (the library clamps the cut to one request per chunk):
    bit-identical to the device-resident step, and the counts match the oracle's definition."""
    dev = _cuda()
    cfg = configs.get("2").with_(B=B)
    bt = inputs.make_batch(cfg)
    g = bt.to(dev)
    bufs = gb.StepBuffers(g, out_dtype=torch.bfloat16)
    O, counts = gb.score_step(g, bufs)
    torch.cuda.synchronize()
    pin = lambda t: t.contiguous().pin_memory()   # noqa: E731
    hb = inputs.Batch(cfg, bt.requests, pin(bt.seq_offsets), pin(bt.cand_offsets), pin(bt.U),
                      pin(bt.T), bt.W_q, bt.W_k, bt.W_v, pin(bt.user_ids), pin(bt.user_offsets),
                      pin(bt.item_ids), pin(bt.item_offsets))
    plan = gb.HostPlan(hb, n_chunks=chunks, out_dtype=torch.bfloat16, device=dev)
    h_O = torch.full(O.shape, float("nan"), dtype=O.dtype).pin_memory()
    h_c = torch.full(counts.shape, -1, dtype=torch.int32).pin_memory()
    plan.run(h_O, h_c)
    torch.cuda.synchronize()
    plan.close()
    assert torch.equal(h_O, O.cpu())
    assert torch.equal(h_c, counts.cpu())
    ref = oracle.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                           bt.cand_offsets, cfg.F)
    assert (h_c.numpy() == ref).all()


@pytest.mark.parametrize("B,kv_splits", [(4, 1), (1, 0)])
def test_back_to_back_steps_keep_stream_order(B, kv_splits):
    """Steps on alternating inputs, enqueued back to back with no host synchronisation, sharing
    ONE K/V cache and work buffer (so a later step's projection overwrites what the previous
    step's attention reads): the hot-path kernels are launched with programmatic dependent
    launch (csrc/kernels.h launch_pdl), so this checks that every kernel still waits for its
    predecessor (read-after-write and write-after-read along the stream, B = 1 with split-L and
    the combine kernel included).  Each step's O and counts must equal its inputs' reference,
    bit for bit."""
    dev = _cuda()
    cfg = configs.get("3h").with_(B=B)
    bts = [inputs.make_batch(cfg, requests=list(range(i * B, (i + 1) * B)), device=dev)
           for i in range(2)]
    K = torch.empty((cfg.H, bts[0].U.shape[0], cfg.d), dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    ws = torch.empty(gb.tasa_workspace_bytes(B, bts[0].total_C, cfg.H, cfg.d, kv_splits),
                     dtype=torch.uint8, device=dev)
    ref = []
    for bt in bts:
        k, v = gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act)
        O, _ = gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, k, v, bt.seq_offsets, cfg.H, cfg.d,
                             cfg.act, kv_splits=kv_splits, out_dtype=torch.bfloat16,
                             want_lse=False)
        c = gb.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                         bt.cand_offsets, cfg.F)
        torch.cuda.synchronize()
        ref.append((O.clone(), c.clone()))
    n = 8
    outs = [torch.empty_like(ref[i % 2][0]) for i in range(n)]
    cnts = [torch.empty_like(ref[i % 2][1]) for i in range(n)]
    torch.cuda.synchronize()
    for i in range(n):
        bt = bts[i % 2]
        gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act, K_cache=K, V_cache=V)
        gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H, cfg.d, cfg.act,
                      kv_splits=kv_splits, O=outs[i], want_lse=False, workspace=ws)
        gb.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets,
                     bt.cand_offsets, cfg.F, counts=cnts[i])
    torch.cuda.synchronize()
    for i in range(n):
        assert torch.equal(outs[i], ref[i % 2][0]), i
        assert torch.equal(cnts[i], ref[i % 2][1]), i


@pytest.mark.parametrize("chunks,out_dtype,cap", [(1, torch.bfloat16, 0),
                                                   (3, torch.bfloat16, 0),
                                                   (2, torch.float32, 3)])
def test_score_host_ids_matches_score_host(chunks, out_dtype, cap):
    """gesr_score_host_ids (host holds table row ids; the device-resident shared table is
    gathered inside the projections) gives exactly gesr_score_host's O and
    counts when E[hist_rows] = U and E[cand_rows] = T (E = a row permutation of [U; T])."""
    dev = _cuda()
    cfg = configs.get("3").with_(B=6, L=("uniform", 0, 300), C=("uniform", 0, 400))
    bt = inputs.make_batch(cfg)
    pin = lambda t: t.contiguous().pin_memory()   # noqa: E731
    hb = inputs.Batch(cfg, bt.requests, pin(bt.seq_offsets), pin(bt.cand_offsets), pin(bt.U),
                      pin(bt.T), bt.W_q, bt.W_k, bt.W_v, pin(bt.user_ids), pin(bt.user_offsets),
                      pin(bt.item_ids), pin(bt.item_offsets))
    nL, nC = bt.U.shape[0], bt.T.shape[0]
    g = torch.Generator().manual_seed(21)
    perm = torch.randperm(nL + nC, generator=g)
    E = torch.cat([bt.U, bt.T])[perm].to(dev)           # row perm[j] of [U; T] at j
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(nL + nC)
    hist_rows = pin(inv[:nL].to(torch.int32))
    cand_rows = pin(inv[nL:].to(torch.int32))
    plan = gb.HostPlan(hb, n_chunks=chunks, out_dtype=out_dtype, cap=cap, device=dev)
    O1 = torch.full((nC, cfg.H * cfg.d), float("nan"), dtype=out_dtype).pin_memory()
    c1 = torch.full((nC, cfg.F), -1, dtype=torch.int32).pin_memory()
    O2, c2 = O1.clone().pin_memory(), c1.clone().pin_memory()
    plan.run(O1, c1)
    plan.run_ids(E, hist_rows, cand_rows, O2, c2)
    torch.cuda.synchronize()
    with pytest.raises(gb.GesrError):          # the table must be device memory
        plan.run_ids(E.cpu(), hist_rows, cand_rows, O2, c2)
    plan.close()
    assert torch.equal(O1, O2) and torch.equal(c1, c2)


def test_kv_cache_shape_is_checked():
    """A K/V cache whose row count differs from the history's would be written with one
    head-major stride and read with another: the binding rejects it."""
    dev = _cuda()
    cfg = configs.get("2").with_(B=2)
    bt = inputs.make_batch(cfg, hma=False, device=dev)
    L = bt.U.shape[0]
    K = torch.empty((cfg.H, L + 1, cfg.d), dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    with pytest.raises(gb.GesrError):
        gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act, K_cache=K, V_cache=V)
