"""Pins for the attention oracle (PAPER.md:335-346 s3.4.2).

Each check pins the oracle to something other than itself:
  * kv_project  == torch.nn.functional.linear (+ silu) in fp64 (a library routine);
  * tasa_score  == torch scaled_dot_product_attention in fp64 per request (library routine);
  * tasa_score  == the brute-force full (L+C)^2 masked attention (mask built from the rules);
  * closed forms: q = 0 -> mean of V (uniform scores), L = 1 -> the V row, [1000, 0] scores ->
    V of the larger without overflow, hard-attention limit -> V of the argmax;
  * invariants: history permutation, candidate isolation,
    head split (identical weight slices -> identical halves), lse = logsumexp (scipy);
  * golden mask fixtures.
"""
import math
import os

import numpy as np
import pytest
import torch
from scipy.special import logsumexp

import oracle
from paper_2511_21095_b200 import configs, inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _bf16(x):
    return torch.as_tensor(x, dtype=torch.float32).to(torch.bfloat16)


def _rand_bf16(gen, *shape, scale=1.0):
    return (torch.randn(*shape, generator=gen, dtype=torch.float32) * scale).to(torch.bfloat16)


def _lin64(X, W, act):
    y = torch.nn.functional.linear(X.to(torch.float64), W.to(torch.float64))
    return torch.nn.functional.silu(y) if act == 1 else y


def _small_problem(seed=0, B=4, H=2, d=16, D_in=32, Ls=(5, 0, 1, 9), Cs=(3, 2, 0, 4)):
    g = torch.Generator().manual_seed(seed)
    so = torch.tensor(np.concatenate([[0], np.cumsum(Ls)]), dtype=torch.int64)
    co = torch.tensor(np.concatenate([[0], np.cumsum(Cs)]), dtype=torch.int64)
    U = _rand_bf16(g, int(so[-1]), D_in)
    T = _rand_bf16(g, int(co[-1]), D_in)
    a = math.sqrt(6.0 / (D_in + H * d))
    Wq, Wk, Wv = [_bf16((torch.rand(H * d, D_in, generator=g) * 2 - 1) * a) for _ in range(3)]
    return so, co, U, T, Wq, Wk, Wv


@pytest.mark.parametrize("act", [0, 1])
def test_kv_project_equals_torch_linear(act):
    so, co, U, T, Wq, Wk, Wv = _small_problem(1)
    H, d = 2, 16
    bk = torch.linspace(-0.5, 0.5, H * d, dtype=torch.float64)
    K, V = oracle.kv_project(U, Wk, Wv, H, d, act=act, b_k=bk.numpy())
    Kt = _lin64(U, Wk, 0) + bk
    Kt = torch.nn.functional.silu(Kt) if act else Kt
    Vt = _lin64(U, Wv, act)
    # head split: head h = columns [h*d, (h+1)*d)  ("flattened across heads")
    Kt = Kt.reshape(-1, H, d).permute(1, 0, 2).numpy()
    Vt = Vt.reshape(-1, H, d).permute(1, 0, 2).numpy()
    np.testing.assert_allclose(K, Kt, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(V, Vt, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("act", [0, 1])
def test_kv_project_gather_pins(act):
    """oracle.kv_project_gather (the history rows are the shared embedding
    table's rows of the history IDs): each output row is torch fp64 linear(+SiLU) of the table
    row its ID names, written out row by row with scalar Python loops on a small case (a wrong
    index, e.g. position m instead of rows[m], or a transposed W fails); repeated IDs give
    identical rows; permuting the IDs permutes the rows."""
    g = torch.Generator().manual_seed(7)
    H, d, D_in, n_E = 2, 4, 8, 11
    E = _rand_bf16(g, n_E, D_in)
    Wk = _rand_bf16(g, H * d, D_in, scale=0.3)
    Wv = _rand_bf16(g, H * d, D_in, scale=0.3)
    rows = np.array([3, 10, 0, 3, 7, 7, 1], dtype=np.int32)
    K, V = oracle.kv_project_gather(E, rows, Wk, Wv, H, d, act=act)
    Ef, Wkf, Wvf = E.double().numpy(), Wk.double().numpy(), Wv.double().numpy()
    for m, r in enumerate(rows):
        for h in range(H):
            for j in range(d):
                n = h * d + j
                yk = sum(Ef[r, k] * Wkf[n, k] for k in range(D_in))
                yv = sum(Ef[r, k] * Wvf[n, k] for k in range(D_in))
                if act:
                    yk, yv = yk / (1 + math.exp(-yk)), yv / (1 + math.exp(-yv))
                assert abs(K[h, m, j] - yk) < 1e-12 and abs(V[h, m, j] - yv) < 1e-12
    assert np.array_equal(K[:, 0], K[:, 3]) and np.array_equal(V[:, 4], V[:, 5])
    perm = np.array([6, 2, 0, 5, 1, 4, 3])
    Kp, Vp = oracle.kv_project_gather(E, rows[perm], Wk, Wv, H, d, act=act)
    assert np.array_equal(Kp, K[:, perm]) and np.array_equal(Vp, V[:, perm])


def _oracle_tasa(so, co, U, T, Wq, Wk, Wv, H, d, act, scale=None):
    K, V = oracle.kv_project(U, Wk, Wv, H, d, act=act)
    return oracle.tasa_score(T, co, Wq, K, V, so, H, d, act=act, scale=scale)


@pytest.mark.parametrize("act", [0, 1])
def test_tasa_equals_torch_sdpa(act):
    H, d = 2, 16
    so, co, U, T, Wq, Wk, Wv = _small_problem(2)
    O, lse = _oracle_tasa(so, co, U, T, Wq, Wk, Wv, H, d, act)
    for b in range(len(so) - 1):
        r0, r1, c0, c1 = int(so[b]), int(so[b + 1]), int(co[b]), int(co[b + 1])
        if c1 == c0:
            continue
        if r1 == r0:   # reading R6: empty history -> O = 0, lse = -inf
            assert np.all(O[c0:c1] == 0) and np.all(np.isneginf(lse[c0:c1]))
            continue
        q = _lin64(T[c0:c1], Wq, act).reshape(-1, H, d).transpose(0, 1)
        k = _lin64(U[r0:r1], Wk, act).reshape(-1, H, d).transpose(0, 1)
        v = _lin64(U[r0:r1], Wv, act).reshape(-1, H, d).transpose(0, 1)
        ref = torch.nn.functional.scaled_dot_product_attention(q, k, v)  # scale 1/sqrt(d)
        ref = ref.transpose(0, 1).reshape(c1 - c0, H * d).numpy()
        np.testing.assert_allclose(O[c0:c1], ref, rtol=1e-12, atol=1e-12)
        s = torch.einsum("hcd,hld->hcl", q, k).numpy() / math.sqrt(d)
        np.testing.assert_allclose(lse[c0:c1], logsumexp(s, axis=2).T, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("act", [0, 1])
def test_tasa_equals_bruteforce_full_mask(act):
    H, d = 2, 16
    so, co, U, T, Wq, Wk, Wv = _small_problem(3, Ls=(8, 1, 3, 0), Cs=(4, 2, 3, 2))
    O, lse = _oracle_tasa(so, co, U, T, Wq, Wk, Wv, H, d, act)
    for b in range(len(so) - 1):
        r0, r1, c0, c1 = int(so[b]), int(so[b + 1]), int(co[b]), int(co[b + 1])
        Ob, lb = oracle.full_masked_attention(U[r0:r1], T[c0:c1], Wq, Wk, Wv, H, d, act=act,
                                              self_key=False)
        np.testing.assert_allclose(O[c0:c1], Ob, rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(np.isneginf(lse[c0:c1]), np.isneginf(lb))
        fin = np.isfinite(lb)
        np.testing.assert_allclose(lse[c0:c1][fin], lb[fin], rtol=1e-12, atol=1e-12)


def _golden_mask(name):
    rows, self_key = [], 0
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            if line.startswith("# self_key="):
                self_key = int(line.split("=")[1])
            elif line.strip() and not line.startswith("#"):
                rows.append([int(x) for x in line.split()])
    return np.array(rows, np.uint8), self_key


@pytest.mark.parametrize("name,N,n", [("mask_N3_n2.txt", 3, 2), ("mask_N0_n2.txt", 0, 2)])
def test_mask_golden(name, N, n):
    want, self_key = _golden_mask(name)
    np.testing.assert_array_equal(oracle.build_mask(N, n, self_key=bool(self_key)), want)
    # hot-path reading (R2): identical except the candidate diagonal is off
    off = oracle.build_mask(N, n, self_key=False)
    want_off = want.copy()
    for i in range(N, N + n):
        want_off[i, i] = 0
    np.testing.assert_array_equal(off, want_off)


def test_mask_rule_predicate_random():
    rng = np.random.default_rng(0)
    for _ in range(20):
        N, n = int(rng.integers(0, 12)), int(rng.integers(1, 6))
        for sk in (False, True):
            m = oracle.build_mask(N, n, self_key=sk)
            for i in range(N + n):
                for j in range(N + n):
                    hist_i, hist_j = i < N, j < N
                    allowed = ((hist_i and hist_j and j <= i) or (not hist_i and hist_j) or
                               (not hist_i and not hist_j and sk and i == j))
                    assert m[i, j] == int(allowed)


def test_self_key_variant_equals_history_plus_diagonal():
    """With the diagonal on, each candidate's softmax also includes its own key/value."""
    H, d = 1, 8
    so, co, U, T, Wq, Wk, Wv = _small_problem(4, B=1, H=H, d=d, D_in=16, Ls=(6,), Cs=(3,))
    O, _ = oracle.full_masked_attention(U, T, Wq, Wk, Wv, H, d, act=1, self_key=True)
    for c in range(3):
        q = _lin64(T[c:c + 1], Wq, 1)
        k = torch.cat([_lin64(U, Wk, 1), _lin64(T[c:c + 1], Wk, 1)])
        v = torch.cat([_lin64(U, Wv, 1), _lin64(T[c:c + 1], Wv, 1)])
        w = torch.softmax(q @ k.T / math.sqrt(d), dim=-1)
        np.testing.assert_allclose(O[c], (w @ v)[0].numpy(), rtol=1e-12, atol=1e-12)


def test_uniform_scores_give_mean_pooling():
    # W_q = 0 -> q = act(0) = 0 for identity and SiLU -> all scores equal -> O = mean V
    H, d = 2, 16
    so, co, U, T, Wq, Wk, Wv = _small_problem(5, Ls=(7, 3, 1, 12))
    Wq = torch.zeros_like(Wq)
    for act in (0, 1):
        O, lse = _oracle_tasa(so, co, U, T, Wq, Wk, Wv, H, d, act)
        Vt = _lin64(U, Wv, act).numpy()
        for b in range(len(so) - 1):
            r0, r1, c0, c1 = int(so[b]), int(so[b + 1]), int(co[b]), int(co[b + 1])
            for c in range(c0, c1):
                np.testing.assert_allclose(O[c], Vt[r0:r1].mean(axis=0), rtol=1e-13, atol=1e-14)
                np.testing.assert_allclose(lse[c], math.log(r1 - r0), atol=1e-14)


def test_single_token_history_returns_v():
    # one KV row v -> output v regardless of the query
    H, d = 2, 16
    so, co, U, T, Wq, Wk, Wv = _small_problem(6, B=2, Ls=(1, 1), Cs=(5, 2))
    K, V = oracle.kv_project(U, Wk, Wv, H, d, act=1)
    O, _ = oracle.tasa_score(T, co, Wq, K, V, so, H, d, act=1)
    for b in range(2):
        for c in range(int(co[b]), int(co[b + 1])):
            for h in range(H):
                assert np.array_equal(O[c, h * d:(h + 1) * d], V[h, b])


def _controlled_scores(svals, Vrows, scale=1.0):
    """One request, one head, d = 2: q = e_0 via identity act, K[:,0] = svals -> s = scale*svals."""
    L = len(svals)
    d, H, D_in = 2, 1, 2
    T = _bf16([[1.0, 0.0]])
    Wq = _bf16([[1.0, 0.0], [0.0, 1.0]])
    K = np.zeros((H, L, d))
    K[0, :, 0] = svals
    V = np.zeros((H, L, d))
    V[0] = Vrows
    return oracle.tasa_score(T, [0, 1], Wq, K, V, [0, L], H, d, act=0, scale=scale)


def test_softmax_spec_examples():
    # SPEC.md:70 row [0,0] -> [0.5, 0.5]: O = average of the two V rows
    O, lse = _controlled_scores([0.0, 0.0], [[2.0, -4.0], [6.0, 8.0]])
    np.testing.assert_array_equal(O[0], [4.0, 2.0])
    assert abs(lse[0, 0] - math.log(2.0)) < 1e-15
    # SPEC.md:71 row [1000, 0] -> [~1, ~0] without overflow: O = V row 0 exactly
    O, lse = _controlled_scores([1000.0, 0.0], [[2.0, -4.0], [6.0, 8.0]])
    assert np.all(np.isfinite(O)) and np.array_equal(O[0], [2.0, -4.0])
    assert lse[0, 0] == 1000.0
    # SPEC.md:72 row [1,2,3] -> exp-normalised values (softmax weights read back through V = I)
    O, _ = _controlled_scores([1.0, 2.0, 3.0], [[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]])
    e = np.exp([1.0, 2.0, 3.0])
    np.testing.assert_allclose(O[0], e[:2] / e.sum(), rtol=1e-15)


def test_hard_attention_limit():
    rng = np.random.default_rng(7)
    s = rng.standard_normal(20)
    Vr = rng.standard_normal((20, 2))
    O, _ = _controlled_scores(s, Vr, scale=1e4)
    np.testing.assert_allclose(O[0], Vr[np.argmax(s)], atol=1e-12)


def test_history_permutation_invariance():
    H, d = 2, 16
    so, co, U, T, Wq, Wk, Wv = _small_problem(8, B=1, Ls=(13,), Cs=(4,))
    O, lse = _oracle_tasa(so, co, U, T, Wq, Wk, Wv, H, d, 1)
    perm = torch.randperm(13, generator=torch.Generator().manual_seed(3))
    O2, lse2 = _oracle_tasa(so, co, U[perm], T, Wq, Wk, Wv, H, d, 1)
    np.testing.assert_allclose(O, O2, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(lse, lse2, rtol=1e-13, atol=1e-14)


def test_candidate_isolation_exact():
    # editing candidate 2 leaves the other rows bit-identical
    H, d = 2, 16
    so, co, U, T, Wq, Wk, Wv = _small_problem(9, B=1, Ls=(10,), Cs=(4,))
    O, _ = _oracle_tasa(so, co, U, T, Wq, Wk, Wv, H, d, 1)
    T2 = T.clone()
    T2[2] = -T2[2] + 1
    O2, _ = _oracle_tasa(so, co, U, T2, Wq, Wk, Wv, H, d, 1)
    keep = [0, 1, 3]
    assert np.array_equal(O[keep], O2[keep]) and not np.array_equal(O[2], O2[2])


def test_head_split_identical_slices():
    # reading R5: heads independent; identical weight slices -> identical halves (exact)
    H, d, D_in = 2, 8, 16
    so, co, U, T, Wq, Wk, Wv = _small_problem(10, B=2, H=H, d=d, D_in=D_in, Ls=(5, 3), Cs=(2, 3))
    for W in (Wq, Wk, Wv):
        W[d:] = W[:d]
    O, lse = _oracle_tasa(so, co, U, T, Wq, Wk, Wv, H, d, 1)
    assert np.array_equal(O[:, :d], O[:, d:]) and np.array_equal(lse[:, 0], lse[:, 1])


def test_rounding_aware_mode_is_close():
    # diagnostic mode (reading R8) differs from pure fp64 only by bf16 quantisation of q/K/V
    cfg = configs.get("1")
    bt = inputs.make_batch(cfg, hma=False)
    K, V = oracle.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, act=1)
    O, _ = oracle.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H, cfg.d)
    Kr, Vr = oracle.round_to_bf16(K), oracle.round_to_bf16(V)
    Or, _ = oracle.tasa_score(bt.T, bt.cand_offsets, bt.W_q, Kr, Vr, bt.seq_offsets, cfg.H, cfg.d,
                              round_q_bf16=True)
    assert 0 < np.abs(O - Or).max() < 2e-2


def test_round_to_bf16_matches_torch():
    x = np.random.default_rng(1).standard_normal(1000) * 10
    ref = torch.tensor(x, dtype=torch.float64).to(torch.float32).to(torch.bfloat16)
    np.testing.assert_array_equal(oracle.round_to_bf16(x), ref.to(torch.float64).numpy())


def test_config1_end_to_end_matches_sdpa():
    """The oracle on the generated config-1 workload equals torch fp64 SDPA."""
    cfg = configs.get("1")
    bt = inputs.make_batch(cfg, hma=False)
    K, V = oracle.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, act=cfg.act)
    O, _ = oracle.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H, cfg.d,
                             act=cfg.act)
    q = _lin64(bt.T, bt.W_q, 1).reshape(-1, cfg.H, cfg.d).transpose(0, 1)
    k = _lin64(bt.U, bt.W_k, 1).reshape(-1, cfg.H, cfg.d).transpose(0, 1)
    v = _lin64(bt.U, bt.W_v, 1).reshape(-1, cfg.H, cfg.d).transpose(0, 1)
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v).transpose(0, 1)
    np.testing.assert_allclose(O, ref.reshape(O.shape).numpy(), rtol=1e-12, atol=1e-12)
