"""Pins for oracle.stu_stack_forward (SPEC.md:298 self_attention_forward, SPEC.md:343 layer
internals, SPEC.md:277 mask; reading R18):
  * one layer equals the composition of the separately pinned oracle functions (torch
    layer_norm, history_attention for the U rows, the C++ full_masked_attention with the
    candidate diagonal for the T rows, stu_output) -- two independent implementations;
  * zero layers is the identity; zero output projections leave the input unchanged (residual);
  * candidate isolation: editing candidate 2 leaves candidate 1's row bit-identical;
  * causality: editing history row N-1 leaves history rows 0..N-2 bit-identical.
"""
import numpy as np
import torch

import oracle


def _case(Ls=(5, 3, 0), Cs=(2, 3, 2), H=2, d=4, seed=0, n_layers=2):
    rng = np.random.default_rng(seed)
    D = H * d
    so = np.concatenate([[0], np.cumsum(Ls)]).astype(np.int64)
    co = np.concatenate([[0], np.cumsum(Cs)]).astype(np.int64)
    U = rng.standard_normal((so[-1], D))
    T = rng.standard_normal((co[-1], D))
    layers = []
    for _ in range(n_layers):
        w = lambda: rng.standard_normal((D, D)) * 0.4   # noqa: E731
        layers.append(dict(W_q=w(), W_k=w(), W_v=w(), W_g=w(), W_o=w(),
                           ln_in=(rng.uniform(0.5, 1.5, D), rng.standard_normal(D) * 0.1),
                           ln_out=(rng.uniform(0.5, 1.5, D), rng.standard_normal(D) * 0.1)))
    return U, T, so, co, layers, H, d


def test_one_layer_equals_composition_of_pinned_oracles():
    # bf16-exact inputs so the C++ oracle (bf16 bit inputs) sees identical values
    U, T, so, co, layers, H, d = _case(n_layers=1, seed=1)
    bf = lambda x: torch.tensor(x).to(torch.bfloat16)   # noqa: E731
    U, T = bf(U).double().numpy(), bf(T).double().numpy()
    lay = layers[0]
    for k in ("W_q", "W_k", "W_v", "W_g", "W_o"):
        lay[k] = bf(lay[k]).double().numpy()
    Uo, To = oracle.stu_stack_forward(U, T, so, co, layers, H, d)
    D = H * d
    ln = lambda X, g, b: torch.nn.functional.layer_norm(   # noqa: E731
        torch.tensor(X), (D,), torch.tensor(g), torch.tensor(b), eps=1e-5).numpy()
    for b in range(len(so) - 1):
        Ub, Tb = U[so[b]:so[b + 1]], T[co[b]:co[b + 1]]
        Un, Tn = ln(Ub, *lay["ln_in"]), ln(Tb, *lay["ln_in"])
        N = Ub.shape[0]
        if N:
            A_U, _ = oracle.history_attention(Un, np.array([0, N]), lay["W_q"], lay["W_k"],
                                              lay["W_v"], H, d, act=1)
            want_U = oracle.stu_output(Un, A_U, lay["W_g"], *lay["ln_out"], lay["W_o"], X_res=Ub)
            np.testing.assert_allclose(Uo[so[b]:so[b + 1]], want_U, rtol=0, atol=1e-10)
        # the candidate rows' masked attention: the stack's numpy attention on bf16-rounded
        # normalised rows agrees with the C++ brute force (which takes bf16 inputs) ...
        Unr, Tnr = bf(Un).double().numpy(), bf(Tn).double().numpy()
        A_T, _ = oracle.full_masked_attention(bf(Unr), bf(Tnr), bf(lay["W_q"]), bf(lay["W_k"]),
                                              bf(lay["W_v"]), H, d, act=1, self_key=True)
        # same T rows from the numpy stack attention on the rounded normalised rows
        X = np.concatenate([Unr, Tnr])
        allowed = oracle.build_mask(N, Tb.shape[0], self_key=True).astype(bool)
        silu = lambda z: z / (1 + np.exp(-z))   # noqa: E731
        Q, K, V = (silu(X @ lay[k].T) for k in ("W_q", "W_k", "W_v"))
        A = np.zeros_like(X)
        for h in range(H):
            cs = slice(h * d, (h + 1) * d)
            S = np.where(allowed, Q[:, cs] @ K[:, cs].T / np.sqrt(d), -np.inf)
            w = np.exp(S - S.max(1, keepdims=True))
            A[:, cs] = w @ V[:, cs] / w.sum(1, keepdims=True)
        np.testing.assert_allclose(A[N:], A_T, rtol=0, atol=1e-12)
        # ... and on the exact rows the stack's T output is stu_output of a scalar-loop attention
        want_T = oracle.stu_output(Tn, _stack_T_attention(Un, Tn, lay, H, d, N), lay["W_g"],
                                   *lay["ln_out"], lay["W_o"], X_res=Tb)
        np.testing.assert_allclose(To[co[b]:co[b + 1]], want_T, rtol=0, atol=1e-10)


def _stack_T_attention(Un, Tn, lay, H, d, N):
    """Candidate rows of the masked attention on unrounded normalised rows, via the numpy
    history_attention oracle's building blocks: each candidate attends to the N history rows
    and itself (the candidate diagonal)."""
    X = np.concatenate([Un, Tn])
    silu = lambda z: z / (1 + np.exp(-z))   # noqa: E731
    Q, K, V = (silu(X @ lay[k].T) for k in ("W_q", "W_k", "W_v"))
    out = np.zeros((Tn.shape[0], H * d))
    for t in range(Tn.shape[0]):
        keys = list(range(N)) + [N + t]
        for h in range(H):
            cs = slice(h * d, (h + 1) * d)
            s = np.array([Q[N + t, cs] @ K[k, cs] for k in keys]) / np.sqrt(d)
            w = np.exp(s - s.max())
            out[t, cs] = sum(w[i] * V[k, cs] for i, k in enumerate(keys)) / w.sum()
    return out


def test_zero_layers_and_zero_projection_are_identity():
    U, T, so, co, layers, H, d = _case(seed=2)
    Uo, To = oracle.stu_stack_forward(U, T, so, co, [], H, d)
    assert np.array_equal(Uo, U) and np.array_equal(To, T)
    for lay in layers:
        lay["W_o"] = np.zeros_like(lay["W_o"])
    Uo, To = oracle.stu_stack_forward(U, T, so, co, layers, H, d)
    assert np.array_equal(Uo, U) and np.array_equal(To, T)


def test_candidate_isolation_and_causality():
    U, T, so, co, layers, H, d = _case(seed=3)
    Uo, To = oracle.stu_stack_forward(U, T, so, co, layers, H, d)
    T2 = T.copy()
    T2[co[1] + 1] += 1.0                      # request 1, candidate 2
    Uo2, To2 = oracle.stu_stack_forward(U, T2, so, co, layers, H, d)
    assert np.array_equal(To2[co[1]], To[co[1]])
    assert np.array_equal(Uo2, Uo)
    assert not np.array_equal(To2[co[1] + 1], To[co[1] + 1])
    U2 = U.copy()
    U2[so[1] - 1] += 1.0                      # request 0, last history row
    Uo3, _ = oracle.stu_stack_forward(U2, T, so, co, layers, H, d)
    assert np.array_equal(Uo3[:so[1] - 1], Uo[:so[1] - 1])
    assert not np.array_equal(Uo3[so[1] - 1], Uo[so[1] - 1])
