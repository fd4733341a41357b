"""Pins for the HMA oracle (PAPER.md:308-312 s3.4.1).

The oracle's brute-force count IS the definition (sum_i sum_j [u_i == t_j]); it is pinned
against things other than itself: the SPEC worked examples (golden file), a second C++
algorithm (multiplicity map), a pure-Python multiset count, and the invariants the paper and
the mathematics fix (symmetry, bound by the shorter duplicate-free list, zero for disjoint IDs,
permutation invariance, monotone under appended matches, the cap).
"""
import os
import random
from collections import Counter

import numpy as np
import pytest

import oracle
from paper_2511_21095_b200 import configs, inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _single(user, item, cap):
    """One request, one candidate, one field."""
    uo = [0, len(user)]
    io = [0, len(item)]
    co = [0, 1]
    return int(oracle.hma_count(np.array(user, np.int64), uo, np.array(item, np.int64), io, co,
                                F=1, cap=cap)[0, 0])


def _read_golden():
    rows = []
    with open(os.path.join(GOLDEN, "hma_spec_examples.txt")) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            u, i, m, e, cite = [p.strip() for p in line.split("|")]
            user = [int(x) for x in u.split(",")] if u else []
            item = [int(x) for x in i.split(",")] if i else []
            rows.append((user, item, int(m), int(e), cite))
    return rows


@pytest.mark.parametrize("row", _read_golden(), ids=lambda r: r[4])
def test_spec_worked_examples(row):
    user, item, cap, expected, _ = row
    assert _single(user, item, cap) == expected
    # the independent algorithm agrees
    got = oracle.hma_count_hash(np.array(user or [0], np.int64)[: len(user)], [0, len(user)],
                                np.array(item, np.int64), [0, len(item)], [0, 1], F=1, cap=cap)
    assert int(got[0, 0]) == expected


def _random_problem(rng, B, F, max_c, max_u, max_i, vocab, dup):
    Cs = [rng.randint(0, max_c) for _ in range(B)]
    co = np.concatenate([[0], np.cumsum(Cs)]).astype(np.int64)
    users, uo = [], [0]
    for b in range(B):
        for f in range(F):
            n = rng.randint(0, max_u)
            seg = [rng.randrange(vocab) for _ in range(n)] if dup else \
                rng.sample(range(vocab), min(n, vocab))
            users += [(f << 40) - 7 + v * 1_000_003 for v in seg]
            uo.append(len(users))
    items, io = [], [0]
    for t in range(int(co[-1])):
        for f in range(F):
            m = rng.randint(0, max_i)
            seg = [rng.randrange(vocab) for _ in range(m)] if dup else \
                rng.sample(range(vocab), min(m, vocab))
            items += [(f << 40) - 7 + v * 1_000_003 for v in seg]
            io.append(len(items))
    return (np.array(users, np.int64), np.array(uo, np.int64), np.array(items, np.int64),
            np.array(io, np.int64), co)


def _python_counts(ui, uo, ii, io, co, F, cap):
    """Pure-Python multiset count: sum over shared values of mult_u(v) * mult_i(v)."""
    B = len(co) - 1
    out = np.zeros((int(co[-1]), F), np.int32)
    for b in range(B):
        for f in range(F):
            cu = Counter(ui[uo[b * F + f]:uo[b * F + f + 1]].tolist())
            for t in range(co[b], co[b + 1]):
                ci = Counter(ii[io[t * F + f]:io[t * F + f + 1]].tolist())
                c = sum(cu[v] * ci[v] for v in ci)
                out[t, f] = min(c, cap) if cap > 0 else c
    return out


@pytest.mark.parametrize("dup", [False, True])
@pytest.mark.parametrize("cap", [0, 3, 16])
def test_three_algorithms_agree(dup, cap):
    rng = random.Random(1234 + cap + 7 * dup)
    args = _random_problem(rng, B=7, F=3, max_c=9, max_u=20, max_i=12, vocab=24, dup=dup)
    a = oracle.hma_count(*args, F=3, cap=cap)
    b = oracle.hma_count_hash(*args, F=3, cap=cap)
    c = _python_counts(*args, F=3, cap=cap)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(a, c)
    if dup:
        assert a.max() > 1   # duplicates exercised


def test_pairwise_reading_with_duplicates():
    # reading R11: pairwise sum, i.e. duplicates on both sides multiply (2 x 3 = 6)
    assert _single([5, 5, 9], [5, 5, 5], cap=0) == 6
    # multiset-intersection (min) would give 2 and set-intersection 1: rejected readings
    assert _single([5, 5, 9], [5, 5, 5], cap=4) == 4


def test_symmetry_bound_disjoint():
    rng = random.Random(99)
    for _ in range(200):
        n, m = rng.randint(0, 30), rng.randint(0, 30)
        u = rng.sample(range(-50, 50), n)
        i = rng.sample(range(-50, 50), m)
        c = _single(u, i, 0)
        assert c == _single(i, u, 0)                     # symmetric
        assert c <= min(n, m)                            # bounded by the shorter dedup'd list
        assert c == len(set(u) & set(i))                 # = set intersection when dup-free
        disjoint = [x + 1000 for x in i]
        assert _single(u, disjoint, 0) == 0              # zero for disjoint IDs


def test_permutation_invariance_and_monotone():
    rng = random.Random(5)
    u = [rng.randrange(40) for _ in range(30)]
    i = [rng.randrange(40) for _ in range(10)]
    base = _single(u, i, 0)
    for _ in range(20):
        u2 = u[:]
        rng.shuffle(u2)
        i2 = i[:]
        rng.shuffle(i2)
        assert _single(u2, i2, 0) == base                # SPEC.md:244 / 241
    # monotone nondecreasing as matching events are appended, until the cap
    prev = _single([], [7], 16)
    seq = []
    for k in range(25):
        seq.append(7)
        c = _single(seq, [7], 16)
        assert c >= prev and c == min(k + 1, 16)
        prev = c


def test_int64_full_range_ids():
    big = [-(1 << 63), (1 << 63) - 1, 0, -1]
    assert _single(big, [-(1 << 63)], 0) == 1
    assert _single(big, [(1 << 63) - 1, -1], 0) == 2
    assert _single(big, [1, -2], 0) == 0


def test_empty_and_degenerate():
    # empty lists count 0; F = 0 / C = 0 are no-ops
    assert _single([], [], 0) == 0
    assert oracle.hma_count([], [0], [], [], [0, 0], F=1).shape == (0, 1)


def test_generator_lists_are_duplicate_free_and_counts_spread():
    cfg = configs.get("2").with_(B=6)
    bt = inputs.make_batch(cfg, attention=False)
    F = cfg.F
    ui, uo = bt.user_ids.numpy(), bt.user_offsets.numpy()
    ii, io = bt.item_ids.numpy(), bt.item_offsets.numpy()
    for s in range(len(uo) - 1):
        seg = ui[uo[s]:uo[s + 1]]
        assert len(set(seg.tolist())) == len(seg)
    for s in range(len(io) - 1):
        seg = ii[io[s]:io[s + 1]]
        assert len(set(seg.tolist())) == len(seg)
    c = oracle.hma_count(ui, uo, ii, io, bt.cand_offsets, F)
    c2 = _python_counts(ui, uo, ii, io, bt.cand_offsets.numpy(), F, 0)
    np.testing.assert_array_equal(c, c2)
    assert c.max() >= 4 and (c == 0).any()


# ---------------------------------------------------------------- offset embedding (f2)

def _offset_examples():
    path = os.path.join(os.path.dirname(__file__), "golden", "hma_offset_examples.txt")
    rows = []
    for ln in open(path):
        if ln.startswith("#") or not ln.strip():
            continue
        c, o, M, want, _ = [x.strip() for x in ln.split("|")]
        rows.append((int(c), int(o), int(M), int(want)))
    return rows


def test_offset_index_spec_examples():
    for c, o, M, want in _offset_examples():
        assert oracle.offset_index(c, o, M) == want


def test_offset_index_exhaustive_collision_free():
    # SPEC.md:232 "exhaustive (c,o) grid for P=3, M=4 -> all indices distinct and in range"
    P, M = 3, 4
    idx = [oracle.offset_index(c, o, M) for o in range(P) for c in range(M + 1)]
    assert sorted(idx) == list(range(P * (M + 1)))
    with pytest.raises(ValueError):
        oracle.offset_index(M + 1, 0, M)


def test_offset_embed_against_one_hot_matmul():
    # the gather equals the one-hot row selection onehot(c + o (M+1)) @ E, built here from the
    # counts without offset_index; pair order is the concatenation order
    rng = np.random.default_rng(7)
    F, M, D_h, C = 3, 5, 8, 11
    counts = rng.integers(0, M + 1, size=(C, F))
    E = rng.standard_normal((F * (M + 1), D_h))
    got = oracle.hma_offset_embed(counts, E, M)
    for t in range(C):
        for o in range(F):
            onehot = np.zeros(F * (M + 1))
            onehot[o * (M + 1) + counts[t, o]] = 1.0
            assert np.array_equal(got[t, o * D_h:(o + 1) * D_h], onehot @ E)

