"""Request-subset rule of SURVEY.md s8(c) for the full-size attention parity checks."""
import numpy as np


def survey_subset(Ls: np.ndarray, Cs: np.ndarray, seed: int = 2511, n_random: int = 32):
    """8 longest-L, 8 shortest-L, 8 largest-C, 8 smallest-C, 32 random
    (distinct; topped up to >= 64 with further random requests).  Ties broken by index."""
    B = len(Ls)
    idx = np.arange(B)
    pick = []
    for key in (-Ls, Ls, -Cs, Cs):
        pick += list(np.lexsort((idx, key))[:8])
    rng = np.random.default_rng(seed)
    pick = list(dict.fromkeys(int(x) for x in pick))
    target = min(B, len(pick) + n_random)
    target = max(target, min(B, 64))
    for r in rng.permutation(B):
        if len(pick) >= target:
            break
        if int(r) not in pick:
            pick.append(int(r))
    return sorted(pick)
