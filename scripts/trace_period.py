"""Median exp-token period (cycles per key tile) of a -DGESR_TRACE pair-kernel build, from the
trace that scripts/trace_attn2.py prints:  python scripts/trace_period.py gpurun_out/trace_X.txt"""
import sys

import numpy as np

for path in sys.argv[1:]:
    lines = open(path).read().split("\n")
    res = []
    for start in [i for i, l in enumerate(lines) if l.startswith("CTA ")]:
        rows = []
        for l in lines[start + 2:start + 42]:
            f = l.split()
            if len(f) == 9 and f[0].isdigit():
                rows.append([int(x) for x in f])
        r = np.array(rows)
        tok, ed = r[:, 5], r[:, 4]
        res.append((np.median(np.diff(tok)), np.median(ed - tok), np.median(tok[1:] - ed[:-1])))
    a = np.array(res)
    print(f"{path}: period {np.median(a[:, 0]):.0f}  exp window {np.median(a[:, 1]):.0f}  "
          f"handoff {np.median(a[:, 2]):.0f}  (CTAs {len(res)})")
