"""Summarise interleaved kbench.py A/B output ("== NAME" headers followed by JSON lines)."""
import json
import sys
from collections import defaultdict

v, rows = None, defaultdict(list)
for line in sys.stdin:
    if line.startswith("=="):
        v = line.split()[1]
    elif line.startswith("{"):
        d = json.loads(line)
        rows[v].append((d["kv_ms"], d["tasa_ms"], d["hma_ms"], d["step_ms"]))
        print(v, *(round(x, 3) for x in rows[v][-1]))
    elif "Error" in line:
        print(line.strip())
for k, r in rows.items():
    med = [sorted(c)[len(c) // 2] for c in zip(*r)]
    print("median", k, "kv/tasa/hma/step ms", *(round(x, 3) for x in med))
