"""A/B timing of gesr_hma_count variants (GESR_LIB selects the library) on config 3h.

    GESR_LIB=build/ab/X.so python scripts/hma_ab.py
Prints ms per call (CUDA events, 20 calls) and a checksum of the counts.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_21095_b200 import binding as gb  # noqa: E402
from paper_2511_21095_b200 import configs, inputs  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "3h")
bt = inputs.make_batch(cfg, attention=False, device=torch.device("cuda"))
args = (bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets, bt.cand_offsets, cfg.F, 0)
c = gb.hma_count(*args)
for _ in range(3):
    gb.hma_count(*args, counts=c)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    gb.hma_count(*args, counts=c)
b.record()
torch.cuda.synchronize()
w = torch.arange(c.numel(), device=c.device, dtype=torch.int64) % 1000003
print(f"{os.environ.get('GESR_LIB', 'default')}: {a.elapsed_time(b) / 20:.4f} ms  "
      f"sum={int(c.sum())} chk={int((c.view(-1).long() * w).sum())}")
