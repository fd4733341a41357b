"""A/B timing of gesr_kv_project (K-PROJ) on a config: ms per call (CUDA events, 20 calls)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_21095_b200 import binding as gb  # noqa: E402
from paper_2511_21095_b200 import configs, inputs  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "3h")
bt = inputs.make_batch(cfg, hma=False, device=torch.device("cuda"))
K, V = gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act)
for _ in range(3):
    gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act, K_cache=K, V_cache=V)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act, K_cache=K, V_cache=V)
b.record()
torch.cuda.synchronize()
w = torch.arange(K.numel(), device=K.device, dtype=torch.int64) % 1000003
chk = int((K.view(torch.int16).view(-1).long() * w).sum()) ^ int((V.view(torch.int16).view(-1).long() * w).sum())
print(f"{os.environ.get('GESR_LIB', 'default')}: "
      f"{a.elapsed_time(b) / 20:.4f} ms  chk={chk}")
