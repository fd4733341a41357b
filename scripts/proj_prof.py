"""K-PROJ wait profile (build with -DGESR_PROJ_PROF; GESR_LIB selects the library): per CTA
cycles the producer waits for a free stage, the MMA issuer waits for loaded stages / a free
accumulator, and epilogue warp 4 waits for a full accumulator, for the K/V projection at 3h."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_21095_b200 import binding as gb  # noqa: E402
from paper_2511_21095_b200 import configs, inputs  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "3h")
bt = inputs.make_batch(cfg, hma=False, device=torch.device("cuda"))
L = gb.lib()
fn = L.gesr_debug_projprof_copy
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((296, 8), np.uint64)
K, V = gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act)
for _ in range(3):
    gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act, K_cache=K, V_cache=V)
torch.cuda.synchronize()
fn(buf.ctypes.data, 1)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act, K_cache=K, V_cache=V)
b.record()
torch.cuda.synchronize()
fn(buf.ctypes.data, 1)
lead = buf[0::2].astype(np.float64)
peer = buf[1::2].astype(np.float64)
tot = lead[:, 3]
used = tot > 0
print(f"{os.environ.get('GESR_LIB', 'default')}: {a.elapsed_time(b):.3f} ms")
print(f"  MMA warp total      {tot[used].mean():.0f} cyc")
print(f"  MMA wait full (ld)  {lead[used, 1].mean():.0f} cyc ({lead[used, 1].mean() / tot[used].mean():.1%})")
print(f"  MMA wait tempty     {lead[used, 2].mean():.0f} cyc ({lead[used, 2].mean() / tot[used].mean():.1%})")
print(f"  producer wait empty {lead[used, 0].mean():.0f} / peer {peer[used, 0].mean():.0f} cyc")
print(f"  epi warp4 wait full {lead[used, 4].mean():.0f} / peer {peer[used, 4].mean():.0f} cyc")
