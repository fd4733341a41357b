"""Debug: timeline of the persistent 1-CTA attention pipeline (-DGESR_TRACE build via GESR_LIB).
Rows are global key tiles of a CTA (16 per unit at L=2048)."""
import ctypes, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_21095_b200 import binding as gb, configs, inputs  # noqa: E402

cfg = configs.get("3h").with_(B=160)
bt = inputs.make_batch(cfg, device="cuda", hma=False)
bufs = gb.StepBuffers(bt, out_dtype=torch.bfloat16)
gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, 1, K_cache=bufs.K, V_cache=bufs.V)
for _ in range(3):
    gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, bufs.K, bufs.V, bt.seq_offsets, cfg.H, cfg.d, 1,
                  O=bufs.O, want_lse=False, workspace=bufs.workspace)
torch.cuda.synchronize()
buf = np.zeros((64, 64, 8), np.uint64)
assert gb.lib().gesr_debug_trace_copy(ctypes.c_void_p(buf.ctypes.data)) == 0
names = ["s0_ready", "s0_max", "p0_done", "s1_ready", "p1_done", "mma_p0", "mma_p1", "epi0_done"]
for cta in (0, 5):
    t = buf[cta].astype(np.int64)
    base = t[0, 0]
    print(f"CTA {cta}: clk relative to s0_ready[0]")
    print("   g " + " ".join(f"{n:>10s}" for n in names))
    for g in range(48):
        print(f"  {g:2d} " + " ".join(f"{int(t[g, e] - base) if t[g, e] else 0:10d}" for e in range(8)))
    s0 = t[:48, 0]
    print("  period (s0_ready diffs):", np.diff(s0[s0 > 0]).tolist())
    print("  softmax0 (s0_ready->p0_done):", (t[:48, 2] - t[:48, 0]).tolist())
    print("  softmax1 (s1_ready->p1_done):", (t[:48, 4] - t[:48, 3]).tolist())
    print("  exp pass0 (s0_ready->s0_max):", (t[:48, 1] - t[:48, 0]).tolist())
