"""Debug: timeline of the CTA-pair attention pipeline (needs a -DGESR_TRACE build via GESR_LIB)."""
import ctypes, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_21095_b200 import binding as gb, configs, inputs  # noqa: E402

cfg = configs.get("3h").with_(B=64)
bt = inputs.make_batch(cfg, device="cuda", hma=False)
bufs = gb.StepBuffers(bt)
gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, 1, K_cache=bufs.K, V_cache=bufs.V)
for _ in range(3):
    gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, bufs.K, bufs.V, bt.seq_offsets, cfg.H, cfg.d, 1,
                  O=bufs.O, want_lse=False, workspace=bufs.workspace)
torch.cuda.synchronize()
buf = np.zeros((64, 32, 8), np.uint64)
assert gb.lib().gesr_debug_trace2_copy(ctypes.c_void_p(buf.ctypes.data)) == 0
names = ["s_ready", "exp_start", "p_done", "mma_step", "mma_sfree", "mma_pfull", "sm_exp_end", "exp_done"]
for cta in (0, 1, 20, 21):
    t = buf[cta].astype(np.int64)
    base = t[0, 0] if t[0, 0] else t[0, 3]
    print(f"CTA {cta} (rank {cta % 2}): clk relative to s_ready[0]")
    print("   j " + " ".join(f"{n:>10s}" for n in names))
    for j in range(16):
        print(f"  {j:2d} " + " ".join(f"{int(t[j, e] - base) if t[j, e] else 0:10d}" for e in range(8)))
    print("  softmax period (s_ready diffs):", np.diff(t[:16, 0]).tolist())
    print("  exp pass (exp_done - exp_start):", (t[1:16, 7] - t[1:16, 1]).tolist())
