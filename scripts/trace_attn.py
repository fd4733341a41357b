"""Debug: timeline of the attention pipeline (needs a -DGESR_TRACE build, GESR_LIB=...)."""
import ctypes, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_21095_b200 import binding as gb, configs, inputs  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "3h").with_(B=64)
bt = inputs.make_batch(cfg, device="cuda", hma=False)
bufs = gb.StepBuffers(bt)
gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, 1, K_cache=bufs.K, V_cache=bufs.V)
for _ in range(3):
    gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, bufs.K, bufs.V, bt.seq_offsets, cfg.H, cfg.d, 1,
                  O=bufs.O, want_lse=False, workspace=bufs.workspace)
torch.cuda.synchronize()
buf = np.zeros((64, 32, 8), np.uint64)
rc = gb.lib().gesr_debug_trace_copy(ctypes.c_void_p(buf.ctypes.data))
assert rc == 0, rc
names = ["s0_ready", "s0_max", "p0_done", "s1_ready", "p1_done", "mma_p0", "mma_p1", "mma_step"]
for cta in (0, 1, 17, 40):
    t = buf[cta].astype(np.int64)
    base = t[0, 7]
    print(f"CTA {cta}: columns relative to mma_step[0] (clk)")
    print("   j " + " ".join(f"{n:>9s}" for n in names))
    for j in range(16):
        print(f"  {j:2d} " + " ".join(f"{int(t[j, e] - base):9d}" for e in range(8)))
    d = np.diff(t[:16, 7])
    print("  step period (mma_step diffs):", d.tolist())
    print("  softmax0 (s0_ready->p0_done):", (t[:16, 2] - t[:16, 0]).tolist())
    print("  softmax1 (s1_ready->p1_done):", (t[:16, 4] - t[:16, 3]).tolist())
