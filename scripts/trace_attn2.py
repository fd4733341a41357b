"""Debug: timeline of the persistent CTA-pair attention pipeline (-DGESR_TRACE build via GESR_LIB,
GESR_ATTN_PAIR=1).  Rows are global key tiles (unit * 16 + j) of a CTA."""
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
assert gb.lib().gesr_debug_trace2_copy(ctypes.c_void_p(buf.ctypes.data)) == 0
names = ["sA_ready", "sB_ready", "pA_done", "pB_done", "mma_pA", "mma_pB", "epiA_end", "epiB_end"]
for cta in (0, 1, 10):
    t = buf[cta].astype(np.int64)
    base = t[0, 0] if t[0, 0] else t[0, 4]
    print(f"CTA {cta}: clk relative to sA_ready[0]")
    print("   g " + " ".join(f"{n:>10s}" for n in names))
    for g in range(48):
        print(f"  {g:2d} " + " ".join(f"{int(t[g, e] - base) if t[g, e] else 0:10d}" for e in range(8)))
    sa = t[:48, 0][::2]
    print("  A period per 2 tiles:", np.diff(sa[sa > 0]).tolist())
    print("  softmax A (s->p):", (t[:48:2, 2] - t[:48:2, 0]).tolist())
    print("  softmax B (s->p):", (t[1:48:2, 3] - t[1:48:2, 1]).tolist())
    print("  A pdone->mma:", (t[:48:2, 4] - t[:48:2, 2]).tolist())
