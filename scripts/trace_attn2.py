"""Debug: timeline of the persistent CTA-pair attention pipeline (-DGESR_TRACE build via GESR_LIB,
GESR_ATTN_PAIR=1).  Rows are global key tiles (unit * 16 + j); softmax events of warpgroup A."""
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
names = ["s_ready", "s_loaded", "s_freed", "exp_done", "token", "p_done", "mma_pv", "mma_s"]
for cta in (0, 1, 10):
    t = buf[cta].astype(np.int64)
    base = t[0, 0]
    print(f"CTA {cta}: clk relative to s_ready[0] (even tiles: warpgroup A, odd: B)")
    print("   g " + " ".join(f"{n:>10s}" for n in names))
    for g in range(40):
        print(f"  {g:2d} " + " ".join(f"{int(t[g, e] - base) if t[g, e] else 0:10d}" for e in range(8)))
    for par in (0, 1):
      ev = t[par:40:2]
      ev = ev[ev[:, 0] > 0]
      print("  warpgroup", "AB"[par])
      for a, b, nm in [(0, 1, "ld"), (1, 2, "sfree"), (2, 4, "tokwait"), (4, 3, "exp"), (3, 5, "fence"), (5, 0, "->next s")]:
        if nm == "->next s":
            d = ev[1:, 0] - ev[:-1, 5]
        else:
            d = ev[:, b] - ev[:, a]
        print(f"    {nm:9s}", d.tolist())
buf3 = np.zeros((64, 16, 8), np.uint64)
assert gb.lib().gesr_debug_trace3_copy(ctypes.c_void_p(buf3.ctypes.data)) == 0
names3 = ["q_full_ok", "o_free_ok", "lastPV_iss", "Qload_iss", "K0_iss", "ml_full", "o_done", "o_free_arr"]
for cta in (0, 1):
    t = buf3[cta].astype(np.int64)
    base = buf[cta, 0, 0].astype(np.int64)
    print(f"CTA {cta} per-unit control events (clk rel. to s_ready[0])")
    print("   u " + " ".join(f"{n:>10s}" for n in names3))
    for u in range(5):
        print(f"  {u:2d} " + " ".join(f"{int(t[u, e] - base) if t[u, e] else 0:10d}" for e in range(8)))
buf4 = np.zeros((64, 16, 16), np.uint64)
assert gb.lib().gesr_debug_trace4_copy(ctypes.c_void_p(buf4.ctypes.data)) == 0
t4 = buf4[0].astype(np.int64)
for u in range(3):
    print(f"unit {u} epilogue chunk loads (clk after o_done):", (t4[u, :4] - buf3[0, u, 6].astype(np.int64)).tolist())
    print(f"unit {u} epilogue chunk stores (clk after o_done):", (t4[u, 8:12] - buf3[0, u, 6].astype(np.int64)).tolist())
