"""Debug: run the pair attention kernel once on a jagged config and check it against the
1-CTA kernel (GESR_ATTN_PAIR is read once per process: run twice)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_21095_b200 import binding as gb, configs, inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cfg = configs.get(name).with_(B=B)
bt = inputs.make_batch(cfg, device="cuda", hma=False)
bufs = gb.StepBuffers(bt, out_dtype=torch.bfloat16)
gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, 1, K_cache=bufs.K, V_cache=bufs.V)
gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, bufs.K, bufs.V, bt.seq_offsets, cfg.H, cfg.d, 1,
              O=bufs.O, want_lse=False, workspace=bufs.workspace)
torch.cuda.synchronize()
out = os.environ.get("REPRO_OUT")
if out:
    torch.save(bufs.O.cpu(), out)
print("ok", name, B, float(bufs.O.float().abs().sum()))
