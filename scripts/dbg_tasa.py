import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2511_21095_b200 import binding as gb, configs, inputs
cfg = configs.get("1")
bt = inputs.make_batch(cfg, hma=False).to("cuda")
K, V = gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, 1)
torch.cuda.synchronize(); print("kv ok", flush=True)
print("ws bytes", gb.tasa_workspace_bytes(1, 16, 1, 32, 0), flush=True)
O, lse = gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H, cfg.d, 1)
torch.cuda.synchronize(); print("tasa ok", float(O.abs().sum()), flush=True)
