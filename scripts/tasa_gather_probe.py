import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2511_21095_b200 import binding as gb, configs, inputs
dev = torch.device('cuda', 0)
cfg = configs.get('3h')
bt = inputs.make_batch(cfg, device=dev, hma=False)
n_E = 8_000_000
g = torch.Generator(device=dev).manual_seed(1)
E = torch.randn(n_E, cfg.D_in, generator=g, device=dev).to(torch.bfloat16)
rows = torch.randint(0, n_E, (bt.total_C,), generator=g, device=dev, dtype=torch.int32)
K, V = gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act)
T = E.index_select(0, rows.long())
for _ in range(2):
    gb.tasa_score_gather(E, rows, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H, cfg.d, cfg.act, want_lse=False, out_dtype=torch.bfloat16)
    gb.tasa_score(T, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H, cfg.d, cfg.act, want_lse=False, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
