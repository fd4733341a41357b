"""PDL stress: 300 steps on alternating inputs sharing one K/V cache and workspace, enqueued with
no host synchronisation; every step's O and counts must equal its inputs' reference."""
import sys, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2511_21095_b200 import binding as gb, configs, inputs
dev = torch.device('cuda', 0)
bad = 0
for name, B, splits in (("3h", 2, 1), ("3h", 1, 0), ("2", 16, 0)):
    # equal shapes across the two batches (the K/V cache and workspace are shared)
    cfg = configs.get(name).with_(B=B, L=("fixed", 300 if name == "2" else 2048))
    bts = [inputs.make_batch(cfg, requests=list(range(i * B, (i + 1) * B)), device=dev) for i in range(2)]
    K = torch.empty((cfg.H, bts[0].U.shape[0], cfg.d), dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    ws = torch.empty(gb.tasa_workspace_bytes(B, bts[0].total_C, cfg.H, cfg.d, splits), dtype=torch.uint8, device=dev)
    ref = []
    for bt in bts:
        k, v = gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act)
        O, _ = gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, k, v, bt.seq_offsets, cfg.H, cfg.d, cfg.act, kv_splits=splits, out_dtype=torch.bfloat16, want_lse=False)
        c = gb.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets, bt.cand_offsets, cfg.F)
        torch.cuda.synchronize(); ref.append((O.clone(), c.clone()))
    n = 300
    outs = [torch.empty_like(ref[i % 2][0]) for i in range(n)]
    cnts = [torch.empty_like(ref[i % 2][1]) for i in range(n)]
    for i in range(n):
        bt = bts[i % 2]
        gb.kv_project(bt.U, bt.W_k, bt.W_v, cfg.H, cfg.d, cfg.act, K_cache=K, V_cache=V)
        gb.tasa_score(bt.T, bt.cand_offsets, bt.W_q, K, V, bt.seq_offsets, cfg.H, cfg.d, cfg.act, kv_splits=splits, O=outs[i], want_lse=False, workspace=ws)
        gb.hma_count(bt.user_ids, bt.user_offsets, bt.item_ids, bt.item_offsets, bt.cand_offsets, cfg.F, counts=cnts[i])
    torch.cuda.synchronize()
    nb = sum(0 if (torch.equal(outs[i], ref[i % 2][0]) and torch.equal(cnts[i], ref[i % 2][1])) else 1 for i in range(n))
    print(name, B, splits, "mismatching steps:", nb, "of", n)
    bad += nb
print("PDL stress", "OK" if bad == 0 else "FAILED")

# the host path: 40 back-to-back gesr_score_host / _ids calls (copy streams, two buffer sets,
# chunk pipeline) into distinct pinned outputs, each compared with the device-resident step
cfg = configs.get("3").with_(B=24)
bt = inputs.make_batch(cfg)
pin = lambda t: t.contiguous().pin_memory()   # noqa: E731
hb = inputs.Batch(cfg, bt.requests, pin(bt.seq_offsets), pin(bt.cand_offsets), pin(bt.U),
                  pin(bt.T), bt.W_q, bt.W_k, bt.W_v, pin(bt.user_ids), pin(bt.user_offsets),
                  pin(bt.item_ids), pin(bt.item_offsets))
g = bt.to(dev)
bufs = gb.StepBuffers(g, out_dtype=torch.bfloat16)
O_ref, c_ref = gb.score_step(g, bufs)
torch.cuda.synchronize()
O_ref, c_ref = O_ref.cpu(), c_ref.cpu()
nL, nC = bt.U.shape[0], bt.T.shape[0]
perm = torch.randperm(nL + nC, generator=torch.Generator().manual_seed(1))
E = torch.cat([bt.U, bt.T])[perm].to(dev)
inv = torch.empty_like(perm)
inv[perm] = torch.arange(nL + nC)
hr, cr = pin(inv[:nL].to(torch.int32)), pin(inv[nL:].to(torch.int32))
plan = gb.HostPlan(hb, n_chunks=5, out_dtype=torch.bfloat16, device=dev)
outs = [(torch.empty_like(O_ref).pin_memory(), torch.empty_like(c_ref).pin_memory()) for _ in range(40)]
for i, (o, c) in enumerate(outs):
    if i % 2:
        plan.run_ids(E, hr, cr, o, c)
    else:
        plan.run(o, c)
torch.cuda.synchronize()
hb_bad = sum(0 if (torch.equal(o, O_ref) and torch.equal(c, c_ref)) else 1 for o, c in outs)
plan.close()
print("host path: mismatching calls:", hb_bad, "of", len(outs))
print("host stress", "OK" if hb_bad == 0 else "FAILED")
