"""Repeat one fused-loss call many times -- alone and beside heavy H2D / D2H
copy traffic on other streams -- and compare every run's statistics and
per-row dlogits checksums bit for bit with the first run."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2505_17826_b200 import RFTLoss, RFTLossConfig
from paper_2505_17826_b200 import _native as N
from paper_2505_17826_b200.packing import PackedBatch

V, K, Lr = 151936, 8, int(sys.argv[1]) if len(sys.argv) > 1 else 2048
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 60
rows = K * Lr
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
x = torch.empty((rows, V), dtype=torch.bfloat16, device=dev).normal_(0, 2.0, generator=g)
rng = np.random.default_rng(99)
tgt = torch.as_tensor(rng.integers(0, V, rows).astype(np.int32), device=dev)
meta = torch.as_tensor(np.stack([rng.normal(-1.0, 0.05, rows), rng.normal(-1.0, 0.1, rows)]).astype(np.float32), device=dev)
so = torch.as_tensor(np.arange(0, rows + 1, Lr, dtype=np.int32), device=dev)
go = torch.as_tensor(np.array([0, K], np.int32), device=dev)
rw = torch.as_tensor(rng.integers(0, 2, K).astype(np.float32), device=dev)
pb = PackedBatch(logits=x, target=tgt, seq_offsets=so, group_offsets=go, reward=rw, old_lp=meta[0],
                 ref_lp=meta[1], vocab=V, n_rows=rows, n_seqs=K, n_groups=1)
cfg = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl",
                    kl_coef=0.001, loss_agg_mode="token-mean", clip_lo=0.2, clip_hi=0.28)
loss = RFTLoss(cfg)
dz = torch.empty_like(x)
host = torch.empty((rows, V), dtype=torch.bfloat16, pin_memory=True)
junk = torch.empty_like(x)
s_cmp, s_cp = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def run(traffic):
    with torch.cuda.stream(s_cmp):
        out = loss(pb, dlogits=dz, n_tok_global=1048576, n_seq_global=512, stream=s_cmp)
    if traffic:
        with torch.cuda.stream(s_cp):
            junk.copy_(host, non_blocking=True)
            host.copy_(junk, non_blocking=True)
    torch.cuda.synchronize()
    ck = dz.view(torch.int32).sum(dim=1, dtype=torch.int64)
    return out.stats.clone(), ck, out.lp.clone()


st0, ck0, lp0 = run(False)
bad = 0
for it in range(iters):
    st, ck, lp = run(traffic=(it % 2 == 1))
    if not torch.equal(st, st0) or not torch.equal(ck, ck0) or not torch.equal(lp, lp0):
        bad += 1
        d = (st != st0).nonzero().flatten().tolist()
        rws = (ck != ck0).nonzero().flatten().tolist()
        lrs = (lp != lp0).nonzero().flatten().tolist()
        print(f"iter {it}: stats {[N.STAT_NAMES[j] for j in d][:6]} rows {rws[:8]} (n={len(rws)}) lp rows {lrs[:8]} (n={len(lrs)})")
        if lrs:
            r = lrs[0]
            print("   lp", float(lp0[r]), float(lp[r]))
print(f"rows={rows} iters={iters} mismatching runs: {bad}")
