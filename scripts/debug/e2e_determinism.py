"""Which calls of the e2e harness differ from the device path, and why:
bitwise determinism of RFTLoss on one 16,384-row batch (repeat, in place vs
new, side stream, concurrent copies), then the bench's 3-stream loop."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2505_17826_b200 import RFTLoss, RFTLossConfig  # noqa: E402
from paper_2505_17826_b200.packing import PackedBatch  # noqa: E402
from paper_2505_17826_b200 import _native as N  # noqa: E402

dev = torch.device("cuda:0")
V, K, Lr = 151936, 8, 2048
rows = K * Lr
loss = RFTLoss(RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip", clip_lo=0.2,
                             clip_hi=0.28, kl_fn="low_var_kl", kl_coef=0.001,
                             loss_agg_mode="token-mean"))
rng = np.random.default_rng(99)
gen = torch.Generator(device=dev)
gen.manual_seed(7)
base = torch.empty((rows, V), dtype=torch.bfloat16, device=dev).normal_(0.0, 2.0, generator=gen)
tgt = torch.as_tensor(rng.integers(0, V, rows).astype(np.int32), device=dev)
meta = torch.as_tensor(np.stack([rng.normal(-1.0, 0.05, rows), rng.normal(-1.0, 0.1, rows)]
                                ).astype(np.float32), device=dev)
so = torch.as_tensor(np.arange(0, rows + 1, Lr, dtype=np.int32), device=dev)
go = torch.as_tensor(np.array([0, K], np.int32), device=dev)
rw = torch.as_tensor(rng.integers(0, 2, K).astype(np.float32), device=dev)
NT = rows * 64


def packed(lg):
    return PackedBatch(logits=lg, target=tgt, seq_offsets=so, group_offsets=go, reward=rw,
                       old_lp=meta[0], ref_lp=meta[1], vocab=V, n_rows=rows, n_seqs=K,
                       n_groups=1, n_rl_rows=rows, n_rl_seqs=K, max_rows_per_seq=Lr)


def diff(a, b):
    d = (a != b).nonzero().flatten().tolist()
    return {N.STAT_NAMES[j]: (float(a[j]), float(b[j])) for j in d[:5]}


ref = loss(packed(base), dlogits="new", n_tok_global=NT, n_seq_global=K * 64)
want = ref.stats.cpu()
lp0 = ref.lp.clone()
res = {}
for i in range(4):
    o = loss(packed(base), dlogits="new", n_tok_global=NT, n_seq_global=K * 64)
    res[f"repeat{i}"] = diff(o.stats.cpu(), want)
    if i == 0:
        res["repeat0_lp_rows_differ"] = int((o.lp != lp0).sum())
buf = base.clone()
o = loss(packed(buf), dlogits="inplace", n_tok_global=NT, n_seq_global=K * 64)
res["inplace"] = diff(o.stats.cpu(), want)
res["inplace_lp_rows_differ"] = int((o.lp != lp0).sum())
res["inplace_dz_equal"] = bool(torch.equal(buf, ref.dlogits))
s = torch.cuda.Stream(dev)
with torch.cuda.stream(s):
    buf.copy_(base)
    o = loss(packed(buf), dlogits="inplace", n_tok_global=NT, n_seq_global=K * 64, stream=s)
torch.cuda.synchronize()
res["side_stream_inplace"] = diff(o.stats.cpu(), want)
# concurrent H2D / D2H traffic on other streams while the loss runs
host = torch.empty((rows, V), dtype=torch.bfloat16, pin_memory=True)
host.copy_(base)
scratch = torch.empty_like(base)
s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
outs = []
for i in range(6):
    with torch.cuda.stream(s_in):
        scratch.copy_(host, non_blocking=True)
    with torch.cuda.stream(s_out):
        host.copy_(scratch, non_blocking=True) if i % 2 else None
    with torch.cuda.stream(s):
        buf.copy_(base)
        o = loss(packed(buf), dlogits="inplace", n_tok_global=NT, n_seq_global=K * 64, stream=s)
        o.stats.record_stream(s)
        outs.append(o)
torch.cuda.synchronize()
for i, o in enumerate(outs):
    res[f"concurrent{i}"] = diff(o.stats.cpu(), want)
    res[f"concurrent{i}_lp_rows_differ"] = int((o.lp != lp0).sum())
for k, v in res.items():
    print(k, v)
