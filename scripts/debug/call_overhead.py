"""Host (CPU) cost of one RFTLoss call at the c1 shape, without syncs."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, pack_arrays
V, G, K, Lr = 32000, 8, 8, 512
T = G * K * Lr
dev = torch.device("cuda", 0)
logits = torch.randn((T, V), device=dev).to(torch.bfloat16)
rng = np.random.default_rng(0)
b = pack_arrays(logits, rng.integers(0, V, T), [Lr] * (G * K), [K] * G, rng.integers(0, 2, G * K),
                old_lp=rng.normal(-1, .1, T), ref_lp=rng.normal(-1, .1, T))
loss = RFTLoss(RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl",
                             kl_coef=0.001, loss_agg_mode="token-mean", clip_lo=0.2, clip_hi=0.28))
dz = torch.empty_like(logits)
out = None
for _ in range(20):
    out = loss(b, dlogits=dz, n_tok_global=T, out=out)
torch.cuda.synchronize()
import cProfile, pstats
t0 = time.perf_counter()
for _ in range(200):
    out = loss(b, dlogits=dz, n_tok_global=T, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue per call {1e6*(t1-t0)/200:.1f} us; wall per call {1e6*(t2-t0)/200:.1f} us")
pr = cProfile.Profile(); pr.enable()
for _ in range(200):
    out = loss(b, dlogits=dz, n_tok_global=T, out=out)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
