"""fp32 logits at Qwen vocabulary: fused route (CL = 4 clusters) vs the two-pass
route.  python scripts/ab_fp32.py [--rows 32768]"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, pack_arrays  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=32768)
p.add_argument("--vocab", type=int, default=151936)
a = p.parse_args()
V, T = a.vocab, a.rows
x = torch.randn(T, V, device="cuda") * 2.0
tgt = np.random.default_rng(0).integers(0, V, T)
lens, gs = [2048] * (T // 2048), [T // 2048 // 2] * 2
b = pack_arrays(x, tgt, lens, gs, np.random.default_rng(1).integers(0, 2, len(lens)).astype(np.float32))
base = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl",
                     kl_coef=0.001, loss_agg_mode="token-mean")
dz = torch.empty_like(x)
for name, cfg in (("fused", base), ("two_pass", base.with_(force_two_pass=True))):
    loss = RFTLoss(cfg)
    for _ in range(3):
        loss(b, dlogits=dz)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        loss(b, dlogits=dz)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name:9s} route {loss.route(b)}: {ms:.3f} ms  {T / ms / 1e3:.2f} M rows/s  "
          f"{T * 8 * V / ms / 1e9:.0f} GB/s-equivalent of the 8V single-pass bytes")
