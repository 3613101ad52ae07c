"""Throughput of the fused AdamW step (tg_adamw_step) on an LM-head weight
against the HBM roofline, with torch.optim.AdamW (fused=True and foreach) on
the same tensors as a reference point.

    python scripts/bench_adamw.py [--vocab 151936] [--dim 1536] [--dtype bf16|fp32]

Algorithmic bytes per parameter: param read + write, grad read, exp_avg and
exp_avg_sq read + write = 2 E_p + E_g + 16 (22 B for bf16 param and grad).
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2505_17826_b200 import adamw_step  # noqa: E402
from scripts.bench_lmhead import timed  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--vocab", type=int, default=151936)
p.add_argument("--dim", type=int, default=1536)
p.add_argument("--dtype", default="bf16")
a = p.parse_args()
dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
V, d = a.vocab, a.dim
w = (torch.randn(V, d, device="cuda") * 0.02).to(dt)
g = (torch.randn(V, d, device="cuda") * 1e-3).to(dt)
m = torch.zeros(V, d, device="cuda")
v = torch.zeros(V, d, device="cuda")
hp = dict(lr=1e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
n = V * d
E = w.element_size()
bytes_per = 2 * E + E + 16
ms = timed(lambda: adamw_step(w, g, m, v, 5, check_finite=False, **hp), reps=20)
ms_chk = timed(lambda: adamw_step(w, g, m, v, 5, check_finite=True, **hp), reps=20)
peak = None
try:
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
except Exception:
    pass
out = {"kernel": "k_adamw", "params": n, "dtype": a.dtype, "ms": ms,
       "gbs": n * bytes_per / ms / 1e6, "bytes_per_param": bytes_per, "peak_gbs": peak,
       "frac": (n * bytes_per / ms / 1e6 / peak) if peak else None,
       "ms_with_finite_check": ms_chk}
# torch.optim.AdamW on the same parameter (fp32 moments are torch's own state)
for kind in ("fused", "foreach"):
    try:
        prm = torch.nn.Parameter(w.clone())
        prm.grad = g.clone()
        opt = torch.optim.AdamW([prm], **hp, **{kind: True})
        out[f"torch_{kind}_ms"] = timed(opt.step, reps=20)
    except Exception as e:  # (fused AdamW may not support every dtype)
        out[f"torch_{kind}_ms"] = f"unavailable: {type(e).__name__}"
print(json.dumps(out))
