"""A/B timing of the fused LM-head forward alone (tg_lmhead_logprob_fwd) and
cuBLAS's GEMM into materialised logits at one shape (CUDA events, 10 launches
after warm-up); the library / switches come from the environment
(TG_LOSS_LIB, TG_LMHEAD_PAIR, TG_LMHEAD_ORDER in the A/B build).

    python scripts/ab_lmhead_fwd.py [--rows 16384] [--dim 3584] [--vocab 151936]
"""
import argparse
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_17826_b200 import lmhead_logprob_fwd  # noqa: E402
from scripts.bench_lmhead import timed  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=16384)
p.add_argument("--dim", type=int, default=3584)
p.add_argument("--vocab", type=int, default=151936)
p.add_argument("--cublas", action="store_true")
a = p.parse_args()
T, d, V = a.rows, a.dim, a.vocab
h = torch.randn(T, d, device="cuda").to(torch.bfloat16)
w = (torch.randn(V, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
y = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
flops = 2.0 * T * V * d
ms = timed(lambda: lmhead_logprob_fwd(h, w, y))
out = {"rows": T, "dim": d, "ms": ms, "tflops": flops / ms / 1e9,
       "env": {k: v for k, v in os.environ.items() if k.startswith("TG_")}}
if a.cublas:
    ms_c = timed(lambda: torch.matmul(h, w.T))
    out.update(cublas_ms=ms_c, cublas_tflops=flops / ms_c / 1e9)
print(json.dumps(out))
