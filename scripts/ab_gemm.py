"""A/B timing of the LM-head backward GEMMs alone (tg_lmhead_grad_hidden /
_weight / _chunk over one 16,384-column chunk) with cuBLAS's two GEMMs timed
in the same process as the box reference; the CTA mode comes from the
environment (TG_GEMM_PAIR in the A/B build).

    python scripts/ab_gemm.py [--rows 16384] [--dim 1536] [--chunk 16384]
"""
import argparse
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_17826_b200 import (lmhead_grad_chunk, lmhead_grad_hidden,  # noqa: E402
                                   lmhead_grad_weight)
from scripts.bench_lmhead import timed  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=16384)
p.add_argument("--dim", type=int, default=1536)
p.add_argument("--chunk", type=int, default=16384)
a = p.parse_args()
T, d, nc = a.rows, a.dim, a.chunk
w = (torch.randn(nc, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
h = torch.randn(T, d, device="cuda").to(torch.bfloat16)
dz = (torch.randn(T, nc, device="cuda") * 1e-3).to(torch.bfloat16)
dh = torch.zeros(T, d, dtype=torch.float32, device="cuda")
dw = torch.empty(nc, d, dtype=torch.bfloat16, device="cuda")
gf = 2.0 * T * nc * d / 1e9
r = {"rows": T, "dim": d, "chunk": nc, "gemm_pair": os.environ.get("TG_GEMM_PAIR", "default")}
r["grad_hidden_tflops"] = gf / timed(lambda: lmhead_grad_hidden(dz, w, 0, dh, accumulate=True))
r["grad_weight_tflops"] = gf / timed(lambda: lmhead_grad_weight(dz, h, dw))
r["grad_chunk_tflops"] = 2 * gf / timed(lambda: lmhead_grad_chunk(dz, h, w, 0, dh, dw, accumulate=True))
ms_c = timed(lambda: torch.addmm(dh, dz, w, out_dtype=torch.float32)) + \
    timed(lambda: torch.mm(dz.t(), h, out=dw))
r["cublas_pair_tflops"] = 2 * gf / ms_c
print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items()}))
