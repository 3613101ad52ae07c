"""TFLOP/s of the LM-head backward chunk kernel (tg_lmhead_dlogits) alone:
recompute of z = hidden x W_chunk^T (2 T n_cols d FLOPs) plus the bf16 dz
epilogue, CUDA events over repeated launches, next to the forward kernel.

    python scripts/bench_lmhead_dz.py [--rows 16384] [--dim 1536] [--chunk 16384]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2505_17826_b200 import lmhead_dlogits, lmhead_logprob_fwd  # noqa: E402
from scripts.bench_lmhead import timed  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=int, default=16384)
    p.add_argument("--dim", type=int, default=1536)
    p.add_argument("--vocab", type=int, default=151936)
    p.add_argument("--chunk", type=int, default=16384)
    a = p.parse_args()
    T, d, V, nc = a.rows, a.dim, a.vocab, a.chunk
    h = torch.randn(T, d, device="cuda").to(torch.bfloat16)
    w = (torch.randn(V, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
    y = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
    _, _, lse = lmhead_logprob_fwd(h, w, y)
    coef = torch.randn(3, T, device="cuda") * 1e-3
    dz = torch.empty(T, nc, dtype=torch.bfloat16, device="cuda")
    ms = timed(lambda: lmhead_dlogits(h, w, y, lse, coef, 0, nc, out=dz), reps=20)
    ms_f = timed(lambda: lmhead_logprob_fwd(h, w[:nc], y), reps=20)
    fl = 2.0 * T * nc * d
    print(json.dumps({"kernel": "k_lmhead_logprob<dz>", "rows": T, "dim": d, "chunk": nc,
                      "ms": ms, "tflops": fl / ms / 1e9, "fwd_same_cols_ms": ms_f,
                      "fwd_tflops": fl / ms_f / 1e9, "dz_write_gbs": T * nc * 2 / ms / 1e6}))


if __name__ == "__main__":
    main()
