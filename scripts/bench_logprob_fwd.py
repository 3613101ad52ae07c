"""Forward-only logprob service (tg_logprob_fwd): read GB/s of
the 2V bytes per row at V = 151,936 over a 40 GB bf16 logits buffer.
    python scripts/bench_logprob_fwd.py [--rows 131072]"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_17826_b200 import logprob_fwd, pack_arrays  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=131072)
p.add_argument("--vocab", type=int, default=151936)
a = p.parse_args()
T, V = a.rows, a.vocab
x = torch.empty((T, V), dtype=torch.bfloat16, device="cuda")
for r in range(0, T, 8192):
    x[r:r + 8192].normal_(0, 2.0)
tgt = np.random.default_rng(0).integers(0, V, T)
b = pack_arrays(x, tgt, [2048] * (T // 2048), [T // 2048], np.zeros(T // 2048, np.float32))
for _ in range(3):
    logprob_fwd(b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
n = 10
for _ in range(n):
    logprob_fwd(b)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(json.dumps({"rows": T, "vocab": V, "ms": ms, "read_gbs": T * (2 * V + 16) / ms / 1e6,
                  "rows_per_s": T / ms * 1e3}))
