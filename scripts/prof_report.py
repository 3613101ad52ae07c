"""Summarise the per-CTA cycle accounting of the instrumented fused kernel
(libtg_loss_prof.so, bench.py with TG_FUSED_PROF_OUT=file.npy)."""
import sys

import numpy as np

NCW = int(sys.argv[1]) if sys.argv[1].isdigit() else 14  # consumer warps
if sys.argv[1].isdigit():
    sys.argv.pop(1)
for f in sys.argv[1:]:
    a = np.load(f).astype(np.float64)
    a = a[a[:, 2] > 0]
    span = a[:, 2]
    print(f"{f}: {len(a)} CTAs, rows/CTA {a[:, 6].mean():.1f}, span {span.mean() / 1e6:.2f} Mcyc")
    names = ["consumer data wait", "consumer bcast wait", None, "producer slot wait",
             "epilogue partial wait", "epilogue cluster wait"]
    for i, n in enumerate(names):
        if n is None:
            continue
        per = a[:, i] / (NCW if i < 2 else 1)
        print(f"  {n:24s} {100 * (per / span).mean():6.2f} % of span "
              f"(min {100 * (per / span).min():.1f}, max {100 * (per / span).max():.1f})")
    rows = a[:, 6]
    print(f"  per row: span {(span / rows).mean():.0f} cyc, epilogue critical path "
          f"{(a[:, 7] / rows).mean():.0f} cyc; first local partial -> epilogue wake "
          f"{(a[:, 9] / rows).mean():.0f} cyc, intra-CTA post skew {(a[:, 10] / rows).mean():.0f} cyc")
    print(f"  checked-path phase-1 chunks per row per warp: {(a[:, 15] / rows / NCW).mean():.3f}")
    if a[:, 11:15].sum() > 0:  # anchor mode 3 (split stash)
        w = [100 * (a[:, 11 + q] / (NCW if q < 2 else 1) / span).mean() for q in range(4)]
        print(f"  mode 3: consumer data wait on TMEM positions {w[0]:.2f} %, on shared positions "
              f"{w[1]:.2f} %; copier waits: free TMEM position {w[2]:.2f} %, landed data {w[3]:.2f} %")
