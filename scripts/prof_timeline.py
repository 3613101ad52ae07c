"""Kernel timeline of the bench step (torch.profiler / CUPTI): per-kernel
durations and the idle gaps between them, to see where a short step's time
goes beyond the fused kernel (profiles/r02_c1_timeline.txt).

    python scripts/prof_timeline.py [--variant c1] [--steps 5]
"""
import argparse
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, pack_arrays  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--vocab", type=int, default=32000)
    ap.add_argument("--groups", type=int, default=8)
    ap.add_argument("--group-size", type=int, default=8)
    ap.add_argument("--resp-len", type=int, default=512)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--graph", action="store_true")
    a = ap.parse_args()
    V, G, K, Lr = a.vocab, a.groups, a.group_size, a.resp_len
    T = G * K * Lr
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    logits = torch.randn((T, V), device=dev, generator=g).mul_(2.0).to(torch.bfloat16)
    rng = np.random.default_rng(0)
    tgt = rng.integers(0, V, T)
    cfg = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl",
                        kl_coef=0.001, loss_agg_mode="token-mean", clip_lo=0.2, clip_hi=0.28)
    b = pack_arrays(logits, tgt, [Lr] * (G * K), [K] * G, rng.integers(0, 2, G * K),
                    old_lp=rng.normal(-1, 0.1, T), ref_lp=rng.normal(-1, 0.1, T))
    loss = RFTLoss(cfg, graphs=a.graph) if a.graph else RFTLoss(cfg)
    dz = torch.empty_like(logits)
    out = None
    for _ in range(5):
        out = loss(b, dlogits=dz, n_tok_global=T, out=out)
    torch.cuda.synchronize()
    acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
    with torch.profiler.profile(activities=acts) as prof:
        for _ in range(a.steps):
            out = loss(b, dlogits=dz, n_tok_global=T, out=out)
            st = out.stats.sum()  # the bench's per-step stack / sum
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    dur = defaultdict(list)
    gaps = []
    for i, e in enumerate(ev):
        dur[e.name[:60]].append(e.time_range.elapsed_us())
        if i:
            gaps.append(e.time_range.start - ev[i - 1].time_range.end)
    span = ev[-1].time_range.end - ev[0].time_range.start
    print(f"V={V} T={T}: {len(ev)} device events over {span:.1f} us "
          f"({span / a.steps:.1f} us per step)")
    for n, d in sorted(dur.items(), key=lambda x: -sum(x[1])):
        print(f"  {sum(d) / a.steps:9.1f} us/step  x{len(d) // a.steps:<3d} {n}")
    gaps = np.array(gaps)
    print(f"  idle between device events: {gaps.sum() / a.steps:.1f} us/step "
          f"(median gap {np.median(gaps):.1f} us, max {gaps.max():.1f} us)")


if __name__ == "__main__":
    main()
