"""Host cost of the reference-record drop-in at configs[4] scale (C5: 256
groups x 16 ragged responses, ~13.6 M trainable rows): flatten_groups over
reference-style records (Python lists, records.py:21-131), the FNV state /
target pass (tg_scored_states, C++), and sample_batch(group_by_task) indexing
(tg_group_by_task, C++) over a buffer of 8,192 experiences -- next to the
GPU step of the same batch (bench.py --variant c5).

    python scripts/bench_host_packing.py [--scale 1.0]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from _golden import Exp, Group  # noqa: E402
from paper_2505_17826_b200.packing import flatten_groups, group_by_task, scored_states  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0, help="fraction of the 256 groups")
    a = ap.parse_args()
    rng = np.random.default_rng(1236)
    G, K = max(1, int(256 * a.scale)), 16
    L = np.clip(np.exp(rng.normal(np.log(3000.0), 0.8, G * K)), 64, 8191).astype(int)
    groups, k = [], 0
    for g in range(G):
        exps = []
        for _ in range(K):
            n = int(L[k]); k += 1
            toks = rng.integers(0, 151936, n + 8).tolist()
            mask = [False] * 8 + [True] * n
            exps.append(Exp(tokens=toks, prompt_length=8, action_mask=mask,
                            logprobs=rng.normal(-1, 0.1, n).tolist(), reward=float(g % 2)))
        groups.append(Group(exps))
    t0 = time.perf_counter()
    h = flatten_groups(groups)
    t1 = time.perf_counter()
    st, tg = scored_states(h, 4096)
    t2 = time.perf_counter()
    n_buf = 2 * G * K
    tasks = rng.integers(0, 2 * G, n_buf)
    ready = rng.uniform(size=n_buf) < 0.9
    t3 = time.perf_counter()
    res = group_by_task(tasks, ready, K, G, "FIFO")
    t4 = time.perf_counter()
    rows = int(h.seq_lengths.sum())
    print(f"C5 x{a.scale}: {G} groups x {K}, {rows} trainable rows, {h.tokens.size} tokens")
    print(f"  flatten_groups (reference records -> arrays): {1e3 * (t1 - t0):9.1f} ms "
          f"({1e9 * (t1 - t0) / h.tokens.size:.1f} ns/token)")
    print(f"  tg_scored_states (FNV states + targets, C++): {1e3 * (t2 - t1):9.1f} ms")
    print(f"  tg_group_by_task over {n_buf} buffered experiences: {1e3 * (t4 - t3):9.3f} ms "
          f"({len(res)} groups)")


if __name__ == "__main__":
    main()
