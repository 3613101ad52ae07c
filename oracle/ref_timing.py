"""Timing harness for the REFERENCE's own CPU loss path (MEASUREMENT
INFRASTRUCTURE -- only bench.py's reference arm / cpu_baseline call it).

Runs triad's ``group_loss`` over a batch of task groups followed by
``combine_reports`` (algorithms.py:351-379; OPMD_SIMPLE, the reference's GRPO
analogue, algorithms.py:220-253 -- the reference has no PPO / k3, so this is
the nearest reference timing), exactly as
``Trainer.step_groups`` calls it (orchestrator.py:299-304) without
``apply_update``.  triad is imported from ``oracle/_ref`` (installed by
``oracle/stage_ref.sh``); nothing here is a restatement.

Workload per worker and step: one group of K rollouts of ``resp_len``
mask-true response tokens over a bucketed logits table of ``buckets`` rows at
the bench's vocabulary (bf16-rounded N(0, 2^2) + a target bump, so row
distributions match the GPU arm's).  Throughput = mask-true tokens / wall
seconds; workers run in separate processes on disjoint groups, mirroring the
GPU sharding (SURVEY.md 8(d) "all-cores figure").
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

REF_DIR = Path(__file__).resolve().parent / "_ref"


def available() -> bool:
    return (REF_DIR / "triad" / "algorithms.py").exists()


def _triad():
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    from triad import algorithms as A
    from triad import policy as P
    from triad.records import Experience, TaskGroup
    return A, P, Experience, TaskGroup


def _bf16(x: np.ndarray) -> np.ndarray:
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def build(seed: int, vocab: int, group_size: int, resp_len: int, buckets: int = 64,
          bump: float = 13.5):
    """(params, groups, config) of one worker-step sample."""
    A, P, Experience, TaskGroup = _triad()
    rng = np.random.default_rng(seed)
    theta = rng.normal(0.0, 2.0, size=(buckets, vocab))
    theta[np.arange(buckets), rng.integers(0, vocab, buckets)] += bump
    params = P.PolicyParams(_bf16(theta), 0, P.Vocabulary(size=vocab, eos_token=vocab - 1))
    exps = []
    for _ in range(group_size):
        prompt = [int(x) for x in rng.integers(0, vocab, 4)]
        resp = [int(x) for x in rng.integers(0, vocab, resp_len)]
        exps.append(Experience(task_key=1, tokens=prompt + resp, prompt_length=len(prompt),
                               action_mask=[False] * len(prompt) + [True] * resp_len,
                               logprobs=list(rng.normal(-1.0, 0.1, resp_len)),
                               reward=float(rng.integers(0, 2)), model_version=0))
    groups = [TaskGroup(1, exps)]
    cfg = A.AlgorithmConfig(A.Variant.OPMD_SIMPLE, tau=1.0)
    return params, groups, cfg


def run(seed: int, vocab: int, group_size: int, resp_len: int, buckets: int = 64):
    """One timed worker-step: returns (mask-true tokens, seconds, loss)."""
    A, _, _, _ = _triad()
    params, groups, cfg = build(seed, vocab, group_size, resp_len, buckets)
    t0 = time.perf_counter()
    reports = [A.group_loss(g, params, cfg) for g in groups]
    combined = A.combine_reports(reports)
    dt = time.perf_counter() - t0
    return group_size * resp_len * len(groups), dt, float(combined.loss)


def _worker(args):
    os.environ.setdefault("OMP_NUM_THREADS", "1")  # one core per worker process
    return run(*args)


def pool_size(vocab: int, buckets: int, group_size: int, resp_len: int) -> int:
    """Worker processes: every core, bounded by a share of host memory (a
    worker holds the table and the group's per-sequence gradient rows,
    algorithms.py:104-109)."""
    cores = os.cpu_count() or 1
    try:
        avail = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_AVPHYS_PAGES")
    except (ValueError, OSError):
        avail = 64 << 30
    per = 8 * vocab * (buckets + 3 * group_size * min(resp_len, buckets)) + (256 << 20)
    return max(1, min(cores, int(0.5 * avail // per), 128))
