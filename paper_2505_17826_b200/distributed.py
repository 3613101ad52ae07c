"""Data parallelism for the loss path: shard by rollout group, allreduce stats.

Every reference loss is intra-group -- advantages, the Kimi baseline and the
pairwise sums read only group members (algorithms.py:118-253) -- and a
batch's report is a plain sum of group losses plus a mean of group metrics
(combine_reports, algorithms.py:368-379).  Gradients w.r.t. logits are
per-row.  So the batch shards by whole groups with no data-path collective;
the only exchange is one allreduce(sum) of the 32-double statistics vector
per step (NCCL over NVLink on GPUs, gloo on CPU in tests).  Denominators that
span the global batch (token-mean's N_tok, sequence means' B, DPO's pair
count) are computed on the host from the global batch layout, which every
rank holds, so no pre-kernel collective is needed.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

try:  # torch.distributed is plumbing; the shard planner itself is pure numpy
    import torch
    import torch.distributed as dist
except Exception:  # pragma: no cover
    torch = None
    dist = None


def group_rows(seq_lengths: Sequence[int], group_sizes: Sequence[int]) -> np.ndarray:
    """Trainable rows per group."""
    seq_lengths = np.asarray(seq_lengths, np.int64)
    go = np.concatenate([[0], np.cumsum(group_sizes)]).astype(np.int64)
    return np.array([seq_lengths[go[g]:go[g + 1]].sum() for g in range(len(group_sizes))],
                    np.int64)


def shard_groups(rows_per_group: Sequence[int], world: int) -> List[List[int]]:
    """Longest-processing-time bin packing of whole groups onto ranks, by row
    count (HBM bytes are proportional to rows).  Deterministic: groups are
    placed largest first (ties by index) on the least-loaded rank (ties by
    rank); each rank's groups are returned in ascending (sample_batch) order.
    Equal-length batches reduce to an even split."""
    if world < 1:
        raise ValueError("world must be >= 1")
    rows = np.asarray(rows_per_group, np.int64)
    order = sorted(range(len(rows)), key=lambda g: (-int(rows[g]), g))
    load = [0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for g in order:
        r = min(range(world), key=lambda i: (load[i], i))
        out[r].append(g)
        load[r] += int(rows[g])
    return [sorted(x) for x in out]


@dataclass
class GlobalCounts:
    """Batch-wide denominators passed to every rank's kernel call."""

    n_tok_rl: int
    n_seq_rl: int
    n_sft_seq: int
    n_groups: int

    @classmethod
    def of(cls, seq_lengths, group_sizes, seq_kind=None) -> "GlobalCounts":
        seq_lengths = np.asarray(seq_lengths, np.int64)
        kind = np.zeros(len(seq_lengths), np.int64) if seq_kind is None else np.asarray(seq_kind)
        rl = kind == 0
        return cls(n_tok_rl=int(seq_lengths[rl].sum()), n_seq_rl=int(rl.sum()),
                   n_sft_seq=int((~rl).sum()), n_groups=len(group_sizes))

    def kwargs(self) -> dict:
        return dict(n_tok_global=self.n_tok_rl, n_seq_global=self.n_seq_rl,
                    n_sft_seq_global=self.n_sft_seq)


@dataclass
class ShardSlice:
    """Index maps of one rank's shard into the global packed layout."""

    groups: np.ndarray      # global group ids, ascending
    seqs: np.ndarray        # global sequence ids, ascending
    rows: np.ndarray        # global row ids, ascending
    seq_lengths: np.ndarray
    group_sizes: np.ndarray


def shard_slice(seq_lengths, group_sizes, groups: Sequence[int]) -> ShardSlice:
    seq_lengths = np.asarray(seq_lengths, np.int64)
    group_sizes = np.asarray(group_sizes, np.int64)
    go = np.concatenate([[0], np.cumsum(group_sizes)])
    so = np.concatenate([[0], np.cumsum(seq_lengths)])
    groups = np.asarray(sorted(groups), np.int64)
    seqs = np.concatenate([np.arange(go[g], go[g + 1]) for g in groups]) if len(groups) else \
        np.zeros(0, np.int64)
    rows = np.concatenate([np.arange(so[i], so[i + 1]) for i in seqs]) if len(seqs) else \
        np.zeros(0, np.int64)
    return ShardSlice(groups=groups, seqs=seqs.astype(np.int64), rows=rows.astype(np.int64),
                      seq_lengths=seq_lengths[seqs] if len(seqs) else np.zeros(0, np.int64),
                      group_sizes=group_sizes[groups] if len(groups) else np.zeros(0, np.int64))


def allreduce_stats(stats, group=None):
    """Sum the statistics vector over ranks in place (no-op when not distributed).
    Stream-ordered on GPUs (NCCL); the only collective on the loss path."""
    if dist is not None and dist.is_available() and dist.is_initialized() and \
            dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def rank_world() -> Tuple[int, int]:
    if dist is not None and dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1
