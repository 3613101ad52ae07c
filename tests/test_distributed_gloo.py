"""Multi-rank host logic on CPU (world_size 2, gloo): group sharding, global
denominators and the statistics allreduce reproduce the single-rank batch.
The per-rank loss values come from the CPU oracle standing in for the kernel
(the kernel itself is covered by the GPU tests; here the subject is the
sharding + collective logic in paper_2505_17826_b200/distributed.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rft_oracle as O
from paper_2505_17826_b200.distributed import (GlobalCounts, allreduce_stats, group_rows,
                                               shard_groups, shard_slice)

WORLD = 2


def full_batch(seed=0, V=40):
    rng = np.random.default_rng(seed)
    group_sizes = [3, 4, 2, 4, 1, 3]
    seq_lengths = [int(rng.integers(0, 9)) for _ in range(sum(group_sizes))]
    T = sum(seq_lengths)
    b = O.Batch(logits=rng.normal(0, 1.5, (T, V)), target=rng.integers(0, V, T),
                seq_offsets=np.concatenate([[0], np.cumsum(seq_lengths)]),
                group_offsets=np.concatenate([[0], np.cumsum(group_sizes)]),
                reward=rng.integers(0, 2, len(seq_lengths)).astype(float),
                old_lp=rng.normal(-1.5, 0.3, T), ref_lp=rng.normal(-1.5, 0.3, T))
    b.seq_ref_lp = np.array([b.old_lp[b.seq_rows(i)].sum() for i in range(b.n_seqs)])
    return b, seq_lengths, group_sizes


def local_batch(b, sl):
    return O.Batch(logits=b.logits[sl.rows], target=b.target[sl.rows],
                   seq_offsets=np.concatenate([[0], np.cumsum(sl.seq_lengths)]),
                   group_offsets=np.concatenate([[0], np.cumsum(sl.group_sizes)]),
                   reward=b.reward[sl.seqs], old_lp=b.old_lp[sl.rows], ref_lp=b.ref_lp[sl.rows],
                   seq_ref_lp=b.seq_ref_lp[sl.seqs])


CFGS = [
    dict(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="k3", kl_coef=0.1,
         entropy_loss_fn="default", entropy_coef=0.01, loss_agg_mode="token-mean"),
    dict(advantage_fn="rloo", policy_loss_fn="vanilla", loss_agg_mode="seq-mean-token-mean"),
    dict(policy_loss_fn="opmd_kimi", tau=0.7),
]


def _worker(rank, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        b, lens, gs = full_batch()
        shards = shard_groups(group_rows(lens, gs), WORLD)
        counts = GlobalCounts.of(lens, gs)
        results = []
        for ci, kw in enumerate(CFGS):
            cfg = O.Config(**kw, n_tok_global=counts.n_tok_rl, n_seq_global=counts.n_seq_rl)
            sl = shard_slice(lens, gs, shards[rank])
            out = O.general_loss(local_batch(b, sl), cfg)
            st = torch.tensor(out["stats"], dtype=torch.float64)
            allreduce_stats(st)
            # per-row gradients and logprobs are row-separable: gather them too
            dz = torch.zeros_like(torch.tensor(b.logits))
            dz[torch.as_tensor(sl.rows)] = torch.tensor(out["dz"])
            dist.all_reduce(dz)
            results.append((st.numpy(), dz.numpy()))
        if rank == 0:
            np.savez(out_path, **{f"st{i}": r[0] for i, r in enumerate(results)},
                     **{f"dz{i}": r[1] for i, r in enumerate(results)})
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_planner_balances_and_preserves_order():
    rows = [5, 9, 1, 7, 7, 3, 2, 8]
    shards = shard_groups(rows, 3)
    assert sorted(g for s in shards for g in s) == list(range(len(rows)))
    loads = [sum(rows[g] for g in s) for s in shards]
    assert max(loads) - min(loads) <= max(rows)
    assert all(s == sorted(s) for s in shards)
    assert shard_groups([4] * 8, 4) == [[0, 4], [1, 5], [2, 6], [3, 7]]


def test_two_rank_gloo_matches_single_rank(tmp_path):
    out = tmp_path / "res.npz"
    mp.spawn(_worker, args=(_free_port(), str(out)), nprocs=WORLD, join=True)
    res = np.load(out)
    b, lens, gs = full_batch()
    counts = GlobalCounts.of(lens, gs)
    for i, kw in enumerate(CFGS):
        cfg = O.Config(**kw, n_tok_global=counts.n_tok_rl, n_seq_global=counts.n_seq_rl)
        ref = O.general_loss(b, cfg)
        np.testing.assert_allclose(res[f"st{i}"], ref["stats"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(res[f"dz{i}"], ref["dz"], rtol=0, atol=1e-15)
