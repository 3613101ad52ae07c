"""Data-parallel loss path with the real kernels: two ranks (gloo; both on
the one GPU reachable here -- on a multi-GPU box each rank owns a device and
the backend is NCCL) each run RFTLoss on their LPT shard of whole groups with
the global denominators, allreduce the 32-double statistics vector, and must
reproduce the single-process full batch: statistics to fp rounding, per-row
dlogits / logprobs row for row."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, pack_arrays
from paper_2505_17826_b200.distributed import (GlobalCounts, allreduce_stats, group_rows,
                                               shard_groups, shard_slice)

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

WORLD = 2
V = 151936
CFGS = [
    dict(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl", kl_coef=0.001,
         entropy_loss_fn="default", entropy_coef=0.001, loss_agg_mode="token-mean"),
    dict(advantage_fn="rloo", policy_loss_fn="vanilla", loss_agg_mode="seq-mean-token-mean"),
    dict(policy_loss_fn="opmd_kimi", tau=0.7),
]


def full_batch(seed=0):
    rng = np.random.default_rng(seed)
    group_sizes = [3, 4, 2, 4, 1, 3]
    seq_lengths = [int(rng.integers(1, 40)) for _ in range(sum(group_sizes))]
    T = sum(seq_lengths)
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = (torch.randn(T, V, device="cuda", generator=g) * 2.0).to(torch.bfloat16)
    tgt = rng.integers(0, V, T)
    reward = rng.integers(0, 2, len(seq_lengths)).astype(np.float32)
    old = rng.normal(-12.0, 0.3, T).astype(np.float32)
    ref = rng.normal(-12.0, 0.3, T).astype(np.float32)
    so = np.concatenate([[0], np.cumsum(seq_lengths)])
    seq_ref = np.array([old[so[i]:so[i + 1]].sum() for i in range(len(seq_lengths))], np.float32)
    return x, tgt, seq_lengths, group_sizes, reward, old, ref, seq_ref


def _worker(rank, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        x, tgt, lens, gs, reward, old, ref, seq_ref = full_batch()
        shards = shard_groups(group_rows(lens, gs), WORLD)
        glob = GlobalCounts.of(lens, gs).kwargs()
        sl = shard_slice(lens, gs, shards[rank])
        rows = torch.as_tensor(sl.rows, device="cuda")
        res = {}
        for i, kw in enumerate(CFGS):
            b = pack_arrays(x[rows].contiguous(), tgt[sl.rows], sl.seq_lengths, sl.group_sizes,
                            reward[sl.seqs], old_lp=old[sl.rows], ref_lp=ref[sl.rows],
                            seq_ref_lp=seq_ref[sl.seqs])
            out = RFTLoss(RFTLossConfig(**kw))(b, **glob)
            st = allreduce_stats(out.stats.clone())
            dz = torch.zeros((x.shape[0], V), dtype=torch.float32, device="cuda")
            dz[rows] = out.dlogits.float()
            lp = torch.zeros(x.shape[0], dtype=torch.float32, device="cuda")
            lp[rows] = out.lp
            dist.all_reduce(dz)
            dist.all_reduce(lp)
            res[f"st{i}"] = st.cpu().numpy()
            res[f"dz{i}"] = dz.cpu().numpy()
            res[f"lp{i}"] = lp.cpu().numpy()
        if rank == 0:
            np.savez(out_path, **res)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_match_single_process(tmp_path):
    out = tmp_path / "res.npz"
    mp.spawn(_worker, args=(_free_port(), str(out)), nprocs=WORLD, join=True)
    res = np.load(out)
    x, tgt, lens, gs, reward, old, ref, seq_ref = full_batch()
    glob = GlobalCounts.of(lens, gs).kwargs()
    for i, kw in enumerate(CFGS):
        b = pack_arrays(x, tgt, lens, gs, reward, old_lp=old, ref_lp=ref, seq_ref_lp=seq_ref)
        want = RFTLoss(RFTLossConfig(**kw))(b, **glob)
        st = want.stats.cpu().numpy()
        np.testing.assert_allclose(res[f"st{i}"], st, rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(res[f"lp{i}"], want.lp.cpu().numpy(), rtol=1e-6, atol=1e-5)
        dz = want.dlogits.float().cpu().numpy()
        assert np.max(np.abs(res[f"dz{i}"] - dz)) <= 2.0 ** -8 * np.max(np.abs(dz))
