"""Synthetic LLM-shaped cases: the same inputs as an oracle Batch (float64 of
the exact bf16 / f32 values) and as a device PackedBatch."""

from __future__ import annotations

import numpy as np
import torch

from oracle import rft_oracle as O
from paper_2505_17826_b200 import RFTLossConfig, pack_arrays


def make_case(seed, V, seq_lens, group_sizes, dtype=torch.bfloat16, scale=2.0, bump=None,
              old=True, ref=True, seq_kind=None, anchor=False, neg_inf=0.0, ld=None,
              seq_ref=True, device="cuda"):
    rng = np.random.default_rng(seed)
    T = int(sum(seq_lens))
    B = len(seq_lens)
    ld = ld or V
    target = rng.integers(0, V, T)
    x = rng.normal(0.0, scale, (T, ld)).astype(np.float32)
    if bump is None:
        bump = 1.5 * scale * np.log(max(V, 2)) ** 0.5
    x[np.arange(T), target] += bump
    if neg_inf > 0:
        m = rng.uniform(size=(T, ld)) < neg_inf
        m[np.arange(T), target] = False
        x[m] = -np.inf
    dev_logits = torch.as_tensor(x, device=device).to(dtype)
    host = dev_logits.float().cpu().numpy().astype(np.float64)[:, :V]
    anc_dev = None
    anc_host = None
    if anchor:
        a = (x + rng.normal(0.0, 0.5, x.shape).astype(np.float32))
        anc_dev = torch.as_tensor(a, device=device).to(dtype)
        anc_host = anc_dev.float().cpu().numpy().astype(np.float64)[:, :V]
    lp_true = O.row_forward(host, target)[1]
    old_lp = (lp_true + rng.normal(0.0, 0.05, T)).astype(np.float32) if old else None
    ref_lp = (lp_true + rng.normal(0.0, 0.1, T)).astype(np.float32) if ref else None
    reward = rng.integers(0, 2, B).astype(np.float32)
    if B:
        reward[: group_sizes[0]] = 1.0  # an all-equal group
    so = np.concatenate([[0], np.cumsum(seq_lens)]).astype(np.int64)
    seq_ref_lp = None
    if seq_ref and old_lp is not None:
        seq_ref_lp = np.array([old_lp[so[i]:so[i + 1]].astype(np.float64).sum()
                               for i in range(B)], np.float32)
    batch = O.Batch(logits=host, target=target, seq_offsets=so,
                    group_offsets=np.concatenate([[0], np.cumsum(group_sizes)]).astype(np.int64),
                    reward=reward.astype(np.float64),
                    seq_ref_lp=None if seq_ref_lp is None else seq_ref_lp.astype(np.float64),
                    old_lp=None if old_lp is None else old_lp.astype(np.float64),
                    ref_lp=None if ref_lp is None else ref_lp.astype(np.float64),
                    seq_kind=None if seq_kind is None else np.asarray(seq_kind, np.int64),
                    anchor_logits=anc_host)
    packed = pack_arrays(dev_logits[:, :V] if ld != V else dev_logits, target, seq_lens,
                         group_sizes, reward, old_lp=old_lp, ref_lp=ref_lp,
                         seq_ref_lp=seq_ref_lp, seq_kind=seq_kind,
                         anchor_logits=None if anc_dev is None else anc_dev[:, :V])
    return batch, packed


def oracle_cfg(cfg: RFTLossConfig, **kw) -> O.Config:
    return O.Config(advantage_fn=cfg.advantage_fn, policy_loss_fn=cfg.policy_loss_fn,
                    kl_fn=cfg.kl_fn, entropy_loss_fn=cfg.entropy_loss_fn,
                    loss_agg_mode=cfg.loss_agg_mode, tau=cfg.tau, clip_lo=cfg.clip_lo,
                    clip_hi=cfg.clip_hi, clip_c=cfg.clip_c, kl_coef=cfg.kl_coef,
                    entropy_coef=cfg.entropy_coef, std_eps=cfg.std_eps,
                    sft_weight=cfg.sft_weight, anchor_beta=cfg.anchor_beta,
                    dpo_beta=cfg.dpo_beta, agg_norm=cfg.agg_norm, **kw)
