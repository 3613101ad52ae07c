"""numpy float64 restatement of the reference loss path (TEST INFRASTRUCTURE).

Two layers:

1. ``ref_*`` functions restate the reference's own variants *in the
   reference's order of operations* so their losses are bit-identical to
   ``triad.algorithms`` on identical inputs (gradients to ~1e-13, because the
   reference accumulates rows per context bucket while we keep one row per
   token):

   - ``ref_logprob_rows``   policy.log_softmax + logprob   (policy.py:164-167, 194-212)
   - ``ref_grad_rows``      policy.softmax + grad_logprob  (policy.py:170-172, 253-270)
   - ``ref_tau_log_zhat``   algorithms.tau_log_zhat       (algorithms.py:93-101)
   - ``ref_opmd_kimi``      algorithms.loss_opmd_kimi     (algorithms.py:118-153)
   - ``ref_opmd_pairwise``  algorithms.loss_opmd_pairwise (algorithms.py:156-190)
   - ``ref_regularizer_g``  algorithms.regularizer_g      (algorithms.py:193-217)
   - ``ref_opmd_simple``    algorithms.loss_opmd_simple   (algorithms.py:220-253)
   - ``ref_sft``            algorithms.loss_sft           (algorithms.py:256-274)
   - ``ref_dpo``            algorithms.loss_dpo           (algorithms.py:277-326)
   - ``ref_combine``        algorithms.combine_reports    (algorithms.py:368-379)

2. ``general_loss`` restates the *unified* per-row formulation that the CUDA
   path implements for every registry combination (advantage_fn x
   policy_loss_fn x kl_fn x entropy x loss_agg_mode, plus the anchor KL and
   the sequence-coupled OPMD/DPO losses).  ``tests/test_oracle.py`` pins it
   to layer 1 through the exact reductions listed in SURVEY.md section 8c.

All inputs use the packed layout of ``include/tg_loss.h``: one logits row per
trainable (mask-true) token, rows of a sequence contiguous, sequences of a
group contiguous, ``seq_offsets[B+1]`` (rows per sequence) and
``group_offsets[G+1]`` (sequences per group).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, Optional, Sequence, Tuple

import numpy as np

# ---------------------------------------------------------------------------
# packed batch + config (mirrors TgBatch / TgConfig in include/tg_loss.h)


@dataclass
class Batch:
    logits: np.ndarray                  # [T, V] float64
    target: np.ndarray                  # [T] int
    seq_offsets: np.ndarray             # [B+1] int
    group_offsets: np.ndarray           # [G+1] int
    reward: np.ndarray                  # [B]
    seq_ref_lp: Optional[np.ndarray] = None   # [B] sequence-level reference logprob
    old_lp: Optional[np.ndarray] = None       # [T] behaviour (rollout) logprob per row
    ref_lp: Optional[np.ndarray] = None       # [T] reference-policy logprob per row
    seq_kind: Optional[np.ndarray] = None     # [B] 0 = RL rollout, 1 = SFT / expert
    anchor_logits: Optional[np.ndarray] = None  # [T, V] frozen anchor policy rows
    advantage: Optional[np.ndarray] = None    # [B] precomputed (advantage_fn "given")
    pg_coef: Optional[np.ndarray] = None      # [T] -d l_t / d lp_t (policy_loss_fn "given")
    pg_loss: Optional[np.ndarray] = None      # [T] l_t (policy_loss_fn "given")

    @property
    def n_rows(self) -> int:
        return int(self.logits.shape[0])

    @property
    def n_seqs(self) -> int:
        return len(self.seq_offsets) - 1

    @property
    def n_groups(self) -> int:
        return len(self.group_offsets) - 1

    def seq_rows(self, i: int) -> slice:
        return slice(int(self.seq_offsets[i]), int(self.seq_offsets[i + 1]))

    def group_seqs(self, g: int) -> range:
        return range(int(self.group_offsets[g]), int(self.group_offsets[g + 1]))


@dataclass
class Config:
    advantage_fn: str = "grpo"        # grpo | rloo | opmd | reinforce | given
    policy_loss_fn: str = "ppo_clip"  # vanilla | ppo_clip | sft | opmd_kimi | opmd_pairwise | dpo
    #                                   | given (a caller-registered per-row loss + coefficient)
    kl_fn: str = "none"               # none | k1 | k2 | k3 (low_var_kl) | abs
    entropy_loss_fn: str = "none"     # none | default
    loss_agg_mode: str = "token-mean"  # seq-sum | token-mean | seq-mean-token-sum |
    #                                    seq-mean-token-mean | seq-mean-token-sum-norm
    tau: float = 0.0
    clip_lo: float = 0.2
    clip_hi: float = 0.2
    clip_c: float = 0.0               # dual-clip constant (0 = off)
    kl_coef: float = 0.0
    entropy_coef: float = 0.0
    std_eps: float = 1e-6
    sft_weight: float = 1.0
    anchor_beta: float = 0.0
    dpo_beta: float = 0.1
    agg_norm: float = 1.0
    n_tok_global: int = 0             # 0 -> local RL row count
    n_seq_global: int = 0             # 0 -> local RL sequence count
    n_sft_seq_global: int = 0         # 0 -> local SFT sequence count


# ---------------------------------------------------------------------------
# layer 1: the reference's own variants, reference order of operations


def ref_logprob_rows(logits: np.ndarray, target: np.ndarray) -> np.ndarray:
    """lp_t = log_softmax(row_t)[y_t]   (policy.py:164-167, 209)."""
    out = np.empty(logits.shape[0])
    for t in range(logits.shape[0]):
        row = logits[t]
        shifted = row - np.max(row)
        out[t] = float((shifted - math.log(np.sum(np.exp(shifted))))[int(target[t])])
    return out


def ref_grad_rows(logits: np.ndarray, target: np.ndarray) -> np.ndarray:
    """e_{y_t} - softmax(row_t)   (policy.py:170-172, 267-269)."""
    out = np.empty_like(logits, dtype=np.float64)
    for t in range(logits.shape[0]):
        shifted = np.exp(logits[t] - np.max(logits[t]))
        vec = -(shifted / np.sum(shifted))
        vec[int(target[t])] += 1.0
        out[t] = vec
    return out


def _seq_total(lp_rows: np.ndarray, batch: Batch, i: int) -> float:
    """Sequential per-sequence sum, as policy.logprob accumulates (policy.py:205-211)."""
    total = 0.0
    for v in lp_rows[batch.seq_rows(i)]:
        total += float(v)
    return total


def ref_tau_log_zhat(rewards: Sequence[float], tau: float) -> float:
    """algorithms.py:93-101."""
    if tau <= 0:
        raise ValueError(f"tau must be > 0, got {tau}")
    if not rewards:
        raise ValueError("rewards must be nonempty")
    m = max(rewards)
    mean_exp = sum(math.exp((r - m) / tau) for r in rewards) / len(rewards)
    return m + tau * math.log(mean_exp)


@dataclass
class Report:
    """LossReport restated with a dense per-row gradient (algorithms.py:59-69)."""

    loss: float
    dz: np.ndarray                      # [T, V]: d loss / d logits row, one row per token
    metrics: Dict[str, float] = field(default_factory=dict)


def _kl_metric(lps: Sequence[float], refs: Sequence[float]) -> float:
    """algorithms.py:112-115."""
    return float(np.mean([r - l for l, r in zip(lps, refs)]))


def _group_lp_grads(batch: Batch, g: int, lp_rows, grad_rows):
    seqs = list(batch.group_seqs(g))
    return seqs, [_seq_total(lp_rows, batch, i) for i in seqs]


def ref_opmd_simple(batch: Batch, g: int, tau: float, beta: float,
                    lp_rows=None, grad_rows=None) -> Report:
    """algorithms.py:220-253 for one group (rows of other groups get zero grad)."""
    lp_rows = ref_logprob_rows(batch.logits, batch.target) if lp_rows is None else lp_rows
    grad_rows = ref_grad_rows(batch.logits, batch.target) if grad_rows is None else grad_rows
    seqs, lps = _group_lp_grads(batch, g, lp_rows, grad_rows)
    rewards = [float(batch.reward[i]) for i in seqs]
    rbar = float(np.mean(rewards))
    coef = 1.0 / (1.0 + tau)
    loss = 0.0
    dz = np.zeros_like(batch.logits, dtype=np.float64)
    for i, r, lp in zip(seqs, rewards, lps):
        loss -= coef * (r - rbar) * lp
        dz[batch.seq_rows(i)] += (-coef * (r - rbar)) * grad_rows[batch.seq_rows(i)]
    if beta > 0:
        g_value, g_dz = ref_regularizer_g(batch, g)
        loss += beta * g_value
        dz += beta * g_dz
    refs = [float(batch.seq_ref_lp[i]) for i in seqs]
    metrics = {
        "mean_reward": rbar,
        "baseline": rbar,
        "kl_estimate": _kl_metric(lps, refs),
        "group_size": float(len(seqs)),
    }
    return Report(loss, dz, metrics)


def ref_regularizer_g(batch: Batch, g: int) -> Tuple[float, np.ndarray]:
    """algorithms.py:193-217: (1/K) sum over visited rows of KL(p || q)."""
    seqs = list(batch.group_seqs(g))
    k = len(seqs)
    total = 0.0
    dz = np.zeros_like(batch.logits, dtype=np.float64)
    for i in seqs:
        for t in range(*batch.seq_rows(i).indices(batch.n_rows)):
            row = batch.logits[t]
            qrow = batch.anchor_logits[t]
            sh = np.exp(row - np.max(row))
            p = sh / np.sum(sh)
            s1 = row - np.max(row)
            log_p = s1 - math.log(np.sum(np.exp(s1)))
            s2 = qrow - np.max(qrow)
            log_q = s2 - math.log(np.sum(np.exp(s2)))
            kl = float(np.sum(p * (log_p - log_q)))
            total += kl / k
            dz[t] += p * ((log_p - log_q) - kl) / k
    return total, dz


def ref_opmd_kimi(batch: Batch, g: int, tau: float, lp_rows=None, grad_rows=None) -> Report:
    """algorithms.py:118-153 (refs = batch.seq_ref_lp)."""
    if tau <= 0:
        raise ValueError("OPMD_KIMI requires tau > 0")
    lp_rows = ref_logprob_rows(batch.logits, batch.target) if lp_rows is None else lp_rows
    grad_rows = ref_grad_rows(batch.logits, batch.target) if grad_rows is None else grad_rows
    seqs, lps = _group_lp_grads(batch, g, lp_rows, grad_rows)
    rewards = [float(batch.reward[i]) for i in seqs]
    refs = [float(batch.seq_ref_lp[i]) for i in seqs]
    zhat = ref_tau_log_zhat(rewards, tau)
    loss = 0.0
    dz = np.zeros_like(batch.logits, dtype=np.float64)
    for i, r, lp, ref in zip(seqs, rewards, lps, refs):
        residual = r - zhat - tau * (lp - ref)
        loss += residual * residual
        dz[batch.seq_rows(i)] += (-2.0 * tau * residual) * grad_rows[batch.seq_rows(i)]
    metrics = {
        "mean_reward": float(np.mean(rewards)),
        "baseline": zhat,
        "kl_estimate": _kl_metric(lps, refs),
        "group_size": float(len(seqs)),
    }
    return Report(loss, dz, metrics)


def ref_opmd_pairwise(batch: Batch, g: int, tau: float, lp_rows=None, grad_rows=None) -> Report:
    """algorithms.py:156-190."""
    if tau <= 0:
        raise ValueError("OPMD_PAIRWISE requires tau > 0")
    lp_rows = ref_logprob_rows(batch.logits, batch.target) if lp_rows is None else lp_rows
    grad_rows = ref_grad_rows(batch.logits, batch.target) if grad_rows is None else grad_rows
    seqs, lps = _group_lp_grads(batch, g, lp_rows, grad_rows)
    k = len(seqs)
    if k < 2:
        raise ValueError("pairwise loss needs a group of at least 2 rollouts")
    rewards = [float(batch.reward[i]) for i in seqs]
    refs = [float(batch.seq_ref_lp[i]) for i in seqs]
    a = [r - tau * (lp - ref) for r, lp, ref in zip(rewards, lps, refs)]
    loss = 0.0
    for i in range(k):
        for j in range(i + 1, k):
            diff = a[i] - a[j]
            loss += diff * diff
    total_a = sum(a)
    dz = np.zeros_like(batch.logits, dtype=np.float64)
    for idx, i in enumerate(seqs):
        dz[batch.seq_rows(i)] += (-2.0 * tau * (k * a[idx] - total_a)) * grad_rows[batch.seq_rows(i)]
    metrics = {
        "mean_reward": float(np.mean(rewards)),
        "baseline": float(np.mean(rewards)),
        "kl_estimate": _kl_metric(lps, refs),
        "group_size": float(k),
    }
    return Report(loss, dz, metrics)


def ref_sft(batch: Batch, seqs: Optional[Sequence[int]] = None,
            lp_rows=None, grad_rows=None) -> Report:
    """algorithms.py:256-274 over the given sequences (default: all)."""
    seqs = list(range(batch.n_seqs)) if seqs is None else list(seqs)
    if not seqs:
        raise ValueError("SFT batch must be nonempty")
    lp_rows = ref_logprob_rows(batch.logits, batch.target) if lp_rows is None else lp_rows
    grad_rows = ref_grad_rows(batch.logits, batch.target) if grad_rows is None else grad_rows
    n = len(seqs)
    loss = 0.0
    dz = np.zeros_like(batch.logits, dtype=np.float64)
    for i in seqs:
        lp = _seq_total(lp_rows, batch, i)
        loss -= lp / n
        dz[batch.seq_rows(i)] += (-1.0 / n) * grad_rows[batch.seq_rows(i)]
    rewards = [float(batch.reward[i]) for i in seqs]
    metrics = {
        "mean_reward": float(np.mean(rewards)) if rewards else 0.0,
        "baseline": 0.0,
        "kl_estimate": 0.0,
        "group_size": float(n),
    }
    return Report(loss, dz, metrics)


def _sigmoid(x: float) -> float:
    """algorithms.py:318-322."""
    if x >= 0:
        return 1.0 / (1.0 + math.exp(-x))
    e = math.exp(x)
    return e / (1.0 + e)


def _softplus(x: float) -> float:
    """algorithms.py:325-326."""
    return math.log1p(math.exp(-abs(x))) + max(x, 0.0)


def ref_dpo(batch: Batch, dpo_beta: float, lp_rows=None, grad_rows=None) -> Report:
    """algorithms.py:277-315.  Every group is one (chosen, rejected) pair, in that
    order; ``seq_ref_lp`` holds the reference policy's sequence logprobs."""
    if batch.n_groups < 1:
        raise ValueError("DPO batch must be nonempty")
    if dpo_beta <= 0:
        raise ValueError(f"dpo_beta must be > 0, got {dpo_beta}")
    lp_rows = ref_logprob_rows(batch.logits, batch.target) if lp_rows is None else lp_rows
    grad_rows = ref_grad_rows(batch.logits, batch.target) if grad_rows is None else grad_rows
    n = batch.n_groups
    loss = 0.0
    dz = np.zeros_like(batch.logits, dtype=np.float64)
    margins = []
    for g in range(n):
        c, r = list(batch.group_seqs(g))
        lpc, lpr = _seq_total(lp_rows, batch, c), _seq_total(lp_rows, batch, r)
        margin = dpo_beta * ((lpc - float(batch.seq_ref_lp[c])) - (lpr - float(batch.seq_ref_lp[r])))
        margins.append(margin)
        loss += _softplus(-margin) / n
        coef = (_sigmoid(margin) - 1.0) * dpo_beta / n
        dz[batch.seq_rows(c)] += coef * grad_rows[batch.seq_rows(c)]
        dz[batch.seq_rows(r)] += (-coef) * grad_rows[batch.seq_rows(r)]
    metrics = {
        "mean_reward": float(np.mean(margins)),
        "baseline": 0.0,
        "kl_estimate": 0.0,
        "group_size": float(n),
    }
    return Report(loss, dz, metrics)


def ref_combine(reports: Sequence[Report]) -> Report:
    """algorithms.py:368-379: losses and gradients summed, metrics averaged."""
    if not reports:
        raise ValueError("cannot combine an empty report list")
    loss = 0.0
    dz = np.zeros_like(reports[0].dz)
    for rep in reports:
        loss += rep.loss
        dz += rep.dz
    keys = reports[0].metrics.keys()
    metrics = {k: float(np.mean([r.metrics[k] for r in reports])) for k in keys}
    return Report(loss, dz, metrics)


def ref_group_batch(batch: Batch, variant: str, tau: float = 1.0, beta: float = 0.0) -> Report:
    """Trainer.step_groups without apply_update (orchestrator.py:299-308)."""
    lp_rows = ref_logprob_rows(batch.logits, batch.target)
    grad_rows = ref_grad_rows(batch.logits, batch.target)
    reps = []
    for g in range(batch.n_groups):
        if variant == "OPMD_SIMPLE":
            reps.append(ref_opmd_simple(batch, g, tau, beta, lp_rows, grad_rows))
        elif variant == "OPMD_KIMI":
            reps.append(ref_opmd_kimi(batch, g, tau, lp_rows, grad_rows))
        elif variant == "OPMD_PAIRWISE":
            reps.append(ref_opmd_pairwise(batch, g, tau, lp_rows, grad_rows))
        else:
            raise ValueError(f"{variant} is not a group-based loss")
    return ref_combine(reps)


# ---------------------------------------------------------------------------
# layer 2: the unified per-row formulation the CUDA path implements

#: Stats vector layout; must match TG_S_* in include/tg_loss.h.
STAT_NAMES = [
    "loss", "pg_loss", "kl_loss", "entropy_loss", "anchor_loss", "sft_loss",
    "n_groups", "sum_mean_reward", "sum_baseline", "sum_kl_estimate", "sum_group_size",
    "n_tok", "n_tok_rl", "clip_count", "sum_entropy", "sum_kl", "sum_ppo_kl",
    "sum_lp", "nonfinite", "n_seqs", "sum_adv", "sum_ratio", "n_sft_seqs",
    "sum_sft_reward", "sum_dpo_margin", "dual_clip_count", "sum_anchor_kl",
    "invalid", "reserved28", "reserved29", "reserved30", "reserved31",
]
STAT = {n: i for i, n in enumerate(STAT_NAMES)}
NSTAT = len(STAT_NAMES)


def row_forward(logits: np.ndarray, target: np.ndarray, block: int = 512):
    """Per-row lse, lp and entropy H = lse - sum_v p_v z_v, in row blocks."""
    T = logits.shape[0]
    lse = np.empty(T)
    lp = np.empty(T)
    ent = np.empty(T)
    for a in range(0, T, block):
        X = np.asarray(logits[a:a + block], dtype=np.float64)
        m = X.max(axis=1)
        e = np.exp(X - m[:, None])
        s = e.sum(axis=1)
        l = m + np.log(s)
        lse[a:a + block] = l
        lp[a:a + block] = X[np.arange(X.shape[0]), target[a:a + block]] - l
        # -inf logits (masked vocabulary entries) carry p = 0 and add nothing
        ent[a:a + block] = l - (e * np.maximum(X, -1e30)).sum(axis=1) / s
    return lse, lp, ent


def advantages(batch: Batch, cfg: Config) -> np.ndarray:
    """Per-sequence advantage A_i for RL sequences (SFT sequences get 0)."""
    A = np.zeros(batch.n_seqs)
    kind = batch.seq_kind if batch.seq_kind is not None else np.zeros(batch.n_seqs, np.int64)
    for g in range(batch.n_groups):
        seqs = [i for i in batch.group_seqs(g) if kind[i] == 0]
        if not seqs:
            continue
        r = np.array([float(batch.reward[i]) for i in seqs])
        k = len(seqs)
        fn = cfg.advantage_fn
        if fn == "opmd":       # algorithms.py:234-242: (r - rbar) / (1 + tau)
            rbar = float(np.mean(r))
            a = (1.0 / (1.0 + cfg.tau)) * (r - rbar)
        elif fn == "grpo":     # (r - mean) / (std_unbiased + eps); K = 1 -> 0
            if k < 2:
                a = np.zeros(k)
            else:
                a = (r - r.mean()) / (r.std(ddof=1) + cfg.std_eps)
        elif fn == "rloo":     # r_i - mean_{j != i} r_j; K = 1 -> 0
            a = np.zeros(k) if k < 2 else (r - (r.sum() - r) / (k - 1))
        elif fn == "reinforce":
            a = r.copy()
        elif fn == "given":
            a = (np.zeros(k) if batch.advantage is None
                 else np.array([float(batch.advantage[i]) for i in seqs]))
        else:
            raise ValueError(f"unknown advantage_fn {fn}")
        A[seqs] = a
    return A


def seq_weights(batch: Batch, cfg: Config) -> np.ndarray:
    """Per-sequence aggregation weight w_i applied to every row of sequence i."""
    kind = batch.seq_kind if batch.seq_kind is not None else np.zeros(batch.n_seqs, np.int64)
    n_rows = np.diff(batch.seq_offsets)
    rl = kind == 0
    n_tok = cfg.n_tok_global or int(n_rows[rl].sum())
    n_seq = cfg.n_seq_global or int(rl.sum())
    n_sft = cfg.n_sft_seq_global or int((~rl).sum())
    w = np.zeros(batch.n_seqs)
    mode = cfg.loss_agg_mode
    for i in range(batch.n_seqs):
        if not rl[i]:
            w[i] = cfg.sft_weight / max(n_sft, 1)
        elif mode == "seq-sum":
            w[i] = 1.0
        elif mode == "token-mean":
            w[i] = 1.0 / max(n_tok, 1)
        elif mode == "seq-mean-token-sum":
            w[i] = 1.0 / max(n_seq, 1)
        elif mode == "seq-mean-token-mean":
            w[i] = 1.0 / (max(n_seq, 1) * max(int(n_rows[i]), 1))
        elif mode == "seq-mean-token-sum-norm":
            w[i] = 1.0 / cfg.agg_norm
        else:
            raise ValueError(f"unknown loss_agg_mode {mode}")
    return w


def _kl_value_grad(kind: str, lp: np.ndarray, ref: np.ndarray):
    """Token KL penalty and its derivative w.r.t. lp."""
    if kind == "k1":
        return lp - ref, np.ones_like(lp)
    if kind == "k2":
        d = lp - ref
        return 0.5 * d * d, d
    if kind in ("k3", "low_var_kl"):
        delta = ref - lp
        dcl = np.clip(delta, -20.0, 20.0)
        ratio = np.exp(dcl)
        raw = ratio - dcl - 1.0
        val = np.clip(raw, -10.0, 10.0)
        live = (delta == dcl) & (raw == val)
        return val, np.where(live, 1.0 - ratio, 0.0)
    if kind == "abs":
        d = lp - ref
        return np.abs(d), np.sign(d)
    raise ValueError(f"unknown kl_fn {kind}")


def general_loss(batch: Batch, cfg: Config, want_dz: bool = True) -> Dict[str, object]:
    """The unified per-row loss that every CUDA entry point computes.

    Returns dict with ``stats`` (NSTAT float64, layout STAT_NAMES), ``dz``
    [T,V] (or None), ``lp``/``entropy``/``lse`` [T], ``seq_lp`` [B],
    ``seq_adv`` [B].
    """
    T, V = batch.logits.shape
    B, G = batch.n_seqs, batch.n_groups
    kind = batch.seq_kind if batch.seq_kind is not None else np.zeros(B, np.int64)
    lse, lp, ent = row_forward(batch.logits, batch.target)
    row_seq = np.repeat(np.arange(B), np.diff(batch.seq_offsets))
    seq_lp = np.array([lp[batch.seq_rows(i)].sum() for i in range(B)])
    st = np.zeros(NSTAT)
    pg = cfg.policy_loss_fn
    coupled = pg in ("opmd_kimi", "opmd_pairwise", "dpo")
    A = advantages(batch, cfg) if not coupled else np.zeros(B)
    w = seq_weights(batch, cfg) if not coupled else np.ones(B)
    old = batch.old_lp if batch.old_lp is not None else lp
    ref = batch.ref_lp if batch.ref_lp is not None else lp
    seq_ref = (batch.seq_ref_lp if batch.seq_ref_lp is not None
               else np.array([old[batch.seq_rows(i)].sum() for i in range(B)]))
    is_rl_row = kind[row_seq] == 0
    s = np.zeros(T)       # s_t = -d loss / d lp_t
    h = np.zeros(T)       # entropy coefficient per row
    loss_rows = np.zeros(T)

    if not coupled:
        At = A[row_seq]
        wt = w[row_seq]
        if pg == "vanilla":
            pg_t = -At * lp
            s_pg = At.copy()
        elif pg == "ppo_clip":
            dlr = lp - old
            logr = np.clip(dlr, -20.0, 20.0)
            rho = np.exp(logr)
            l1 = -At * rho
            l2 = -At * np.clip(rho, 1.0 - cfg.clip_lo, 1.0 + cfg.clip_hi)
            pg_t = np.maximum(l1, l2)
            clipped = l2 > l1
            # the log-ratio clamp is a torch.clamp (verl): zero gradient when active
            s_pg = np.where(clipped | (logr != dlr), 0.0, At * rho)
            if cfg.clip_c > 0:
                l3 = -At * cfg.clip_c
                dual = (At < 0) & (l3 < pg_t)
                pg_t = np.where(dual, l3, pg_t)
                s_pg = np.where(dual, 0.0, s_pg)
                st[STAT["dual_clip_count"]] = float((dual & is_rl_row).sum())
            st[STAT["clip_count"]] = float((clipped & is_rl_row).sum())
            st[STAT["sum_ratio"]] = float(rho[is_rl_row].sum())
            st[STAT["sum_ppo_kl"]] = float((old - lp)[is_rl_row].sum())
        elif pg == "sft":
            pg_t = -lp
            s_pg = np.ones(T)
        elif pg == "given":  # a registered Python policy loss, evaluated by the caller
            pg_t = np.asarray(batch.pg_loss, np.float64)
            s_pg = np.asarray(batch.pg_coef, np.float64)
        else:
            raise ValueError(f"unknown policy_loss_fn {pg}")
        kl_t = np.zeros(T)
        s_kl = np.zeros(T)
        if cfg.kl_fn != "none":
            kl_t, dkl = _kl_value_grad(cfg.kl_fn, lp, ref)
            s_kl = -cfg.kl_coef * dkl
        ent_on = cfg.entropy_loss_fn != "none"
        c_ent = cfg.entropy_coef if ent_on else 0.0
        # RL rows
        s = np.where(is_rl_row, wt * (s_pg + s_kl), wt * 1.0)
        h = np.where(is_rl_row, c_ent * wt, 0.0)
        pg_loss = np.where(is_rl_row, wt * pg_t, 0.0)
        kl_loss = np.where(is_rl_row, wt * cfg.kl_coef * kl_t, 0.0)
        ent_loss = np.where(is_rl_row, -c_ent * wt * ent, 0.0)
        sft_loss = np.where(is_rl_row, 0.0, -wt * lp)
        loss_rows = pg_loss + kl_loss + ent_loss + sft_loss
        st[STAT["pg_loss"]] = pg_loss.sum()
        st[STAT["kl_loss"]] = kl_loss.sum()
        st[STAT["entropy_loss"]] = ent_loss.sum()
        st[STAT["sft_loss"]] = sft_loss.sum()
        st[STAT["sum_kl"]] = float(kl_t[is_rl_row].sum())
        st[STAT["sum_adv"]] = float(A[kind == 0].sum())
    else:
        coef_seq = np.zeros(B)    # s_i: per-sequence -d loss / d LP_i
        total = 0.0
        if pg == "dpo":
            n = G
            for g in range(G):
                c, r = list(batch.group_seqs(g))
                margin = cfg.dpo_beta * ((seq_lp[c] - seq_ref[c]) - (seq_lp[r] - seq_ref[r]))
                total += _softplus(-margin) / n
                sig1 = (1.0 - _sigmoid(margin)) * cfg.dpo_beta / n
                coef_seq[c] = sig1
                coef_seq[r] = -sig1
                st[STAT["sum_dpo_margin"]] += margin
        else:
            tau = cfg.tau
            for g in range(G):
                seqs = list(batch.group_seqs(g))
                r = np.array([float(batch.reward[i]) for i in seqs])
                lps = seq_lp[seqs]
                refs = seq_ref[seqs]
                if pg == "opmd_kimi":
                    zhat = ref_tau_log_zhat(list(r), tau)
                    res = r - zhat - tau * (lps - refs)
                    total += float((res * res).sum())
                    coef_seq[seqs] = 2.0 * tau * res
                else:
                    a = r - tau * (lps - refs)
                    k = len(seqs)
                    total += float(k * (a * a).sum() - a.sum() ** 2)
                    coef_seq[seqs] = 2.0 * tau * (k * a - a.sum())
        s = coef_seq[row_seq]
        st[STAT["pg_loss"]] = total
        loss_rows[:] = 0.0

    # anchor KL regularizer (algorithms.py:193-217), beta * (1/K) sum kl_t per group
    anchor_loss = 0.0
    akl = None
    if cfg.anchor_beta > 0:
        if batch.anchor_logits is None:
            raise ValueError("anchor_beta > 0 requires anchor_logits")
        ksize = np.zeros(B)
        for g in range(G):
            seqs = list(batch.group_seqs(g))
            ksize[seqs] = len(seqs)
        qlse, _, _ = row_forward(batch.anchor_logits, batch.target)
        X = batch.logits
        Q = batch.anchor_logits
        p = np.exp(X - lse[:, None])
        d = (X - lse[:, None]) - (Q - qlse[:, None])
        akl = (p * d).sum(axis=1)
        coefa = cfg.anchor_beta / ksize[row_seq]
        anchor_loss = float((coefa * akl).sum())
        st[STAT["anchor_loss"]] = anchor_loss
        st[STAT["sum_anchor_kl"]] = float(akl.sum())

    dz = None
    if want_dz:
        X = np.maximum(batch.logits, -1e30)   # p = 0 exactly where a logit is -inf
        p = np.exp(X - lse[:, None])
        dz = p * (s[:, None] + h[:, None] * ((X - lse[:, None]) + ent[:, None]))
        dz[np.arange(T), batch.target] -= s
        if akl is not None:
            dz += coefa[:, None] * p * (d - akl[:, None])

    st[STAT["loss"]] = st[STAT["pg_loss"]] + st[STAT["kl_loss"]] + st[STAT["entropy_loss"]] \
        + st[STAT["sft_loss"]] + anchor_loss
    # bookkeeping + per-group metrics (mean_reward, baseline, kl_estimate, group_size)
    st[STAT["n_tok"]] = T
    st[STAT["n_tok_rl"]] = float(is_rl_row.sum())
    st[STAT["n_seqs"]] = B
    st[STAT["n_sft_seqs"]] = float((kind != 0).sum())
    st[STAT["sum_sft_reward"]] = float(batch.reward[kind != 0].sum())
    st[STAT["sum_lp"]] = lp.sum()
    st[STAT["sum_entropy"]] = float(ent[is_rl_row].sum())
    nonfinite = (~np.isfinite(lp)).sum() + (~np.isfinite(lse)).sum()
    if dz is not None:
        nonfinite += (~np.isfinite(dz).all(axis=1)).sum()
    st[STAT["nonfinite"]] = float(nonfinite)
    for g in range(G):
        seqs = [i for i in batch.group_seqs(g) if kind[i] == 0]
        if not seqs:
            continue
        r = np.array([float(batch.reward[i]) for i in seqs])
        st[STAT["n_groups"]] += 1
        st[STAT["sum_mean_reward"]] += float(np.mean(r))
        if pg == "opmd_kimi":
            st[STAT["sum_baseline"]] += ref_tau_log_zhat(list(r), cfg.tau)
        elif pg == "dpo":
            pass
        else:
            st[STAT["sum_baseline"]] += float(np.mean(r))
        st[STAT["sum_kl_estimate"]] += float(np.mean(seq_ref[seqs] - seq_lp[seqs]))
        st[STAT["sum_group_size"]] += len(seqs)
    return {
        "stats": st, "dz": dz, "lp": lp, "entropy": ent, "lse": lse,
        "seq_lp": seq_lp, "seq_adv": A, "seq_w": w, "s": s,
    }


def stats_dict(st: np.ndarray) -> Dict[str, float]:
    return {n: float(st[i]) for i, n in enumerate(STAT_NAMES) if not n.startswith("reserved")}


def single_pass_blocked(batch: Batch, cfg: Config, dz_out: Optional[np.ndarray] = None,
                        block: int = 64) -> Dict[str, object]:
    """Memory-bounded restatement of ``general_loss`` for the single-pass
    policy losses (vanilla / ppo_clip / sft, any advantage / KL / entropy /
    aggregation, no anchor): rows are processed in blocks, so Qwen-vocab
    samples fit in host RAM.  Used as the timed CPU baseline (bench.py) and
    checked against ``general_loss`` in tests/test_oracle.py."""
    if cfg.policy_loss_fn not in ("vanilla", "ppo_clip", "sft") or cfg.anchor_beta > 0:
        raise ValueError("single_pass_blocked handles single-pass losses without anchor")
    T = batch.n_rows
    B = batch.n_seqs
    kind = batch.seq_kind if batch.seq_kind is not None else np.zeros(B, np.int64)
    A = advantages(batch, cfg)
    w = seq_weights(batch, cfg)
    row_seq = np.repeat(np.arange(B), np.diff(batch.seq_offsets))
    is_rl = kind[row_seq] == 0
    lse = np.empty(T)
    lp = np.empty(T)
    ent = np.empty(T)
    loss = np.zeros(4)  # pg, kl, ent, sft
    c_ent = cfg.entropy_coef if cfg.entropy_loss_fn != "none" else 0.0
    for a in range(0, T, block):
        b = min(a + block, T)
        X = np.maximum(np.asarray(batch.logits[a:b], dtype=np.float64), -1e30)
        y = batch.target[a:b]
        m = X.max(axis=1)
        e = np.exp(X - m[:, None])
        s_ = e.sum(axis=1)
        l = m + np.log(s_)
        lpb = X[np.arange(b - a), y] - l
        hb = l - (e * X).sum(axis=1) / s_
        lse[a:b], lp[a:b], ent[a:b] = l, lpb, hb
        At, wt, rl = A[row_seq[a:b]], w[row_seq[a:b]], is_rl[a:b]
        if cfg.policy_loss_fn == "ppo_clip":
            old = batch.old_lp[a:b] if batch.old_lp is not None else lpb
            dlr = lpb - old
            logr = np.clip(dlr, -20.0, 20.0)
            rho = np.exp(logr)
            l1 = -At * rho
            l2 = -At * np.clip(rho, 1.0 - cfg.clip_lo, 1.0 + cfg.clip_hi)
            pg = np.maximum(l1, l2)
            s_pg = np.where((l2 > l1) | (logr != dlr), 0.0, At * rho)
            if cfg.clip_c > 0:
                l3 = -At * cfg.clip_c
                dual = (At < 0) & (l3 < pg)
                pg = np.where(dual, l3, pg)
                s_pg = np.where(dual, 0.0, s_pg)
        elif cfg.policy_loss_fn == "sft":
            pg, s_pg = -lpb, np.ones(b - a)
        else:
            pg, s_pg = -At * lpb, At.copy()
        klv = np.zeros(b - a)
        s_kl = np.zeros(b - a)
        if cfg.kl_fn != "none":
            ref = batch.ref_lp[a:b] if batch.ref_lp is not None else lpb
            klv, dkl = _kl_value_grad(cfg.kl_fn, lpb, ref)
            s_kl = -cfg.kl_coef * dkl
        s = np.where(rl, wt * (s_pg + s_kl), wt)
        h = np.where(rl, c_ent * wt, 0.0)
        loss += [np.where(rl, wt * pg, 0).sum(), np.where(rl, wt * cfg.kl_coef * klv, 0).sum(),
                 np.where(rl, -c_ent * wt * hb, 0).sum(), np.where(rl, 0, -wt * lpb).sum()]
        p = e / s_[:, None]
        dz = p * (s[:, None] + h[:, None] * ((X - l[:, None]) + hb[:, None]))
        dz[np.arange(b - a), y] -= s
        if dz_out is not None:
            dz_out[a:b] = dz
    return {"loss": float(loss.sum()), "pg_loss": loss[0], "kl_loss": loss[1],
            "entropy_loss": loss[2], "sft_loss": loss[3], "lp": lp, "entropy": ent, "lse": lse}
