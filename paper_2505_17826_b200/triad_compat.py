"""Reference-shaped drop-in: ``group_loss`` / ``loss_sft`` / ``loss_dpo`` /
``combine_reports`` / ``Trainer`` with the reference's signatures and error
behaviour, computed by the CUDA path.

The reference (``triad``) scores tokens with a bucketed logits *table*
(policy.py:59-94): each mask-true token t reads row
``state_t = FNV1a(context, t, prev) mod S`` (policy.py:152-191).  Here the
states come from the C host helper ``tg_scored_states`` and the table is
read in place by the kernels through ``row_index`` (no gather copy); the
per-token gradient rows are scatter-added back by state into a dense table
gradient, which is what ``SparseGrad.to_dense`` holds in the reference
(policy.py:215-250).

Gradients stay on the GPU: ``SparseGrad`` holds the touched states and
their rows as device tensors (the reference's ``{state: row}`` dict is
materialised only when ``.rows`` is read), ``combine_reports`` merges them on
the device, and ``apply_update`` / ``Trainer`` step the table with
``tg_apply_update``.  ``Trainer`` keeps the policy table resident on the GPU;
``params`` materialises the host table when read.

Objects are duck-typed: ``params`` needs ``logits`` [S, V], ``num_buckets``,
``vocab.size`` (and ``version`` for the Trainer); groups / experiences as in
records.py.  Arithmetic is fp32 on the device (tables are uploaded as f32),
so results match the reference's float64 to ~1e-6 relative, not bit-exactly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, Sequence, Tuple

import numpy as np
import torch

from .config import AlgorithmError, RFTLossConfig, Variant
from .loss import RFTLoss, logprob_fwd, stats_to_metrics
from .packing import HostGroups, PolicyError, flatten_groups, pack_arrays, scored_states


@dataclass
class AlgorithmConfig:
    """algorithms.py:36-56, same validation."""

    variant: Variant = Variant.OPMD_SIMPLE
    tau: float = 1.0
    beta: float = 0.0
    dpo_beta: float = 0.1
    learning_rate: float = 0.1

    def __post_init__(self) -> None:
        if isinstance(self.variant, str):
            self.variant = Variant(self.variant)
        if self.tau < 0:
            raise AlgorithmError(f"tau must be >= 0, got {self.tau}")
        if self.variant in (Variant.OPMD_KIMI, Variant.OPMD_PAIRWISE) and self.tau <= 0:
            raise AlgorithmError(f"{self.variant.value} requires tau > 0")
        if self.beta < 0:
            raise AlgorithmError(f"beta must be >= 0, got {self.beta}")
        if self.dpo_beta <= 0:
            raise AlgorithmError(f"dpo_beta must be > 0, got {self.dpo_beta}")
        if self.learning_rate <= 0:
            raise AlgorithmError(f"learning_rate must be > 0, got {self.learning_rate}")


class SparseGrad:
    """policy.SparseGrad (policy.py:215-250): the touched rows of a table
    gradient, held on the GPU as ascending state ids ``ids`` [n] int64 and
    float64 rows ``vals`` [n, V].  The reference's methods are kept; ``rows``
    gives the reference's {state: row} dict (a host copy, made on access)."""

    def __init__(self, ids=None, vals=None) -> None:
        self.ids = ids
        self.vals = vals

    @classmethod
    def from_token_rows(cls, dz: torch.Tensor, states) -> "SparseGrad":
        """Per-token gradient rows -> per-state sums (grad_logprob's add_row
        per scored token, policy.py:253-270), on the device."""
        dev = dz.device
        st = torch.as_tensor(np.asarray(states, np.int64), device=dev)
        ids, inv = torch.unique(st, sorted=True, return_inverse=True)
        vals = torch.zeros((ids.numel(), dz.shape[1]), dtype=torch.float64, device=dev)
        vals.index_add_(0, inv, dz.double())
        return cls(ids, vals)

    def _merge(self, ids: torch.Tensor, vals: torch.Tensor) -> None:
        if self.ids is None:
            self.ids, self.vals = ids, vals
            return
        cat = torch.cat([self.ids, ids])
        u, inv = torch.unique(cat, sorted=True, return_inverse=True)
        out = torch.zeros((u.numel(), vals.shape[1]), dtype=torch.float64, device=vals.device)
        out.index_add_(0, inv, torch.cat([self.vals, vals]))
        self.ids, self.vals = u, out

    def add_row(self, state: int, vec) -> None:
        dev = self.vals.device if self.vals is not None else _device()
        v = torch.as_tensor(np.asarray(vec, np.float64), device=dev).reshape(1, -1)
        self._merge(torch.tensor([int(state)], device=dev), v)

    def axpy(self, coef: float, other: "SparseGrad") -> None:
        if other.ids is not None:
            self._merge(other.ids, coef * other.vals)

    def scaled(self, coef: float) -> "SparseGrad":
        return SparseGrad(self.ids, None if self.vals is None else coef * self.vals)

    @property
    def rows(self) -> Dict[int, np.ndarray]:
        if self.ids is None:
            return {}
        return dict(zip(self.ids.cpu().tolist(), self.vals.cpu().numpy()))

    def to_dense(self, shape: Tuple[int, int]) -> np.ndarray:
        dense = np.zeros(shape)
        if self.ids is not None:
            dense[self.ids.cpu().numpy()] += self.vals.cpu().numpy()
        return dense

    def is_finite(self) -> bool:
        return self.vals is None or bool(torch.isfinite(self.vals).all())

    def max_abs(self) -> float:
        return 0.0 if self.vals is None or self.vals.numel() == 0 else \
            float(self.vals.abs().max())


@dataclass
class LossReport:
    """algorithms.py:59-69."""

    loss: float
    gradient: SparseGrad
    metrics: Dict[str, float] = field(default_factory=dict)

    def __post_init__(self) -> None:
        if not math.isfinite(self.loss):
            raise AlgorithmError(f"loss must be finite, got {self.loss}")
        if not self.gradient.is_finite():
            raise AlgorithmError("gradient must be finite")


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the RFT loss runs only on CUDA devices (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _table(params, dev) -> torch.Tensor:
    return torch.as_tensor(np.asarray(params.logits, dtype=np.float32), device=dev).contiguous()


def _check_vocab(h: HostGroups, target: np.ndarray, V: int) -> None:
    """policy._check_generated_tokens (policy.py:175-178)."""
    if target.size and (target.min() < 0 or target.max() >= V):
        bad = int(target[(target < 0) | (target >= V)][0])
        raise PolicyError(f"token {bad} outside vocabulary of size {V}")


def _seq_logprob(table: torch.Tensor, states: np.ndarray, target: np.ndarray,
                 seq_lengths: np.ndarray) -> np.ndarray:
    """experience_logprob for every sequence under a table (algorithms.py:81-85)."""
    dev = table.device
    b = pack_arrays(table, target, seq_lengths, [len(seq_lengths)], np.zeros(len(seq_lengths)),
                    row_index=states)
    _, _, _, seq_lp = logprob_fwd(b)
    return seq_lp.double().cpu().numpy()


def _run(groups, params, cfg: RFTLossConfig, *, anchor=None, seq_ref_override=None,
         seq_kind=None, metrics_override=None, table=None, anchor_table=None, keep_rows=False):
    dev = _device()
    h = flatten_groups(groups)
    S, V = int(params.num_buckets), int(params.vocab.size)
    states, target = scored_states(h, S)
    _check_vocab(h, target, V)
    if table is None:
        table = _table(params, dev)
    seq_ref = h.seq_ref_lp if seq_ref_override is None else seq_ref_override
    anchor_rows = None
    if anchor is not None:
        if tuple(np.shape(anchor.logits)) != tuple(np.shape(params.logits)):
            raise AlgorithmError(f"parameter shapes differ: {np.shape(params.logits)} vs "
                                 f"{np.shape(anchor.logits)}")
        if anchor_table is None:
            anchor_table = _table(anchor, dev)
        anchor_rows = anchor_table[torch.as_tensor(states, device=dev)].contiguous()
    batch = pack_arrays(table, target, h.seq_lengths, h.group_sizes, h.reward, old_lp=h.old_lp,
                        seq_ref_lp=seq_ref, seq_kind=seq_kind, anchor_logits=anchor_rows,
                        row_index=states)
    out = RFTLoss(cfg)(batch, dlogits="new")
    st = out.stats_dict()
    if st["invalid"] > 0:
        raise AlgorithmError("invalid group shape for this loss")
    grad = SparseGrad.from_token_rows(out.dlogits, states)
    m = stats_to_metrics(st, check=False)
    metrics = {k: m[k] for k in ("mean_reward", "baseline", "kl_estimate", "group_size")}
    if metrics_override:
        metrics.update(metrics_override(st))
    report = LossReport(loss=float(st["loss"]), gradient=grad, metrics=metrics)
    if keep_rows:
        return report, out.dlogits, states
    return report


def group_losses(groups: Sequence, params, config: AlgorithmConfig,
                 sft_params=None, ref_params=None) -> LossReport:
    """``combine_reports([group_loss(g, ...) for g in groups])`` in one kernel
    pipeline (orchestrator.py:299-304)."""
    if config.variant not in (Variant.OPMD_KIMI, Variant.OPMD_PAIRWISE, Variant.OPMD_SIMPLE):
        raise AlgorithmError(f"{config.variant.value} is not a group-based loss")
    if not groups:
        raise AlgorithmError("cannot combine an empty report list")
    cfg = RFTLossConfig.from_variant(config.variant, config.tau, config.beta, config.dpo_beta)
    anchor = None
    if config.variant == Variant.OPMD_SIMPLE:
        if config.beta > 0 and sft_params is None:
            raise AlgorithmError("beta > 0 requires sft_params")
        anchor = sft_params if config.beta > 0 else None
    if config.variant == Variant.OPMD_PAIRWISE and any(len(g.experiences) < 2 for g in groups):
        raise AlgorithmError("pairwise loss needs a group of at least 2 rollouts")
    seq_ref = None
    if config.variant == Variant.OPMD_KIMI and ref_params is not None:
        h = flatten_groups(groups)
        st, tg = scored_states(h, int(ref_params.num_buckets))
        seq_ref = _seq_logprob(_table(ref_params, _device()), st, tg, h.seq_lengths)
    return _run(groups, params, cfg, anchor=anchor, seq_ref_override=seq_ref)


def group_loss(group, params, config: AlgorithmConfig, sft_params=None,
               ref_params=None) -> LossReport:
    """algorithms.py:351-365."""
    return group_losses([group], params, config, sft_params=sft_params, ref_params=ref_params)


# ---- the per-variant entry points and helpers of algorithms.py ----------------

def loss_opmd_kimi(group, params, config: AlgorithmConfig, ref_params=None) -> LossReport:
    """algorithms.py:118-153 (ref_logprobs from the group unless ref_params)."""
    if config.tau <= 0:
        raise AlgorithmError("OPMD_KIMI requires tau > 0")
    if ref_params is None and getattr(group, "ref_logprobs", None) is None:
        raise AlgorithmError("OPMD_KIMI requires ref_logprobs")
    return group_losses([group], params, _as_variant(config, Variant.OPMD_KIMI),
                        ref_params=ref_params)


def loss_opmd_pairwise(group, params, config: AlgorithmConfig) -> LossReport:
    """algorithms.py:156-190."""
    return group_losses([group], params, _as_variant(config, Variant.OPMD_PAIRWISE))


def loss_opmd_simple(group, params, config: AlgorithmConfig, sft_params=None) -> LossReport:
    """algorithms.py:220-253 (plus beta * regularizer_g with an anchor table)."""
    return group_losses([group], params, _as_variant(config, Variant.OPMD_SIMPLE),
                        sft_params=sft_params)


def _as_variant(config: AlgorithmConfig, variant: Variant) -> AlgorithmConfig:
    return AlgorithmConfig(variant, tau=config.tau, beta=config.beta, dpo_beta=config.dpo_beta,
                           learning_rate=config.learning_rate)


def tau_log_zhat(rewards: Sequence[float], tau: float) -> float:
    """algorithms.py:93-101 (host helper; the kernels compute it per group)."""
    if tau <= 0:
        raise AlgorithmError(f"tau must be > 0, got {tau}")
    if not rewards:
        raise AlgorithmError("rewards must be nonempty")
    m = max(rewards)
    mean_exp = sum(math.exp((r - m) / tau) for r in rewards) / len(rewards)
    return m + tau * math.log(mean_exp)


def experience_logprob(params, exp) -> float:
    """algorithms.py:81-85: total logprob of a stored experience under params
    (tg_logprob_fwd over the table rows it scores)."""
    dev = _device()
    h = flatten_groups([_OneGroup([exp if exp.reward is not None else _with_reward(exp)])])
    S, V = int(params.num_buckets), int(params.vocab.size)
    states, target = scored_states(h, S)
    _check_vocab(h, target, V)
    if target.size == 0:
        return 0.0
    return float(_seq_logprob(_table(params, dev), states, target, h.seq_lengths)[0])


def experience_grad(params, exp) -> SparseGrad:
    """algorithms.py:88-90: d logprob / d table rows (e_y - p per scored token)
    -- the negated gradient of SFT's loss over the single experience."""
    rep = loss_sft([exp], params)
    return rep.gradient.scaled(-1.0)


def regularizer_g(params, sft_params, group) -> Tuple[float, SparseGrad]:
    """algorithms.py:193-217: the anchor KL term alone -- OPMD_SIMPLE with
    beta = 1 over the group with its rewards zeroed (the centred policy term
    then vanishes identically)."""
    if tuple(np.shape(params.logits)) != tuple(np.shape(sft_params.logits)):
        raise AlgorithmError(f"parameter shapes differ: {np.shape(params.logits)} vs "
                             f"{np.shape(sft_params.logits)}")
    zeroed = _OneGroup([_with_reward(e) for e in group.experiences],
                       getattr(group, "ref_logprobs", None))
    cfg = RFTLossConfig.from_variant(Variant.OPMD_SIMPLE, 0.0, 1.0)
    rep = _run([zeroed], params, cfg, anchor=sft_params)
    return rep.loss, rep.gradient


class _OneGroup:
    def __init__(self, exps, ref=None):
        self.experiences = list(exps)
        self.ref_logprobs = ref


def loss_sft(batch: Sequence, params) -> LossReport:
    """algorithms.py:256-274: mean over sequences of -sum_t lp."""
    return _sft(batch, params)


def _sft(batch, params, table=None, keep_rows=False):
    if not batch:
        raise AlgorithmError("SFT batch must be nonempty")
    cfg = RFTLossConfig.from_variant(Variant.SFT)
    n = len(batch)
    rewards = [e.reward for e in batch if e.reward is not None]

    def metrics(st):
        return {"mean_reward": float(np.mean(rewards)) if rewards else 0.0, "baseline": 0.0,
                "kl_estimate": 0.0, "group_size": float(n)}

    exps = [e if e.reward is not None else _with_reward(e) for e in batch]
    return _run([_OneGroup(exps)], params, cfg, metrics_override=metrics, table=table,
                keep_rows=keep_rows)


def _with_reward(e):
    class _E:
        pass
    x = _E()
    x.tokens, x.prompt_length, x.action_mask, x.logprobs = (e.tokens, e.prompt_length,
                                                            e.action_mask, e.logprobs)
    x.reward = 0.0
    return x


def loss_dpo(pairs: Sequence[Tuple], params, ref, dpo_beta: float) -> LossReport:
    """algorithms.py:277-315."""
    return _dpo(pairs, params, ref, dpo_beta)


def _dpo(pairs, params, ref, dpo_beta, table=None, ref_table=None, keep_rows=False):
    if not pairs:
        raise AlgorithmError("DPO batch must be nonempty")
    if dpo_beta <= 0:
        raise AlgorithmError(f"dpo_beta must be > 0, got {dpo_beta}")
    for c, r in pairs:
        if list(c.tokens[: c.prompt_length]) != list(r.tokens[: r.prompt_length]):
            raise AlgorithmError("chosen and rejected must share a prompt")
    groups = [_OneGroup([c if c.reward is not None else _with_reward(c),
                         r if r.reward is not None else _with_reward(r)]) for c, r in pairs]
    h = flatten_groups(groups)
    st, tg = scored_states(h, int(ref.num_buckets))
    seq_ref = _seq_logprob(ref_table if ref_table is not None else _table(ref, _device()), st, tg,
                           h.seq_lengths)
    cfg = RFTLossConfig.from_variant(Variant.DPO, dpo_beta=dpo_beta)
    n = len(pairs)

    def metrics(s):
        return {"mean_reward": s["sum_dpo_margin"] / n, "baseline": 0.0, "kl_estimate": 0.0,
                "group_size": float(n)}

    return _run(groups, params, cfg, seq_ref_override=seq_ref, metrics_override=metrics,
                table=table, keep_rows=keep_rows)


def combine_reports(reports: Sequence[LossReport]) -> LossReport:
    """algorithms.py:368-379: losses summed, gradients merged on the device
    (SparseGrad), metrics averaged over the reports."""
    if not reports:
        raise AlgorithmError("cannot combine an empty report list")
    grad = SparseGrad()
    for rep in reports:
        grad.axpy(1.0, rep.gradient)
    metrics = {k: float(np.mean([r.metrics[k] for r in reports])) for k in reports[0].metrics}
    return LossReport(loss=float(sum(r.loss for r in reports)), gradient=grad, metrics=metrics)


def apply_update(params, gradient: SparseGrad, learning_rate: float):
    """algorithms.py:329-348: SGD step returning new params with version + 1,
    computed by tg_apply_update on an fp32 device copy of the table (refuses
    a non-finite gradient or a row outside the table, before any write)."""
    dev = _device()
    table = _table(params, dev)
    if gradient.ids is not None and gradient.ids.numel():
        apply_update_rows(table, gradient.vals.float(), gradient.ids.cpu().numpy(),
                          learning_rate)
    return type(params)(logits=table.double().cpu().numpy(), version=params.version + 1,
                        vocab=params.vocab, num_buckets=params.num_buckets)


def apply_update_rows(table: torch.Tensor, dlogits: torch.Tensor, states: np.ndarray,
                      learning_rate: float) -> None:
    """algorithms.apply_update (algorithms.py:329-348) on the device, straight
    from the loss kernels' per-token gradient rows: ``table[s] -= lr * sum of
    the dlogits rows scored by state s`` (``tg_apply_update``; per-state f64
    sums in row order).  ``table`` is the fp32 [S, V] device table, updated in
    place.  Raises AlgorithmError like the reference -- non-finite gradient,
    state outside the table -- and then the table is unchanged."""
    from . import _native as N

    states = np.asarray(states, dtype=np.int64)
    dev = table.device
    if table.dtype != torch.float32 or table.dim() != 2 or table.stride(1) != 1:
        raise ValueError("table must be a 2-D fp32 tensor with unit column stride")
    if dlogits.dim() != 2 or dlogits.shape[0] != states.size or dlogits.stride(1) != 1:
        raise ValueError("dlogits must hold one row per state entry")
    order = np.argsort(states, kind="stable")  # rows grouped by state, row order kept
    uniq, starts = np.unique(states[order], return_index=True)
    offsets = np.append(starts, states.size).astype(np.int64)
    i64 = dict(dtype=torch.int64, device=dev)
    ids_d = torch.as_tensor(uniq, **i64)
    off_d = torch.as_tensor(offsets, **i64)
    ord_d = torch.as_tensor(order.astype(np.int64), **i64)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    dtype = N.TG_DTYPE_BF16 if dlogits.dtype == torch.bfloat16 else N.TG_DTYPE_F32
    L = N.lib()
    with torch.cuda.device(dev):
        N.check(L.tg_apply_update(table.data_ptr(), table.stride(0), table.shape[0],
                                  table.shape[1], dlogits.data_ptr(), dtype, dlogits.stride(0),
                                  ids_d.data_ptr(), off_d.data_ptr(), ord_d.data_ptr(),
                                  uniq.size, states.size, float(learning_rate),
                                  status.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
    code = int(status.item())
    if code & 2:
        bad = int(uniq[(uniq < 0) | (uniq >= table.shape[0])][0])
        raise AlgorithmError(f"gradient row {bad} outside the logits table")
    if code & 1:
        raise AlgorithmError("refusing to apply a non-finite gradient")


class Trainer:
    """orchestrator.Trainer (orchestrator.py:288-322) on the CUDA path with the
    policy table resident on the GPU: the loss kernels read it in place
    (row_index) and the SGD step runs on the device from the per-token
    gradient rows (tg_apply_update), so only the LossReport crosses PCIe.  The
    anchor / reference snapshot (orchestrator.py:292-296) is frozen on the
    device too.  ``params`` materialises the host table when read (version
    counted like apply_update, algorithms.py:343-348)."""

    def __init__(self, params, algo: AlgorithmConfig) -> None:
        dev = _device()
        self._host = params
        self.algo = algo
        self.anchor = params
        self.table = _table(params, dev)
        self.anchor_table = self.table.clone()
        self.version = int(getattr(params, "version", 0))

    @property
    def params(self):
        p = self._host
        return type(p)(logits=self.table.double().cpu().numpy(), version=self.version,
                       vocab=p.vocab, num_buckets=p.num_buckets)

    def _apply(self, dz: torch.Tensor, states: np.ndarray) -> None:
        apply_update_rows(self.table, dz, states, self.algo.learning_rate)
        self.version += 1

    def step_groups(self, groups) -> LossReport:
        config = self.algo
        if config.variant not in (Variant.OPMD_KIMI, Variant.OPMD_PAIRWISE, Variant.OPMD_SIMPLE):
            raise AlgorithmError(f"{config.variant.value} is not a group-based loss")
        if not groups:
            raise AlgorithmError("cannot combine an empty report list")
        if config.variant == Variant.OPMD_PAIRWISE and any(len(g.experiences) < 2 for g in groups):
            raise AlgorithmError("pairwise loss needs a group of at least 2 rollouts")
        cfg = RFTLossConfig.from_variant(config.variant, config.tau, config.beta, config.dpo_beta)
        anchor = self.anchor if (config.variant == Variant.OPMD_SIMPLE and config.beta > 0) else None
        report, dz, states = _run(groups, self._host, cfg, anchor=anchor, table=self.table,
                                  anchor_table=self.anchor_table, keep_rows=True)
        self._apply(dz, states)
        return report

    def step_sft(self, batch) -> LossReport:
        report, dz, states = _sft(batch, self._host, table=self.table, keep_rows=True)
        self._apply(dz, states)
        return report

    def step_dpo(self, pairs) -> LossReport:
        report, dz, states = _dpo(pairs, self._host, self.anchor, self.algo.dpo_beta,
                                  table=self.table, ref_table=self.anchor_table, keep_rows=True)
        self._apply(dz, states)
        return report


DeviceTrainer = Trainer  # round-1 name
