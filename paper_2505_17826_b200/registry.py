"""Loss-component registries: advantage_fn, policy_loss_fn, kl_fn,
entropy_loss_fn and loss_agg_mode.

Same idiom as the reference's string registries (``REWARD_FNS`` /
``register_reward_fn``, workflows.py:188-197; ``WORKFLOWS``, 241-246): a
module-level dict from name to component, filled by a decorator.

Two kinds of entries:

* built-ins -- each names one branch of the fused CUDA epilogue
  (``csrc/tg_rowcoef.cuh``, ``csrc/tg_group.cu``) by its TG_* code; no Python
  runs for them;
* user components registered from Python with ``register_advantage_fn`` /
  ``register_policy_loss_fn``.  They run as torch code on the batch's device
  and feed the kernels through the C ABI's GIVEN routes:

  - an advantage function returns one advantage per sequence
    (``fn(AdvantageInputs) -> Tensor[B]``), passed as ``TgBatch.advantage``
    with ``TG_ADV_GIVEN`` -- the single-pass route is unchanged (4V bytes/row);
  - a policy loss returns one loss per trainable row, differentiable in the
    row's logprob (``fn(PolicyLossInputs) -> Tensor[T]``, row-separable: row
    t's loss may depend on lp_t only).  ``RFTLoss`` evaluates it on the lp of a
    forward pass, takes -d l_t / d lp_t with torch.autograd, and the fused
    kernel (``TG_PG_GIVEN``) writes dlogits once with the registry's token KL,
    entropy bonus, aggregation weights and SFT rows around it: 2V + 4V bytes
    per row instead of 4V.

Reference variants map onto registry combinations (RFTLossConfig.from_variant):

    OPMD_SIMPLE   advantage "opmd"   + policy_loss "vanilla"       + agg "seq-sum"
                  (+ anchor_beta -> regularizer_g)       algorithms.py:220-253
    OPMD_KIMI     policy_loss "opmd_kimi"                algorithms.py:118-153
    OPMD_PAIRWISE policy_loss "opmd_pairwise"            algorithms.py:156-190
    SFT           policy_loss "sft" + agg "seq-mean-token-sum"   :256-274
    DPO           policy_loss "dpo"                      algorithms.py:277-315
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Callable, Dict, Optional, Tuple

from . import _native as N


@dataclass(frozen=True)
class Component:
    name: str
    code: int
    doc: str
    aliases: Tuple[str, ...] = field(default_factory=tuple)
    fn: Optional[Callable] = None   # a Python component (runs through a GIVEN route)

    @property
    def builtin(self) -> bool:
        return self.fn is None


ADVANTAGE_FNS: Dict[str, Component] = {}
POLICY_LOSS_FNS: Dict[str, Component] = {}
KL_FNS: Dict[str, Component] = {}
ENTROPY_LOSS_FNS: Dict[str, Component] = {}
LOSS_AGG_MODES: Dict[str, Component] = {}


def _add(table: Dict[str, Component], comp: Component) -> None:
    for key in (comp.name, *comp.aliases):
        if key in table:
            raise ValueError(f"{key!r} is already registered (as {table[key].name!r})")
    for key in (comp.name, *comp.aliases):
        table[key] = comp


# ---- built-ins: (name, TG code, math, aliases) ----------------------------------

_BUILTINS = (
    (ADVANTAGE_FNS, [
        ("grpo", N.TG_ADV_GRPO,
         "A_i = (r_i - mean_g r) / (std_g r + std_eps), unbiased std; a group of one gets 0.", ()),
        ("rloo", N.TG_ADV_RLOO,
         "A_i = r_i - mean_{j != i} r_j (leave-one-out baseline); a group of one gets 0.", ()),
        ("opmd", N.TG_ADV_OPMD,
         "A_i = (r_i - mean_g r) / (1 + tau) -- OPMD_SIMPLE, algorithms.py:234-242.",
         ("opmd_simple", "mean_baseline")),
        ("reinforce", N.TG_ADV_REINFORCE, "A_i = r_i (no baseline).", ()),
        ("given", N.TG_ADV_GIVEN, "A_i supplied by the caller per sequence (batch.advantage).",
         ("precomputed",)),
    ]),
    (POLICY_LOSS_FNS, [
        ("vanilla", N.TG_PG_VANILLA,
         "loss_t = -A_i lp_t; d/d lp = -A_i.  With agg 'seq-sum' this is OPMD_SIMPLE.",
         ("pg", "opmd_simple")),
        ("ppo_clip", N.TG_PG_PPO_CLIP,
         "rho = exp(clamp(lp - old_lp, -20, 20)); loss_t = max(-A rho, -A clip(rho, 1-clip_lo, "
         "1+clip_hi)), optionally dual-clipped at -A*clip_c for A < 0; zero gradient on clipped "
         "tokens and through a clamped log-ratio.", ("ppo", "grpo")),
        ("sft", N.TG_PG_SFT,
         "loss_t = -lp_t (loss_sft, algorithms.py:256-274 with agg 'seq-mean-token-sum').",
         ("nll",)),
        ("opmd_kimi", N.TG_PG_OPMD_KIMI,
         "sum_i (r_i - tau log Zhat - tau (LP_i - ref_i))^2 per group (algorithms.py:118-153).",
         ("kimi",)),
        ("opmd_pairwise", N.TG_PG_OPMD_PAIRWISE,
         "sum_{i<j} (a_i - a_j)^2, a_i = r_i - tau (LP_i - ref_i) (algorithms.py:156-190).",
         ("pairwise",)),
        ("dpo", N.TG_PG_DPO,
         "mean over (chosen, rejected) groups of softplus(-beta margin) (algorithms.py:277-315).",
         ()),
    ]),
    (KL_FNS, [
        ("none", N.TG_KL_NONE, "No token KL penalty.", ()),
        ("k1", N.TG_KL_K1, "kl = lp - ref_lp.", ()),
        ("k2", N.TG_KL_K2, "kl = (lp - ref_lp)^2 / 2.", ("mse",)),
        ("k3", N.TG_KL_K3, "kl = clamp(e^d - d - 1, -10, 10), d = clamp(ref_lp - lp, -20, 20).",
         ("low_var_kl",)),
        ("abs", N.TG_KL_ABS, "kl = |lp - ref_lp|.", ()),
    ]),
    (ENTROPY_LOSS_FNS, [
        ("none", N.TG_ENT_NONE, "No entropy bonus.", ()),
        ("default", N.TG_ENT_DEFAULT,
         "loss -= entropy_coef * agg(H_t), H_t = lse_t - sum_v p_tv z_tv (full-vocab entropy).",
         ("entropy",)),
    ]),
    (LOSS_AGG_MODES, [
        ("seq-sum", N.TG_AGG_SEQ_SUM,
         "w = 1: tokens summed per sequence, sequences and groups summed (the reference).",
         ("seq_sum", "sum")),
        ("token-mean", N.TG_AGG_TOKEN_MEAN,
         "w = 1 / N_tok over all RL tokens of the global batch (masked token mean).",
         ("token_mean",)),
        ("seq-mean-token-sum", N.TG_AGG_SEQ_MEAN_TOKEN_SUM,
         "w = 1 / B: token sums averaged over sequences.", ()),
        ("seq-mean-token-mean", N.TG_AGG_SEQ_MEAN_TOKEN_MEAN,
         "w = 1 / (B n_i): token means averaged over sequences.", ()),
        ("seq-mean-token-sum-norm", N.TG_AGG_SEQ_MEAN_TOKEN_SUM_NORM,
         "w = 1 / agg_norm (token sums over a fixed normaliser, e.g. max response length).", ()),
    ]),
)
for _table, _entries in _BUILTINS:
    for _name, _code, _doc, _aliases in _entries:
        _add(_table, Component(_name, _code, _doc, tuple(_aliases)))


# ---- user components -------------------------------------------------------------

@dataclass
class AdvantageInputs:
    """What a registered advantage function sees (device tensors of one call)."""

    reward: Any            # [B] float32
    group_index: Any       # [B] int64: the group of each sequence (0 .. G-1, ascending)
    group_offsets: Any     # [G+1] int32 sequence prefix sums
    seq_lengths: Any       # [B] int32 trainable rows per sequence
    is_rl: Any             # [B] bool (False: SFT / expert sequence)
    n_groups: int
    config: Any            # the RFTLossConfig


@dataclass
class PolicyLossInputs:
    """What a registered policy loss sees: one entry per trainable row."""

    lp: Any                # [T] float32, requires_grad: the current policy's logprob
    old_lp: Any            # [T] float32 behaviour logprob (or None)
    ref_lp: Any            # [T] float32 reference logprob (or None)
    advantage: Any         # [T] float32: the row's sequence advantage (advantage_fn)
    entropy: Any           # [T] float32 (detached)
    seq_index: Any         # [T] int64: the row's sequence
    config: Any            # the RFTLossConfig


def register_advantage_fn(name: str, aliases=()) -> Callable:
    """Register ``fn(AdvantageInputs) -> Tensor[B]`` (float, on the batch's
    device) under ``name``.  Runs before the kernels; the values reach them as
    ``TgBatch.advantage`` with ``TG_ADV_GIVEN``.  Names must be new."""

    def deco(fn: Callable) -> Callable:
        _add(ADVANTAGE_FNS, Component(name, N.TG_ADV_GIVEN, (fn.__doc__ or "").strip(),
                                      tuple(aliases), fn))
        return fn

    return deco


def register_policy_loss_fn(name: str, aliases=()) -> Callable:
    """Register ``fn(PolicyLossInputs) -> Tensor[T]``: the per-row policy loss
    l_t (before the aggregation weight), differentiable w.r.t. ``inputs.lp``
    and row-separable.  Lowered to ``TG_PG_GIVEN``: the kernels receive l_t and
    -d l_t / d lp_t per row.  Names must be new."""

    def deco(fn: Callable) -> Callable:
        _add(POLICY_LOSS_FNS, Component(name, N.TG_PG_GIVEN, (fn.__doc__ or "").strip(),
                                        tuple(aliases), fn))
        return fn

    return deco


def unregister(table: Dict[str, Component], name: str) -> None:
    """Remove a user component (and its aliases); built-ins cannot be removed."""
    comp = table[name]
    if comp.builtin:
        raise ValueError(f"{name!r} is a built-in component")
    for key in (comp.name, *comp.aliases):
        table.pop(key, None)


def lookup(table: Dict[str, Component], name: str, kind: str) -> Component:
    try:
        return table[name]
    except KeyError:
        raise KeyError(f"{kind} {name!r} is not registered; known: "
                       f"{sorted({c.name for c in table.values()})}") from None
