"""Loss-component registries: advantage_fn, policy_loss_fn, kl_fn,
entropy_loss_fn and loss_agg_mode.

Same idiom as the reference's string registries (``REWARD_FNS`` /
``register_reward_fn``, workflows.py:188-197; ``WORKFLOWS``, 241-246): a
module-level dict filled by a decorator.  Each entry names one branch of the
fused CUDA epilogue (``csrc/tg_rowcoef.cuh``, ``csrc/tg_group.cu``) by its
TG_* code and documents its math; there is no Python compute behind it.

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
from typing import Callable, Dict, Tuple

from . import _native as N


@dataclass(frozen=True)
class Component:
    name: str
    code: int
    doc: str
    aliases: Tuple[str, ...] = field(default_factory=tuple)


ADVANTAGE_FNS: Dict[str, Component] = {}
POLICY_LOSS_FNS: Dict[str, Component] = {}
KL_FNS: Dict[str, Component] = {}
ENTROPY_LOSS_FNS: Dict[str, Component] = {}
LOSS_AGG_MODES: Dict[str, Component] = {}


def _register(table: Dict[str, Component], name: str, code: int, aliases=()) -> Callable:
    def deco(fn):
        comp = Component(name, code, (fn.__doc__ or "").strip(), tuple(aliases))
        table[name] = comp
        for a in aliases:
            table[a] = comp
        return fn

    return deco


def register_advantage_fn(name, code, aliases=()):
    return _register(ADVANTAGE_FNS, name, code, aliases)


def register_policy_loss_fn(name, code, aliases=()):
    return _register(POLICY_LOSS_FNS, name, code, aliases)


def register_kl_fn(name, code, aliases=()):
    return _register(KL_FNS, name, code, aliases)


def register_entropy_loss_fn(name, code, aliases=()):
    return _register(ENTROPY_LOSS_FNS, name, code, aliases)


def register_loss_agg_mode(name, code, aliases=()):
    return _register(LOSS_AGG_MODES, name, code, aliases)


# ---- advantage_fn ------------------------------------------------------------

@register_advantage_fn("grpo", N.TG_ADV_GRPO)
def _grpo():
    """A_i = (r_i - mean_g r) / (std_g r + std_eps), unbiased std; a group of one gets 0."""


@register_advantage_fn("rloo", N.TG_ADV_RLOO)
def _rloo():
    """A_i = r_i - mean_{j != i} r_j (leave-one-out baseline); a group of one gets 0."""


@register_advantage_fn("opmd", N.TG_ADV_OPMD, aliases=("opmd_simple", "mean_baseline"))
def _opmd():
    """A_i = (r_i - mean_g r) / (1 + tau) -- OPMD_SIMPLE, algorithms.py:234-242."""


@register_advantage_fn("reinforce", N.TG_ADV_REINFORCE)
def _reinforce():
    """A_i = r_i (no baseline)."""


@register_advantage_fn("given", N.TG_ADV_GIVEN, aliases=("precomputed",))
def _given():
    """A_i supplied by the caller per sequence (batch.advantage)."""


# ---- policy_loss_fn ----------------------------------------------------------

@register_policy_loss_fn("vanilla", N.TG_PG_VANILLA, aliases=("pg", "opmd_simple"))
def _vanilla():
    """loss_t = -A_i lp_t; d/d lp = -A_i.  With agg 'seq-sum' this is OPMD_SIMPLE."""


@register_policy_loss_fn("ppo_clip", N.TG_PG_PPO_CLIP, aliases=("ppo", "grpo"))
def _ppo():
    """rho = exp(lp - old_lp); loss_t = max(-A rho, -A clip(rho, 1-clip_lo, 1+clip_hi)),
    optionally dual-clipped at -A*clip_c for A < 0; zero gradient on clipped tokens."""


@register_policy_loss_fn("sft", N.TG_PG_SFT, aliases=("nll",))
def _sft():
    """loss_t = -lp_t (loss_sft, algorithms.py:256-274 with agg 'seq-mean-token-sum')."""


@register_policy_loss_fn("opmd_kimi", N.TG_PG_OPMD_KIMI, aliases=("kimi",))
def _kimi():
    """sum_i (r_i - tau log Zhat - tau (LP_i - ref_i))^2 per group (algorithms.py:118-153)."""


@register_policy_loss_fn("opmd_pairwise", N.TG_PG_OPMD_PAIRWISE, aliases=("pairwise",))
def _pairwise():
    """sum_{i<j} (a_i - a_j)^2, a_i = r_i - tau (LP_i - ref_i) (algorithms.py:156-190)."""


@register_policy_loss_fn("dpo", N.TG_PG_DPO)
def _dpo():
    """mean over (chosen, rejected) groups of softplus(-beta margin) (algorithms.py:277-315)."""


# ---- kl_fn --------------------------------------------------------------------

@register_kl_fn("none", N.TG_KL_NONE)
def _kl_none():
    """No token KL penalty."""


@register_kl_fn("k1", N.TG_KL_K1)
def _k1():
    """kl = lp - ref_lp."""


@register_kl_fn("k2", N.TG_KL_K2, aliases=("mse",))
def _k2():
    """kl = (lp - ref_lp)^2 / 2."""


@register_kl_fn("k3", N.TG_KL_K3, aliases=("low_var_kl",))
def _k3():
    """kl = clamp(e^d - d - 1, -10, 10), d = clamp(ref_lp - lp, -20, 20)."""


@register_kl_fn("abs", N.TG_KL_ABS)
def _kl_abs():
    """kl = |lp - ref_lp|."""


# ---- entropy_loss_fn ----------------------------------------------------------

@register_entropy_loss_fn("none", N.TG_ENT_NONE)
def _ent_none():
    """No entropy bonus."""


@register_entropy_loss_fn("default", N.TG_ENT_DEFAULT, aliases=("entropy",))
def _ent_default():
    """loss -= entropy_coef * agg(H_t), H_t = lse_t - sum_v p_tv z_tv (full-vocab entropy)."""


# ---- loss_agg_mode -------------------------------------------------------------

@register_loss_agg_mode("seq-sum", N.TG_AGG_SEQ_SUM, aliases=("seq_sum", "sum"))
def _seq_sum():
    """w = 1: tokens summed per sequence, sequences and groups summed (the reference)."""


@register_loss_agg_mode("token-mean", N.TG_AGG_TOKEN_MEAN, aliases=("token_mean",))
def _token_mean():
    """w = 1 / N_tok over all RL tokens of the global batch (masked token mean)."""


@register_loss_agg_mode("seq-mean-token-sum", N.TG_AGG_SEQ_MEAN_TOKEN_SUM)
def _smts():
    """w = 1 / B: token sums averaged over sequences."""


@register_loss_agg_mode("seq-mean-token-mean", N.TG_AGG_SEQ_MEAN_TOKEN_MEAN)
def _smtm():
    """w = 1 / (B n_i): token means averaged over sequences."""


@register_loss_agg_mode("seq-mean-token-sum-norm", N.TG_AGG_SEQ_MEAN_TOKEN_SUM_NORM)
def _smtsn():
    """w = 1 / agg_norm (token sums over a fixed normaliser, e.g. max response length)."""


def lookup(table: Dict[str, Component], name: str, kind: str) -> Component:
    try:
        return table[name]
    except KeyError:
        raise KeyError(f"{kind} {name!r} is not registered; known: "
                       f"{sorted({c.name for c in table.values()})}") from None
