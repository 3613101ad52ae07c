"""Loss configuration: registry names + scalars, validated like the reference's
AlgorithmConfig (algorithms.py:36-56) and lowered to the C ABI's TgConfig."""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, replace
from typing import Optional

from . import _native as N
from .registry import (ADVANTAGE_FNS, ENTROPY_LOSS_FNS, KL_FNS, LOSS_AGG_MODES,
                       POLICY_LOSS_FNS, lookup)


class AlgorithmError(ValueError):
    """Invalid algorithm configuration or loss input (algorithms.py:24-25)."""


class Variant(str, enum.Enum):
    """The reference's loss variants (algorithms.py:28-33)."""

    OPMD_KIMI = "OPMD_KIMI"
    OPMD_PAIRWISE = "OPMD_PAIRWISE"
    OPMD_SIMPLE = "OPMD_SIMPLE"
    SFT = "SFT"
    DPO = "DPO"


COUPLED = ("opmd_kimi", "opmd_pairwise", "dpo")


@dataclass
class RFTLossConfig:
    advantage_fn: str = "grpo"
    policy_loss_fn: str = "ppo_clip"
    kl_fn: str = "none"
    entropy_loss_fn: str = "none"
    loss_agg_mode: Optional[str] = None   # None: "seq-sum" for coupled losses, else "token-mean"
    tau: float = 0.0
    clip_lo: float = 0.2
    clip_hi: float = 0.2
    clip_c: float = 0.0
    kl_coef: float = 0.0
    entropy_coef: float = 0.0
    std_eps: float = 1e-6
    sft_weight: float = 1.0
    anchor_beta: float = 0.0
    dpo_beta: float = 0.1
    agg_norm: float = 1.0
    force_two_pass: bool = False

    def __post_init__(self) -> None:
        # registry names resolve (aliases allowed) -- canonicalise
        self.advantage_fn = lookup(ADVANTAGE_FNS, self.advantage_fn, "advantage_fn").name
        self.policy_loss_fn = lookup(POLICY_LOSS_FNS, self.policy_loss_fn, "policy_loss_fn").name
        self.kl_fn = lookup(KL_FNS, self.kl_fn, "kl_fn").name
        self.entropy_loss_fn = lookup(ENTROPY_LOSS_FNS, self.entropy_loss_fn,
                                      "entropy_loss_fn").name
        if self.loss_agg_mode is None:
            self.loss_agg_mode = "seq-sum" if self.policy_loss_fn in COUPLED else "token-mean"
        self.loss_agg_mode = lookup(LOSS_AGG_MODES, self.loss_agg_mode, "loss_agg_mode").name
        # scalar rules (algorithms.py:47-56 and the north_star pieces)
        if not self.tau >= 0:
            raise AlgorithmError(f"tau must be >= 0, got {self.tau}")
        if self.policy_loss_fn in ("opmd_kimi", "opmd_pairwise") and not self.tau > 0:
            name = "OPMD_KIMI" if self.policy_loss_fn == "opmd_kimi" else "OPMD_PAIRWISE"
            raise AlgorithmError(f"{name} requires tau > 0")
        if not self.anchor_beta >= 0:
            raise AlgorithmError(f"beta must be >= 0, got {self.anchor_beta}")
        if not self.dpo_beta > 0:
            raise AlgorithmError(f"dpo_beta must be > 0, got {self.dpo_beta}")
        if not (self.clip_lo >= 0 and self.clip_hi >= 0):
            raise AlgorithmError("clip ranges must be >= 0")
        if self.clip_c != 0 and not self.clip_c > 1:
            raise AlgorithmError("clip_c must be 0 (off) or > 1")
        if not self.std_eps >= 0:
            raise AlgorithmError("std_eps must be >= 0")
        if not self.sft_weight >= 0:
            raise AlgorithmError("sft_weight must be >= 0")
        if self.loss_agg_mode == "seq-mean-token-sum-norm" and not self.agg_norm > 0:
            raise AlgorithmError("agg_norm must be > 0")
        if self.policy_loss_fn in COUPLED:
            # the sequence-coupled losses are whole-sequence objectives (algorithms.py:
            # 118-190, 277-315): a token KL, an entropy bonus or a token aggregation
            # would have no defined gradient there -- refuse instead of dropping them
            if self.kl_fn != "none" and self.kl_coef != 0:
                raise AlgorithmError(f"{self.policy_loss_fn} takes no token KL penalty "
                                     f"(kl_fn={self.kl_fn!r}, kl_coef={self.kl_coef})")
            if self.entropy_loss_fn != "none" and self.entropy_coef != 0:
                raise AlgorithmError(f"{self.policy_loss_fn} takes no entropy bonus")
            if self.loss_agg_mode != "seq-sum":
                raise AlgorithmError(f"{self.policy_loss_fn} sums over groups; loss_agg_mode "
                                     f"{self.loss_agg_mode!r} does not apply")
        for k in ("tau", "clip_lo", "clip_hi", "clip_c", "kl_coef", "entropy_coef", "std_eps",
                  "sft_weight", "anchor_beta", "dpo_beta", "agg_norm"):
            if not math.isfinite(getattr(self, k)):
                raise AlgorithmError(f"{k} must be finite")

    @property
    def coupled(self) -> bool:
        return self.policy_loss_fn in COUPLED

    @property
    def advantage_callable(self):
        """The registered Python advantage function, or None for a built-in."""
        return ADVANTAGE_FNS[self.advantage_fn].fn

    @property
    def policy_loss_callable(self):
        """The registered Python policy loss, or None for a built-in."""
        return POLICY_LOSS_FNS[self.policy_loss_fn].fn

    @classmethod
    def from_variant(cls, variant, tau: float = 1.0, beta: float = 0.0,
                     dpo_beta: float = 0.1) -> "RFTLossConfig":
        """The reference's AlgorithmConfig(variant, tau, beta, dpo_beta) as registry entries."""
        v = Variant(variant)
        if v == Variant.OPMD_SIMPLE:
            return cls(advantage_fn="opmd", policy_loss_fn="vanilla", loss_agg_mode="seq-sum",
                       tau=tau, anchor_beta=beta, dpo_beta=dpo_beta)
        if v == Variant.OPMD_KIMI:
            return cls(policy_loss_fn="opmd_kimi", tau=tau, dpo_beta=dpo_beta)
        if v == Variant.OPMD_PAIRWISE:
            return cls(policy_loss_fn="opmd_pairwise", tau=tau, dpo_beta=dpo_beta)
        if v == Variant.SFT:
            return cls(advantage_fn="given", policy_loss_fn="sft",
                       loss_agg_mode="seq-mean-token-sum", dpo_beta=dpo_beta)
        return cls(policy_loss_fn="dpo", dpo_beta=dpo_beta)

    def with_(self, **kw) -> "RFTLossConfig":
        return replace(self, **kw)

    def to_c(self, n_tok_global: int = 0, n_seq_global: int = 0,
             n_sft_seq_global: int = 0) -> N.TgConfig:
        c = N.TgConfig()
        c.advantage_fn = ADVANTAGE_FNS[self.advantage_fn].code
        c.policy_loss_fn = POLICY_LOSS_FNS[self.policy_loss_fn].code
        c.kl_fn = KL_FNS[self.kl_fn].code
        c.entropy_loss_fn = ENTROPY_LOSS_FNS[self.entropy_loss_fn].code
        c.loss_agg_mode = LOSS_AGG_MODES[self.loss_agg_mode].code
        c.flags = N.TG_FLAG_FORCE_TWO_PASS if self.force_two_pass else 0
        for k in ("tau", "clip_lo", "clip_hi", "clip_c", "kl_coef", "entropy_coef", "std_eps",
                  "sft_weight", "anchor_beta", "dpo_beta", "agg_norm"):
            setattr(c, k, float(getattr(self, k)))
        c.n_tok_global = int(n_tok_global)
        c.n_seq_global = int(n_seq_global)
        c.n_sft_seq_global = int(n_sft_seq_global)
        return c
