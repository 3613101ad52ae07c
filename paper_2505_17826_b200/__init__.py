"""B200-native (sm_100a) RFT trainer loss path of Trinity-RFT (arXiv 2505.17826).

logits -> logprob -> group advantage -> policy loss (+ KL, entropy, anchor KL)
-> dlogits, fused into hand-written CUDA kernels behind the C ABI in
``include/tg_loss.h``; Python registries select the loss components.

    from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, pack_arrays
"""

from .config import AlgorithmError, RFTLossConfig, Variant
from .loss import (LossOutput, RFTLoss, lmhead_dlogits, lmhead_grad_chunk, lmhead_grad_hidden,
                   lmhead_grad_weight,
                   lmhead_logprob_fwd, lmhead_loss_fwd, lmhead_loss_fwd_bwd, logprob_fwd,
                   stats_to_metrics)
from .optim import LMHeadAdamW, adamw_step
from .packing import PackedBatch, PolicyError, group_by_task, pack_arrays
from .registry import (ADVANTAGE_FNS, ENTROPY_LOSS_FNS, KL_FNS, LOSS_AGG_MODES,
                       POLICY_LOSS_FNS)

__all__ = [
    "AlgorithmError", "PolicyError", "RFTLossConfig", "Variant", "RFTLoss", "LossOutput",
    "logprob_fwd", "lmhead_logprob_fwd", "lmhead_loss_fwd", "lmhead_loss_fwd_bwd",
    "lmhead_dlogits", "lmhead_grad_chunk", "lmhead_grad_hidden", "lmhead_grad_weight", "stats_to_metrics", "PackedBatch", "pack_arrays", "group_by_task",
    "adamw_step", "LMHeadAdamW",
    "ADVANTAGE_FNS", "POLICY_LOSS_FNS", "KL_FNS", "ENTROPY_LOSS_FNS", "LOSS_AGG_MODES",
]
