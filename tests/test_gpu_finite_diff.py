"""Finite-difference audit of the CUDA gradients themselves (the reference's
test style: test_algorithms.py:304-389, test_acceptance.py A3 167-253), on the
fp32-logits kernels: for a few (row, column) entries -- each row's target
column, its largest logit, and a random one -- the central difference
(L(z + h e_tv) - L(z - h e_tv)) / 2h of the kernel's own loss must match the
kernel's dlogits[t, v].

Tolerance: |fd - g| <= 2e-5 + 2e-2 |g| with h = 2e-2.  The loss is computed in
fp32 rows + f64 reductions (relative error ~1e-7), so the FD noise is
~1e-7 |L| / h ~ 1e-5; the O(h^2) truncation term of these smooth losses is
below 1e-2 relative at h = 2e-2 (PPO ratios are kept away from the clip
kinks: old_lp = lp + N(0, 0.05^2) inside [0.8, 1.28])."""

import numpy as np
import pytest
import torch

from _cases import make_case
from paper_2505_17826_b200 import RFTLoss, RFTLossConfig

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

CASES = {
    "grpo_ppo_k3_entropy_token_mean": (
        dict(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl", kl_coef=0.05,
             entropy_loss_fn="default", entropy_coef=0.02, loss_agg_mode="token-mean"),
        dict()),
    "rloo_dual_clip_k2_seq_mean_token_mean": (
        dict(advantage_fn="rloo", policy_loss_fn="ppo_clip", clip_c=3.0, kl_fn="k2",
             kl_coef=0.05, loss_agg_mode="seq-mean-token-mean"),
        dict()),
    "opmd_simple_seq_sum": (dict(advantage_fn="opmd", policy_loss_fn="vanilla", tau=0.5,
                                 loss_agg_mode="seq-sum"), dict()),
    "opmd_kimi": (dict(policy_loss_fn="opmd_kimi", tau=0.7), dict()),
    "opmd_pairwise": (dict(policy_loss_fn="opmd_pairwise", tau=0.5), dict()),
    "dpo": (dict(policy_loss_fn="dpo", dpo_beta=0.3), dict(group_sizes=[2, 2])),
    "anchor_kl": (dict(advantage_fn="opmd", policy_loss_fn="vanilla", tau=0.5,
                       loss_agg_mode="seq-sum", anchor_beta=0.2), dict(anchor=True)),
    "mixed_sft": (dict(advantage_fn="grpo", policy_loss_fn="ppo_clip",
                       loss_agg_mode="token-mean", sft_weight=0.7),
                  dict(seq_kind=[0, 0, 1, 1])),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_kernel_gradient_matches_central_differences(name):
    cfg_kw, case_kw = CASES[name]
    group_sizes = case_kw.pop("group_sizes", [2, 2])
    V = 96
    seq_lens = [6, 5, 7, 4]
    _, packed = make_case(17, V, seq_lens, group_sizes, dtype=torch.float32, scale=1.0,
                          **case_kw)
    loss = RFTLoss(RFTLossConfig(**cfg_kw))
    z = packed.logits
    grad = loss(packed, dlogits="new").dlogits.clone()

    def L():
        return loss(packed, dlogits=None).stats_dict()["loss"]

    rng = np.random.default_rng(3)
    T = z.shape[0]
    h = 2e-2
    checked = 0
    worst = 0.0
    for t in rng.choice(T, 8, replace=False):
        cols = {int(packed.target[t]), int(torch.argmax(z[t])), int(rng.integers(0, V))}
        for v in cols:
            z0 = float(z[t, v])
            z[t, v] = z0 + h
            lp = L()
            z[t, v] = z0 - h
            lm = L()
            z[t, v] = z0
            fd = (lp - lm) / (2 * h)
            g = float(grad[t, v])
            worst = max(worst, abs(fd - g) / (2e-5 + 2e-2 * abs(g)))
            assert abs(fd - g) <= 2e-5 + 2e-2 * abs(g), (name, int(t), v, fd, g)
            checked += 1
    print(f"{name}: worst |fd - g| / tol = {worst:.3f}")
    assert checked >= 16
    # the gradient is not trivially zero
    assert float(grad.abs().max()) > 1e-4
