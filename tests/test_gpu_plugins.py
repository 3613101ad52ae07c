"""Python-registered loss components (registry.register_advantage_fn /
register_policy_loss_fn, the reference's register_reward_fn idiom,
workflows.py:188-197) through the CUDA path, against the oracle.

* a torch restatement of PPO clip registered as a policy loss must give the
  built-in ppo_clip's loss and dlogits (TG_PG_GIVEN route vs the fused
  built-in), and the oracle's loss / dlogits for the per-row (l_t, -dl/dlp)
  it was handed;
* a registered advantage function (group-median baseline) must match the
  oracle with those advantages given.
Tolerances as in test_gpu_parity.py."""

import numpy as np
import pytest
import torch

from _cases import make_case, oracle_cfg
from oracle import rft_oracle as O
from paper_2505_17826_b200 import AlgorithmError, RFTLoss, RFTLossConfig
from paper_2505_17826_b200.registry import (ADVANTAGE_FNS, POLICY_LOSS_FNS,
                                            register_advantage_fn, register_policy_loss_fn,
                                            unregister)

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from test_gpu_parity import compare  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def components():
    @register_policy_loss_fn("ppo_torch")
    def ppo_torch(x):
        """PPO clip in torch (the built-in ppo_clip, restated)."""
        c = x.config
        ratio = torch.exp(torch.clamp(x.lp - x.old_lp, -20.0, 20.0))
        l1 = -x.advantage * ratio
        l2 = -x.advantage * torch.clamp(ratio, 1.0 - c.clip_lo, 1.0 + c.clip_hi)
        return torch.maximum(l1, l2)

    @register_policy_loss_fn("gspo_like")
    def gspo_like(x):
        """A loss the kernels do not have: -A tanh(lp - old) (row-separable)."""
        return -x.advantage * torch.tanh(x.lp - x.old_lp)

    @register_advantage_fn("median_baseline")
    def median_baseline(x):
        """A_i = r_i - median of the group's rewards (equal group sizes)."""
        k = x.reward.numel() // x.n_groups
        r = x.reward.view(x.n_groups, k)
        return (r - r.median(dim=1, keepdim=True).values).reshape(-1)

    yield
    unregister(POLICY_LOSS_FNS, "ppo_torch")
    unregister(POLICY_LOSS_FNS, "gspo_like")
    unregister(ADVANTAGE_FNS, "median_baseline")


BASE = dict(advantage_fn="grpo", kl_fn="low_var_kl", kl_coef=0.01, entropy_loss_fn="default",
            entropy_coef=0.005, loss_agg_mode="token-mean", clip_lo=0.2, clip_hi=0.28)


@pytest.mark.parametrize("V,dtype", [(1000, torch.float32), (32000, torch.bfloat16),
                                     (151936, torch.bfloat16)])
def test_registered_ppo_equals_builtin_and_oracle(V, dtype):
    lens = [13, 9, 21, 7] if V == 151936 else [17, 33, 5, 12, 20, 9]
    gs = [2, 2] if V == 151936 else [3, 3]
    batch, packed = make_case(31, V, lens, gs, dtype=dtype)
    builtin = RFTLoss(RFTLossConfig(policy_loss_fn="ppo_clip", **BASE))
    custom = RFTLoss(RFTLossConfig(policy_loss_fn="ppo_torch", **BASE))
    assert custom.route(packed) == 1   # the fused kernel writes dlogits once
    a = builtin(packed, dlogits="new")
    b = custom(packed, dlogits="new")
    sa, sb = a.stats_dict(), b.stats_dict()
    for k in ("loss", "pg_loss", "kl_loss", "entropy_loss"):
        assert sb[k] == pytest.approx(sa[k], rel=1e-4, abs=1e-6), k
    da, db = a.dlogits.float(), b.dlogits.float()
    assert float((da - db).abs().max()) <= 2.0 ** -8 * float(da.abs().max())
    # the oracle, given the per-row loss / coefficient the plugin produced
    given = custom._plugins(packed, torch.cuda.current_stream(), {})
    batch.pg_coef = given.pg_coef.double().cpu().numpy()
    batch.pg_loss = given.pg_loss.double().cpu().numpy()
    ocfg = oracle_cfg(custom.cfg.with_(policy_loss_fn="ppo_clip"))
    ocfg.policy_loss_fn = "given"
    ref = O.general_loss(batch, ocfg)
    compare(b, ref, dtype)


def test_registered_policy_loss_the_kernels_do_not_have():
    batch, packed = make_case(32, 32000, [17, 33, 5, 12], [2, 2], dtype=torch.bfloat16)
    loss = RFTLoss(RFTLossConfig(policy_loss_fn="gspo_like", **BASE))
    out = loss(packed, dlogits="new")
    given = loss._plugins(packed, torch.cuda.current_stream(), {})
    # d/dlp of -A tanh(lp - old) = -A (1 - tanh^2): the coefficient handed over
    lp = out.lp.double()
    adv = out.seq_adv.double().repeat_interleave(torch.as_tensor([17, 33, 5, 12], device="cuda"))
    want = adv * (1 - torch.tanh(lp - packed.old_lp.double()) ** 2)
    assert torch.allclose(given.pg_coef.double(), want, rtol=1e-4, atol=1e-6)
    batch.pg_coef = given.pg_coef.double().cpu().numpy()
    batch.pg_loss = given.pg_loss.double().cpu().numpy()
    ocfg = oracle_cfg(RFTLossConfig(policy_loss_fn="vanilla", **BASE))
    ocfg.policy_loss_fn = "given"
    ref = O.general_loss(batch, ocfg)
    compare(out, ref, torch.bfloat16)


def test_registered_advantage_fn_matches_oracle():
    batch, packed = make_case(33, 1000, [17, 33, 5, 12, 20, 9], [3, 3], dtype=torch.float32)
    cfg = RFTLossConfig(advantage_fn="median_baseline", policy_loss_fn="ppo_clip",
                        loss_agg_mode="token-mean")
    out = RFTLoss(cfg)(packed, dlogits="new")
    r = batch.reward.reshape(2, 3)
    adv = (r - np.median(r, axis=1, keepdims=True)).reshape(-1)
    np.testing.assert_allclose(out.seq_adv.double().cpu().numpy(), adv, rtol=1e-6, atol=1e-7)
    batch.advantage = adv
    compare(out, O.general_loss(batch, oracle_cfg(cfg.with_(advantage_fn="given"))),
            torch.float32)


def test_registered_component_errors():
    @register_policy_loss_fn("bad_shape")
    def bad_shape(x):
        return x.lp.sum()

    try:
        _, packed = make_case(34, 64, [5, 7], [2])
        with pytest.raises(AlgorithmError, match="one loss per row"):
            RFTLoss(RFTLossConfig(policy_loss_fn="bad_shape"))(packed)
    finally:
        unregister(POLICY_LOSS_FNS, "bad_shape")
