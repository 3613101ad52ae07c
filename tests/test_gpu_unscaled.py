"""Sequence-coupled losses in one pass (TG_FLAG_UNSCALED_GRAD, route 4): the
fused kernel writes p - e_y and the per-row scale s_t comes out of the
coupled epilogue, d loss / d z_t = s_t (p_t - e_y) (hard part 3).
Checked against the two-pass coupled route (route 3, itself parity-tested
against the oracle in test_gpu_parity.py) on the same inputs.

Tolerances: statistics rel 1e-5 with an absolute floor of 2e-6 sum|lp|, per-row
lp / lse rel 1e-5 (the two routes sum the row in different orders); s_t * unscaled vs the scaled dlogits: bf16
2^-8 max|dz| + 1e-2 |dz| (two bf16 roundings vs one), fp32 1e-5 max + 1e-3 |dz|
(the coupled coefficient carries the sequence-sum difference)."""

import numpy as np
import pytest
import torch

from _cases import make_case
from paper_2505_17826_b200 import RFTLoss, RFTLossConfig

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

CFGS = {
    "kimi": (dict(policy_loss_fn="opmd_kimi", tau=0.7), [4, 4]),
    "pairwise": (dict(policy_loss_fn="opmd_pairwise", tau=0.5), [4, 4]),
    "dpo": (dict(policy_loss_fn="dpo", dpo_beta=0.3), [2, 2, 2, 2]),
}


@pytest.mark.parametrize("V,dtype", [(32000, torch.bfloat16), (151936, torch.bfloat16),
                                     (151936, torch.float32)], ids=["v32k_bf16", "v152k_bf16",
                                                                    "v152k_f32"])
@pytest.mark.parametrize("name", sorted(CFGS))
def test_unscaled_single_pass_matches_two_pass(name, V, dtype):
    cfg_kw, groups = CFGS[name]
    lens = [23, 17, 31, 9, 40, 12, 25, 19]
    _, batch = make_case(31, V, lens, groups, dtype=dtype)
    loss = RFTLoss(RFTLossConfig(**cfg_kw))
    assert loss.route(batch) == 3
    assert loss.route(batch, unscaled=True) == 4
    ref = loss(batch, dlogits="new")
    got = loss(batch, dlogits="new", unscaled=True)
    again = loss(batch, dlogits="new", unscaled=True)
    torch.cuda.synchronize()
    assert torch.equal(again.stats, got.stats) and torch.equal(again.dlogits, got.dlogits)
    a, b = got.stats_dict(), ref.stats_dict()
    # sequence-level statistics difference sums of ~25 per-row values of ~1: the
    # absolute floor scales with sum |lp| (the rows' rounding differences add up)
    floor = 2e-6 * max(1.0, abs(b["sum_lp"]))
    for k, v in b.items():
        assert a[k] == pytest.approx(v, rel=1e-5, abs=floor), k
    torch.testing.assert_close(got.lp, ref.lp, rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(got.lse, ref.lse, rtol=1e-6, atol=1e-5)
    # the coupled coefficients are differences of sequence sums (LP_i - ref_i):
    # same absolute floor as the statistics
    torch.testing.assert_close(got.seq_adv, ref.seq_adv, rtol=1e-5,
                               atol=2e-6 * float(ref.seq_lp.abs().max()) + 1e-6)
    scaled = got.dlogits.float() * got.row_scale[:, None]
    want = ref.dlogits.float()
    if dtype == torch.bfloat16:
        tol = 2.0 ** -8 * float(want.abs().max()) + 1e-2 * want.abs()
    else:
        # fp32 rows are exact to ~1e-6, but the coupled coefficient inherits the
        # sequence-sum difference above (up to ~3e-4 relative)
        tol = 1e-5 * float(want.abs().max()) + 1e-3 * want.abs()
    assert bool(((scaled - want).abs() <= tol).all())
    # the unscaled rows are p - e_y: each sums to ~0 and has -1 + p_y at the target
    rows = got.dlogits.float().sum(1)
    assert float(rows.abs().max()) < 5e-2


def test_unscaled_in_place_and_errors():
    from paper_2505_17826_b200._native import NativeError
    lens = [30, 20, 25, 35]
    _, batch = make_case(5, 32000, lens, [2, 2])
    kimi = RFTLoss(RFTLossConfig(policy_loss_fn="opmd_kimi", tau=0.5))
    new = kimi(batch, dlogits="new", unscaled=True)
    torch.cuda.synchronize()
    first = new.dlogits.clone()
    inplace = kimi(batch, dlogits="inplace", unscaled=True)
    torch.cuda.synchronize()
    assert torch.equal(inplace.dlogits, first)
    _, b2 = make_case(6, 32000, lens, [2, 2])
    grpo = RFTLoss(RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip"))
    with pytest.raises(NativeError):
        grpo(b2, dlogits="new", unscaled=True)  # not a coupled loss
    with pytest.raises(NativeError):
        kimi(b2, dlogits=None, unscaled=True)  # needs dlogits


def test_unscaled_on_a_layout_without_single_pass_plan():
    """An unaligned row pitch has no fused plan: the unscaled gradient still
    comes out (route 3 with a unit-coefficient backward), matching the scaled
    two-pass result row by row."""
    lens = [21, 13, 30, 8]
    _, batch = make_case(9, 4097, lens, [2, 2])  # 4,097 x 2 B rows: not 16-byte aligned
    kimi = RFTLoss(RFTLossConfig(policy_loss_fn="opmd_kimi", tau=0.6))
    assert kimi.route(batch, unscaled=True) == 3
    ref = kimi(batch, dlogits="new")
    got = kimi(batch, dlogits="new", unscaled=True)
    torch.cuda.synchronize()
    assert torch.equal(got.stats, ref.stats)
    scaled = got.dlogits.float() * got.row_scale[:, None]
    want = ref.dlogits.float()
    assert bool(((scaled - want).abs() <= 2.0 ** -8 * float(want.abs().max())
                 + 1e-2 * want.abs()).all())
