"""The reference's invariance / identity tests (test_algorithms.py:194-246),
restated on the CUDA path at LLM shapes (V = 151,936, bf16 logits): they hold
for any size, so they check the kernels where the CPU oracle is too slow.

  * reward-shift invariance: adding a constant to every reward of a group
    leaves OPMD_SIMPLE / KIMI / PAIRWISE and GRPO losses and gradients
    unchanged (test_algorithms.py:194-227);
  * pairwise / simple identity at the reference point: grad[pairwise] /
    (1 + tau)^2 == (2 tau K / (1 + tau)) grad[simple]  (test_algorithms.py:230-246);
  * dlogits rows sum to zero (softmax gradient, test_policy.py:444-451), to
    fp32 accuracy.
Tolerances: bf16 dlogits, |a - b| <= 2^-7 max|b| (two bf16 roundings)."""

import numpy as np
import pytest
import torch

from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, logprob_fwd, pack_arrays

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

V = 151936


def batch(seed, lens, groups, reward, seq_ref_lp=None, fp32=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    T = int(sum(lens))
    x = torch.randn(T, V, device="cuda", generator=g) * 2.0
    tgt = np.random.default_rng(seed).integers(0, V, T)
    x[torch.arange(T, device="cuda"), torch.as_tensor(tgt, device="cuda")] += 13.5
    x = x if fp32 else x.to(torch.bfloat16)
    return pack_arrays(x, tgt, lens, groups, np.asarray(reward, np.float32),
                       seq_ref_lp=seq_ref_lp)


def close(a, b, rel=2.0 ** -7):
    a, b = a.float(), b.float()
    scale = float(b.abs().max())
    assert float((a - b).abs().max()) <= rel * scale + 1e-12


@pytest.mark.parametrize("cfg", [RFTLossConfig.from_variant("OPMD_SIMPLE", tau=0.6),
                                 RFTLossConfig.from_variant("OPMD_KIMI", tau=0.6),
                                 RFTLossConfig.from_variant("OPMD_PAIRWISE", tau=0.6),
                                 RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip",
                                               loss_agg_mode="token-mean")],
                         ids=["simple", "kimi", "pairwise", "grpo_ppo"])
def test_reward_shift_invariance(cfg):
    lens, groups = [40, 25, 33, 18, 27, 31], [3, 3]
    reward = [0.9, 0.1, 0.4, 1.0, 0.0, 0.5]
    a = RFTLoss(cfg)(batch(1, lens, groups, reward))
    b = RFTLoss(cfg)(batch(1, lens, groups, [r + 7.5 for r in reward]))
    la, lb = a.stats_dict()["loss"], b.stats_dict()["loss"]
    assert lb == pytest.approx(la, rel=1e-5, abs=1e-6)
    close(b.dlogits, a.dlogits)


def test_pairwise_simple_gradient_identity_at_reference_point():
    tau, lens, groups = 0.8, [30, 22, 41, 17], [4]
    reward = [1.3, -0.2, 0.6, 0.9]
    probe = batch(2, lens, groups, reward, fp32=True)
    seq_lp = logprob_fwd(probe)[3].double().cpu().numpy()  # LP_i: the reference point
    b = batch(2, lens, groups, reward, seq_ref_lp=seq_lp.astype(np.float32), fp32=True)
    pair = RFTLoss(RFTLossConfig.from_variant("OPMD_PAIRWISE", tau=tau))(b)
    simple = RFTLoss(RFTLossConfig.from_variant("OPMD_SIMPLE", tau=tau))(b)
    k = len(lens)
    lhs = pair.dlogits / (1.0 + tau) ** 2
    rhs = simple.dlogits * (2.0 * tau * k / (1.0 + tau))
    close(lhs, rhs, rel=1e-4)  # fp32 logits and dlogits


def test_dlogits_rows_sum_to_zero():
    lens, groups = [64, 64, 64, 64], [2, 2]
    out = RFTLoss(RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip",
                                kl_fn="low_var_kl", kl_coef=0.001,
                                loss_agg_mode="token-mean"))(
        batch(3, lens, groups, [1.0, 0.0, 0.0, 1.0], fp32=True))
    # a row sums to s (sum_v p_v - 1): fp32 with ex2.approx over 151,936 terms
    # keeps |sum p - 1| at a few 1e-6 (the reference's f64 bound is 1e-12)
    rows = out.dlogits.double().sum(1)
    assert float(rows.abs().max()) <= 1e-5 * float(out.dlogits.abs().max())


def test_baseline_size_micro_batch_properties():
    """One full micro-batch of BASELINE configs[1] (8 groups x 8 x 2,048 =
    131,072 rows x V = 151,936 bf16: 40 GB in, 40 GB out) -- sizes the oracle
    cannot reach, checked through properties: the fused kernel and the
    two-pass route agree, its lp equals the forward-only kernel's, dz[y] =
    s (e^lp - 1) on every row, statistics are exact counts, and reruns are
    bit-identical."""
    T, lens, groups = 131072, [2048] * 64, [8] * 8
    x = torch.empty((T, V), dtype=torch.bfloat16, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(11)
    for r in range(0, T, 8192):
        x[r:r + 8192].normal_(0.0, 2.0, generator=g)
    tgt = np.random.default_rng(11).integers(0, V, T)
    tgt_d = torch.as_tensor(tgt, device="cuda")
    x[torch.arange(T, device="cuda"), tgt_d] += 13.5
    reward = np.random.default_rng(12).integers(0, 2, 64).astype(np.float32)
    b = pack_arrays(x, tgt, lens, groups, reward)
    cfg = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="vanilla", loss_agg_mode="token-mean")
    loss = RFTLoss(cfg)
    assert loss.route(b) == 1
    dz = torch.empty_like(x)
    out = loss(b, dlogits=dz)
    st = out.stats_dict()
    assert st["n_tok"] == T and st["n_seqs"] == 64 and st["n_groups"] == 8
    assert st["nonfinite"] == 0 and st["invalid"] == 0
    lp_fwd = logprob_fwd(b)[0]
    assert float((out.lp - lp_fwd).abs().max()) <= 1e-4
    s = out.seq_adv.repeat_interleave(2048) / T  # token-mean weight
    dzy = dz[torch.arange(T, device="cuda"), tgt_d].float()
    expect = s * (torch.exp(out.lp) - 1.0)
    assert torch.all((dzy - expect).abs() <= 1e-2 * expect.abs() + 1e-9)
    again = loss(b, dlogits=torch.empty_like(x))
    assert torch.equal(again.dlogits, dz) and torch.equal(again.stats, out.stats)
    del again
    two = RFTLoss(cfg.with_(force_two_pass=True))(b, dlogits=torch.empty_like(x))
    scale = max(float(dz[r:r + 8192].float().abs().max()) for r in range(0, T, 8192))
    diff = max(float((two.dlogits[r:r + 8192].float() - dz[r:r + 8192].float()).abs().max())
               for r in range(0, T, 8192))  # chunked: a full fp32 copy would be 80 GB
    assert diff <= 2.0 ** -8 * scale
    assert two.stats_dict()["loss"] == pytest.approx(st["loss"], rel=1e-5, abs=1e-9)


@pytest.mark.parametrize("V,cfg_kw", [
    (151936, dict(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl",
                  kl_coef=1e-3, loss_agg_mode="token-mean")),
    (32000, dict(policy_loss_fn="opmd_kimi", tau=0.5)),
], ids=["fused_cl2", "coupled_v32k"])
def test_loss_call_captures_into_a_cuda_graph(V, cfg_kw):
    """The library call is stream-ordered with no host sync or allocation once
    the workspace is cached, so a training step can capture it in a CUDA graph
    and replay it on new logits (static input / output buffers): the replay
    matches an eager call bit for bit."""
    rng = np.random.default_rng(9)
    lens, groups = [40, 33, 57, 20], [2, 2]
    T = sum(lens)
    y = rng.integers(0, V, T)
    rew = np.array([1.0, 0.0, 1.0, 1.0], np.float32)
    old = rng.normal(-9.0, 0.3, T).astype(np.float32)
    logits = (torch.randn(T, V, device="cuda") * 2).to(torch.bfloat16)
    batch = pack_arrays(logits, y, lens, groups, rew, old_lp=old, ref_lp=old)
    loss = RFTLoss(RFTLossConfig(**cfg_kw))
    dz = torch.empty_like(logits)
    out = loss(batch, dlogits=dz)  # warm-up: caches the workspace
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        loss(batch, dlogits=dz, out=out)
    new = (torch.randn(T, V, device="cuda") * 2).to(torch.bfloat16)
    logits.copy_(new)
    g.replay()
    torch.cuda.synchronize()
    got_stats, got_dz = out.stats.clone(), dz.clone()
    eager = loss(pack_arrays(new.clone(), y, lens, groups, rew, old_lp=old, ref_lp=old),
                 dlogits="new")
    torch.cuda.synchronize()
    assert torch.equal(got_stats, eager.stats)
    assert torch.equal(got_dz, eager.dlogits)
