"""Pin the CPU oracle to the reference: golden fixtures produced by the
reference itself (tests/golden/make_golden.py), the reference tests' frozen
known-answer values, and the exact reductions of SURVEY.md section 8c."""

import math

import numpy as np
import pytest

from _golden import groups_of, load, metrics_of
from oracle import rft_oracle as O
from oracle import toy_policy as TP

GROUP_CASES = ["simple_tau05", "simple_tau0", "simple_anchor", "kimi", "pairwise",
               "simple_bf16_v512", "kimi_bf16_v512", "simple_v4_uniform"]


def packed(fx, with_anchor=True):
    groups = groups_of(fx)
    anchor = fx.get("anchor") if with_anchor else None
    batch, states = TP.pack_groups(groups, fx["theta"], anchor)
    return batch, states


@pytest.mark.parametrize("name", GROUP_CASES)
def test_states_and_token_logprobs_match_reference(name):
    fx = load(name)
    batch, states = packed(fx)
    assert np.array_equal(states, fx["states"])              # group indexing / hashing: exact
    assert np.array_equal(batch.target, fx["target"])
    lp = O.ref_logprob_rows(batch.logits, batch.target)
    assert np.array_equal(lp, fx["lp_tok"])                    # bit-exact per-token logprob


@pytest.mark.parametrize("name", GROUP_CASES)
def test_reference_variants_bit_exact(name):
    fx = load(name)
    batch, states = packed(fx)
    variant = str(fx["variant"])
    rep = O.ref_group_batch(batch, variant, float(fx["tau"]), float(fx["beta"]))
    assert rep.loss == float(fx["loss"])                       # bit-exact loss
    S = fx["theta"].shape[0]
    grad = TP.scatter_rows(rep.dz, states, S)
    assert np.max(np.abs(grad - fx["grad"])) <= 1e-12
    gm = metrics_of(fx)
    for k, v in rep.metrics.items():
        assert v == pytest.approx(gm[k], abs=1e-12), k


def _cfg_for(variant, tau, beta):
    if variant == "OPMD_SIMPLE":
        return O.Config(advantage_fn="opmd", policy_loss_fn="vanilla", loss_agg_mode="seq-sum",
                        tau=tau, anchor_beta=beta)
    if variant == "OPMD_KIMI":
        return O.Config(policy_loss_fn="opmd_kimi", tau=tau)
    return O.Config(policy_loss_fn="opmd_pairwise", tau=tau)


@pytest.mark.parametrize("name", GROUP_CASES)
def test_general_loss_reproduces_reference(name):
    fx = load(name)
    batch, states = packed(fx)
    cfg = _cfg_for(str(fx["variant"]), float(fx["tau"]), float(fx["beta"]))
    out = O.general_loss(batch, cfg)
    st = O.stats_dict(out["stats"])
    assert st["loss"] == pytest.approx(float(fx["loss"]), rel=1e-12, abs=1e-12)
    grad = TP.scatter_rows(out["dz"], states, fx["theta"].shape[0])
    assert np.max(np.abs(grad - fx["grad"])) <= 1e-12
    gm = metrics_of(fx)
    n = st["n_groups"]
    assert st["sum_mean_reward"] / n == pytest.approx(gm["mean_reward"], abs=1e-12)
    assert st["sum_baseline"] / n == pytest.approx(gm["baseline"], abs=1e-12)
    assert st["sum_kl_estimate"] / n == pytest.approx(gm["kl_estimate"], abs=1e-12)
    assert st["sum_group_size"] / n == pytest.approx(gm["group_size"], abs=1e-12)
    assert st["nonfinite"] == 0


def test_sft_matches_reference():
    fx = load("sft")
    batch, states = packed(fx, with_anchor=False)
    rep = O.ref_sft(batch)
    assert rep.loss == float(fx["loss"])
    S = fx["theta"].shape[0]
    assert np.max(np.abs(TP.scatter_rows(rep.dz, states, S) - fx["grad"])) <= 1e-12
    for cfg_kind in ("sft_rows", "pg_sft"):
        if cfg_kind == "sft_rows":
            batch.seq_kind = np.ones(batch.n_seqs, np.int64)
            cfg = O.Config(policy_loss_fn="vanilla", advantage_fn="reinforce")
        else:
            batch.seq_kind = None
            cfg = O.Config(policy_loss_fn="sft", loss_agg_mode="seq-mean-token-sum")
        out = O.general_loss(batch, cfg)
        assert out["stats"][O.STAT["loss"]] == pytest.approx(float(fx["loss"]), rel=1e-12)
        grad = TP.scatter_rows(out["dz"], states, S)
        assert np.max(np.abs(grad - fx["grad"])) <= 1e-12


def test_dpo_matches_reference():
    fx = load("dpo")
    batch, states = packed(fx)
    batch.seq_ref_lp = fx["ref_seq_lp"]
    beta = float(fx["dpo_beta"])
    rep = O.ref_dpo(batch, beta)
    assert rep.loss == float(fx["loss"])
    S = fx["theta"].shape[0]
    assert np.max(np.abs(TP.scatter_rows(rep.dz, states, S) - fx["grad"])) <= 1e-12
    assert rep.metrics["mean_reward"] == pytest.approx(metrics_of(fx)["mean_reward"], abs=1e-14)
    out = O.general_loss(batch, O.Config(policy_loss_fn="dpo", dpo_beta=beta))
    assert out["stats"][O.STAT["loss"]] == pytest.approx(float(fx["loss"]), rel=1e-12)
    assert np.max(np.abs(TP.scatter_rows(out["dz"], states, S) - fx["grad"])) <= 1e-12
    n = batch.n_groups
    assert out["stats"][O.STAT["sum_dpo_margin"]] / n == pytest.approx(
        metrics_of(fx)["mean_reward"], abs=1e-12)


def test_regularizer_g_matches_reference():
    fx = load("regularizer_g")
    batch, states = packed(fx)
    value, dz = O.ref_regularizer_g(batch, 0)
    assert value == pytest.approx(float(fx["value"]), abs=1e-13)
    S = fx["theta"].shape[0]
    assert np.max(np.abs(TP.scatter_rows(dz, states, S) - fx["grad"])) <= 1e-12
    # unified path: anchor term alone (zero rewards -> zero policy-gradient part)
    batch.reward = np.zeros(batch.n_seqs)
    out = O.general_loss(batch, O.Config(advantage_fn="opmd", policy_loss_fn="vanilla",
                                         loss_agg_mode="seq-sum", anchor_beta=1.0))
    assert out["stats"][O.STAT["anchor_loss"]] == pytest.approx(float(fx["value"]), rel=1e-12)
    assert np.max(np.abs(TP.scatter_rows(out["dz"], states, S) - fx["grad"])) <= 1e-12


# ---------------------------------------------------------------------------
# frozen known answers from the reference tests (test_algorithms.py:109-188)


def uniform_batch(seq_lens, V, rewards, group_sizes):
    T = sum(seq_lens)
    off = np.concatenate([[0], np.cumsum(seq_lens)])
    goff = np.concatenate([[0], np.cumsum(group_sizes)])
    lp_seq = np.array([-n * math.log(V) for n in seq_lens])
    return O.Batch(logits=np.zeros((T, V)), target=np.zeros(T, np.int64), seq_offsets=off,
                   group_offsets=goff, reward=np.array(rewards, float), seq_ref_lp=lp_seq,
                   old_lp=np.full(T, -math.log(V)))


def test_known_answers():
    fx = load("known_answers")
    ka = dict(zip(fx["names"], fx["values"]))
    assert O.ref_tau_log_zhat([0.0, math.log(9.0)], 1.0) == pytest.approx(math.log(5.0), abs=1e-12)
    assert O.ref_tau_log_zhat([0.0, math.log(9.0)], 1.0) == ka["tau_log_zhat_ln5"]
    assert O.ref_tau_log_zhat([0.0, 0.0, 0.0], 2.0) == 0.0
    assert O.ref_tau_log_zhat([1000.0, 1000.0], 1.0) == ka["tau_log_zhat_1000"]
    assert O.ref_tau_log_zhat([5.0], 0.5) == pytest.approx(5.0, abs=1e-12)
    # Kimi K=2 on-policy fixture (test_algorithms.py:135-148)
    b = uniform_batch([3, 3], 4, [1.0, 0.0], [2])
    out = O.general_loss(b, O.Config(policy_loss_fn="opmd_kimi", tau=1.0))
    st = O.stats_dict(out["stats"])
    assert st["sum_baseline"] == pytest.approx(0.6201145069582775, abs=1e-12)
    assert st["loss"] == pytest.approx(0.5288549895636602, abs=1e-9)
    assert st["sum_kl_estimate"] == pytest.approx(0.0, abs=1e-12)
    # Pairwise K=2 -> 1.0 (151-158)
    out = O.general_loss(b, O.Config(policy_loss_fn="opmd_pairwise", tau=1.0))
    assert out["stats"][O.STAT["loss"]] == pytest.approx(1.0, abs=1e-12)
    # Simple at uniform logits -> 0, baseline 0.5 (161-169)
    b3 = uniform_batch([3, 3, 3], 4, [1.0, 0.0, 0.5], [3])
    out = O.general_loss(b3, O.Config(advantage_fn="opmd", policy_loss_fn="vanilla",
                                      loss_agg_mode="seq-sum", tau=0.0))
    assert out["stats"][O.STAT["loss"]] == pytest.approx(0.0, abs=1e-12)
    assert out["stats"][O.STAT["sum_baseline"]] == pytest.approx(0.5)
    # SFT uniform V=4, three tokens -> 3 ln 4 (172-178)
    b1 = uniform_batch([3], 4, [0.0], [1])
    out = O.general_loss(b1, O.Config(policy_loss_fn="sft", loss_agg_mode="seq-mean-token-sum"))
    assert out["stats"][O.STAT["loss"]] == pytest.approx(4.1588830833596715, abs=1e-12)
    # DPO at the reference -> ln 2 (181-188)
    b2 = uniform_batch([2, 2], 4, [0.0, 0.0], [2])
    out = O.general_loss(b2, O.Config(policy_loss_fn="dpo", dpo_beta=0.1))
    assert out["stats"][O.STAT["loss"]] == pytest.approx(0.6931471805599453, abs=1e-12)


# ---------------------------------------------------------------------------
# north_star pieces: exact reductions to reference variants


def _base():
    fx = load("simple_tau0")
    batch, states = packed(fx)
    return fx, batch, states


def test_grpo_reduces_to_opmd_with_std_scaled_rewards():
    fx, batch, states = _base()
    out = O.general_loss(batch, O.Config(advantage_fn="grpo", policy_loss_fn="vanilla",
                                         loss_agg_mode="seq-sum"))
    scaled = O.Batch(**{**batch.__dict__})
    r = batch.reward.copy()
    for g in range(batch.n_groups):
        s = list(batch.group_seqs(g))
        r[s] = r[s] / (np.std(batch.reward[s], ddof=1) + 1e-6)
    scaled.reward = r
    ref = O.ref_group_batch(scaled, "OPMD_SIMPLE", 0.0, 0.0)
    assert out["stats"][O.STAT["loss"]] == pytest.approx(ref.loss, rel=1e-10, abs=1e-12)
    assert np.max(np.abs(out["dz"] - ref.dz)) <= 1e-12


def test_rloo_reduces_to_opmd_with_scaled_rewards():
    fx, batch, states = _base()
    out = O.general_loss(batch, O.Config(advantage_fn="rloo", policy_loss_fn="vanilla",
                                         loss_agg_mode="seq-sum"))
    scaled = O.Batch(**{**batch.__dict__})
    r = batch.reward.copy()
    for g in range(batch.n_groups):
        s = list(batch.group_seqs(g))
        k = len(s)
        r[s] = r[s] * k / (k - 1)
    scaled.reward = r
    ref = O.ref_group_batch(scaled, "OPMD_SIMPLE", 0.0, 0.0)
    assert out["stats"][O.STAT["loss"]] == pytest.approx(ref.loss, rel=1e-10, abs=1e-12)
    assert np.max(np.abs(out["dz"] - ref.dz)) <= 1e-12


def test_ppo_at_ratio_one_has_opmd_gradient_and_token_mean_scales():
    fx, batch, states = _base()
    lp = O.ref_logprob_rows(batch.logits, batch.target)
    batch.old_lp = lp.copy()      # rho = 1 everywhere
    ref = O.ref_group_batch(batch, "OPMD_SIMPLE", 0.0, 0.0)
    out = O.general_loss(batch, O.Config(advantage_fn="opmd", policy_loss_fn="ppo_clip",
                                         loss_agg_mode="seq-sum"))
    assert np.max(np.abs(out["dz"] - ref.dz)) <= 1e-12
    assert out["stats"][O.STAT["clip_count"]] == 0
    out = O.general_loss(batch, O.Config(advantage_fn="opmd", policy_loss_fn="ppo_clip",
                                         loss_agg_mode="token-mean"))
    assert np.max(np.abs(out["dz"] - ref.dz / batch.n_rows)) <= 1e-14


def test_k3_gradient_vanishes_at_reference():
    fx, batch, states = _base()
    lp = O.ref_logprob_rows(batch.logits, batch.target)
    batch.ref_lp = lp.copy()
    batch.reward = np.zeros(batch.n_seqs)
    # (abs is non-differentiable at lp == ref; it is covered by finite differences)
    for kl in ("k1", "k2", "k3"):
        out = O.general_loss(batch, O.Config(advantage_fn="opmd", policy_loss_fn="vanilla",
                                             kl_fn=kl, kl_coef=0.5))
        if kl == "k1":
            assert np.max(np.abs(out["dz"])) > 1e-3     # k1 has a constant gradient
        else:
            assert np.max(np.abs(out["dz"])) <= 1e-15, kl
            assert out["stats"][O.STAT["kl_loss"]] == pytest.approx(0.0, abs=1e-15)


def _fd_check(batch, cfg, h=1e-6, tol=1e-6, rows=None):
    out = O.general_loss(batch, cfg)
    dz = out["dz"]
    T, V = batch.logits.shape
    rows = range(T) if rows is None else rows
    for t in rows:
        for v in range(V):
            up = O.Batch(**{**batch.__dict__})
            up.logits = batch.logits.copy()
            up.logits[t, v] += h
            lu = O.general_loss(up, cfg, want_dz=False)["stats"][O.STAT["loss"]]
            up.logits[t, v] -= 2 * h
            ld = O.general_loss(up, cfg, want_dz=False)["stats"][O.STAT["loss"]]
            fd = (lu - ld) / (2 * h)
            assert abs(fd - dz[t, v]) <= tol * max(1.0, abs(fd)), (t, v, fd, dz[t, v])


def _small_batch(seed=0, V=6):
    rng = np.random.default_rng(seed)
    seq_lens = [2, 3, 1, 2]
    T = sum(seq_lens)
    b = O.Batch(logits=rng.normal(0, 1.0, (T, V)), target=rng.integers(0, V, T),
                seq_offsets=np.concatenate([[0], np.cumsum(seq_lens)]),
                group_offsets=np.array([0, 2, 4]), reward=rng.uniform(-1, 1, 4),
                old_lp=rng.normal(-1.5, 0.3, T), ref_lp=rng.normal(-1.5, 0.3, T))
    b.seq_ref_lp = np.array([b.old_lp[b.seq_rows(i)].sum() for i in range(4)])
    b.anchor_logits = rng.normal(0, 1.0, (T, V))
    return b


@pytest.mark.parametrize("kl", ["k1", "k2", "k3", "abs"])
@pytest.mark.parametrize("agg", ["token-mean", "seq-mean-token-mean", "seq-mean-token-sum",
                                 "seq-mean-token-sum-norm", "seq-sum"])
def test_finite_difference_ppo_kl_entropy(kl, agg):
    b = _small_batch()
    cfg = O.Config(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn=kl, kl_coef=0.3,
                   entropy_loss_fn="default", entropy_coef=0.05, loss_agg_mode=agg,
                   clip_lo=0.2, clip_hi=0.28, agg_norm=4.0)
    _fd_check(b, cfg)


@pytest.mark.parametrize("pg", ["opmd_kimi", "opmd_pairwise", "dpo"])
def test_finite_difference_coupled(pg):
    b = _small_batch(1)
    b.group_offsets = np.array([0, 2, 4])
    _fd_check(b, O.Config(policy_loss_fn=pg, tau=0.7, dpo_beta=0.4))


def test_finite_difference_anchor_and_mixed_sft():
    b = _small_batch(2)
    b.seq_kind = np.array([0, 0, 1, 1])
    cfg = O.Config(advantage_fn="rloo", policy_loss_fn="vanilla", loss_agg_mode="token-mean",
                   anchor_beta=0.6, sft_weight=0.5)
    _fd_check(b, cfg)


def test_dual_clip_counts_and_zero_gradient():
    b = _small_batch(3)
    b.old_lp = b.old_lp - 3.0  # rho >> 1
    cfg = O.Config(advantage_fn="reinforce", policy_loss_fn="ppo_clip", clip_c=3.0,
                   loss_agg_mode="token-mean")
    out = O.general_loss(b, cfg)
    st = O.stats_dict(out["stats"])
    assert st["clip_count"] + st["dual_clip_count"] > 0
    _fd_check(b, cfg)


def test_ppo_log_ratio_clamp_has_no_gradient():
    """|lp - old| > 20: the ratio is clamped like torch.clamp, so the row has
    no policy gradient even on the unclipped (A < 0, rho >> 1) branch."""
    b = _small_batch(4)
    b.old_lp = b.old_lp - 25.0
    b.reward = -np.abs(b.reward) - 1.0  # reinforce: A < 0 everywhere
    cfg = O.Config(advantage_fn="reinforce", policy_loss_fn="ppo_clip", loss_agg_mode="seq-sum")
    out = O.general_loss(b, cfg)
    assert np.all(out["s"] == 0.0) and np.all(out["dz"] == 0.0)
    assert out["stats"][O.STAT["clip_count"]] == 0
    _fd_check(b, cfg)
    dz = np.zeros_like(b.logits)
    O.single_pass_blocked(b, cfg, dz_out=dz)
    assert np.all(dz == 0.0)


@pytest.mark.parametrize("cfg", [
    O.Config(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="k3", kl_coef=0.1,
             entropy_loss_fn="default", entropy_coef=0.05, loss_agg_mode="token-mean"),
    O.Config(advantage_fn="opmd", policy_loss_fn="vanilla", loss_agg_mode="seq-sum", tau=0.5),
    O.Config(advantage_fn="rloo", policy_loss_fn="sft", loss_agg_mode="seq-mean-token-mean",
             clip_c=3.0),
])
def test_blocked_single_pass_matches_general(cfg):
    b = _small_batch(7, V=50)
    b.seq_kind = np.array([0, 0, 0, 1])
    ref = O.general_loss(b, cfg)
    dz = np.zeros_like(b.logits)
    out = O.single_pass_blocked(b, cfg, dz_out=dz, block=3)
    assert out["loss"] == pytest.approx(ref["stats"][O.STAT["loss"]], rel=1e-12, abs=1e-14)
    assert np.max(np.abs(dz - ref["dz"])) <= 1e-14
    assert np.max(np.abs(out["lp"] - ref["lp"])) <= 1e-14


@pytest.mark.parametrize("name", ["trainer_simple_anchor", "trainer_kimi"])
def test_oracle_group_steps_reproduce_reference_trainer(name):
    """Pins the trainer fixtures (the reference's own orchestrator.Trainer):
    the oracle's reference-order group loss, scattered by state and applied as
    theta -= lr * grad (algorithms.py:329-348), reproduces every step_groups
    loss of the reference to the last bit (the later SFT / DPO steps are
    covered by their own fixtures)."""
    fx = load(name)
    theta = fx["theta"].copy()
    anchor = fx["theta"]
    lr = float(fx["lr"])
    for step in range(int(fx["steps"])):
        batch, states = TP.pack_groups(groups_of(fx), theta, anchor)
        rep = O.ref_group_batch(batch, str(fx["variant"]), float(fx["tau"]), float(fx["beta"]))
        assert rep.loss == float(fx["losses"][step]), step
        theta = theta - lr * TP.scatter_rows(rep.dz, states, theta.shape[0])
