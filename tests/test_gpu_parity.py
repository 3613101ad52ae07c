"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same inputs, plus the reference's own golden fixtures.

Tolerances (stated here, per the north_star: bf16 input, fp32 accumulate,
rtol 1e-3 on the loss):
  * loss and every loss component: |a - b| <= 1e-3 * max(|b|, floor), floor
    = 1e-3 * sum_t |s_t lp_t| (guards cancelling sums);
  * per-row lp / lse / entropy: 1e-4 absolute + 1e-5 relative (fp32 math);
  * dlogits: bf16 outputs |a - b| <= 2^-8 * max|b| + 1e-2 |b|;
    fp32 outputs 1e-5 * max|b| + 1e-4 |b|;
  * integer / index work (states, group indexing, counts): exact.
"""

import math

import numpy as np
import pytest
import torch

from _cases import make_case, oracle_cfg
from _golden import groups_of, load
from oracle import rft_oracle as O
from paper_2505_17826_b200 import AlgorithmError, RFTLoss, RFTLossConfig, logprob_fwd, pack_arrays
from paper_2505_17826_b200 import triad_compat as C

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - the marker keeps these off CPU runs
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _close_loss(a, b, floor):
    assert abs(a - b) <= 1e-3 * max(abs(b), floor), (a, b, floor)


def compare(out, ref, dtype, dz=True, rtol_dz=None):
    st = out.stats_dict()
    rs = O.stats_dict(ref["stats"])
    floor = 1e-3 * float(np.sum(np.abs(ref["s"] * ref["lp"]))) + 1e-6
    for k in ("loss", "pg_loss", "kl_loss", "entropy_loss", "anchor_loss", "sft_loss"):
        _close_loss(st[k], rs[k], floor)
    for k in ("n_groups", "n_tok", "n_tok_rl", "n_seqs", "n_sft_seqs", "nonfinite", "invalid"):
        assert st[k] == rs[k], k
    for k in ("sum_mean_reward", "sum_baseline", "sum_group_size", "sum_lp", "sum_entropy",
              "sum_kl_estimate", "sum_adv", "sum_ratio", "sum_kl", "sum_ppo_kl"):
        assert st[k] == pytest.approx(rs[k], rel=1e-4, abs=1e-3 + 1e-5 * rs["n_tok"]), k
    # clip decisions can flip for tokens sitting on the clip boundary in fp32
    assert abs(st["clip_count"] - rs["clip_count"]) <= max(2, 1e-3 * rs["n_tok"])
    lp = out.lp.double().cpu().numpy()
    np.testing.assert_allclose(lp, ref["lp"], rtol=1e-5, atol=1e-4)
    np.testing.assert_allclose(out.entropy.double().cpu().numpy(), ref["entropy"], rtol=1e-5,
                               atol=1e-4)
    np.testing.assert_allclose(out.seq_lp.double().cpu().numpy(), ref["seq_lp"], rtol=1e-5,
                               atol=1e-3)
    if dz:
        d = out.dlogits.float().cpu().numpy().astype(np.float64)
        r = ref["dz"]
        scale = float(np.max(np.abs(r))) if r.size else 0.0
        if dtype == torch.bfloat16:
            tol = 2.0 ** -8 * scale + (rtol_dz or 1e-2) * np.abs(r)
        else:
            tol = 1e-5 * scale + (rtol_dz or 1e-4) * np.abs(r)
        err = np.abs(d[:, : r.shape[1]] - r)
        assert np.all(err <= tol), float(np.max(err - tol))


CONFIGS = {
    "grpo_ppo_tokmean": RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip",
                                      loss_agg_mode="token-mean", clip_lo=0.2, clip_hi=0.28),
    "grpo_ppo_k3_ent": RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip",
                                     kl_fn="low_var_kl", kl_coef=0.001, entropy_loss_fn="default",
                                     entropy_coef=0.001, loss_agg_mode="token-mean",
                                     clip_lo=0.2, clip_hi=0.28),
    "rloo_vanilla_smtm": RFTLossConfig(advantage_fn="rloo", policy_loss_fn="vanilla",
                                       loss_agg_mode="seq-mean-token-mean", kl_fn="k2",
                                       kl_coef=0.05),
    "opmd_simple": RFTLossConfig.from_variant("OPMD_SIMPLE", tau=1.0),
    "dualclip_k1_smts": RFTLossConfig(advantage_fn="reinforce", policy_loss_fn="ppo_clip",
                                      clip_c=3.0, kl_fn="k1", kl_coef=0.02,
                                      loss_agg_mode="seq-mean-token-sum"),
    "abs_norm_ent": RFTLossConfig(advantage_fn="grpo", policy_loss_fn="vanilla", kl_fn="abs",
                                  kl_coef=0.01, entropy_loss_fn="default", entropy_coef=0.01,
                                  loss_agg_mode="seq-mean-token-sum-norm", agg_norm=64.0),
    "sft": RFTLossConfig.from_variant("SFT"),
    "kimi": RFTLossConfig.from_variant("OPMD_KIMI", tau=0.7),
    "pairwise": RFTLossConfig.from_variant("OPMD_PAIRWISE", tau=1.3),
}

SHAPES = {  # V, seq_lens, group_sizes
    "v64": (64, [5, 0, 7, 3, 1, 9, 2, 4], [4, 4]),
    "v1000": (1000, [17, 33, 5, 12, 20, 9], [3, 3]),
    "v32000": (32000, [40, 24, 31, 17, 22, 38, 9, 11], [4, 4]),
    "v151936": (151936, [13, 9, 21, 7], [2, 2]),
}


def run_case(cfg, shape, dtype, seed=0, force_two_pass=False, **case_kw):
    V, lens, gs = SHAPES[shape]
    batch, packed = make_case(seed, V, lens, gs, dtype=dtype, **case_kw)
    c = cfg.with_(force_two_pass=force_two_pass)
    out = RFTLoss(c)(packed, dlogits="new")
    ref = O.general_loss(batch, oracle_cfg(c))
    return out, ref, packed


@pytest.mark.parametrize("shape", list(SHAPES))
@pytest.mark.parametrize("name", list(CONFIGS))
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_parity_matrix(name, shape, dtype):
    if shape == "v151936" and dtype == torch.float32 and name not in ("grpo_ppo_k3_ent", "kimi"):
        pytest.skip("fp32 at V=152k covered by two configs")
    out, ref, _ = run_case(CONFIGS[name], shape, dtype)
    compare(out, ref, dtype)


@pytest.mark.parametrize("shape", list(SHAPES))
@pytest.mark.parametrize("name", ["kimi", "pairwise"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_unscaled_single_pass_coupled_matches_oracle(name, shape, dtype):
    """Route 4 (TG_FLAG_UNSCALED_GRAD): one pass writes p - e_y, the per-row
    scale comes from the coupled epilogue; scale x unscaled = the oracle's
    d loss / d z within the same tolerances as every other route."""
    if shape == "v151936" and dtype == torch.float32 and name != "kimi":
        pytest.skip("fp32 at V=152k covered by kimi")
    V, lens, gs = SHAPES[shape]
    batch, packed = make_case(0, V, lens, gs, dtype=dtype)
    loss = RFTLoss(CONFIGS[name])
    assert loss.route(packed, unscaled=True) == 4
    out = loss(packed, dlogits="new", unscaled=True)
    out.dlogits = out.dlogits.float() * out.row_scale[:, None]
    compare(out, O.general_loss(batch, oracle_cfg(CONFIGS[name])), dtype)


@pytest.mark.parametrize("shape", ["v1000", "v32000", "v151936"])
@pytest.mark.parametrize("name", ["grpo_ppo_k3_ent", "opmd_simple", "sft"])
def test_two_pass_route_matches_oracle(name, shape):
    out, ref, packed = run_case(CONFIGS[name], shape, torch.bfloat16, force_two_pass=True)
    compare(out, ref, torch.bfloat16)


def test_routes():
    _, _, packed = run_case(CONFIGS["grpo_ppo_tokmean"], "v151936", torch.bfloat16)
    assert RFTLoss(CONFIGS["grpo_ppo_tokmean"]).route(packed) == 1
    assert RFTLoss(CONFIGS["kimi"]).route(packed) == 3
    assert RFTLoss(CONFIGS["grpo_ppo_tokmean"].with_(force_two_pass=True)).route(packed) == 2


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_anchor_kl_regularizer(dtype):
    cfg = RFTLossConfig.from_variant("OPMD_SIMPLE", tau=0.4, beta=0.9)
    out, ref, _ = run_case(cfg, "v1000", dtype, anchor=True)
    compare(out, ref, dtype)


@pytest.mark.parametrize("shape,case_kw", [
    ("v1000", {}), ("v32000", {}), ("v151936", {}), ("v1000", dict(ld=1008)),
], ids=["v1000", "v32000", "v151936", "v1000_tail_vector"])
def test_fused_anchor_kl_route_matches_oracle(shape, case_kw):
    """regularizer_g in one pass (route 1 with the anchor rows on the fused
    kernel's ring, 6V bytes per row) against the oracle; forced two-pass
    (10V) on the same inputs agrees too."""
    if shape == "v1000" and "ld" in case_kw:
        V, lens, gs = 1001, SHAPES["v1000"][1], SHAPES["v1000"][2]
    else:
        V, lens, gs = SHAPES[shape]
    cfg = RFTLossConfig.from_variant("OPMD_SIMPLE", tau=0.4, beta=0.9)
    batch, packed = make_case(3, V, lens, gs, dtype=torch.bfloat16, anchor=True, **case_kw)
    assert RFTLoss(cfg).route(packed) == 1
    out = RFTLoss(cfg)(packed, dlogits="new")
    ref = O.general_loss(batch, oracle_cfg(cfg))
    compare(out, ref, torch.bfloat16)
    again = RFTLoss(cfg)(packed, dlogits="new")  # fixed-order reductions: bitwise rerun
    assert torch.equal(again.stats, out.stats) and torch.equal(again.dlogits, out.dlogits)
    two = RFTLoss(cfg.with_(force_two_pass=True))(packed, dlogits="new")
    a, b = out.stats_dict(), two.stats_dict()
    assert a["anchor_loss"] == pytest.approx(b["anchor_loss"], rel=1e-4, abs=1e-6)
    assert a["sum_anchor_kl"] == pytest.approx(b["sum_anchor_kl"], rel=1e-4, abs=1e-5)


@pytest.mark.parametrize("shape,route", [("v1000", 1), ("v32000", 1), ("v151936", 1)])
def test_fp32_anchor_kl_routes_match_oracle(shape, route):
    """fp32 rows take the fused anchor path: both slices in the TMEM stash
    (V up to ~65 k), or the split TMEM + shared-memory stash (Qwen vocabulary,
    4-CTA clusters); against the oracle."""
    V, lens, gs = SHAPES[shape]
    cfg = RFTLossConfig.from_variant("OPMD_SIMPLE", tau=0.4, beta=0.9)
    batch, packed = make_case(7, V, lens, gs, dtype=torch.float32, anchor=True)
    assert RFTLoss(cfg).route(packed) == route
    out = RFTLoss(cfg)(packed, dlogits="new")
    compare(out, O.general_loss(batch, oracle_cfg(cfg)), torch.float32)


@pytest.mark.parametrize("shape", ["v32000", "v151936"])
def test_fused_anchor_kl_with_masked_vocabulary_matches_two_pass(shape):
    """-inf logits (masked vocabulary, in both the policy and the anchor rows)
    take the fused anchor path's checked branch (V = 151,936: the split
    stash, phase 2 clamps them from TMEM and shared-memory positions); the oracle cannot evaluate
    KL(p || q) there (inf - inf), so the two-pass route -- which clamps -inf
    the same way -- is the reference."""
    V, lens, gs = SHAPES[shape]
    cfg = RFTLossConfig.from_variant("OPMD_SIMPLE", tau=0.4, beta=0.9)
    _, packed = make_case(4, V, lens, gs, dtype=torch.bfloat16, anchor=True, neg_inf=0.02)
    assert RFTLoss(cfg).route(packed) == 1
    out = RFTLoss(cfg)(packed, dlogits="new")
    two = RFTLoss(cfg.with_(force_two_pass=True))(packed, dlogits="new")
    a, b = out.stats_dict(), two.stats_dict()
    assert a["nonfinite"] == 0
    for k in ("loss", "anchor_loss", "sum_anchor_kl", "sum_lp", "sum_entropy"):
        assert a[k] == pytest.approx(b[k], rel=1e-4, abs=1e-5), k
    d, r = out.dlogits.float(), two.dlogits.float()
    assert bool(((d - r).abs() <= 2.0 ** -8 * float(r.abs().max()) + 1e-2 * r.abs()).all())


def test_mixed_rl_sft_batch():
    cfg = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip",
                        loss_agg_mode="token-mean", sft_weight=0.5)
    V, lens, gs = SHAPES["v32000"]
    kind = [0, 0, 0, 0, 1, 1, 1, 1]
    batch, packed = make_case(3, V, lens, gs, seq_kind=kind)
    out = RFTLoss(cfg)(packed)
    ref = O.general_loss(batch, oracle_cfg(cfg))
    compare(out, ref, torch.bfloat16)


def test_dpo_pairs():
    cfg = RFTLossConfig.from_variant("DPO", dpo_beta=0.3)
    batch, packed = make_case(4, 1000, [6, 9, 4, 4, 11, 3], [2, 2, 2])
    out = RFTLoss(cfg)(packed)
    ref = O.general_loss(batch, oracle_cfg(cfg))
    compare(out, ref, torch.bfloat16)


@pytest.mark.parametrize("ld", [1008, 1024])
def test_padded_pitch_and_tail_vector(ld):
    cfg = CONFIGS["grpo_ppo_k3_ent"]
    batch, packed = make_case(5, 1001, [10, 20, 30, 5], [2, 2], ld=ld)
    assert packed.logits.stride(0) == ld
    out = RFTLoss(cfg)(packed)
    compare(out, O.general_loss(batch, oracle_cfg(cfg)), torch.bfloat16)


def test_unaligned_vocab_scalar_path():
    cfg = CONFIGS["grpo_ppo_k3_ent"]
    batch, packed = make_case(6, 999, [10, 20, 30, 5], [2, 2])   # ld*2 not a multiple of 16
    out = RFTLoss(cfg)(packed)
    assert RFTLoss(cfg).route(packed) == 2
    compare(out, O.general_loss(batch, oracle_cfg(cfg)), torch.bfloat16)


def test_inplace_dlogits():
    cfg = CONFIGS["grpo_ppo_k3_ent"]
    V, lens, gs = SHAPES["v151936"]
    batch, packed = make_case(7, V, lens, gs)
    ref = O.general_loss(batch, oracle_cfg(cfg))
    out = RFTLoss(cfg)(packed, dlogits="inplace")
    assert out.dlogits.data_ptr() == packed.logits.data_ptr()
    compare(out, ref, torch.bfloat16)


def test_masked_vocab_neg_inf_logits():
    cfg = CONFIGS["grpo_ppo_k3_ent"]
    for shape in ("v1000", "v32000"):
        V, lens, gs = SHAPES[shape]
        batch, packed = make_case(8, V, lens, gs, neg_inf=0.3)
        out = RFTLoss(cfg)(packed)
        ref = O.general_loss(batch, oracle_cfg(cfg))
        assert out.stats_dict()["nonfinite"] == 0
        compare(out, ref, torch.bfloat16)


def test_forward_only_loss():
    cfg = CONFIGS["grpo_ppo_k3_ent"]
    V, lens, gs = SHAPES["v32000"]
    batch, packed = make_case(9, V, lens, gs)
    out = RFTLoss(cfg)(packed, dlogits=None)
    assert out.dlogits is None
    compare(out, O.general_loss(batch, oracle_cfg(cfg)), torch.bfloat16, dz=False)


def test_logprob_fwd_matches_oracle():
    for shape in ("v64", "v151936"):
        V, lens, gs = SHAPES[shape]
        batch, packed = make_case(10, V, lens, gs)
        lp, ent, lse, seq_lp = logprob_fwd(packed)
        l_ref, lp_ref, ent_ref = O.row_forward(batch.logits, batch.target)
        np.testing.assert_allclose(lp.double().cpu().numpy(), lp_ref, rtol=1e-5, atol=1e-4)
        np.testing.assert_allclose(lse.double().cpu().numpy(), l_ref, rtol=1e-6, atol=1e-4)
        np.testing.assert_allclose(ent.double().cpu().numpy(), ent_ref, rtol=1e-5, atol=1e-4)
        seq = [lp_ref[batch.seq_rows(i)].sum() for i in range(batch.n_seqs)]
        np.testing.assert_allclose(seq_lp.double().cpu().numpy(), seq, rtol=1e-5, atol=1e-3)


def test_deterministic_bitwise():
    cfg = CONFIGS["grpo_ppo_k3_ent"]
    _, _, packed = run_case(cfg, "v151936", torch.bfloat16)
    a = RFTLoss(cfg)(packed)
    b = RFTLoss(cfg)(packed)
    assert torch.equal(a.stats, b.stats)
    assert torch.equal(a.dlogits, b.dlogits)
    assert torch.equal(a.lp, b.lp)


def test_invalid_target_and_group_shapes_reported():
    cfg = CONFIGS["grpo_ppo_tokmean"]
    V, lens, gs = SHAPES["v64"]
    batch, packed = make_case(11, V, lens, gs)
    packed.target[3] = V + 5  # bypasses the host packer's check
    out = RFTLoss(cfg)(packed)
    assert out.stats_dict()["invalid"] == 1
    with pytest.raises(AlgorithmError):
        out.metrics()
    # pairwise needs K >= 2
    batch, packed = make_case(12, 64, [3, 4, 5], [1, 2])
    out = RFTLoss(CONFIGS["pairwise"])(packed)
    assert out.stats_dict()["invalid"] >= 1


def test_empty_batch_and_singleton_groups():
    cfg = CONFIGS["grpo_ppo_tokmean"]
    batch, packed = make_case(13, 64, [0, 0], [1, 1])
    out = RFTLoss(cfg)(packed)
    st = out.stats_dict()
    assert st["n_tok"] == 0 and st["loss"] == 0.0 and st["n_groups"] == 2
    batch, packed = make_case(14, 1000, [4, 6, 3], [1, 1, 1])   # GRPO K=1 -> A = 0
    out = RFTLoss(cfg)(packed)
    assert torch.all(out.seq_adv == 0)
    compare(out, O.general_loss(batch, oracle_cfg(cfg)), torch.bfloat16)


def test_large_vocab_properties():
    """Size-independent properties at Qwen vocabulary with many rows: vanilla
    gradient rows sum to ~0 (sum_v p - 1 = 0; test_policy.py:444-451),
    dz[y] = s (e^lp - 1), lp <= 0, 0 <= H <= log V, fused == two-pass."""
    V, T = 151936, 2048
    lens = [256] * 8
    cfg = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="vanilla", loss_agg_mode="seq-sum")
    batch, packed = make_case(15, V, lens, [4, 4], ref=False)
    out = RFTLoss(cfg)(packed)
    dz = out.dlogits.float()
    s = out.seq_adv.repeat_interleave(256)
    rowsum = dz.double().sum(dim=1)
    assert torch.all(rowsum.abs() <= 2e-2 * s.abs().double() + 1e-6)
    tgt = packed.target.long()
    dzy = dz[torch.arange(T, device=dz.device), tgt]
    expect = s * (torch.exp(out.lp) - 1.0)
    assert torch.all((dzy - expect).abs() <= 1e-2 * expect.abs() + 1e-3)
    assert torch.all(out.lp <= 1e-6)
    assert torch.all(out.entropy >= -1e-4) and torch.all(out.entropy <= math.log(V) + 1e-3)
    two = RFTLoss(cfg.with_(force_two_pass=True))(packed)
    assert (two.dlogits.float() - dz).abs().max().item() <= 2.0 ** -8 * dz.abs().max().item()
    assert two.stats_dict()["loss"] == pytest.approx(out.stats_dict()["loss"], rel=1e-5)


# ---------------------------------------------------------------------------
# the reference's own golden fixtures through the reference-shaped API


class _Vocab:
    def __init__(self, n):
        self.size = n


class _Params:
    def __init__(self, logits, version=0, vocab=None, num_buckets=0):
        self.logits = np.asarray(logits)
        self.version = version
        self.vocab = vocab or _Vocab(self.logits.shape[1])
        self.num_buckets = num_buckets or self.logits.shape[0]


def _grad_close(report, fx):
    g = report.gradient.to_dense(fx["theta"].shape)
    scale = max(1.0, float(np.max(np.abs(fx["grad"]))))
    assert float(np.max(np.abs(g - fx["grad"]))) / scale <= 1e-5


@pytest.mark.parametrize("name", ["simple_tau05", "simple_tau0", "simple_anchor", "kimi",
                                  "pairwise", "simple_bf16_v512", "kimi_bf16_v512",
                                  "simple_v4_uniform"])
def test_reference_golden_group_losses(name):
    fx = load(name)
    params = _Params(fx["theta"])
    anchor = _Params(fx["anchor"])
    algo = C.AlgorithmConfig(str(fx["variant"]), tau=float(fx["tau"]), beta=float(fx["beta"]))
    rep = C.group_losses(groups_of(fx), params, algo, sft_params=anchor)
    assert rep.loss == pytest.approx(float(fx["loss"]), rel=1e-4, abs=1e-5)
    _grad_close(rep, fx)
    for k, v in zip(fx["metric_names"], fx["metric_values"]):
        assert rep.metrics[str(k)] == pytest.approx(float(v), rel=1e-4, abs=1e-5), k


def test_reference_golden_sft_and_dpo():
    fx = load("sft")
    rep = C.loss_sft(groups_of(fx)[0].experiences, _Params(fx["theta"]))
    assert rep.loss == pytest.approx(float(fx["loss"]), rel=1e-5)
    _grad_close(rep, fx)
    fx = load("dpo")
    g = groups_of(fx)
    pairs = [(x.experiences[0], x.experiences[1]) for x in g]
    rep = C.loss_dpo(pairs, _Params(fx["theta"]), _Params(fx["anchor"]), float(fx["dpo_beta"]))
    assert rep.loss == pytest.approx(float(fx["loss"]), rel=1e-5)
    _grad_close(rep, fx)
    assert rep.metrics["mean_reward"] == pytest.approx(
        dict(zip(fx["metric_names"], fx["metric_values"]))["mean_reward"], rel=1e-4, abs=1e-6)


def test_reference_errors_through_compat():
    fx = load("kimi")
    params = _Params(fx["theta"])
    groups = groups_of(fx)
    with pytest.raises(AlgorithmError):
        C.AlgorithmConfig("OPMD_KIMI", tau=0.0)
    with pytest.raises(AlgorithmError):
        C.group_losses(groups, params, C.AlgorithmConfig("OPMD_SIMPLE", beta=0.5))
    with pytest.raises(AlgorithmError):
        C.group_losses(groups, params, C.AlgorithmConfig("SFT"))
    with pytest.raises(AlgorithmError):
        C.group_losses([type(groups[0])(groups[0].experiences[:1])], params,
                       C.AlgorithmConfig("OPMD_PAIRWISE", tau=1.0))
    with pytest.raises(AlgorithmError):
        C.loss_sft([], params)


# ---------------------------------------------------------------------------
# BASELINE.json configs[2..4] as parity cases (reduced row counts, full vocab)


def test_config3_ppo_k3_entropy_full_vocab_row_sample():
    """configs[2]: PPO clip + low_var_kl + entropy at Qwen vocabulary.  Per-row
    results are checked against the oracle on a sample of rows (the oracle is
    row-separable given the sequence advantages the kernel reports)."""
    V = 151936
    lens, gs = [192] * 8, [4, 4]
    cfg = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl",
                        kl_coef=0.001, entropy_loss_fn="default", entropy_coef=0.001,
                        loss_agg_mode="token-mean", clip_lo=0.2, clip_hi=0.28)
    batch, packed = make_case(21, V, lens, gs)
    out = RFTLoss(cfg)(packed)
    rows = np.random.default_rng(0).choice(batch.n_rows, 48, replace=False)
    sub = O.Batch(logits=batch.logits[rows], target=batch.target[rows],
                  seq_offsets=np.arange(len(rows) + 1), group_offsets=np.array([0, len(rows)]),
                  reward=np.zeros(len(rows)), old_lp=batch.old_lp[rows], ref_lp=batch.ref_lp[rows],
                  advantage=np.repeat(out.seq_adv.double().cpu().numpy(), 192)[rows])
    ref = O.general_loss(sub, oracle_cfg(cfg.with_(advantage_fn="given"),
                                         n_tok_global=batch.n_rows))
    np.testing.assert_allclose(out.lp.double().cpu().numpy()[rows], ref["lp"], rtol=1e-5,
                               atol=1e-4)
    np.testing.assert_allclose(out.entropy.double().cpu().numpy()[rows], ref["entropy"],
                               rtol=1e-5, atol=1e-4)
    d = out.dlogits.float().cpu().numpy()[rows].astype(np.float64)
    r = ref["dz"]
    assert np.all(np.abs(d - r) <= 2.0 ** -8 * np.abs(r).max() + 1e-2 * np.abs(r))
    # GRPO advantages are standardised within each group (an all-equal group -> 0)
    a = out.seq_adv.double().cpu().numpy()
    for g in range(2):
        rew = batch.reward[4 * g:4 * g + 4]
        want = (rew - rew.mean()) / (rew.std(ddof=1) + 1e-6) if rew.std() > 0 else 0 * rew
        np.testing.assert_allclose(a[4 * g:4 * g + 4], want, rtol=1e-5, atol=1e-6)


def test_config4_mixed_grpo_sft_full_vocab():
    """configs[3]: GRPO loss plus SFT NLL on expert trajectories in one batch,
    50/50 mix, vocab 151,936 (the reference runs step_groups and step_sft
    separately; the combined loss is their sum, orchestrator.py:299-315)."""
    V = 151936
    lens = [24] * 8
    kind = [0, 0, 0, 0, 1, 1, 1, 1]
    cfg = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip",
                        loss_agg_mode="token-mean", clip_lo=0.2, clip_hi=0.28, sft_weight=1.0)
    batch, packed = make_case(22, V, lens, [4, 4], seq_kind=kind)
    out = RFTLoss(cfg)(packed)
    ref = O.general_loss(batch, oracle_cfg(cfg))
    compare(out, ref, torch.bfloat16)
    st = out.stats_dict()
    assert st["n_sft_seqs"] == 4 and st["n_tok_rl"] == 96
    # the SFT half equals loss_sft over the expert sequences (algorithms.py:256-274)
    sft = O.ref_sft(batch, seqs=[4, 5, 6, 7])
    assert st["sft_loss"] == pytest.approx(sft.loss, rel=1e-4)


def test_config5_ragged_multiturn_row_index_gather():
    """configs[4]: ragged long-CoT responses with interior mask-false spans.
    The trainable rows are gathered in place from a padded [B*L, V] logits
    tensor through row_index (no compaction copy); results equal the
    compacted layout's."""
    V = 32000
    rng = np.random.default_rng(23)
    B, L = 8, 96
    full = torch.randn((B * L, V), device="cuda", dtype=torch.float32).mul_(2.0).to(torch.bfloat16)
    mask = rng.uniform(size=(B, L)) < 0.85
    for b in range(B):  # ragged: responses end early
        mask[b, int(rng.integers(L // 3, L)):] = False
    lens = mask.sum(axis=1).tolist()
    idx = np.concatenate([np.nonzero(mask[b])[0] + b * L for b in range(B)])
    tgt = rng.integers(0, V, idx.size)
    reward = rng.integers(0, 2, B).astype(np.float32)
    cfg = CONFIGS["grpo_ppo_k3_ent"]
    gathered = pack_arrays(full, tgt, lens, [4, 4], reward, row_index=idx)
    compact = pack_arrays(full[torch.as_tensor(idx, device="cuda")].contiguous(), tgt, lens,
                          [4, 4], reward)
    a = RFTLoss(cfg)(gathered)
    b = RFTLoss(cfg)(compact)
    assert torch.equal(a.lp, b.lp) and torch.equal(a.dlogits, b.dlogits)
    assert torch.equal(a.stats, b.stats)
    lp, _, _, seq_lp = logprob_fwd(gathered)
    assert torch.allclose(lp, a.lp, atol=1e-4)


def _neg_inf_in_some_rows(batch, packed, every=5, fill=-5.0):
    """Keep the -inf logits (and anchor logits) only in rows r % every == 2; the
    other rows get a finite `fill` there, on the host and on the device alike --
    rows with and without masked vocabulary interleave in every warp's stream."""
    keep = (np.arange(batch.logits.shape[0]) % every) == 2
    for host, dev in ((batch.logits, packed.logits),
                      (getattr(batch, "anchor_logits", None), packed.anchor_logits)):
        if host is None or dev is None:
            continue
        m = np.isinf(host) & ~keep[:, None]
        host[m] = fill
        dev.copy_(torch.as_tensor(host, device=dev.device).to(dev.dtype))
    return keep


@pytest.mark.parametrize("shape", ["v32000", "v151936"])
def test_masked_vocab_in_some_rows_only(shape):
    """Rows with and without masked vocabulary interleaved in every warp's row
    stream (the speculative phase 1 holds on the finite rows and falls back to
    the checked path on the others), entropy bonus on (hz z)."""
    cfg = CONFIGS["grpo_ppo_k3_ent"]
    V, lens, gs = SHAPES[shape]
    batch, packed = make_case(12, V, lens, gs, neg_inf=0.2)
    _neg_inf_in_some_rows(batch, packed)
    out = RFTLoss(cfg)(packed, dlogits="new")
    ref = O.general_loss(batch, oracle_cfg(cfg))
    assert out.stats_dict()["nonfinite"] == 0
    assert bool(torch.isfinite(out.dlogits.float()).all())
    compare(out, ref, torch.bfloat16)


def test_fused_anchor_kl_masked_vocabulary_in_some_rows():
    """The anchor path's phase 2 (split stash at V = 151,936) with -inf in a few
    rows of both the logits and the anchor logits, against the two-pass route."""
    V, lens, gs = SHAPES["v151936"]
    cfg = RFTLossConfig.from_variant("OPMD_SIMPLE", tau=0.4, beta=0.9)
    batch, packed = make_case(13, V, [61, 47, 70, 55], gs, dtype=torch.bfloat16, anchor=True,
                              neg_inf=0.02)
    _neg_inf_in_some_rows(batch, packed)
    out = RFTLoss(cfg)(packed, dlogits="new")
    two = RFTLoss(cfg.with_(force_two_pass=True))(packed, dlogits="new")
    a, b = out.stats_dict(), two.stats_dict()
    assert a["nonfinite"] == 0
    for k in ("loss", "anchor_loss", "sum_anchor_kl", "sum_lp", "sum_entropy"):
        assert a[k] == pytest.approx(b[k], rel=1e-4, abs=1e-5), k
    d, r = out.dlogits.float(), two.dlogits.float()
    assert bool(torch.isfinite(d).all())
    assert bool(((d - r).abs() <= 2.0 ** -8 * float(r.abs().max()) + 1e-2 * r.abs()).all())
