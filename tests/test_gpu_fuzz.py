"""Randomised parity sweep: 160 seeded combinations of the registry components
(advantage x policy loss x KL x entropy x aggregation), anchor KL, mixed SFT
sequences, dtype, vocabulary size, padded pitch and the unscaled coupled
route, each against the oracle with the tolerances of test_gpu_parity.py.
Pins the interactions the per-feature tests do not enumerate (e.g. the fused
anchor path under PPO + entropy + token-mean).  TG_FUZZ_SEEDS=n widens the
sweep (profiles/r02_fuzz_1000.txt: 1,000 seeds on the round-2 final tree)."""

import numpy as np
import pytest
import torch

from _cases import make_case, oracle_cfg
from oracle import rft_oracle as O
from paper_2505_17826_b200 import RFTLoss, RFTLossConfig

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

from test_gpu_parity import compare  # noqa: E402

AGGS = ["seq-sum", "token-mean", "seq-mean-token-sum", "seq-mean-token-mean",
        "seq-mean-token-sum-norm"]


def draw(seed):
    r = np.random.default_rng(1000 + seed)
    pg = str(r.choice(["vanilla", "ppo_clip", "ppo_clip", "sft", "opmd_kimi", "opmd_pairwise"]))
    coupled = pg in ("opmd_kimi", "opmd_pairwise")
    kl = str(r.choice(["none", "k1", "k2", "k3", "abs"]))
    ent = str(r.choice(["none", "default"]))
    kw = dict(advantage_fn=str(r.choice(["grpo", "rloo", "opmd", "reinforce"])),
              policy_loss_fn=pg, kl_fn=kl, kl_coef=0.0 if kl == "none" else float(r.choice([0.01, 0.1])),
              entropy_loss_fn=ent, entropy_coef=0.0 if ent == "none" else float(r.choice([0.001, 0.01])),
              loss_agg_mode=str(r.choice(AGGS)), agg_norm=64.0,
              tau=float(r.choice([0.5, 1.0])) if coupled else float(r.choice([0.0, 0.5])),
              clip_lo=0.2, clip_hi=float(r.choice([0.2, 0.28])),
              clip_c=float(r.choice([0.0, 3.0])) if pg == "ppo_clip" else 0.0)
    if coupled:  # the coupled losses take no token KL / entropy bonus / aggregation
        kw.update(kl_fn="none", kl_coef=0.0, entropy_loss_fn="none", entropy_coef=0.0,
                  loss_agg_mode="seq-sum")
    anchor = bool(r.random() < 0.3)
    if anchor:
        kw["anchor_beta"] = float(r.choice([0.1, 0.5]))
    dtype = torch.float32 if r.random() < 0.25 else torch.bfloat16
    V = int(r.choice([64, 1000, 4097, 32000, 32000, 151936]))
    K = int(r.choice([2, 3, 4]))
    G = int(r.choice([1, 2, 3])) if V < 151936 else 1
    lens = [int(x) for x in r.integers(0 if V < 151936 else 1, 41 if V < 151936 else 9, K * G)]
    seq_kind = None
    if not coupled and r.random() < 0.3:
        seq_kind = [int(x) for x in r.integers(0, 2, K * G)]
        kw["sft_weight"] = float(r.choice([0.5, 1.0]))
    ld = None
    if r.random() < 0.3:
        ld = V + int(r.choice([8, 64]))
    unscaled = coupled and not anchor and r.random() < 0.5
    return kw, anchor, dtype, V, K, G, lens, seq_kind, ld, unscaled


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("TG_FUZZ_SEEDS", 160))))
def test_random_configuration_matches_oracle(seed):
    kw, anchor, dtype, V, K, G, lens, seq_kind, ld, unscaled = draw(seed)
    cfg = RFTLossConfig(**kw)
    batch, packed = make_case(seed, V, lens, [K] * G, dtype=dtype, anchor=anchor,
                              seq_kind=seq_kind, ld=ld)
    loss = RFTLoss(cfg)
    if unscaled:
        out = loss(packed, dlogits="new", unscaled=True)
        out.dlogits = out.dlogits.float() * out.row_scale[:, None]
    else:
        out = loss(packed, dlogits="new")
    # sequence-coupled coefficients are differences of sequence sums of fp32 row
    # logprobs (pairwise: a_i - a_j), so near-cancelling groups carry ~1e-4
    # relative error in fp32; per-row losses keep the parity-matrix bar
    coupled = cfg.policy_loss_fn in ("opmd_kimi", "opmd_pairwise")
    compare(out, O.general_loss(batch, oracle_cfg(cfg)), dtype,
            rtol_dz=1e-3 if coupled and dtype == torch.float32 else None)
