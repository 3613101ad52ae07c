"""Run in a subprocess by test_gpu_alt_paths.py: the environment selects an
alternative kernel (TG_FUSED_IMPL=2: the L2-reread fused kernel;
TG_LMHEAD_PAIR=0: the single-CTA LM-head kernel), read once per process.  Exits
non-zero on a parity failure."""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402


def fused():
    from _cases import make_case, oracle_cfg
    from test_gpu_parity import CONFIGS, compare

    from oracle import rft_oracle as O
    from paper_2505_17826_b200 import RFTLoss

    for name in ("grpo_ppo_k3_ent", "opmd_simple"):
        for V, lens in ((32000, [64] * 8), (151936, [24] * 4)):
            cfg = CONFIGS[name]
            batch, packed = make_case(5, V, lens, [len(lens) // 2] * 2)
            loss = RFTLoss(cfg)
            assert loss.route(packed) == 1
            out = loss(packed)
            compare(out, O.general_loss(batch, oracle_cfg(cfg)), torch.bfloat16)


def anchor():
    """The fused anchor KL's other stash modes at Qwen vocabulary (the default
    there is mode 3, the split stash): TG_FUSED_ANCHOR_MODE=1 (z + za in TMEM,
    4-CTA clusters) or 2 (z in TMEM, za re-read from L2, 2-CTA clusters)."""
    import os

    from _cases import make_case, oracle_cfg
    from test_gpu_parity import compare

    from oracle import rft_oracle as O
    from paper_2505_17826_b200 import RFTLoss, RFTLossConfig

    cfg = RFTLossConfig.from_variant("OPMD_SIMPLE", tau=0.4, beta=0.9)
    mode = os.environ["TG_FUSED_ANCHOR_MODE"]
    # mode 1 holds a bf16 row in 4-CTA slices only (fp32 rows do not fit it);
    # mode 2: bf16 on 2-CTA, fp32 on 4-CTA clusters
    cases = {"1": [(torch.bfloat16, 4)], "2": [(torch.bfloat16, 2), (torch.float32, 4)]}[mode]
    for dtype, want_cl in cases:
        lens = [24] * 8 if dtype == torch.bfloat16 else [12] * 4
        batch, packed = make_case(6, 151936, lens, [len(lens) // 2] * 2, dtype=dtype,
                                  anchor=True)
        loss = RFTLoss(cfg)
        assert loss.route(packed) == 1 and loss.cluster_size(packed) == want_cl
        compare(loss(packed, dlogits="new"), O.general_loss(batch, oracle_cfg(cfg)), dtype)


def lmhead():
    from paper_2505_17826_b200 import lmhead_logprob_fwd

    torch.backends.cuda.matmul.allow_tf32 = False
    for T, V, d in ((300, 1000, 128), (1000, 32000, 512), (37888, 1000, 64)):
        g = torch.Generator(device="cuda").manual_seed(T)
        h = torch.randn(T, d, device="cuda", generator=g).to(torch.bfloat16)
        w = (torch.randn(V, d, device="cuda", generator=g) / d ** 0.5 * 3).to(torch.bfloat16)
        y = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
        lp, ent, lse = lmhead_logprob_fwd(h, w, y)
        z = h.float() @ w.float().T
        rlse = torch.logsumexp(z, 1)
        torch.testing.assert_close(lse, rlse, atol=2e-4, rtol=1e-5)
        torch.testing.assert_close(lp, z.gather(1, y.long()[:, None])[:, 0] - rlse, atol=2e-4,
                                   rtol=1e-5)
        rent = rlse - (torch.softmax(z, 1) * z).sum(1)
        torch.testing.assert_close(ent, rent, atol=2e-4, rtol=1e-4)


if __name__ == "__main__":
    {"fused": fused, "lmhead": lmhead, "anchor": anchor}[sys.argv[1]]()
    print("ok")
