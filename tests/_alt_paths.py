"""Run in a subprocess by test_gpu_alt_paths.py: the environment selects an
alternative kernel (TG_FUSED_IMPL=2: the L2-reread fused kernel;
TG_LMHEAD_PAIR=1: the 2-CTA LM-head kernel), read once per process.  Exits
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
    {"fused": fused, "lmhead": lmhead}[sys.argv[1]]()
    print("ok")
