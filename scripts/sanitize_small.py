"""Small invocations of every kernel in libtg_loss.so, for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_small.py

Covers the fused single-pass kernel (bf16 CL = 2 and CL = 1, fp32 CL = 4), the
two-pass and coupled routes, the forward-only logprob kernels, the anchor KL,
the LM-head forward (single and 2-CTA) and backward chunk kernels, the
backward GEMMs, the packer, the update kernel and the fused AdamW.  Exits non-zero on a result mismatch against the
fp32 torch reference computed here."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2505_17826_b200 import (RFTLoss, RFTLossConfig, lmhead_dlogits,  # noqa: E402
                                   lmhead_logprob_fwd, lmhead_loss_fwd_bwd, logprob_fwd,
                                   pack_arrays)


def loss_paths():
    rng = np.random.default_rng(0)
    for V, dtype in ((151936, torch.bfloat16), (32000, torch.bfloat16), (151936, torch.float32)):
        lens, groups = [5, 3, 4, 2], [2, 2]
        T = sum(lens)
        z = (torch.randn(T, V, device="cuda") * 2).to(dtype)
        y = rng.integers(0, V, T)
        rew = rng.integers(0, 2, len(lens)).astype(np.float32)
        old = rng.normal(-8, 0.5, T).astype(np.float32)
        for kw in (dict(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl",
                        kl_coef=1e-3, loss_agg_mode="token-mean"),
                   dict(advantage_fn="grpo", policy_loss_fn="ppo_clip", entropy_loss_fn="default",
                        entropy_coef=1e-3, loss_agg_mode="token-mean"),
                   dict(policy_loss_fn="opmd_kimi", tau=0.5)):
            loss = RFTLoss(RFTLossConfig(**kw))
            b = pack_arrays(z.clone(), y, lens, groups, rew, old_lp=old, ref_lp=old)
            out = loss(b, dlogits="new")
            out2 = loss(b, dlogits="inplace")
            torch.cuda.synchronize()
            assert torch.equal(out.dlogits, b.logits), "in-place dlogits differ"
            out.metrics()
            if loss.cfg.coupled:  # route 4: one pass, unscaled gradient + row scales
                loss(pack_arrays(z.clone(), y, lens, groups, rew, old_lp=old, ref_lp=old),
                     dlogits="new", unscaled=True).metrics()
        logprob_fwd(pack_arrays(z, y, lens, groups, rew))


def anchor_paths():
    rng = np.random.default_rng(1)
    # anchor KL (regularizer_g): mode 1 (V = 4096) and the split stash (mode 3:
    # bf16 2-CTA and fp32 4-CTA clusters at V = 151,936; enough rows per cluster
    # for the 13-position period to wrap)
    for V, dtype, T in ((4096, torch.bfloat16, 6), (151936, torch.bfloat16, 300),
                        (151936, torch.float32, 140)):
        z = torch.randn(T, V, device="cuda").to(dtype)
        q = torch.randn(T, V, device="cuda").to(dtype)
        loss = RFTLoss(RFTLossConfig(policy_loss_fn="opmd_simple", anchor_beta=0.1))
        lens = [T // 2, T - T // 2]
        loss(pack_arrays(z, rng.integers(0, V, T), lens, [2], np.array([0., 1.], np.float32),
                         anchor_logits=q), dlogits="new").metrics()


def lmhead_paths():
    T, V, d = 300, 1000, 128
    h = torch.randn(T, d, device="cuda").to(torch.bfloat16)
    w = (torch.randn(V, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
    y = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
    lp, ent, lse = lmhead_logprob_fwd(h, w, y)
    z = h.float() @ w.float().T
    torch.testing.assert_close(lse, torch.logsumexp(z, 1), atol=2e-4, rtol=1e-5)
    loss = RFTLoss(RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip",
                                 loss_agg_mode="token-mean"))
    out, dh, dw = lmhead_loss_fwd_bwd(h, w, loss, y.cpu().numpy(), [100, 100, 100], [3],
                                      np.array([0., 1., 1.], np.float32), chunk_cols=384)
    lmhead_dlogits(h, w, out.target, out.lse, out.row_coef, 333, 500)
    torch.cuda.synchronize()
    assert torch.isfinite(dh).all()


def optim_paths():
    from paper_2505_17826_b200 import adamw_step
    for dt in (torch.bfloat16, torch.float32):
        for cols in (256, 77):  # vector units / the scalar path
            w = torch.randn(33, cols, device="cuda").to(dt)
            g = torch.randn(33, cols, device="cuda").to(dt)
            m, v = torch.zeros(33, cols, device="cuda"), torch.zeros(33, cols, device="cuda")
            adamw_step(w, g, m, v, 1, check_finite=True)
            adamw_step(w, g, m, v, 2, check_finite=False)
    torch.cuda.synchronize()


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "loss"):
        loss_paths()
    if which in ("all", "loss", "anchor"):
        anchor_paths()
    if which in ("all", "lmhead"):
        lmhead_paths()
    if which in ("all", "optim"):
        optim_paths()
    torch.cuda.synchronize()
    print("sanitize_small ok", os.environ.get("TG_LMHEAD_PAIR", ""))
