"""The fused AdamW step (tg_adamw_step) against
torch.optim.AdamW: fp32 parameters over several steps, bf16 parameters and
gradients against the same update in fp32 arithmetic, row pitches (a column
slice of the LM head), the scalar path (cols not a multiple of 8), the
non-finite refusal (apply_update's rule, algorithms.py:337-338) and the
argument checks."""

import numpy as np
import pytest
import torch

from paper_2505_17826_b200 import AlgorithmError, LMHeadAdamW, adamw_step
from paper_2505_17826_b200._native import NativeError

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

HP = dict(lr=3e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)


def _ref_fp32(p, g, m, v, step, lr, betas, eps, weight_decay):
    """torch.optim.AdamW's single-tensor update in fp32 (the restatement the
    bf16 case is checked against: same inputs, fp32 arithmetic)."""
    b1, b2 = betas
    p = p * (1 - lr * weight_decay)
    m = m.lerp(g, 1 - b1)
    v = v * b2 + (1 - b2) * g * g
    denom = v.sqrt() / (1 - b2 ** step) ** 0.5 + eps
    return p - lr / (1 - b1 ** step) * m / denom, m, v


@pytest.mark.parametrize("rows,cols", [(300, 1536), (77, 1000), (5, 13)])
def test_fp32_matches_torch_adamw_over_steps(rows, cols):
    g = torch.Generator(device="cuda").manual_seed(rows + cols)
    w0 = torch.randn(rows, cols, device="cuda", generator=g)
    ref = torch.nn.Parameter(w0.clone())
    opt = torch.optim.AdamW([ref], foreach=False, **HP)
    w = w0.clone()
    m = torch.zeros_like(w)
    v = torch.zeros_like(w)
    for step in range(1, 5):
        grad = torch.randn(rows, cols, device="cuda", generator=g) * 10 ** (step - 3)
        ref.grad = grad.clone()
        opt.step()
        adamw_step(w, grad, m, v, step, **HP)
        st = opt.state[ref]
        # (m + (1 - b1)(g - m) in one FMA here, a multiply and an add in torch:
        # an ulp of the operands apart, absolute where m nearly cancels)
        torch.testing.assert_close(m, st["exp_avg"], rtol=1e-6,
                                   atol=1e-6 * float(st["exp_avg"].abs().max()))
        torch.testing.assert_close(v, st["exp_avg_sq"], rtol=1e-6,
                                   atol=1e-6 * float(st["exp_avg_sq"].abs().max()))
        torch.testing.assert_close(w, ref.detach(), rtol=2e-6, atol=1e-7)


@pytest.mark.parametrize("cols", [1536, 1000, 77])
def test_bf16_param_and_grad_match_fp32_arithmetic(cols):
    rows = 129
    g = torch.Generator(device="cuda").manual_seed(cols)
    # a column slice of a wider LM head: row pitch > cols
    full = (torch.randn(rows, cols + 24, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    w = full[:, 8:8 + cols]
    grad = (torch.randn(rows, cols, device="cuda", generator=g) * 1e-2).to(torch.bfloat16)
    m = torch.randn(rows, cols, device="cuda", generator=g) * 1e-3
    v = torch.rand(rows, cols, device="cuda", generator=g) * 1e-4
    want_p, want_m, want_v = _ref_fp32(w.float(), grad.float(), m.clone(), v.clone(), 7, **HP)
    before = full.clone()
    adamw_step(w, grad, m, v, 7, **HP)
    torch.testing.assert_close(m, want_m, rtol=1e-6, atol=1e-6 * float(want_m.abs().max()))
    torch.testing.assert_close(v, want_v, rtol=1e-6, atol=1e-6 * float(want_v.abs().max()))
    # bf16 rounding of the same fp32 update: equal, or one rounding step apart
    # where the fp32 values straddle a bf16 rounding boundary
    exact = (w == want_p.to(torch.bfloat16)).float().mean().item()
    assert exact >= 0.99, exact
    torch.testing.assert_close(w.float(), want_p, rtol=2 ** -7, atol=1e-6)
    # the columns outside the slice are untouched
    assert torch.equal(full[:, :8], before[:, :8]) and torch.equal(full[:, 8 + cols:],
                                                                     before[:, 8 + cols:])


def test_mixed_dtypes_bf16_param_fp32_grad():
    g = torch.Generator(device="cuda").manual_seed(3)
    w = (torch.randn(64, 256, device="cuda", generator=g)).to(torch.bfloat16)
    grad = torch.randn(64, 256, device="cuda", generator=g)
    m, v = torch.zeros(64, 256, device="cuda"), torch.zeros(64, 256, device="cuda")
    want_p, _, _ = _ref_fp32(w.float(), grad, m.clone(), v.clone(), 1, **HP)
    adamw_step(w, grad, m, v, 1, **HP)
    torch.testing.assert_close(w.float(), want_p, rtol=2 ** -7, atol=1e-6)


@pytest.mark.parametrize("bad", [float("nan"), float("inf")])
def test_non_finite_gradient_is_refused_before_any_write(bad):
    w = torch.randn(40, 96, device="cuda").to(torch.bfloat16)
    grad = torch.randn(40, 96, device="cuda").to(torch.bfloat16)
    grad[17, 33] = bad
    m, v = torch.rand(40, 96, device="cuda"), torch.rand(40, 96, device="cuda")
    w0, m0, v0 = w.clone(), m.clone(), v.clone()
    with pytest.raises(AlgorithmError):
        adamw_step(w, grad, m, v, 3, **HP)
    assert torch.equal(w, w0) and torch.equal(m, m0) and torch.equal(v, v0)
    opt = LMHeadAdamW(w, **HP)
    with pytest.raises(AlgorithmError):
        opt.step(grad)
    assert opt.t == 0 and torch.equal(w, w0)


def test_argument_errors():
    w = torch.zeros(8, 16, device="cuda")
    g = torch.zeros(8, 16, device="cuda")
    m, v = torch.zeros_like(w), torch.zeros_like(w)
    with pytest.raises(NativeError):
        adamw_step(w, g, m, v, 1, lr=1e-3, betas=(1.0, 0.999))
    with pytest.raises(NativeError):
        adamw_step(w, g, m, v, 0)
    with pytest.raises(NativeError):
        adamw_step(w, g, m, v, 1, lr=-1.0)
    with pytest.raises(ValueError):
        adamw_step(w, g[:, :8], m, v, 1)
    with pytest.raises(ValueError):
        adamw_step(w, g, m.to(torch.bfloat16), v, 1)


def test_lmhead_training_steps_with_fused_adamw():
    """Two training steps of an LM head from hidden states: the logits-free
    loss + backward (tcgen05) feeding the fused AdamW; the loss goes down."""
    from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, lmhead_loss_fwd_bwd
    T, V, d = 512, 4096, 256
    g = torch.Generator(device="cuda").manual_seed(11)
    h = torch.randn(T, d, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(V, d, device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    y = np.random.default_rng(0).integers(0, V, T)
    loss = RFTLoss(RFTLossConfig(advantage_fn="grpo", policy_loss_fn="vanilla",
                                 loss_agg_mode="token-mean"))
    opt = LMHeadAdamW(w, lr=1e-2, weight_decay=0.0)
    losses = []
    for _ in range(3):
        out, dh, dw = lmhead_loss_fwd_bwd(h, w, loss, y, [T // 4] * 4, [4],
                                          np.array([1., 0., 1., 0.], np.float32))
        losses.append(out.stats_dict()["loss"])
        opt.step(dw)
    assert opt.t == 3 and all(np.isfinite(losses))
    assert losses[-1] < losses[0], losses


def test_checkpoint_resume_is_bitwise():
    """state_dict / load_state_dict: 2 steps, checkpoint (weight + optimizer
    state through torch.save), resume in a fresh optimizer, 2 more steps ==
    4 uninterrupted steps, bit for bit."""
    import io
    g = torch.Generator(device="cuda").manual_seed(21)
    w0 = (torch.randn(96, 512, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    grads = [(torch.randn(96, 512, device="cuda", generator=g) * 1e-2).to(torch.bfloat16)
             for _ in range(4)]
    w_a = w0.clone()
    opt_a = LMHeadAdamW(w_a, **HP)
    for gr in grads:
        opt_a.step(gr)
    w_b = w0.clone()
    opt_b = LMHeadAdamW(w_b, **HP)
    for gr in grads[:2]:
        opt_b.step(gr)
    buf = io.BytesIO()
    torch.save({"weight": w_b, "opt": opt_b.state_dict()}, buf)
    buf.seek(0)
    ck = torch.load(buf)
    w_c = ck["weight"].clone()
    opt_c = LMHeadAdamW(w_c)  # default hyper-parameters, restored from the checkpoint
    opt_c.load_state_dict(ck["opt"])
    assert opt_c.t == 2 and opt_c.betas == HP["betas"]
    for gr in grads[2:]:
        opt_c.step(gr)
    assert torch.equal(w_c, w_a)
    assert torch.equal(opt_c.exp_avg, opt_a.exp_avg) and torch.equal(opt_c.exp_avg_sq,
                                                                     opt_a.exp_avg_sq)
