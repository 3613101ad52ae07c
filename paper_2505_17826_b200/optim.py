"""The optimizer step after the loss path.

``adamw_step`` is one fused AdamW update of a 2-D parameter block on the device
(``tg_adamw_step``: torch.optim.AdamW semantics, decoupled weight decay, one
HBM pass); ``LMHeadAdamW`` keeps the fp32 moments of an LM-head weight and
steps it from the d W that ``lmhead_loss_fwd_bwd`` / ``lmhead_grad_*`` produce.
The reference's own optimizer is plain SGD on its logits table
(algorithms.apply_update, algorithms.py:329-348: ``tg_apply_update``,
``triad_compat.Trainer``); this is its LLM-scale counterpart, and it refuses
a non-finite gradient the same way (nothing written, AlgorithmError).
"""

from __future__ import annotations

from typing import Optional, Tuple

import torch

from . import _native as N
from .config import AlgorithmError

_DT = {torch.bfloat16: N.TG_DTYPE_BF16, torch.float32: N.TG_DTYPE_F32}


def _check_2d(name: str, t: torch.Tensor, dev, dtypes) -> None:
    if t.device != dev or t.dim() != 2 or t.stride(1) != 1 or t.dtype not in dtypes:
        raise ValueError(f"{name} must be a 2-D {'/'.join(map(str, dtypes))} tensor on {dev} "
                         "with unit column stride")


def adamw_step(param: torch.Tensor, grad: torch.Tensor, exp_avg: torch.Tensor,
               exp_avg_sq: torch.Tensor, step: int, lr: float = 1e-3,
               betas: Tuple[float, float] = (0.9, 0.999), eps: float = 1e-8,
               weight_decay: float = 1e-2, check_finite: bool = True,
               stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """One AdamW step of ``param`` ([rows, cols], bf16 or fp32, any row pitch)
    from ``grad`` (bf16 or fp32, same shape) with fp32 moments ``exp_avg`` /
    ``exp_avg_sq`` (contiguous, same shape), in place; ``step`` is the 1-based
    step count (bias correction).  ``check_finite``: a non-finite gradient
    raises AlgorithmError and leaves all three tensors unchanged (this reads
    the status word back, i.e. synchronises the stream)."""
    dev = param.device
    _check_2d("param", param, dev, _DT)
    _check_2d("grad", grad, dev, _DT)
    for name, t in (("exp_avg", exp_avg), ("exp_avg_sq", exp_avg_sq)):
        if t.device != dev or t.dtype != torch.float32 or not t.is_contiguous() or \
                t.shape != param.shape:
            raise ValueError(f"{name} must be a contiguous float32 tensor of shape "
                             f"{tuple(param.shape)} on {dev}")
    if grad.shape != param.shape:
        raise ValueError(f"grad shape {tuple(grad.shape)} != param shape {tuple(param.shape)}")
    rows, cols = param.shape
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.device(dev), torch.cuda.stream(s):
        status = torch.zeros(1, dtype=torch.int32, device=dev) if check_finite else None
        N.check(N.lib().tg_adamw_step(
            param.data_ptr(), _DT[param.dtype], param.stride(0), grad.data_ptr(),
            _DT[grad.dtype], grad.stride(0), exp_avg.data_ptr(), exp_avg_sq.data_ptr(), rows,
            cols, float(lr), float(betas[0]), float(betas[1]), float(eps), float(weight_decay),
            int(step), status.data_ptr() if status is not None else None, s.cuda_stream))
        if status is not None and int(status.item()) != 0:
            raise AlgorithmError("refusing to apply a non-finite gradient")
    return param


class LMHeadAdamW:
    """AdamW state of one LM-head weight ``[V, d]`` (fp32 moments on the same
    device): ``step(d_weight)`` applies one fused update in place.  Mirrors
    ``torch.optim.AdamW(params=[weight], lr, betas, eps, weight_decay)`` for a
    single parameter, without autograd."""

    def __init__(self, weight: torch.Tensor, lr: float = 1e-3,
                 betas: Tuple[float, float] = (0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 1e-2, check_finite: bool = True) -> None:
        self.weight = weight
        self.lr, self.betas, self.eps, self.weight_decay = lr, betas, eps, weight_decay
        self.check_finite = check_finite
        self.exp_avg = torch.zeros(weight.shape, dtype=torch.float32, device=weight.device)
        self.exp_avg_sq = torch.zeros_like(self.exp_avg)
        self.t = 0

    def step(self, d_weight: torch.Tensor) -> None:
        adamw_step(self.weight, d_weight, self.exp_avg, self.exp_avg_sq, self.t + 1, self.lr,
                   self.betas, self.eps, self.weight_decay, self.check_finite)
        self.t += 1  # only after a successful (non-refused) step

    def state_dict(self) -> dict:
        """Checkpoint of the optimizer state (moments cloned, on their device),
        the counterpart of torch.optim.Optimizer.state_dict for this parameter."""
        return {"step": self.t, "exp_avg": self.exp_avg.clone(),
                "exp_avg_sq": self.exp_avg_sq.clone(),
                "hyper": {"lr": self.lr, "betas": tuple(self.betas), "eps": self.eps,
                          "weight_decay": self.weight_decay}}

    def load_state_dict(self, state: dict) -> None:
        """Resume from ``state_dict()``: the next step continues the bias
        correction at step + 1 with the saved moments."""
        for k in ("exp_avg", "exp_avg_sq"):
            if tuple(state[k].shape) != tuple(self.weight.shape):
                raise ValueError(f"{k} shape {tuple(state[k].shape)} does not match the weight")
        self.exp_avg.copy_(state["exp_avg"])
        self.exp_avg_sq.copy_(state["exp_avg_sq"])
        self.t = int(state["step"])
        h = state.get("hyper", {})
        self.lr = h.get("lr", self.lr)
        self.betas = tuple(h.get("betas", self.betas))
        self.eps = h.get("eps", self.eps)
        self.weight_decay = h.get("weight_decay", self.weight_decay)
