"""Public API: the fused RFT loss over packed device tensors.

``RFTLoss(cfg)(batch)`` enqueues the CUDA pipeline of ``tg_loss_fwd_bwd`` on
the current torch stream and returns device tensors (loss statistics,
per-row logprob / entropy, per-sequence LP and advantage, and dlogits).
Nothing synchronises until ``LossOutput.metrics()`` reads the 256-byte stats
vector back.  Replaces ``group_loss`` over a batch + ``combine_reports``
(algorithms.py:351-379) -- see triad_compat.py for the reference-shaped
wrappers.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Dict, Optional, Union

import numpy as np
import torch

from . import _native as N
from .config import AlgorithmError, RFTLossConfig
from .packing import PackedBatch

_DTYPES = {torch.bfloat16: N.TG_DTYPE_BF16, torch.float32: N.TG_DTYPE_F32}


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _check_dev(t: Optional[torch.Tensor], dev: torch.device, name: str, dtype=None):
    if t is None:
        return
    if t.device != dev:
        raise ValueError(f"{name} is on {t.device}, expected {dev}")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def c_batch(b: PackedBatch) -> N.TgBatch:
    """PackedBatch -> TgBatch (device pointers, no copies)."""
    lg = b.logits
    if lg.dim() != 2:
        raise ValueError("logits must be 2-D [rows, ld] (flatten [B, L, V] first)")
    if lg.dtype not in _DTYPES:
        raise ValueError(f"logits dtype {lg.dtype} unsupported (bf16 or f32)")
    if lg.numel() and lg.stride(1) != 1:
        raise ValueError("logits rows must be contiguous (stride(1) == 1)")
    dev = lg.device
    if dev.type != "cuda":
        raise RuntimeError("the RFT loss runs only on CUDA devices (no CPU fallback)")
    _check_dev(b.target, dev, "target", torch.int32)
    _check_dev(b.seq_offsets, dev, "seq_offsets", torch.int32)
    _check_dev(b.group_offsets, dev, "group_offsets", torch.int32)
    _check_dev(b.reward, dev, "reward", torch.float32)
    for name in ("old_lp", "ref_lp", "seq_ref_lp", "advantage", "pg_coef", "pg_loss"):
        _check_dev(getattr(b, name), dev, name, torch.float32)
    _check_dev(b.seq_kind, dev, "seq_kind", torch.uint8)
    _check_dev(b.row_index, dev, "row_index", torch.int64)
    # element counts the C ABI cannot see (plain pointers; ranges of device
    # values are the packer's job -- checking them here would sync)
    T, B, G = b.n_rows, b.n_seqs, b.n_groups
    for name, n in (("target", T), ("seq_offsets", B + 1), ("group_offsets", G + 1),
                    ("reward", B), ("old_lp", T), ("ref_lp", T), ("seq_ref_lp", B),
                    ("advantage", B), ("seq_kind", B), ("row_index", T), ("pg_coef", T),
                    ("pg_loss", T)):
        t = getattr(b, name)
        if t is not None and t.numel() != n:
            raise ValueError(f"{name} has {t.numel()} entries, expected {n}")
    if b.row_index is None and lg.numel() and lg.shape[0] < T:
        raise ValueError(f"logits has {lg.shape[0]} rows for {T} trainable rows")
    if b.anchor_logits is not None and (b.anchor_logits.shape[0] < T or
                                        b.anchor_logits.shape[1] < b.vocab):
        raise ValueError("anchor_logits must hold one row of >= vocab columns per trainable row")
    c = N.TgBatch()
    c.dtype = _DTYPES[lg.dtype]
    c.n_seqs, c.n_groups = b.n_seqs, b.n_groups
    c.n_rows, c.vocab = b.n_rows, b.vocab
    c.ld = lg.stride(0) if lg.numel() else max(b.vocab, 1)
    c.logits = lg.data_ptr()
    c.row_index = _ptr(b.row_index)
    if b.anchor_logits is not None:
        a = b.anchor_logits
        if a.dtype != lg.dtype or a.device != dev or a.stride(1) != 1:
            raise ValueError("anchor_logits must match logits' dtype / device / row layout")
        c.anchor_logits = a.data_ptr()
        c.ld_anchor = a.stride(0)
    c.target = b.target.data_ptr()
    c.old_lp, c.ref_lp = _ptr(b.old_lp), _ptr(b.ref_lp)
    c.seq_offsets, c.group_offsets = b.seq_offsets.data_ptr(), b.group_offsets.data_ptr()
    c.reward = b.reward.data_ptr()
    c.seq_ref_lp, c.advantage, c.seq_kind = _ptr(b.seq_ref_lp), _ptr(b.advantage), _ptr(b.seq_kind)
    c.pg_coef, c.pg_loss = _ptr(b.pg_coef), _ptr(b.pg_loss)
    return c


def _coupled_rows(cfg: RFTLossConfig, batch: PackedBatch, cb: N.TgBatch) -> None:
    """Sequence-coupled losses take RL rollouts only (the C ABI refuses a
    seq_kind array for them): SFT sequences are an error, an all-RL seq_kind
    is dropped."""
    if cfg.coupled:
        if batch.n_sft_seqs > 0:
            raise AlgorithmError(f"{cfg.policy_loss_fn} takes no SFT sequences "
                                 f"({batch.n_sft_seqs} in the batch)")
        cb.seq_kind = None


@dataclass
class LossOutput:
    stats: torch.Tensor                   # [32] float64 (layout _native.STAT_NAMES)
    lp: torch.Tensor                      # [T] f32
    entropy: torch.Tensor                 # [T] f32
    lse: torch.Tensor                     # [T] f32
    seq_lp: torch.Tensor                  # [B] f32
    seq_adv: torch.Tensor                 # [B] f32 (advantage, or coupled coefficient)
    dlogits: Optional[torch.Tensor] = None
    row_coef: Optional[torch.Tensor] = None  # [3, T] f32 (a, hz, s), when requested
    target: Optional[torch.Tensor] = None    # [T] i32 packed targets (loss from hidden states)

    @property
    def row_scale(self) -> Optional[torch.Tensor]:
        """Per-row factor of an unscaled gradient (``unscaled=True``): s_t."""
        return None if self.row_coef is None else self.row_coef[2]

    def stats_dict(self) -> Dict[str, float]:
        """Device -> host read of the statistics (the only sync)."""
        host = self.stats.detach().cpu().tolist()
        return {n: host[i] for i, n in enumerate(N.STAT_NAMES) if not n.startswith("reserved")}

    def metrics(self, check: bool = True) -> Dict[str, float]:
        """combine_reports-style metrics (algorithms.py:377-378): group means."""
        return stats_to_metrics(self.stats_dict(), check=check)


def stats_to_metrics(s: Dict[str, float], check: bool = True) -> Dict[str, float]:
    if check:
        if s["invalid"] > 0:
            raise AlgorithmError(f"{int(s['invalid'])} invalid rows/groups in the batch "
                                 "(target outside the vocabulary or bad group shape)")
        if s["nonfinite"] > 0:
            raise AlgorithmError(f"loss must be finite, got {s['loss']} "
                                 f"({int(s['nonfinite'])} non-finite rows)")
    ng = max(s["n_groups"], 1.0)
    ntok = max(s["n_tok_rl"], 1.0)
    out = dict(s)
    out.update({
        "mean_reward": s["sum_mean_reward"] / ng,
        "baseline": s["sum_baseline"] / ng,
        "kl_estimate": s["sum_kl_estimate"] / ng,
        "group_size": s["sum_group_size"] / ng,
        "clipfrac": s["clip_count"] / ntok,
        "entropy": s["sum_entropy"] / ntok,
        "token_kl": s["sum_kl"] / ntok,
        "ppo_kl": s["sum_ppo_kl"] / ntok,
        "mean_ratio": s["sum_ratio"] / ntok,
    })
    return out


class _Workspace:
    """One workspace per (device, stream), allocated ON that stream: the caching
    allocator then only recycles it (or a grown-out buffer) for work ordered
    after the kernels that use it on the same stream."""

    def __init__(self):
        self.buf: Dict[tuple, torch.Tensor] = {}

    def get(self, dev: torch.device, nbytes: int, stream: torch.cuda.Stream) -> torch.Tensor:
        key = (dev.index if dev.index is not None else torch.cuda.current_device(),
               stream.cuda_stream)
        t = self.buf.get(key)
        if t is None or t.numel() < nbytes:
            with torch.cuda.stream(stream):
                t = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=dev)
            self.buf[key] = t
        return t


class RFTLoss:
    """Fused RFT loss (advantage -> logprob -> loss -> dlogits) on B200.

    ``dlogits``: "inplace" (overwrite logits with d loss / d logits), None
    (forward-only loss), "new" (allocate), or a preallocated tensor of the
    logits' dtype with rows of the same length.
    """

    def __init__(self, cfg: Optional[RFTLossConfig] = None, **kw):
        self.cfg = cfg if cfg is not None else RFTLossConfig(**kw)
        self._ws = _Workspace()
        self._probe: Optional["RFTLoss"] = None

    # ---- registered Python components (registry.register_*) -------------------

    def _plugins(self, batch: PackedBatch, s: torch.cuda.Stream, glob: dict,
                 rows=None) -> PackedBatch:
        """Run the config's registered Python components on the batch's device
        and return the batch with their outputs attached: ``advantage``
        (TG_ADV_GIVEN) and ``pg_coef`` / ``pg_loss`` (TG_PG_GIVEN)."""
        from dataclasses import replace

        from .registry import AdvantageInputs, PolicyLossInputs
        adv_fn, pg_fn = self.cfg.advantage_callable, self.cfg.policy_loss_callable
        if adv_fn is None and pg_fn is None:
            return batch
        dev, B, T = batch.device, batch.n_seqs, batch.n_rows
        with torch.cuda.stream(s):
            seq_len = (batch.seq_offsets[1:] - batch.seq_offsets[:-1]).to(torch.int32)
            if adv_fn is not None:
                grp = torch.repeat_interleave(
                    torch.arange(batch.n_groups, device=dev),
                    (batch.group_offsets[1:] - batch.group_offsets[:-1]).long(), output_size=B)
                is_rl = (torch.ones(B, dtype=torch.bool, device=dev) if batch.seq_kind is None
                         else batch.seq_kind == 0)
                a = adv_fn(AdvantageInputs(reward=batch.reward, group_index=grp,
                                           group_offsets=batch.group_offsets, seq_lengths=seq_len,
                                           is_rl=is_rl, n_groups=batch.n_groups, config=self.cfg))
                a = torch.as_tensor(a, device=dev).to(torch.float32).reshape(-1).contiguous()
                if a.numel() != B:
                    raise AlgorithmError(f"advantage_fn {self.cfg.advantage_fn!r} returned "
                                         f"{a.numel()} values for {B} sequences")
                batch = replace(batch, advantage=a)
            if pg_fn is not None:
                # forward pass (2V bytes / row): lp, entropy and the sequence advantages
                if self._probe is None:
                    self._probe = RFTLoss(self.cfg.with_(policy_loss_fn="vanilla", kl_fn="none",
                                                         entropy_loss_fn="none", anchor_beta=0.0))
                if rows is None:
                    fwd = self._probe(batch, dlogits=None, stream=s, **glob)
                else:  # per-row lp / entropy / lse given (LM-head path): no logits pass
                    fwd = self._probe.from_rows(batch, *rows, stream=s, **glob)
                seq = torch.repeat_interleave(torch.arange(B, device=dev), seq_len.long(),
                                              output_size=T)
                lp = fwd.lp.detach().clone().requires_grad_(True)
                with torch.enable_grad():
                    loss_t = pg_fn(PolicyLossInputs(
                        lp=lp, old_lp=batch.old_lp, ref_lp=batch.ref_lp,
                        advantage=fwd.seq_adv[seq], entropy=fwd.entropy, seq_index=seq,
                        config=self.cfg))
                    if not torch.is_tensor(loss_t) or loss_t.shape != (T,):
                        raise AlgorithmError(f"policy_loss_fn {self.cfg.policy_loss_fn!r} must "
                                             f"return one loss per row ([{T}])")
                    (g,) = torch.autograd.grad(loss_t.sum(), lp, allow_unused=True)
                coef = (torch.zeros_like(lp) if g is None else -g).detach().float().contiguous()
                batch = replace(batch, pg_coef=coef,
                                pg_loss=loss_t.detach().float().contiguous())
        return batch

    def route(self, batch: PackedBatch, unscaled: bool = False) -> int:
        """1 = fused single pass, 2 = forward+backward streaming, 3 = sequence-coupled,
        4 = sequence-coupled in one pass with an unscaled gradient."""
        cc = self.cfg.to_c()
        if unscaled:
            cc.flags |= N.TG_FLAG_UNSCALED_GRAD
        return N.lib().tg_route(ctypes.byref(c_batch(batch)), ctypes.byref(cc))

    def cluster_size(self, batch: PackedBatch, unscaled: bool = False) -> int:
        """CL of the k_fused_tma<T, CL> instantiation this batch runs on (0 = a
        streaming route); introspection for tests and benchmarks."""
        cc = self.cfg.to_c()
        if unscaled:
            cc.flags |= N.TG_FLAG_UNSCALED_GRAD
        return N.lib().tg_fused_cluster_size(ctypes.byref(c_batch(batch)), ctypes.byref(cc))

    def __call__(self, batch: PackedBatch, dlogits: Union[str, torch.Tensor, None] = "new", *,
                 n_tok_global: int = 0, n_seq_global: int = 0, n_sft_seq_global: int = 0,
                 out: Optional[LossOutput] = None, stream: Optional[torch.cuda.Stream] = None,
                 unscaled: bool = False) -> LossOutput:
        """Loss, metrics and d loss / d logits of a packed batch.

        ``unscaled=True`` (sequence-coupled losses only: OPMD_KIMI / OPMD_PAIRWISE
        / DPO) reads the logits once instead of twice: ``out.dlogits`` holds
        the unscaled ``p - e_y`` rows and ``out.row_scale`` the per-row factor,
        d loss / d z_t = row_scale[t] * dlogits[t] -- for a caller that folds
        the row scale into its LM-head backward."""
        L = N.lib()
        dev = batch.device
        # outputs and workspace are allocated on the launch stream (see _Workspace)
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        batch = self._plugins(batch, s, dict(n_tok_global=n_tok_global,
                                             n_seq_global=n_seq_global,
                                             n_sft_seq_global=n_sft_seq_global))
        cb = c_batch(batch)
        cfg = self.cfg
        if cfg.coupled and cfg.policy_loss_fn == "dpo" and n_seq_global == 0:
            n_seq_global = batch.n_seqs
        cc = cfg.to_c(n_tok_global, n_seq_global, n_sft_seq_global)
        if unscaled:
            cc.flags |= N.TG_FLAG_UNSCALED_GRAD
        _coupled_rows(cfg, batch, cb)
        T, B = batch.n_rows, batch.n_seqs
        with torch.cuda.stream(s):
            if out is None:
                f32 = dict(dtype=torch.float32, device=dev)
                out = LossOutput(stats=torch.empty(N.NSTAT, dtype=torch.float64, device=dev),
                                 lp=torch.empty(T, **f32), entropy=torch.empty(T, **f32),
                                 lse=torch.empty(T, **f32), seq_lp=torch.empty(B, **f32),
                                 seq_adv=torch.empty(B, **f32))
            if isinstance(dlogits, str):
                if dlogits == "inplace":
                    if batch.row_index is not None:
                        raise ValueError("in-place dlogits needs logits rows == trainable rows")
                    dz = batch.logits
                elif dlogits == "new":
                    dz = torch.empty((T, batch.vocab), dtype=batch.logits.dtype, device=dev)
                else:
                    raise ValueError(f"dlogits must be 'inplace', 'new', None or a tensor")
            else:
                dz = dlogits
            if unscaled and (out.row_coef is None or out.row_coef.shape != (3, T)):
                out.row_coef = torch.empty(3, T, dtype=torch.float32, device=dev)
        co = N.TgOut()
        if dz is not None:
            if dz.dtype != batch.logits.dtype or dz.device != dev or dz.stride(1) != 1:
                raise ValueError("dlogits must match logits' dtype / device with contiguous rows")
            if dz.shape[0] < T or dz.shape[1] < batch.vocab:
                raise ValueError("dlogits too small")
            co.dlogits, co.ld_out = dz.data_ptr(), dz.stride(0)
        co.lp, co.entropy, co.lse = out.lp.data_ptr(), out.entropy.data_ptr(), out.lse.data_ptr()
        co.seq_lp, co.seq_adv, co.stats = (out.seq_lp.data_ptr(), out.seq_adv.data_ptr(),
                                           out.stats.data_ptr())
        if unscaled:
            co.row_coef = out.row_coef.data_ptr()
        nbytes = L.tg_workspace_size(ctypes.byref(cb), ctypes.byref(cc))
        ws = self._ws.get(dev, nbytes, s)
        with torch.cuda.device(dev):
            N.check(L.tg_loss_fwd_bwd(ctypes.byref(cb), ctypes.byref(cc), ctypes.byref(co),
                                      ws.data_ptr(), ws.numel(), s.cuda_stream))
        out.dlogits = dz
        return out

    def from_rows(self, batch: PackedBatch, lp: torch.Tensor, entropy: torch.Tensor,
                  lse: torch.Tensor, *, n_tok_global: int = 0, n_seq_global: int = 0,
                  n_sft_seq_global: int = 0, stream: Optional[torch.cuda.Stream] = None,
                  row_coef: bool = False) -> LossOutput:
        """Forward-only loss and metrics from precomputed per-row lp / entropy /
        lse (``TG_FLAG_ROWS_GIVEN``), e.g. from ``lmhead_logprob_fwd``: no
        logits are read, so a batch built with ``rows_batch`` (empty logits)
        suffices.  Anchor KL needs logits and is rejected.  ``row_coef=True``
        also returns the per-row gradient coefficients ``out.row_coef`` [3, T]
        (a, hz, s: dz = p (a + hz z) - s [v = y]) for ``lmhead_dlogits``."""
        L = N.lib()
        s = stream if stream is not None else torch.cuda.current_stream(batch.device)
        batch = self._plugins(batch, s, dict(n_tok_global=n_tok_global,
                                             n_seq_global=n_seq_global,
                                             n_sft_seq_global=n_sft_seq_global),
                              rows=(lp, entropy, lse))
        cb = c_batch(batch)
        cfg = self.cfg
        if cfg.coupled and cfg.policy_loss_fn == "dpo" and n_seq_global == 0:
            n_seq_global = batch.n_seqs
        cc = cfg.to_c(n_tok_global, n_seq_global, n_sft_seq_global)
        cc.flags |= N.TG_FLAG_ROWS_GIVEN
        _coupled_rows(cfg, batch, cb)
        dev = batch.device
        T, B = batch.n_rows, batch.n_seqs
        for name, t in (("lp", lp), ("entropy", entropy), ("lse", lse)):
            if t.dtype != torch.float32 or t.device != dev or t.shape != (T,) or \
                    not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous float32 [{T}] tensor on {dev}")
        f32 = dict(dtype=torch.float32, device=dev)
        with torch.cuda.stream(s):
            out = LossOutput(stats=torch.empty(N.NSTAT, dtype=torch.float64, device=dev), lp=lp,
                             entropy=entropy, lse=lse, seq_lp=torch.empty(B, **f32),
                             seq_adv=torch.empty(B, **f32))
            if row_coef:
                out.row_coef = torch.empty(3, T, **f32)
        co = N.TgOut()
        co.lp, co.entropy, co.lse = lp.data_ptr(), entropy.data_ptr(), lse.data_ptr()
        co.seq_lp, co.seq_adv, co.stats = (out.seq_lp.data_ptr(), out.seq_adv.data_ptr(),
                                           out.stats.data_ptr())
        if row_coef:
            co.row_coef = out.row_coef.data_ptr()
        nbytes = L.tg_workspace_size(ctypes.byref(cb), ctypes.byref(cc))
        ws = self._ws.get(dev, nbytes, s)
        with torch.cuda.device(dev):
            N.check(L.tg_loss_fwd_bwd(ctypes.byref(cb), ctypes.byref(cc), ctypes.byref(co),
                                      ws.data_ptr(), ws.numel(), s.cuda_stream))
        out.dlogits = None
        return out


def logprob_fwd(batch: PackedBatch, stream: Optional[torch.cuda.Stream] = None):
    """Forward-only per-row logprob / entropy / lse and per-sequence LP
    (experience_logprob, algorithms.py:81-85): 2V bytes per row."""
    L = N.lib()
    cb = c_batch(batch)
    dev = batch.device
    f32 = dict(dtype=torch.float32, device=dev)
    nbytes = L.tg_workspace_size(ctypes.byref(cb), None)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.stream(s):  # outputs + workspace belong to the launch stream
        lp, ent, lse = (torch.empty(batch.n_rows, **f32) for _ in range(3))
        seq_lp = torch.empty(batch.n_seqs, **f32)
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    co = N.TgOut()
    co.lp, co.entropy, co.lse, co.seq_lp = (lp.data_ptr(), ent.data_ptr(), lse.data_ptr(),
                                            seq_lp.data_ptr())
    with torch.cuda.device(dev):
        N.check(L.tg_logprob_fwd(ctypes.byref(cb), ctypes.byref(co), ws.data_ptr(), ws.numel(),
                                 s.cuda_stream))
    return lp, ent, lse, seq_lp


def lmhead_logprob_fwd(hidden: torch.Tensor, weight: torch.Tensor,
                       target: Optional[torch.Tensor] = None,
                       stream: Optional[torch.cuda.Stream] = None):
    """Fused LM-head + log-softmax forward on the tensor cores
    (``tg_lmhead_logprob_fwd``): for hidden [T, d] and weight [V, d] (bf16,
    d a multiple of 64) returns per-row ``(lp, entropy, lse)`` of
    ``z = hidden @ weight.T`` without materialising the [T, V] logits
    (policy.logprob, policy.py:194-212, behind an LM head).  ``lp`` is None
    when no target is given."""
    _check_lmhead(hidden, weight)
    L = N.lib()
    dev = hidden.device
    T, d = hidden.shape
    V = weight.shape[0]
    f32 = dict(dtype=torch.float32, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.stream(s):  # outputs + workspace belong to the launch stream
        ent, lse = torch.empty(T, **f32), torch.empty(T, **f32)
        lp = tgt = None
        if target is not None:
            tgt = target.to(device=dev, dtype=torch.int32).contiguous()
            if tgt.shape != (T,):
                raise ValueError(f"target must have shape ({T},)")
            lp = torch.empty(T, **f32)
        ws = torch.empty(max(L.tg_lmhead_workspace_size(T, V), 16), dtype=torch.uint8,
                         device=dev)
    with torch.cuda.device(dev):
        N.check(L.tg_lmhead_logprob_fwd(
            hidden.data_ptr(), hidden.stride(0), weight.data_ptr(), weight.stride(0), T, V, d,
            tgt.data_ptr() if tgt is not None else None, lp.data_ptr() if lp is not None else None,
            ent.data_ptr(), lse.data_ptr(), ws.data_ptr(), ws.numel(), s.cuda_stream))
    return lp, ent, lse


def _check_lmhead(hidden: torch.Tensor, weight: torch.Tensor) -> None:
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise TypeError("hidden and weight must be bfloat16")
    if hidden.dim() != 2 or weight.dim() != 2 or hidden.shape[1] != weight.shape[1]:
        raise ValueError(f"shape mismatch: hidden {tuple(hidden.shape)}, weight "
                         f"{tuple(weight.shape)}")
    if not hidden.is_cuda or hidden.device != weight.device:
        raise ValueError("hidden and weight must be on the same CUDA device")
    if hidden.stride(1) != 1 or weight.stride(1) != 1:
        raise ValueError("hidden and weight need unit stride along d")


def lmhead_dlogits(hidden: torch.Tensor, weight: torch.Tensor, target: torch.Tensor,
                   lse: torch.Tensor, row_coef: torch.Tensor, col0: int, n_cols: int,
                   out: Optional[torch.Tensor] = None,
                   stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """d loss / d logits of the vocabulary chunk [col0, col0 + n_cols) as bf16
    [T, n_cols], recomputed from hidden states on the tensor cores
    (``tg_lmhead_dlogits``; policy.grad_logprob, policy.py:253-270, behind an
    LM head).  ``lse`` comes from the forward, ``row_coef`` from
    ``RFTLoss.from_rows(..., row_coef=True)``.  ``out`` may be a column slice of
    a wider buffer (row pitch a multiple of 8)."""
    _check_lmhead(hidden, weight)
    L = N.lib()
    dev = hidden.device
    T, d = hidden.shape
    V = weight.shape[0]
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.stream(s):
        if out is None:  # row pitch a multiple of 8 elements (16-byte vector stores)
            out = torch.empty(T, (n_cols + 7) // 8 * 8, dtype=torch.bfloat16,
                              device=dev)[:, :n_cols]
        tgt = target.to(device=dev, dtype=torch.int32).contiguous()
    if out.dtype != torch.bfloat16 or out.shape != (T, n_cols) or out.stride(1) != 1:
        raise ValueError(f"out must be a bf16 [{T}, {n_cols}] tensor with unit column stride")
    for name, t, shape in (("lse", lse, (T,)), ("row_coef", row_coef, (3, T))):
        if t.dtype != torch.float32 or t.shape != shape or not t.is_contiguous() or \
                t.device != dev:
            raise ValueError(f"{name} must be a contiguous float32 {list(shape)} tensor on {dev}")
    with torch.cuda.device(dev):
        N.check(L.tg_lmhead_dlogits(
            hidden.data_ptr(), hidden.stride(0), weight.data_ptr(), weight.stride(0), T, V, d,
            int(col0), int(n_cols), tgt.data_ptr(), lse.data_ptr(), row_coef.data_ptr(),
            out.data_ptr(), out.stride(0), s.cuda_stream))
    return out


def _check_bf16_2d(name: str, t: torch.Tensor, dev: torch.device) -> None:
    if t.dtype != torch.bfloat16 or t.dim() != 2 or t.stride(1) != 1 or t.device != dev:
        raise ValueError(f"{name} must be a 2-D bf16 tensor with unit column stride on {dev}")


def lmhead_grad_hidden(dz: torch.Tensor, weight: torch.Tensor, col0: int,
                       out: torch.Tensor, accumulate: bool = True,
                       stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """``out [T, d] fp32 (+)= dz [T, n] . weight[col0 : col0 + n]`` on the tensor
    cores (``tg_lmhead_grad_hidden``): d hidden from one vocabulary chunk of
    d loss / d logits."""
    dev = dz.device
    _check_bf16_2d("dz", dz, dev)
    _check_bf16_2d("weight", weight, dev)
    T, n = dz.shape
    V, d = weight.shape
    if out.dtype != torch.float32 or out.shape != (T, d) or out.stride(1) != 1:
        raise ValueError(f"out must be a float32 [{T}, {d}] tensor with unit column stride")
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        N.check(N.lib().tg_lmhead_grad_hidden(
            dz.data_ptr(), dz.stride(0), weight.data_ptr(), weight.stride(0), T, V, d, int(col0),
            n, out.data_ptr(), out.stride(0), int(bool(accumulate)), s.cuda_stream))
    return out


def lmhead_grad_weight(dz: torch.Tensor, hidden: torch.Tensor, out: torch.Tensor,
                       stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """``out [n, d] bf16 = dz [T, n]^T . hidden [T, d]`` on the tensor cores
    (``tg_lmhead_grad_weight``): the rows of d W for one vocabulary chunk."""
    dev = dz.device
    _check_bf16_2d("dz", dz, dev)
    _check_bf16_2d("hidden", hidden, dev)
    T, n = dz.shape
    d = hidden.shape[1]
    if hidden.shape[0] != T:
        raise ValueError("dz and hidden must have the same rows")
    _check_bf16_2d("out", out, dev)
    if out.shape != (n, d):
        raise ValueError(f"out must be [{n}, {d}]")
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        N.check(N.lib().tg_lmhead_grad_weight(
            dz.data_ptr(), dz.stride(0), hidden.data_ptr(), hidden.stride(0), T, d, n,
            out.data_ptr(), out.stride(0), s.cuda_stream))
    return out


def lmhead_grad_chunk(dz: torch.Tensor, hidden: torch.Tensor, weight: torch.Tensor, col0: int,
                      d_hidden: torch.Tensor, d_weight_rows: torch.Tensor,
                      accumulate: bool = True,
                      stream: Optional[torch.cuda.Stream] = None) -> None:
    """Both gradient GEMMs of one vocabulary chunk in one tcgen05 launch
    (``tg_lmhead_grad_chunk``): ``d_hidden (+)= dz . weight[col0 : col0 + n]``
    (fp32) and ``d_weight_rows = dz^T . hidden`` (bf16 [n, d])."""
    dev = dz.device
    for name, t in (("dz", dz), ("hidden", hidden), ("weight", weight),
                    ("d_weight_rows", d_weight_rows)):
        _check_bf16_2d(name, t, dev)
    T, n = dz.shape
    V, d = weight.shape
    if hidden.shape != (T, d) or d_weight_rows.shape != (n, d):
        raise ValueError(f"hidden must be [{T}, {d}] and d_weight_rows [{n}, {d}]")
    if d_hidden.dtype != torch.float32 or d_hidden.shape != (T, d) or d_hidden.stride(1) != 1:
        raise ValueError(f"d_hidden must be a float32 [{T}, {d}] tensor with unit column stride")
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        N.check(N.lib().tg_lmhead_grad_chunk(
            dz.data_ptr(), dz.stride(0), hidden.data_ptr(), hidden.stride(0), weight.data_ptr(),
            weight.stride(0), T, V, d, int(col0), n, d_hidden.data_ptr(), d_hidden.stride(0),
            int(bool(accumulate)), d_weight_rows.data_ptr(), d_weight_rows.stride(0),
            s.cuda_stream))


def lmhead_loss_fwd_bwd(hidden: torch.Tensor, weight: torch.Tensor, loss: "RFTLoss", target,
                        seq_lengths, group_sizes, reward, *, chunk_cols: int = 16384,
                        grad_weight: bool = True, **pack_kw):
    """RFT loss and its gradients w.r.t. the hidden states and the LM-head
    weight, without the [T, V] logits (vocabulary-chunked):

    1. ``tg_lmhead_logprob_fwd``: per-row lp / entropy / lse on the tensor cores;
    2. the loss epilogue on those rows (``TG_FLAG_ROWS_GIVEN``), which also
       returns the per-row gradient coefficients;
    3. per vocabulary chunk of ``chunk_cols`` columns: ``tg_lmhead_dlogits``
       recomputes the chunk's logits and writes its bf16 d loss / d z, then the
       two tcgen05 GEMMs d hidden += dz . W_chunk (fp32) and d W_chunk = dz^T .
       hidden in one launch (``tg_lmhead_grad_chunk``).

    Peak extra memory is T x chunk_cols bf16.  Returns ``(LossOutput,
    d_hidden [T, d] fp32, d_weight [V, d] bf16 or None)``."""
    _check_lmhead(hidden, weight)
    out = lmhead_loss_fwd(hidden, weight, loss, target, seq_lengths, group_sizes, reward,
                          row_coef=True, **pack_kw)
    T, d = hidden.shape
    V = int(weight.shape[0])
    dev = hidden.device
    d_hidden = torch.empty(T, d, dtype=torch.float32, device=dev)
    d_weight = torch.empty(V, d, dtype=torch.bfloat16, device=dev) if grad_weight else None
    if T == 0:
        if d_weight is not None:
            d_weight.zero_()
        return out, d_hidden, d_weight
    chunk = max(8, min(int(chunk_cols), V))
    pitch = (chunk + 7) // 8 * 8
    buf = torch.empty(T, pitch, dtype=torch.bfloat16, device=dev)
    tgt = out.target
    for c0 in range(0, V, chunk):
        nc = min(chunk, V - c0)
        dz = lmhead_dlogits(hidden, weight, tgt, out.lse, out.row_coef, c0, nc, out=buf[:, :nc])
        if d_weight is not None:  # both GEMMs in one launch
            lmhead_grad_chunk(dz, hidden, weight, c0, d_hidden, d_weight[c0:c0 + nc],
                              accumulate=c0 > 0)
        else:
            lmhead_grad_hidden(dz, weight, c0, d_hidden, accumulate=c0 > 0)
    return out, d_hidden, d_weight


def lmhead_loss_fwd(hidden: torch.Tensor, weight: torch.Tensor, loss: "RFTLoss", target,
                    seq_lengths, group_sizes, reward, *, row_coef: bool = False,
                    **pack_kw) -> LossOutput:
    """RFT loss and metrics straight from hidden states: the fused LM-head
    kernel gives per-row lp / entropy / lse (no [T, V] logits anywhere), then
    the loss epilogue runs on those rows (``RFTLoss.from_rows``).  ``pack_kw``
    takes pack_arrays' side inputs (old_lp, ref_lp, seq_ref_lp, seq_kind, ...)
    and the global denominators (n_tok_global, ...).  ``row_coef=True`` also
    returns the per-row gradient coefficients (``out.row_coef``) that
    ``lmhead_dlogits`` needs; ``out.target`` holds the packed device targets."""
    from .packing import pack_arrays
    glob = {k: pack_kw.pop(k) for k in ("n_tok_global", "n_seq_global", "n_sft_seq_global")
            if k in pack_kw}
    V = int(weight.shape[0])
    # the packer validates targets on the host: pass a host array (a device
    # tensor costs one synchronising copy here)
    tgt_host = target.cpu().numpy() if torch.is_tensor(target) else np.asarray(target)
    rows = torch.empty((0, V), dtype=torch.bfloat16, device=hidden.device)
    batch = pack_arrays(rows, tgt_host, seq_lengths, group_sizes, reward, vocab=V, **pack_kw)
    lp, ent, lse = lmhead_logprob_fwd(hidden, weight, batch.target)
    out = loss.from_rows(batch, lp, ent, lse, row_coef=row_coef, **glob)
    out.target = batch.target
    return out
