"""Experience batch -> packed device tensors in the TgBatch layout.

The packed layout (include/tg_loss.h): one row per trainable (mask-true)
token, rows of a sequence contiguous, sequences of a group contiguous, with
prefix-sum ``seq_offsets[B+1]`` and ``group_offsets[G+1]``.  Group order and
in-group order are preserved exactly as ``ExperienceBuffer.sample_batch``
returns them (buffer.py:251-264); ``group_by_task`` restates that indexing for
callers that hold a flat experience list.

Inputs are duck-typed against the reference records (records.py:21-131):
experiences need ``tokens``, ``prompt_length``, ``action_mask``,
``logprobs`` (compact: one per mask-true token, records.py:47-49) and
``reward``; groups need ``experiences`` and optionally ``ref_logprobs``
(default: each experience's summed stored logprobs, records.py:119-121).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .config import AlgorithmError


class PolicyError(ValueError):
    """Invalid input to a policy operation (policy.py:35-36)."""


@dataclass
class PackedBatch:
    """Device tensors of one call (all on the same CUDA device)."""

    logits: torch.Tensor                      # [R, ld] bf16 / f32; row t (or row_index[t]) scores target[t]
    target: torch.Tensor                      # [T] int32
    seq_offsets: torch.Tensor                 # [B+1] int32
    group_offsets: torch.Tensor               # [G+1] int32
    reward: torch.Tensor                      # [B] f32
    old_lp: Optional[torch.Tensor] = None     # [T] f32
    ref_lp: Optional[torch.Tensor] = None     # [T] f32
    seq_ref_lp: Optional[torch.Tensor] = None  # [B] f32
    advantage: Optional[torch.Tensor] = None  # [B] f32
    seq_kind: Optional[torch.Tensor] = None   # [B] uint8 (0 RL, 1 SFT)
    anchor_logits: Optional[torch.Tensor] = None  # [T, ld_a]
    row_index: Optional[torch.Tensor] = None  # [T] int64
    pg_coef: Optional[torch.Tensor] = None    # [T] f32 (registered policy loss: -d l / d lp)
    pg_loss: Optional[torch.Tensor] = None    # [T] f32 (registered policy loss: l)
    vocab: int = 0
    # host-side shape facts (known to the packer; no device sync needed)
    n_rows: int = 0
    n_seqs: int = 0
    n_groups: int = 0
    n_rl_rows: int = 0
    n_rl_seqs: int = 0
    n_sft_seqs: int = 0
    max_rows_per_seq: int = 0

    def __post_init__(self) -> None:
        if self.vocab == 0:
            self.vocab = int(self.logits.shape[-1])

    @property
    def device(self) -> torch.device:
        return self.logits.device


def _i32(x, device):
    return torch.as_tensor(np.asarray(x, dtype=np.int32), device=device)


def _f32(x, device):
    return None if x is None else torch.as_tensor(np.asarray(x, dtype=np.float32), device=device)


def offsets_from_lengths(lengths: Sequence[int]) -> np.ndarray:
    return np.concatenate([[0], np.cumsum(np.asarray(lengths, dtype=np.int64))]).astype(np.int64)


def pack_arrays(logits: torch.Tensor, target, seq_lengths, group_sizes, reward, *,
                old_lp=None, ref_lp=None, seq_ref_lp=None, advantage=None, seq_kind=None,
                anchor_logits=None, row_index=None, vocab: int = 0) -> PackedBatch:
    """Build a PackedBatch from host (numpy / list) side arrays + device logits."""
    dev = logits.device
    seq_lengths = np.asarray(seq_lengths, dtype=np.int64)
    group_sizes = np.asarray(group_sizes, dtype=np.int64)
    so = offsets_from_lengths(seq_lengths)
    go = offsets_from_lengths(group_sizes)
    B, G = len(seq_lengths), len(group_sizes)
    if go[-1] != B:
        raise AlgorithmError(f"group sizes sum to {go[-1]} but there are {B} sequences")
    T = int(so[-1])
    target = np.asarray(target)
    if target.shape[0] != T:
        raise AlgorithmError(f"{target.shape[0]} targets for {T} trainable rows")
    kind = None if seq_kind is None else np.asarray(seq_kind, dtype=np.uint8)
    rl = np.ones(B, bool) if kind is None else kind == 0
    V = vocab or int(logits.shape[-1])
    if T and (target.min() < 0 or target.max() >= V):
        bad = int(target[(target < 0) | (target >= V)][0])
        raise PolicyError(f"token {bad} outside vocabulary of size {V}")
    # shapes the C ABI cannot check (plain pointers): a short array would be
    # read out of bounds on the device, a long one silently misaligned
    for name, arr, n in (("reward", reward, B), ("seq_ref_lp", seq_ref_lp, B),
                         ("advantage", advantage, B), ("seq_kind", kind, B),
                         ("old_lp", old_lp, T), ("ref_lp", ref_lp, T)):
        if arr is not None and int(np.size(arr)) != n:
            raise AlgorithmError(f"{name} has {int(np.size(arr))} entries, expected {n} "
                                 f"({'one per sequence' if n == B else 'one per trainable row'})")
    n_logit_rows = int(logits.shape[0]) if logits.dim() == 2 else 0
    if row_index is not None:
        row_index = np.asarray(row_index, dtype=np.int64)
        if row_index.shape != (T,):
            raise AlgorithmError(f"row_index has {row_index.size} entries, expected {T}")
        if T and logits.numel() and (row_index.min() < 0 or row_index.max() >= n_logit_rows):
            raise AlgorithmError(f"row_index outside the {n_logit_rows} logits rows")
    elif logits.numel() and n_logit_rows < T:
        raise AlgorithmError(f"{n_logit_rows} logits rows for {T} trainable rows")
    if anchor_logits is not None:
        if anchor_logits.dim() != 2 or anchor_logits.shape[0] < T or anchor_logits.shape[1] < V:
            raise AlgorithmError(f"anchor_logits {tuple(anchor_logits.shape)} must cover "
                                 f"[{T}, {V}] (one row per trainable row)")
    return PackedBatch(
        logits=logits, target=_i32(target, dev), seq_offsets=_i32(so, dev),
        group_offsets=_i32(go, dev), reward=_f32(reward, dev), old_lp=_f32(old_lp, dev),
        ref_lp=_f32(ref_lp, dev), seq_ref_lp=_f32(seq_ref_lp, dev),
        advantage=_f32(advantage, dev),
        seq_kind=None if kind is None else torch.as_tensor(kind, device=dev),
        anchor_logits=anchor_logits,
        row_index=None if row_index is None else torch.as_tensor(
            np.asarray(row_index, dtype=np.int64), device=dev),
        vocab=V, n_rows=T, n_seqs=B, n_groups=G,
        n_rl_rows=int(seq_lengths[rl].sum()), n_rl_seqs=int(rl.sum()),
        n_sft_seqs=int((~rl).sum()),
        max_rows_per_seq=int(seq_lengths.max()) if B else 0)


@dataclass
class HostGroups:
    """Host-side flattening of TaskGroups (the parts the kernels need)."""

    tokens: np.ndarray
    mask: np.ndarray
    tok_off: np.ndarray
    prompt_len: np.ndarray
    old_lp: np.ndarray
    seq_lengths: np.ndarray
    group_sizes: np.ndarray
    reward: np.ndarray
    seq_ref_lp: np.ndarray
    experiences: List = field(default_factory=list)


def flatten_groups(groups) -> HostGroups:
    """TaskGroups -> flat host arrays: each experience's token / mask / logprob
    lists become numpy arrays in one C-level conversion each (no per-token
    Python), then one concatenation per field.  Validation as records.py:21-131."""
    toks, masks, olds, plen, lens, gsz, rew, refs, exps = [], [], [], [], [], [], [], [], []
    for g in groups:
        gexps = list(g.experiences)
        if not gexps:
            raise AlgorithmError("a task group needs at least one experience")
        gref = getattr(g, "ref_logprobs", None)
        if gref is not None and len(gref) != len(gexps):
            raise AlgorithmError("ref_logprobs length must match the group size")
        gsz.append(len(gexps))
        for j, e in enumerate(gexps):
            t = np.asarray(e.tokens, dtype=np.int64).reshape(-1)
            m = np.asarray(e.action_mask, dtype=bool).reshape(-1)
            lp = np.asarray(e.logprobs, dtype=np.float64).reshape(-1)
            if t.size != m.size:
                raise AlgorithmError("action_mask length must match tokens")
            n_true = int(np.count_nonzero(m))
            if lp.size != n_true:
                raise AlgorithmError("logprobs length must match mask-true count")
            if e.reward is None:
                raise AlgorithmError("READY experience requires a reward")
            toks.append(t)
            masks.append(m)
            olds.append(lp)
            plen.append(int(e.prompt_length))
            lens.append(n_true)
            rew.append(float(e.reward))
            # records.py:64-66, 119-121: Experience.total_logprob = float(sum(logprobs)),
            # a sequential left-to-right sum (kept bit-exact)
            refs.append(float(gref[j]) if gref is not None else float(sum(e.logprobs)))
            exps.append(e)
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt, copy=False) if xs
           else np.zeros(0, dt))
    tok_off = np.concatenate([[0], np.cumsum([t.size for t in toks], dtype=np.int64)])
    return HostGroups(
        tokens=cat(toks, np.int64), mask=cat(masks, np.uint8), tok_off=tok_off.astype(np.int64),
        prompt_len=np.asarray(plen, np.int64), old_lp=cat(olds, np.float64),
        seq_lengths=np.asarray(lens, np.int64), group_sizes=np.asarray(gsz, np.int64),
        reward=np.asarray(rew, np.float64), seq_ref_lp=np.asarray(refs, np.float64),
        experiences=exps)


def scored_states(h: HostGroups, num_buckets: int):
    """Row -> (context bucket, target) for the toy-table policy (C helper:
    policy.py:152-161, 181-191 restated in csrc/tg_host.cpp)."""
    L = N.lib()
    cap = int(h.mask.sum())
    states = np.empty(cap, np.int64)
    target = np.empty(cap, np.int32)
    tokens = np.ascontiguousarray(h.tokens)
    mask = np.ascontiguousarray(h.mask)
    n = L.tg_scored_states(tokens.ctypes.data, mask.ctypes.data, h.tok_off.ctypes.data,
                           h.prompt_len.ctypes.data, len(h.prompt_len), int(num_buckets),
                           states.ctypes.data, target.ctypes.data, cap)
    if n != cap:
        raise PolicyError("malformed experience (prompt_length / offsets)")
    return states, target


def group_by_task(task_keys: Sequence[int], ready: Sequence[bool], group_size: int, n: int,
                  policy: str = "FIFO", priority: Optional[Sequence[float]] = None,
                  id_rank: Optional[Sequence[int]] = None) -> List[List[int]]:
    """ExperienceBuffer.sample_batch(n, policy, group_by_task=True) indexing
    (buffer.py:240-264) over experiences in insertion order; returns groups
    of indices into the input order."""
    L = N.lib()
    if group_size < 1:
        raise ValueError("group_by_task requires group_size >= 1")
    if n < 1:
        raise ValueError("batch size must be >= 1")
    tk = np.ascontiguousarray(np.asarray(task_keys, np.int64))
    rd = np.ascontiguousarray(np.asarray(ready, np.uint8))
    m = len(tk)
    pr = np.ascontiguousarray(np.asarray(priority if priority is not None else np.zeros(m),
                                         np.float64))
    rk = np.ascontiguousarray(np.asarray(id_rank if id_rank is not None else np.arange(m),
                                         np.int64))
    out = np.empty(max(n, 1) * group_size, np.int64)
    pol = {"FIFO": 0, "PRIORITY": 1}[str(policy).upper()]
    k = L.tg_group_by_task(tk.ctypes.data, pr.ctypes.data, rk.ctypes.data, rd.ctypes.data, m,
                           group_size, n, pol, out.ctypes.data)
    if k < 0:
        raise ValueError("invalid group_by_task arguments")
    return out[: k * group_size].reshape(k, group_size).tolist()


def pack_token_batch(logits: torch.Tensor, input_ids: torch.Tensor, loss_mask: torch.Tensor,
                     rewards, group_sizes, *, old_logprobs: Optional[torch.Tensor] = None,
                     ref_logprobs: Optional[torch.Tensor] = None, seq_kind=None,
                     seq_ref_lp=None, advantage=None) -> PackedBatch:
    """LLM-layout batch already on the device -> PackedBatch, packed on the GPU
    (tg_pack_rows): `logits` [B, L, V] (or [B*L, V]) is read in place through
    row_index with the HF shift (logits at l - 1 score input_ids[l]);
    `loss_mask` [B, L] marks trainable target positions; `old_logprobs` /
    `ref_logprobs` are dense [B, L] aligned with `input_ids`.  One 8-byte + 4B
    byte device->host read sizes the batch."""
    L_ = N.lib()
    if input_ids.dim() != 2 or loss_mask.shape != input_ids.shape:
        raise ValueError("input_ids and loss_mask must be [B, L]")
    B, Lx = input_ids.shape
    dev = input_ids.device
    V = int(logits.shape[-1])
    flat = logits.reshape(B * Lx, V)
    if flat.data_ptr() != logits.data_ptr():
        raise ValueError("logits must be viewable as [B*L, V] without a copy")
    ids = input_ids.contiguous()
    if ids.dtype not in (torch.int32, torch.int64):
        raise ValueError("input_ids must be int32 or int64")
    mask = loss_mask.to(torch.uint8).contiguous()
    cap = B * Lx
    row_index = torch.empty(cap, dtype=torch.int64, device=dev)
    target = torch.empty(cap, dtype=torch.int32, device=dev)
    old_out = torch.empty(cap, dtype=torch.float32, device=dev) if old_logprobs is not None else None
    ref_out = torch.empty(cap, dtype=torch.float32, device=dev) if ref_logprobs is not None else None
    old_in = None if old_logprobs is None else old_logprobs.float().contiguous()
    ref_in = None if ref_logprobs is None else ref_logprobs.float().contiguous()
    seq_off = torch.empty(B + 1, dtype=torch.int32, device=dev)
    n_rows = torch.empty(1, dtype=torch.int64, device=dev)
    ws = torch.empty(max(4 * B, 4), dtype=torch.uint8, device=dev)

    def p(t):
        return None if t is None else t.data_ptr()

    with torch.cuda.device(dev):
        N.check(L_.tg_pack_rows(mask.data_ptr(), ids.data_ptr(), int(ids.dtype == torch.int64),
                                B, Lx, p(old_in), p(ref_in), row_index.data_ptr(),
                                target.data_ptr(), p(old_out), p(ref_out), cap, seq_off.data_ptr(),
                                n_rows.data_ptr(), ws.data_ptr(), ws.numel(),
                                torch.cuda.current_stream(dev).cuda_stream))
    so = seq_off.cpu().numpy().astype(np.int64)
    T = int(so[-1])
    seq_lengths = np.diff(so)
    group_sizes = np.asarray(group_sizes, np.int64)
    go = offsets_from_lengths(group_sizes)
    if go[-1] != B:
        raise AlgorithmError(f"group sizes sum to {go[-1]} but there are {B} sequences")
    kind = None if seq_kind is None else np.asarray(seq_kind, dtype=np.uint8)
    rl = np.ones(B, bool) if kind is None else kind == 0
    return PackedBatch(
        logits=flat, target=target[:T], seq_offsets=seq_off, group_offsets=_i32(go, dev),
        reward=_f32(rewards, dev) if not torch.is_tensor(rewards) else rewards.float(),
        old_lp=None if old_out is None else old_out[:T],
        ref_lp=None if ref_out is None else ref_out[:T], seq_ref_lp=_f32(seq_ref_lp, dev),
        advantage=_f32(advantage, dev),
        seq_kind=None if kind is None else torch.as_tensor(kind, device=dev),
        row_index=row_index[:T], vocab=V, n_rows=T, n_seqs=B, n_groups=len(group_sizes),
        n_rl_rows=int(seq_lengths[rl].sum()), n_rl_seqs=int(rl.sum()),
        n_sft_seqs=int((~rl).sum()), max_rows_per_seq=int(seq_lengths.max()) if B else 0)
