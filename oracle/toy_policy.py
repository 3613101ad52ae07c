"""Gather adapter: the reference's bucketed-table policy -> packed per-token rows.

TEST INFRASTRUCTURE ONLY.  The reference's "model forward" is a table gather:
each mask-true position t of an experience scores row
``state_t = FNV1a(context_key, t, prev_tok) mod S`` of the logits table
(policy.py:152-161, 181-191; encoding.py:19-35).  Materialising
``X[t, :] = theta[state_t, :]`` turns the reference's per-token arithmetic into
the LLM-shaped ``[T, V]`` logits the CUDA path consumes; scatter-adding the
kernel's per-row gradient back by ``state_t`` reproduces the reference's
``SparseGrad.to_dense``.

This is an independent restatement (the product has its own C version in
``paper_2505_17826_b200/csrc/tg_host.cpp``); tests cross-check the two.
"""

from __future__ import annotations

import struct
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .rft_oracle import Batch

_FNV_OFFSET = 0xCBF29CE484222325
_FNV_PRIME = 0x100000001B3
_MASK64 = 0xFFFFFFFFFFFFFFFF
CONTEXT_SENTINEL = -1  # policy.py:29


def fnv1a64(data: bytes) -> int:
    """encoding.py:19-25."""
    h = _FNV_OFFSET
    for b in data:
        h ^= b
        h = (h * _FNV_PRIME) & _MASK64
    return h


def sequence_key(tokens: Sequence[int]) -> int:
    """encoding.py:28-35: FNV-1a over little-endian signed 64-bit words."""
    return fnv1a64(b"".join(struct.pack("<q", int(t)) for t in tokens))


def state_index(task_key: int, position: int, prev_token: int, num_buckets: int) -> int:
    """policy.py:152-161."""
    data = struct.pack("<Qqq", task_key & _MASK64, position, prev_token)
    return fnv1a64(data) % num_buckets


def scored_states(context_key: int, tokens: Sequence[int], mask: Sequence[bool],
                  num_buckets: int) -> List[Tuple[int, int, int]]:
    """policy.py:181-191: (position, state, token) for every mask-true position."""
    out = []
    prev = CONTEXT_SENTINEL
    for pos, tok in enumerate(tokens):
        if mask[pos]:
            out.append((pos, state_index(context_key, pos, prev, num_buckets), int(tok)))
            prev = int(tok)
        else:
            prev = CONTEXT_SENTINEL
    return out


def experience_states(exp, num_buckets: int) -> Tuple[List[int], List[int]]:
    """States and targets of one experience's mask-true rows (algorithms.py:81-90)."""
    prompt = exp.tokens[: exp.prompt_length]
    key = sequence_key(prompt)
    sc = scored_states(key, exp.tokens, exp.action_mask, num_buckets)
    return [s for _, s, _ in sc], [t for _, _, t in sc]


def pack_groups(groups, table: np.ndarray, anchor: Optional[np.ndarray] = None,
                seq_kind: Optional[Sequence[int]] = None,
                ref_lp_seq: Optional[Sequence[float]] = None) -> Tuple[Batch, np.ndarray]:
    """TaskGroup list (duck-typed) -> (Batch, states[T]).

    ``groups`` is a list of objects with ``experiences`` (each with tokens,
    prompt_length, action_mask, logprobs, reward) and optional
    ``ref_logprobs``; group order and in-group order are preserved exactly
    (buffer.py:251-264).  ``old_lp`` is the experience's compact stored
    logprobs (records.py:47-49); ``seq_ref_lp`` defaults to the group's
    ``ref_logprobs`` (records.py:119-121).
    """
    S = table.shape[0]
    states, targets, old = [], [], []
    seq_off, grp_off, reward, seq_ref = [0], [0], [], []
    for g in groups:
        refs = getattr(g, "ref_logprobs", None)
        for j, e in enumerate(g.experiences):
            st, tg = experience_states(e, S)
            states += st
            targets += tg
            old += list(e.logprobs)
            seq_off.append(len(states))
            reward.append(float(e.reward) if e.reward is not None else 0.0)
            seq_ref.append(float(refs[j]) if refs is not None else float(sum(e.logprobs)))
        grp_off.append(len(seq_off) - 1)
    states_a = np.array(states, dtype=np.int64)
    X = table[states_a] if len(states) else np.zeros((0, table.shape[1]))
    batch = Batch(
        logits=np.array(X, dtype=np.float64),
        target=np.array(targets, dtype=np.int64),
        seq_offsets=np.array(seq_off, dtype=np.int64),
        group_offsets=np.array(grp_off, dtype=np.int64),
        reward=np.array(reward),
        seq_ref_lp=np.array(ref_lp_seq if ref_lp_seq is not None else seq_ref),
        old_lp=np.array(old),
        seq_kind=None if seq_kind is None else np.array(seq_kind, dtype=np.int64),
        anchor_logits=None if anchor is None else np.array(anchor[states_a], dtype=np.float64),
    )
    return batch, states_a


def scatter_rows(dz: np.ndarray, states: np.ndarray, num_buckets: int) -> np.ndarray:
    """Per-row gradient -> dense table gradient (SparseGrad.to_dense, policy.py:238-242)."""
    out = np.zeros((num_buckets, dz.shape[1]))
    np.add.at(out, states, dz)
    return out
