"""Helpers to rebuild reference inputs from the committed golden fixtures."""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path
from typing import List, Optional

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@dataclass
class Exp:
    """Duck-typed stand-in for triad.records.Experience (records.py:21-49)."""

    tokens: List[int]
    prompt_length: int
    action_mask: List[bool]
    logprobs: List[float]
    reward: Optional[float]
    task_key: int = 0


@dataclass
class Group:
    """Duck-typed stand-in for triad.records.TaskGroup (records.py:104-131)."""

    experiences: List[Exp]
    ref_logprobs: Optional[List[float]] = None
    task_key: int = 0

    @property
    def size(self) -> int:
        return len(self.experiences)


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def groups_of(fx: dict, prefix: str = "") -> List[Group]:
    fx = {k[len(prefix):]: v for k, v in fx.items() if k.startswith(prefix)}
    exps = []
    for i in range(len(fx["prompt_len"])):
        a, b = int(fx["tok_off"][i]), int(fx["tok_off"][i + 1])
        la, lb = int(fx["lp_off"][i]), int(fx["lp_off"][i + 1])
        exps.append(Exp(
            tokens=[int(t) for t in fx["tokens"][a:b]],
            prompt_length=int(fx["prompt_len"][i]),
            action_mask=[bool(m) for m in fx["mask"][a:b]],
            logprobs=[float(x) for x in fx["logprobs"][la:lb]],
            reward=float(fx["reward"][i]),
        ))
    groups, k = [], 0
    refs = fx.get("ref_logprobs")
    for gs in fx["group_size"]:
        gs = int(gs)
        groups.append(Group(exps[k:k + gs],
                            None if refs is None else [float(x) for x in refs[k:k + gs]]))
        k += gs
    return groups


def metrics_of(fx: dict) -> dict:
    return {str(k): float(v) for k, v in zip(fx["metric_names"], fx["metric_values"])}
