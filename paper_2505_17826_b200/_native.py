"""ctypes binding of libtg_loss.so (the C ABI declared in include/tg_loss.h).

There is no fallback: if the library is missing this module raises on import
of any entry point, telling the user to build it.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_void_p
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libtg_loss.so"

# ---- enums (must match include/tg_loss.h) -----------------------------------
TG_OK, TG_EINVAL, TG_ECUDA, TG_EUNSUPPORTED, TG_EWORKSPACE = 0, 1, 2, 3, 4
TG_DTYPE_BF16, TG_DTYPE_F32 = 0, 1
TG_ADV_GIVEN, TG_ADV_GRPO, TG_ADV_RLOO, TG_ADV_OPMD, TG_ADV_REINFORCE = 0, 1, 2, 3, 4
(TG_PG_VANILLA, TG_PG_PPO_CLIP, TG_PG_SFT, TG_PG_OPMD_KIMI, TG_PG_OPMD_PAIRWISE,
 TG_PG_DPO, TG_PG_GIVEN) = 0, 1, 2, 3, 4, 5, 6
TG_KL_NONE, TG_KL_K1, TG_KL_K2, TG_KL_K3, TG_KL_ABS = 0, 1, 2, 3, 4
TG_ENT_NONE, TG_ENT_DEFAULT = 0, 1
(TG_AGG_SEQ_SUM, TG_AGG_TOKEN_MEAN, TG_AGG_SEQ_MEAN_TOKEN_SUM, TG_AGG_SEQ_MEAN_TOKEN_MEAN,
 TG_AGG_SEQ_MEAN_TOKEN_SUM_NORM) = 0, 1, 2, 3, 4
TG_FLAG_FORCE_TWO_PASS = 1
TG_FLAG_ROWS_GIVEN = 4
TG_FLAG_UNSCALED_GRAD = 8

STAT_NAMES = [
    "loss", "pg_loss", "kl_loss", "entropy_loss", "anchor_loss", "sft_loss",
    "n_groups", "sum_mean_reward", "sum_baseline", "sum_kl_estimate", "sum_group_size",
    "n_tok", "n_tok_rl", "clip_count", "sum_entropy", "sum_kl", "sum_ppo_kl",
    "sum_lp", "nonfinite", "n_seqs", "sum_adv", "sum_ratio", "n_sft_seqs",
    "sum_sft_reward", "sum_dpo_margin", "dual_clip_count", "sum_anchor_kl",
    "invalid", "reserved28", "reserved29", "reserved30", "reserved31",
]
STAT = {n: i for i, n in enumerate(STAT_NAMES)}
NSTAT = 32


class TgConfig(ctypes.Structure):
    _fields_ = [
        ("advantage_fn", c_int32), ("policy_loss_fn", c_int32), ("kl_fn", c_int32),
        ("entropy_loss_fn", c_int32), ("loss_agg_mode", c_int32), ("flags", c_int32),
        ("tau", c_double), ("clip_lo", c_double), ("clip_hi", c_double), ("clip_c", c_double),
        ("kl_coef", c_double), ("entropy_coef", c_double), ("std_eps", c_double),
        ("sft_weight", c_double), ("anchor_beta", c_double), ("dpo_beta", c_double),
        ("agg_norm", c_double),
        ("n_tok_global", c_int64), ("n_seq_global", c_int64), ("n_sft_seq_global", c_int64),
    ]


class TgBatch(ctypes.Structure):
    _fields_ = [
        ("dtype", c_int32), ("n_seqs", c_int32), ("n_groups", c_int32), ("reserved0", c_int32),
        ("n_rows", c_int64), ("vocab", c_int64), ("ld", c_int64),
        ("logits", c_void_p), ("row_index", c_void_p), ("anchor_logits", c_void_p),
        ("ld_anchor", c_int64),
        ("target", c_void_p), ("old_lp", c_void_p), ("ref_lp", c_void_p),
        ("seq_offsets", c_void_p), ("group_offsets", c_void_p), ("reward", c_void_p),
        ("seq_ref_lp", c_void_p), ("advantage", c_void_p), ("seq_kind", c_void_p),
        ("pg_coef", c_void_p), ("pg_loss", c_void_p),
    ]


class TgOut(ctypes.Structure):
    _fields_ = [
        ("dlogits", c_void_p), ("ld_out", c_int64), ("lp", c_void_p), ("entropy", c_void_p),
        ("lse", c_void_p), ("seq_lp", c_void_p), ("seq_adv", c_void_p), ("stats", c_void_p),
        ("row_coef", c_void_p),
    ]


EXPORTED = [
    "tg_workspace_size", "tg_loss_fwd_bwd", "tg_logprob_fwd", "tg_route", "tg_strerror",
    "tg_last_error", "tg_abi_version", "tg_scored_states", "tg_group_by_task",
    "tg_set_timing_events", "tg_launch_count", "tg_pack_rows", "tg_lmhead_logprob_fwd",
    "tg_lmhead_workspace_size", "tg_apply_update", "tg_lmhead_dlogits", "tg_fused_cluster_size",
    "tg_lmhead_grad_hidden", "tg_lmhead_grad_weight", "tg_lmhead_grad_chunk", "tg_adamw_step",
]

ABI_VERSION = 5  # include/tg_loss.h TG_ABI_VERSION

_lib = None


class NativeError(RuntimeError):
    """A libtg_loss call failed (bad argument, CUDA error, workspace too small)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"{msg} (code {code})")
        self.code = code


def lib_path() -> Path:
    return Path(os.environ.get("TG_LOSS_LIB", _LIB_PATH))


def lib() -> ctypes.CDLL:
    """Load libtg_loss.so once; raise loudly if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not path.exists():
        raise RuntimeError(
            f"{path} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    L = ctypes.CDLL(str(path))
    L.tg_workspace_size.restype = c_size_t
    L.tg_workspace_size.argtypes = [POINTER(TgBatch), POINTER(TgConfig)]
    L.tg_loss_fwd_bwd.restype = c_int
    L.tg_loss_fwd_bwd.argtypes = [POINTER(TgBatch), POINTER(TgConfig), POINTER(TgOut), c_void_p,
                                  c_size_t, c_void_p]
    L.tg_logprob_fwd.restype = c_int
    L.tg_logprob_fwd.argtypes = [POINTER(TgBatch), POINTER(TgOut), c_void_p, c_size_t, c_void_p]
    L.tg_route.restype = c_int
    L.tg_route.argtypes = [POINTER(TgBatch), POINTER(TgConfig)]
    L.tg_fused_cluster_size.restype = c_int
    L.tg_fused_cluster_size.argtypes = [POINTER(TgBatch), POINTER(TgConfig)]
    L.tg_strerror.restype = c_char_p
    L.tg_strerror.argtypes = [c_int]
    L.tg_last_error.restype = c_char_p
    L.tg_last_error.argtypes = []
    L.tg_abi_version.restype = c_int
    L.tg_scored_states.restype = c_int64
    L.tg_scored_states.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                   c_void_p, c_void_p, c_int64]
    L.tg_group_by_task.restype = c_int64
    L.tg_group_by_task.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                   c_int64, c_int32, c_void_p]
    L.tg_set_timing_events.restype = c_int
    L.tg_set_timing_events.argtypes = [c_void_p, c_void_p]
    L.tg_launch_count.restype = c_int64
    L.tg_launch_count.argtypes = []
    L.tg_pack_rows.restype = c_int
    L.tg_pack_rows.argtypes = [c_void_p, c_void_p, c_int, c_int32, c_int32, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                               c_void_p, c_void_p, c_size_t, c_void_p]
    L.tg_lmhead_logprob_fwd.restype = c_int
    L.tg_lmhead_logprob_fwd.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
                                        c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_size_t, c_void_p]
    L.tg_apply_update.restype = c_int
    L.tg_apply_update.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int, c_int64,
                                  c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_double,
                                  c_void_p, c_void_p]
    L.tg_lmhead_workspace_size.restype = c_size_t
    L.tg_lmhead_workspace_size.argtypes = [c_int64, c_int64]
    L.tg_lmhead_dlogits.restype = c_int
    L.tg_lmhead_dlogits.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
                                    c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_int64, c_void_p]
    L.tg_lmhead_grad_hidden.restype = c_int
    L.tg_lmhead_grad_hidden.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
                                        c_int64, c_int64, c_int64, c_void_p, c_int64, c_int,
                                        c_void_p]
    L.tg_lmhead_grad_weight.restype = c_int
    L.tg_lmhead_grad_weight.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
                                        c_int64, c_void_p, c_int64, c_void_p]
    L.tg_lmhead_grad_chunk.restype = c_int
    L.tg_lmhead_grad_chunk.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64,
                                       c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p,
                                       c_int64, c_int, c_void_p, c_int64, c_void_p]
    L.tg_adamw_step.restype = c_int
    L.tg_adamw_step.argtypes = [c_void_p, c_int, c_int64, c_void_p, c_int, c_int64, c_void_p,
                                c_void_p, c_int64, c_int64, c_double, c_double, c_double,
                                c_double, c_double, c_int64, c_void_p, c_void_p]
    if L.tg_abi_version() != ABI_VERSION:
        raise RuntimeError("libtg_loss ABI mismatch")
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != TG_OK:
        L = lib()
        raise NativeError(rc, f"{L.tg_strerror(rc).decode()}: {L.tg_last_error().decode()}")
