"""CPU-side checks of the C ABI library: it loads, exports every symbol the
header declares, its structs match ctypes, host helpers reproduce the
reference's integer work bit-exactly, and argument validation mirrors the
reference's errors (no device work is launched by any of these)."""

import ctypes
import re
import subprocess
import tempfile
from pathlib import Path

import numpy as np
import pytest

from _golden import groups_of, load
from paper_2505_17826_b200 import _native as N
from paper_2505_17826_b200 import AlgorithmError, RFTLossConfig
from paper_2505_17826_b200.packing import flatten_groups, group_by_task, scored_states
from paper_2505_17826_b200.registry import (ADVANTAGE_FNS, ENTROPY_LOSS_FNS, KL_FNS,
                                            LOSS_AGG_MODES, POLICY_LOSS_FNS)
from oracle import rft_oracle as O

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "tg_loss.h"


def header_functions():
    src = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(tg_[a-z_]+)\(", src, re.M)))


def test_library_exports_every_header_symbol():
    L = N.lib()
    names = header_functions()
    assert set(names) == set(N.EXPORTED), names
    for n in names:
        assert hasattr(L, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", str(N.lib_path())], capture_output=True,
                        text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", nm), n


def test_struct_layout_matches_header():
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "tg_loss.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(TgConfig), sizeof(TgBatch), sizeof(TgOut),
         offsetof(TgBatch, seq_kind), offsetof(TgConfig, n_sft_seq_global), offsetof(TgOut, stats));
  printf("%d %d %d\n", TG_NSTAT, TG_S_INVALID, TG_S_SUM_ANCHOR_KL);
  printf("%zu %d %d %d %d\n", offsetof(TgOut, row_coef), TG_FLAG_FORCE_TWO_PASS,
         TG_FLAG_ROWS_GIVEN, TG_FLAG_UNSCALED_GRAD, TG_ABI_VERSION);
  printf("%zu %d\n", offsetof(TgBatch, pg_loss), TG_PG_GIVEN);
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = Path(d) / "p.c"
        c.write_text(prog)
        exe = Path(d) / "p"
        subprocess.run(["gcc", "-I", str(ROOT / "include"), str(c), "-o", str(exe)], check=True)
        out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    sizes = list(map(int, out))
    assert sizes[0] == ctypes.sizeof(N.TgConfig)
    assert sizes[1] == ctypes.sizeof(N.TgBatch)
    assert sizes[2] == ctypes.sizeof(N.TgOut)
    assert sizes[3] == N.TgBatch.seq_kind.offset
    assert sizes[4] == N.TgConfig.n_sft_seq_global.offset
    assert sizes[5] == N.TgOut.stats.offset
    assert sizes[6] == N.NSTAT == O.NSTAT
    assert sizes[7] == N.STAT["invalid"] == O.STAT["invalid"]
    assert sizes[8] == N.STAT["sum_anchor_kl"]
    assert N.STAT_NAMES == O.STAT_NAMES
    assert sizes[9] == N.TgOut.row_coef.offset
    assert (sizes[10], sizes[11], sizes[12]) == (N.TG_FLAG_FORCE_TWO_PASS, N.TG_FLAG_ROWS_GIVEN,
                                                 N.TG_FLAG_UNSCALED_GRAD)
    assert sizes[13] == N.ABI_VERSION
    assert (sizes[14], sizes[15]) == (N.TgBatch.pg_loss.offset, N.TG_PG_GIVEN)


@pytest.mark.parametrize("name", ["simple_tau05", "kimi", "pairwise", "simple_bf16_v512",
                                  "simple_v4_uniform", "sft", "dpo", "regularizer_g"])
def test_scored_states_match_reference(name):
    fx = load(name)
    h = flatten_groups(groups_of(fx))
    states, target = scored_states(h, fx["theta"].shape[0])
    assert np.array_equal(states, fx["states"])   # FNV bucket indexing: bit-exact
    assert np.array_equal(target, fx["target"])


@pytest.mark.parametrize("name", ["buffer_fifo", "buffer_priority"])
def test_group_by_task_matches_reference_buffer(name):
    fx = load(name)
    ready = fx["ready"].astype(bool)
    groups = group_by_task(fx["tasks"], ready, int(fx["group_size"]), int(fx["n_take"]),
                           policy=str(fx["policy"]), priority=fx["priority"],
                           id_rank=np.arange(len(ready)))
    assert np.array_equal(np.array(groups, np.int64).reshape(-1, int(fx["group_size"])),
                          fx["groups"])


def _dummy_batch():
    b = N.TgBatch()
    b.dtype, b.n_seqs, b.n_groups = N.TG_DTYPE_BF16, 2, 1
    b.n_rows, b.vocab, b.ld = 4, 32, 32
    b.logits = b.target = b.seq_offsets = b.group_offsets = b.reward = 0x1000
    o = N.TgOut()
    o.stats = 0x2000
    return b, o


@pytest.mark.parametrize("mut,code", [
    (lambda b, c: setattr(c, "tau", -1.0), N.TG_EINVAL),
    (lambda b, c: (setattr(c, "policy_loss_fn", N.TG_PG_OPMD_KIMI), setattr(c, "tau", 0.0)),
     N.TG_EINVAL),
    (lambda b, c: setattr(c, "anchor_beta", 0.5), N.TG_EINVAL),      # beta > 0 needs anchor
    (lambda b, c: setattr(c, "dpo_beta", 0.0), N.TG_EINVAL),
    (lambda b, c: setattr(c, "kl_fn", 9), N.TG_EINVAL),
    (lambda b, c: setattr(b, "ld", 16), N.TG_EINVAL),                 # ld < vocab
    (lambda b, c: setattr(b, "dtype", 7), N.TG_EINVAL),
    (lambda b, c: setattr(c, "clip_c", 0.5), N.TG_EINVAL),
    (lambda b, c: None, N.TG_EWORKSPACE),                             # workspace too small
    # sequence-coupled losses refuse token-level terms instead of dropping them
    (lambda b, c: (setattr(c, "policy_loss_fn", N.TG_PG_OPMD_KIMI), setattr(c, "tau", 1.0),
                   setattr(c, "loss_agg_mode", 0), setattr(c, "kl_fn", N.TG_KL_K3),
                   setattr(c, "kl_coef", 0.1)), N.TG_EINVAL),
    (lambda b, c: (setattr(c, "policy_loss_fn", N.TG_PG_DPO), setattr(c, "loss_agg_mode", 0),
                   setattr(c, "entropy_loss_fn", N.TG_ENT_DEFAULT),
                   setattr(c, "entropy_coef", 0.01)), N.TG_EINVAL),
    (lambda b, c: (setattr(c, "policy_loss_fn", N.TG_PG_OPMD_PAIRWISE), setattr(c, "tau", 1.0),
                   setattr(c, "loss_agg_mode", N.TG_AGG_TOKEN_MEAN)), N.TG_EINVAL),
    (lambda b, c: (setattr(c, "policy_loss_fn", N.TG_PG_OPMD_PAIRWISE), setattr(c, "tau", 1.0),
                   setattr(c, "loss_agg_mode", 0), setattr(b, "seq_kind", 0x1000)), N.TG_EINVAL),
])
def test_validation_mirrors_reference_errors(mut, code):
    L = N.lib()
    b, o = _dummy_batch()
    c = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip").to_c()
    mut(b, c)
    rc = L.tg_loss_fwd_bwd(ctypes.byref(b), ctypes.byref(c), ctypes.byref(o), 0x3000, 16, None)
    assert rc == code, L.tg_last_error()
    assert L.tg_last_error().decode()


def test_config_validation_and_registry():
    for tbl in (ADVANTAGE_FNS, POLICY_LOSS_FNS, KL_FNS, ENTROPY_LOSS_FNS, LOSS_AGG_MODES):
        assert tbl and all(c.doc for c in tbl.values())
    assert RFTLossConfig(kl_fn="low_var_kl").kl_fn == "k3"
    with pytest.raises(AlgorithmError):
        RFTLossConfig(tau=-1)
    with pytest.raises(AlgorithmError):
        RFTLossConfig(policy_loss_fn="opmd_kimi", tau=0.0)
    with pytest.raises(AlgorithmError):
        RFTLossConfig(dpo_beta=0.0)
    with pytest.raises(KeyError):
        RFTLossConfig(advantage_fn="nope")
    c = RFTLossConfig.from_variant("OPMD_SIMPLE", tau=0.5, beta=0.2)
    assert (c.advantage_fn, c.policy_loss_fn, c.loss_agg_mode, c.anchor_beta) == \
        ("opmd", "vanilla", "seq-sum", 0.2)
    assert RFTLossConfig.from_variant("SFT").loss_agg_mode == "seq-mean-token-sum"
    assert RFTLossConfig.from_variant("DPO").coupled
    # coupled losses: aggregation defaults to the reference's group sum, and
    # token-level terms are refused rather than silently dropped
    assert RFTLossConfig(policy_loss_fn="opmd_kimi", tau=1.0).loss_agg_mode == "seq-sum"
    assert RFTLossConfig().loss_agg_mode == "token-mean"
    for bad in (dict(kl_fn="k3", kl_coef=0.1), dict(entropy_loss_fn="default", entropy_coef=0.01),
                dict(loss_agg_mode="token-mean")):
        for pg in ("opmd_kimi", "opmd_pairwise", "dpo"):
            with pytest.raises(AlgorithmError):
                RFTLossConfig(policy_loss_fn=pg, tau=1.0, **bad)
    RFTLossConfig(policy_loss_fn="dpo", kl_fn="k3", kl_coef=0.0)  # a zero coefficient is no term


def test_lmhead_and_update_argument_validation():
    """tg_lmhead_logprob_fwd / tg_apply_update reject bad arguments before any
    device work (no GPU needed)."""
    L = N.lib()
    p = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    # dim not a multiple of 64
    rc = L.tg_lmhead_logprob_fwd(p, 96, p, 96, 128, 1000, 96, None, None, p, p, None, 0, None)
    assert rc == N.TG_EINVAL and b"multiple of 64" in L.tg_last_error()
    # row pitch below dim
    rc = L.tg_lmhead_logprob_fwd(p, 64, p, 64, 128, 1000, 128, None, None, p, p, None, 0, None)
    assert rc == N.TG_EINVAL and b"pitch" in L.tg_last_error()
    # lp without target
    rc = L.tg_lmhead_logprob_fwd(p, 128, p, 128, 128, 1000, 128, None, p, p, p, None, 0, None)
    assert rc == N.TG_EINVAL and b"target" in L.tg_last_error()
    # zero rows: nothing to do
    assert L.tg_lmhead_logprob_fwd(p, 128, p, 128, 0, 1000, 128, None, None, p, p, None, 0,
                                   None) == N.TG_OK
    # apply_update: learning rate, pitch, dtype, too many touched states
    args = dict(ld_table=100, n_states=8, vocab=100, dtype=N.TG_DTYPE_F32, ld_grad=100,
                n_touched=2, n_rows=4, lr=0.1)

    def upd(**kw):
        a = {**args, **kw}
        return L.tg_apply_update(p, a["ld_table"], a["n_states"], a["vocab"], p, a["dtype"],
                                 a["ld_grad"], p, p, p, a["n_touched"], a["n_rows"], a["lr"], p,
                                 None)

    assert upd(lr=0.0) == N.TG_EINVAL and b"learning_rate" in L.tg_last_error()
    assert upd(ld_grad=50) == N.TG_EINVAL
    assert upd(dtype=7) == N.TG_EINVAL
    assert upd(n_touched=70000) == N.TG_EINVAL


def test_rows_given_flag_validation():
    """TG_FLAG_ROWS_GIVEN (loss from precomputed rows) is forward-only and
    needs lp / entropy / lse as inputs; rejected before any device work."""
    L = N.lib()
    b = N.TgBatch()
    b.dtype, b.n_rows, b.vocab, b.ld, b.n_seqs, b.n_groups = N.TG_DTYPE_BF16, 4, 100, 100, 1, 1
    cfg = N.TgConfig()
    cfg.flags = N.TG_FLAG_ROWS_GIVEN
    cfg.dpo_beta = 0.1
    o = N.TgOut()
    o.stats = 16
    rc = L.tg_loss_fwd_bwd(ctypes.byref(b), ctypes.byref(cfg), ctypes.byref(o), None, 0, None)
    assert rc == N.TG_EINVAL and b"out.lp" in L.tg_last_error()
    o.lp = o.entropy = o.lse = 16
    o.dlogits, o.ld_out = 16, 100
    rc = L.tg_loss_fwd_bwd(ctypes.byref(b), ctypes.byref(cfg), ctypes.byref(o), None, 0, None)
    assert rc == N.TG_EINVAL and b"forward-only" in L.tg_last_error()


def test_pack_arrays_rejects_misshaped_side_inputs():
    """Host-side shape checks the C ABI cannot do: short arrays
    would be read out of bounds on the device, long ones silently misaligned."""
    import torch
    from paper_2505_17826_b200 import pack_arrays

    logits = torch.zeros(10, 16)
    tgt = np.arange(10) % 16
    ok = dict(old_lp=np.zeros(10), ref_lp=np.zeros(10), seq_ref_lp=np.zeros(3),
              advantage=np.zeros(3), seq_kind=[0, 0, 1])
    b = pack_arrays(logits, tgt, [4, 3, 3], [3], np.zeros(3), **ok)
    assert (b.n_rows, b.n_seqs, b.n_sft_seqs) == (10, 3, 1)
    for name, bad in (("old_lp", np.zeros(30)), ("ref_lp", np.zeros(9)),
                      ("seq_ref_lp", np.zeros(2)), ("advantage", np.zeros(10)),
                      ("seq_kind", [0, 1])):
        with pytest.raises(AlgorithmError, match=name):
            pack_arrays(logits, tgt, [4, 3, 3], [3], np.zeros(3), **{**ok, name: bad})
    with pytest.raises(AlgorithmError, match="reward"):
        pack_arrays(logits, tgt, [4, 3, 3], [3], np.zeros(4))
    with pytest.raises(AlgorithmError, match="row_index"):
        pack_arrays(logits, tgt, [4, 3, 3], [3], np.zeros(3), row_index=np.arange(10) + 1)
    with pytest.raises(AlgorithmError, match="row_index"):
        pack_arrays(logits, tgt, [4, 3, 3], [3], np.zeros(3), row_index=np.arange(9))
    with pytest.raises(AlgorithmError, match="logits rows"):
        pack_arrays(logits[:8], tgt, [4, 3, 3], [3], np.zeros(3))
    with pytest.raises(AlgorithmError, match="anchor_logits"):
        pack_arrays(logits, tgt, [4, 3, 3], [3], np.zeros(3), anchor_logits=torch.zeros(10, 8))


def test_registry_user_components_and_errors():
    """Python components lower to the GIVEN codes; names are unique; built-ins
    cannot be shadowed or removed (no silent aliasing)."""
    from paper_2505_17826_b200.registry import (register_advantage_fn, register_policy_loss_fn,
                                                unregister)

    @register_policy_loss_fn("cpu_test_pg", aliases=("cpu_test_pg_alias",))
    def pg(x):
        """doc"""
        return -x.advantage * x.lp

    @register_advantage_fn("cpu_test_adv")
    def adv(x):
        return x.reward

    try:
        cfg = RFTLossConfig(advantage_fn="cpu_test_adv", policy_loss_fn="cpu_test_pg_alias")
        assert cfg.policy_loss_fn == "cpu_test_pg" and cfg.policy_loss_callable is pg
        assert cfg.advantage_callable is adv
        c = cfg.to_c()
        assert (c.policy_loss_fn, c.advantage_fn) == (N.TG_PG_GIVEN, N.TG_ADV_GIVEN)
        assert RFTLossConfig().policy_loss_callable is None
        with pytest.raises(ValueError, match="already registered"):
            register_policy_loss_fn("ppo_clip")(pg)
        with pytest.raises(ValueError, match="already registered"):
            register_advantage_fn("x", aliases=("grpo",))(adv)
        assert "x" not in ADVANTAGE_FNS  # nothing half-registered
        with pytest.raises(ValueError, match="built-in"):
            unregister(POLICY_LOSS_FNS, "ppo_clip")
    finally:
        unregister(POLICY_LOSS_FNS, "cpu_test_pg")
        unregister(ADVANTAGE_FNS, "cpu_test_adv")
    assert "cpu_test_pg_alias" not in POLICY_LOSS_FNS


def test_adamw_argument_validation():
    """tg_adamw_step checks torch.optim.AdamW's arguments (same messages) and
    the shapes before any device work; an empty block is a no-op."""
    L = N.lib()
    p = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    base = dict(pdt=N.TG_DTYPE_BF16, ldp=64, gdt=N.TG_DTYPE_BF16, ldg=64, rows=8, cols=64,
                lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, wd=0.01, step=1)

    def step(**kw):
        a = {**base, **kw}
        return L.tg_adamw_step(p, a["pdt"], a["ldp"], p, a["gdt"], a["ldg"], p, p, a["rows"],
                               a["cols"], a["lr"], a["b1"], a["b2"], a["eps"], a["wd"],
                               a["step"], None, None)

    cases = [(dict(lr=-1.0), b"Invalid learning rate"), (dict(eps=-1.0), b"Invalid epsilon"),
             (dict(b1=1.0), b"Invalid beta parameter at index 0"),
             (dict(b2=-0.1), b"Invalid beta parameter at index 1"),
             (dict(wd=-0.5), b"Invalid weight_decay"), (dict(step=0), b"step must be >= 1"),
             (dict(pdt=7), b"unknown dtype"), (dict(ldp=32), b"row pitch"),
             (dict(rows=-1), b"bad sizes")]
    for kw, msg in cases:
        assert step(**kw) == N.TG_EINVAL, kw
        assert msg in L.tg_last_error(), (kw, L.tg_last_error())
    assert step(rows=0) == N.TG_OK  # nothing to update, no device work
