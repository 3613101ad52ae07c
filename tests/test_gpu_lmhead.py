"""Fused LM-head + log-softmax forward (tcgen05, tg_lmhead_logprob_fwd) against
a plain PyTorch fp32 reference of the same op (logits = hidden @ weight.T in
fp32 from the bf16 inputs, then log-softmax / entropy / target gather).

Tolerances: the tensor cores multiply bf16 exactly and accumulate in fp32, so
the only difference from the fp32 reference is summation order over d terms:
lse / lp within 2e-4 abs + 1e-5 rel, entropy within 2e-4 abs."""

import numpy as np
import pytest
import torch

from paper_2505_17826_b200 import lmhead_logprob_fwd

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)


def reference(h, w, y):
    torch.backends.cuda.matmul.allow_tf32 = False
    z = h.float() @ w.float().T
    lse = torch.logsumexp(z, dim=1)
    p = torch.softmax(z, dim=1)
    ent = lse - (p * z).sum(1)
    lp = z.gather(1, y.long()[:, None])[:, 0] - lse
    return lp, ent, lse


def make(T, V, d, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    h = (torch.randn(T, d, device="cuda", generator=g) * scale).to(torch.bfloat16)
    w = (torch.randn(V, d, device="cuda", generator=g) / d ** 0.5 * 3.0).to(torch.bfloat16)
    y = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
    return h, w, y


# small row counts take the vocabulary-split + merge path; 37,888 rows = 2 full
# waves of 128-row blocks on 148 SMs takes the unsplit one
@pytest.mark.parametrize("T,V,d", [(128, 256, 64), (300, 1000, 128), (257, 4097, 256),
                                   (512, 32000, 512), (200, 151936, 1536), (37888, 1000, 64)])
def test_lmhead_matches_torch_fp32(T, V, d):
    h, w, y = make(T, V, d, seed=T + V + d)
    lp, ent, lse = lmhead_logprob_fwd(h, w, y)
    torch.cuda.synchronize()
    rlp, rent, rlse = reference(h, w, y)
    assert torch.isfinite(lse).all() and torch.isfinite(ent).all()
    torch.testing.assert_close(lse, rlse, atol=2e-4, rtol=1e-5)
    torch.testing.assert_close(lp, rlp, atol=2e-4, rtol=1e-5)
    torch.testing.assert_close(ent, rent, atol=2e-4, rtol=1e-4)


def test_lmhead_without_target_and_padded_pitch():
    T, V, d = 130, 2000, 192
    h, w, y = make(T, V, d, seed=7)
    hp = torch.zeros(T, d + 64, dtype=torch.bfloat16, device="cuda")
    hp[:, :d] = h
    lp, ent, lse = lmhead_logprob_fwd(hp[:, :d], w)
    assert lp is None
    _, rent, rlse = reference(h, w, y)
    torch.testing.assert_close(lse, rlse, atol=2e-4, rtol=1e-5)
    torch.testing.assert_close(ent, rent, atol=2e-4, rtol=1e-4)


def test_lmhead_peaked_rows_and_determinism():
    # large logits (one dominant column per row) exercise the running-max rescale
    T, V, d = 256, 5000, 256
    h, w, y = make(T, V, d, seed=11, scale=4.0)
    a = lmhead_logprob_fwd(h, w, y)
    b = lmhead_logprob_fwd(h, w, y)
    for x, z in zip(a, b):
        assert torch.equal(x, z)
    rlp, rent, rlse = reference(h, w, y)
    torch.testing.assert_close(a[2], rlse, atol=5e-4, rtol=1e-5)
    torch.testing.assert_close(a[0], rlp, atol=5e-4, rtol=1e-5)


def test_lmhead_argument_errors():
    h, w, y = make(128, 512, 64, seed=3)
    with pytest.raises(Exception):
        lmhead_logprob_fwd(h[:, :32].contiguous(), w[:, :32].contiguous(), y)  # d % 64 != 0
    with pytest.raises(ValueError):
        lmhead_logprob_fwd(h, w[:, :32].contiguous(), y)
    with pytest.raises(TypeError):
        lmhead_logprob_fwd(h.float(), w, y)


@pytest.mark.parametrize("cfg_kw", [
    dict(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl", kl_coef=0.001,
         entropy_loss_fn="default", entropy_coef=0.001, loss_agg_mode="token-mean"),
    dict(policy_loss_fn="opmd_kimi", tau=0.7),
    dict(advantage_fn="grpo", policy_loss_fn="ppo_clip", loss_agg_mode="token-mean",
         sft_weight=1.0),
], ids=["grpo_ppo_k3_ent", "kimi", "mixed_sft"])
def test_loss_from_hidden_states_matches_logits_path(cfg_kw):
    """RFT loss straight from hidden states (LM-head kernel + loss epilogue on
    the rows, TG_FLAG_ROWS_GIVEN) equals the loss computed from fp32 logits."""
    from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, lmhead_loss_fwd, pack_arrays
    T_seq, B, d, V = 64, 8, 256, 32000
    T = T_seq * B
    h, w, y = make(T, V, d, seed=5)
    rng = np.random.default_rng(5)
    reward = rng.integers(0, 2, B).astype(np.float32)
    old = (rng.normal(-8.0, 0.5, T)).astype(np.float32)
    ref = (rng.normal(-8.0, 0.5, T)).astype(np.float32)
    seq_ref = rng.normal(-500.0, 10.0, B).astype(np.float32)
    kind = np.array([0, 0, 0, 0, 1, 1, 1, 1], np.uint8) if cfg_kw.get("sft_weight") else None
    side = dict(old_lp=old, ref_lp=ref, seq_ref_lp=seq_ref, seq_kind=kind)
    cfg = RFTLossConfig(**cfg_kw)
    loss = RFTLoss(cfg)
    got = lmhead_loss_fwd(h, w, loss, y.cpu().numpy(), [T_seq] * B, [4, 4], reward, **side)
    torch.backends.cuda.matmul.allow_tf32 = False
    z = (h.float() @ w.float().T).contiguous()
    want = loss(pack_arrays(z, y.cpu().numpy(), [T_seq] * B, [4, 4], reward, **side),
                dlogits=None)
    a, b = got.stats_dict(), want.stats_dict()
    for k in ("loss", "pg_loss", "kl_loss", "entropy_loss", "sft_loss", "sum_lp",
              "sum_entropy", "clip_count", "n_tok"):
        assert a[k] == pytest.approx(b[k], rel=1e-4, abs=1e-5), k
    torch.testing.assert_close(got.seq_lp, want.seq_lp, atol=2e-3, rtol=1e-5)
    assert got.dlogits is None


@pytest.mark.parametrize("cfg_kw", [
    dict(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl", kl_coef=0.001,
         entropy_loss_fn="default", entropy_coef=0.001, loss_agg_mode="token-mean"),
    dict(policy_loss_fn="opmd_kimi", tau=0.7),
    dict(advantage_fn="grpo", policy_loss_fn="ppo_clip", loss_agg_mode="token-mean",
         sft_weight=1.0),
], ids=["grpo_ppo_k3_ent", "kimi", "mixed_sft"])
def test_loss_backward_from_hidden_states_matches_fp32(cfg_kw):
    """Vocabulary-chunked backward from hidden states (tg_lmhead_dlogits +
    two GEMMs per chunk) against the fp32-logits path: dlogits of the fp32
    logits (the parity-tested fp32 kernel path), then d hidden = dz W and
    d W = dz^T h in fp32.  The chunk (1,000 columns) is not a multiple of the
    256-column tile and V = 3,000 is not either.

    Tolerances: dz is stored in bf16 (relative rounding 2^-9 per element), so
    per element 2^-8 max|dz| + 1e-2 |dz| (the parity bar of the dlogits
    tests); d hidden / d W as relative Frobenius error <= 1e-2."""
    from paper_2505_17826_b200 import (RFTLoss, RFTLossConfig, lmhead_dlogits,
                                       lmhead_loss_fwd_bwd, pack_arrays)
    T_seq, B, d, V = 48, 8, 256, 3000
    T = T_seq * B
    h, w, y = make(T, V, d, seed=11)
    rng = np.random.default_rng(11)
    reward = rng.integers(0, 2, B).astype(np.float32)
    old = (rng.normal(-8.0, 0.5, T)).astype(np.float32)
    ref = (rng.normal(-8.0, 0.5, T)).astype(np.float32)
    seq_ref = rng.normal(-400.0, 10.0, B).astype(np.float32)
    kind = np.array([0, 0, 0, 0, 1, 1, 1, 1], np.uint8) if cfg_kw.get("sft_weight") else None
    side = dict(old_lp=old, ref_lp=ref, seq_ref_lp=seq_ref, seq_kind=kind)
    loss = RFTLoss(RFTLossConfig(**cfg_kw))
    got, dh, dw = lmhead_loss_fwd_bwd(h, w, loss, y.cpu().numpy(), [T_seq] * B, [4, 4], reward,
                                      chunk_cols=1000, **side)
    torch.backends.cuda.matmul.allow_tf32 = False
    z = (h.float() @ w.float().T).contiguous()
    want = loss(pack_arrays(z, y.cpu().numpy(), [T_seq] * B, [4, 4], reward, **side),
                dlogits="new")
    a, b = got.stats_dict(), want.stats_dict()
    for k in ("loss", "pg_loss", "kl_loss", "entropy_loss", "sft_loss", "sum_lp"):
        assert a[k] == pytest.approx(b[k], rel=1e-4, abs=1e-5), k
    dl = want.dlogits
    dh_ref = dl @ w.float()
    dw_ref = dl.T @ h.float()
    assert torch.isfinite(dh).all() and torch.isfinite(dw.float()).all()
    assert float((dh - dh_ref).norm() / dh_ref.norm()) < 1e-2
    assert float((dw.float() - dw_ref).norm() / dw_ref.norm()) < 1e-2
    # one chunk directly, at an offset that is not tile aligned
    dz = lmhead_dlogits(h, w, got.target, got.lse, got.row_coef, 1234, 777).float()
    want_c = dl[:, 1234:1234 + 777]
    tol = 2.0 ** -8 * float(want_c.abs().max()) + 1e-2 * want_c.abs()
    assert bool(((dz - want_c).abs() <= tol).all())


def test_lmhead_dlogits_argument_errors():
    from paper_2505_17826_b200 import lmhead_dlogits
    from paper_2505_17826_b200._native import NativeError
    h, w, y = make(128, 512, 64, seed=4)
    lse = torch.zeros(128, device="cuda")
    coef = torch.zeros(3, 128, device="cuda")
    with pytest.raises(NativeError):
        lmhead_dlogits(h, w, y, lse, coef, 500, 100)  # chunk past the vocabulary
    buf = torch.empty(128, 100, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(NativeError):
        lmhead_dlogits(h, w, y, lse, coef, 0, 99, out=buf[:, 1:])  # misaligned out
    with pytest.raises(ValueError):
        lmhead_dlogits(h, w, y, lse, coef[:2], 0, 64)


@pytest.mark.parametrize("T,V,d,col0,n_cols", [(1, 700, 64, 0, 700), (129, 1000, 128, 37, 601),
                                               (300, 4097, 192, 4000, 97),
                                               (513, 2048, 256, 256, 1792)])
def test_lmhead_dlogits_matches_formula(T, V, d, col0, n_cols):
    """tg_lmhead_dlogits against the formula in fp32 torch, with arbitrary row
    coefficients: dz = exp(z - lse) (a + hz z) - s [v = y] over the chunk.
    Row counts off the 128-row tile, chunk offsets / widths off the 256-column
    tile and the 8-column store granule."""
    from paper_2505_17826_b200 import lmhead_dlogits
    h, w, y = make(T, V, d, seed=T + col0)
    torch.backends.cuda.matmul.allow_tf32 = False
    z = h.float() @ w.float().T
    lse = torch.logsumexp(z, 1).contiguous()
    g = torch.Generator(device="cuda").manual_seed(5)
    coef = (torch.randn(3, T, device="cuda", generator=g) * 0.3).contiguous()
    got = lmhead_dlogits(h, w, y, lse, coef, col0, n_cols).float()
    zc = z[:, col0:col0 + n_cols]
    want = torch.exp(zc - lse[:, None]) * (coef[0][:, None] + coef[1][:, None] * zc)
    onehot = (y.long()[:, None] == torch.arange(col0, col0 + n_cols, device="cuda")[None, :])
    want = want - coef[2][:, None] * onehot.float()
    tol = 2.0 ** -8 * float(want.abs().max()) + 1e-2 * want.abs()
    assert bool(((got - want).abs() <= tol).all())


@pytest.mark.skipif(bool(__import__("os").environ.get("TG_LMHEAD_PAIR")),
                    reason="already pinned to one CTA mode by the environment")
@pytest.mark.parametrize("pair", ["0", "1"])
def test_lmhead_backward_in_both_cta_modes(pair):
    """The LM-head kernels (forward, backward chunks) and the backward GEMMs run
    as 2-CTA pairs by default and as single CTAs with TG_LMHEAD_PAIR=0 /
    TG_GEMM_PAIR=0; the mode is read once per process, so each runs the parity
    tests in a subprocess."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    ab = Path(__file__).resolve().parents[1] / "paper_2505_17826_b200" / "_lib" / "libtg_loss_ab.so"
    assert ab.exists(), "build the A/B variant (__graft_entry__.build())"
    env = dict(os.environ, TG_LMHEAD_PAIR=pair, TG_GEMM_PAIR=pair,
               TG_LOSS_LIB=str(ab))  # switches: A/B build
    r = subprocess.run([sys.executable, "-m", "pytest", __file__, "-q", "-x", "-p",
                        "no:cacheprovider", "-k", "matches_torch_fp32 or backward_from_hidden or "
                        "matches_formula or matches_float64 or random_shapes"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("TG_LMHEAD_SEEDS", 24))))
def test_lmhead_random_shapes(seed):
    """Seeded random shapes for both LM-head kernels: row counts off the tile
    grid (including 1), vocabularies off the 256-column tile, several d, and a
    random vocabulary chunk for the backward -- forward lse / entropy against
    torch fp32 and dz against the formula."""
    from paper_2505_17826_b200 import lmhead_dlogits
    r = np.random.default_rng(500 + seed)
    T = int(r.choice([1, 7, 128, 129, 300, 777]))
    V = int(r.integers(64, 5000))
    d = int(r.choice([64, 128, 256, 512]))
    h, w, y = make(T, V, d, seed=seed)
    lp, ent, lse = lmhead_logprob_fwd(h, w, y)
    rlp, rent, rlse = reference(h, w, y)
    torch.testing.assert_close(lse, rlse, atol=2e-4, rtol=1e-5)
    torch.testing.assert_close(ent, rent, atol=2e-4, rtol=1e-4)
    col0 = int(r.integers(0, V - 1))
    n = int(r.integers(1, V - col0 + 1))
    coef = (torch.randn(3, T, device="cuda", generator=torch.Generator(device="cuda")
                        .manual_seed(seed)) * 0.3).contiguous()
    got = lmhead_dlogits(h, w, y, rlse.contiguous(), coef, col0, n).float()
    z = (h.float() @ w.float().T)[:, col0:col0 + n]
    want = torch.exp(z - rlse[:, None]) * (coef[0][:, None] + coef[1][:, None] * z)
    want -= coef[2][:, None] * (y.long()[:, None] ==
                                torch.arange(col0, col0 + n, device="cuda")).float()
    tol = 2.0 ** -8 * float(want.abs().max()) + 1e-2 * want.abs()
    assert bool(((got - want).abs() <= tol).all())


# ---------------------------------------------------------------------------
# the backward GEMMs on tcgen05 (tg_lmhead_grad_hidden / tg_lmhead_grad_weight)
# against float64 torch products of the same bf16 operands.  The tensor cores
# multiply bf16 exactly and accumulate in fp32: the bar is fp32 summation
# noise, |a - b| <= 1e-5 (|A| |B|) + 1e-6 elementwise (plus bf16 rounding of
# the d W output, 2^-8 |b|).


def _gemm_operands(T, n, d, V, col0, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    pitch = (n + 7) // 8 * 8 + 8  # dz as a column slice of a wider buffer
    dz = torch.randn(T, pitch, device="cuda", generator=g).to(torch.bfloat16)[:, :n]
    w = torch.randn(V, d, device="cuda", generator=g).to(torch.bfloat16)
    h = torch.randn(T, d, device="cuda", generator=g).to(torch.bfloat16)
    return dz, w, h


@pytest.mark.parametrize("T,n,d,col0", [(128, 256, 256, 0), (300, 1000, 192, 100), (37, 72, 64, 5),
                                        (1024, 4096, 1536, 2048), (129, 65, 3584, 7)])
def test_grad_hidden_gemm_matches_float64(T, n, d, col0):
    from paper_2505_17826_b200 import lmhead_grad_hidden
    V = col0 + n + 3
    dz, w, h = _gemm_operands(T, n, d, V, col0, seed=T + n + d)
    wc = w[col0:col0 + n].double()
    want = dz.double() @ wc
    bound = dz.double().abs() @ wc.abs()
    base = torch.full((T, d), 0.25, device="cuda")
    got = lmhead_grad_hidden(dz, w, col0, base.clone(), accumulate=True).double()
    assert bool(((got - 0.25 - want).abs() <= 1e-5 * bound + 1e-6).all())
    got = lmhead_grad_hidden(dz, w, col0, base.clone(), accumulate=False).double()
    assert bool(((got - want).abs() <= 1e-5 * bound + 1e-6).all())


@pytest.mark.parametrize("T,n,d", [(128, 256, 256), (300, 1000, 192), (37, 72, 64), (2048, 4096, 1536),
                                   (777, 130, 3584)])
def test_grad_weight_gemm_matches_float64(T, n, d):
    from paper_2505_17826_b200 import lmhead_grad_weight
    dz, _, h = _gemm_operands(T, n, d, 1, 0, seed=7 * T + n)
    want = dz.double().T @ h.double()
    bound = dz.double().abs().T @ h.double().abs()
    out = torch.full((n + 2, d), 7.0, device="cuda").to(torch.bfloat16)
    got = lmhead_grad_weight(dz, h, out[1:n + 1]).double()
    assert bool(((got - want).abs() <= 2.0 ** -8 * want.abs() + 1e-5 * bound + 1e-6).all())
    assert bool((out[0] == 7.0).all() and (out[n + 1] == 7.0).all())  # rows outside untouched


def test_grad_gemm_argument_errors():
    from paper_2505_17826_b200 import lmhead_grad_hidden, lmhead_grad_weight
    from paper_2505_17826_b200._native import NativeError
    dz, w, h = _gemm_operands(64, 128, 64, 256, 0, seed=1)
    with pytest.raises(NativeError):  # chunk past the vocabulary
        lmhead_grad_hidden(dz, w, 200, torch.zeros(64, 64, device="cuda"))
    with pytest.raises(ValueError):   # wrong output shape
        lmhead_grad_hidden(dz, w, 0, torch.zeros(64, 32, device="cuda"))
    with pytest.raises(ValueError):
        lmhead_grad_weight(dz, h[:10], torch.empty(128, 64, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(NativeError):  # d W row pitch must be a multiple of 8 elements
        lmhead_grad_weight(dz, h, torch.empty(128, 68, dtype=torch.bfloat16, device="cuda")[:, :64])


@pytest.mark.parametrize("T,n,d,col0", [(300, 1000, 192, 100), (1024, 4096, 1536, 2048),
                                        (4096, 640, 256, 0), (37, 72, 64, 5)])
def test_grad_chunk_one_launch_matches_float64(T, n, d, col0):
    """tg_lmhead_grad_chunk: both GEMMs of a chunk on one tile queue (the job
    with the longer K first) give the two single-GEMM results."""
    from paper_2505_17826_b200 import lmhead_grad_chunk
    V = col0 + n + 9
    dz, w, h = _gemm_operands(T, n, d, V, col0, seed=3 * T + n)
    wc = w[col0:col0 + n].double()
    want_h = dz.double() @ wc
    bound_h = dz.double().abs() @ wc.abs()
    want_w = dz.double().T @ h.double()
    bound_w = dz.double().abs().T @ h.double().abs()
    dh = torch.full((T, d), -1.0, device="cuda")
    dw = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    lmhead_grad_chunk(dz, h, w, col0, dh, dw, accumulate=True)
    assert bool(((dh.double() + 1.0 - want_h).abs() <= 1e-5 * bound_h + 1e-6).all())
    err_w = (dw.double() - want_w).abs()
    assert bool((err_w <= 2.0 ** -8 * want_w.abs() + 1e-5 * bound_w + 1e-6).all())


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("TG_LMHEAD_SEEDS", 24))))
def test_grad_chunk_random_shapes(seed):
    """Seeded random shapes for the backward GEMM pair in one launch: rows,
    chunk widths and d off the 256 / 128 tile grids (tail-split half tiles
    and partial pair tiles included), against float64 products."""
    from paper_2505_17826_b200 import lmhead_grad_chunk
    r = np.random.default_rng(900 + seed)
    T = int(r.integers(1, 1200))
    n = int(r.integers(1, 400)) * 8
    d = int(r.choice([64, 128, 192, 256, 320, 512, 1536]))  # (d % 64 == 0: the API rule)
    col0 = int(r.integers(0, 64))
    V = col0 + n + int(r.integers(0, 9))
    dz, w, h = _gemm_operands(T, n, d, V, col0, seed=seed)
    wc = w[col0:col0 + n].double()
    want_h = dz.double() @ wc
    bound_h = dz.double().abs() @ wc.abs()
    want_w = dz.double().T @ h.double()
    bound_w = dz.double().abs().T @ h.double().abs()
    dh = torch.zeros(T, d, device="cuda")
    dw = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    lmhead_grad_chunk(dz, h, w, col0, dh, dw, accumulate=bool(seed % 2))
    assert bool(((dh.double() - want_h).abs() <= 1e-5 * bound_h + 1e-6).all()), (T, n, d)
    err_w = (dw.double() - want_w).abs()
    assert bool((err_w <= 2.0 ** -8 * want_w.abs() + 1e-5 * bound_w + 1e-6).all()), (T, n, d)
