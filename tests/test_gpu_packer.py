"""On-device packer (tg_pack_rows) against a numpy restatement of the packing
rule, and the loss through packed rows against the compacted layout."""

import numpy as np
import pytest
import torch

from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, pack_arrays
from paper_2505_17826_b200.packing import pack_token_batch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _batch(seed, B=6, L=77, V=1000):
    rng = np.random.default_rng(seed)
    ids = rng.integers(0, V, (B, L))
    mask = np.zeros((B, L), bool)
    for b in range(B):  # prompt, then multi-turn response spans with env text between
        p = int(rng.integers(2, 12))
        l = p
        while l < L:
            span = int(rng.integers(1, 15))
            mask[b, l:min(L, l + span)] = True
            l += span + int(rng.integers(1, 6))
    mask[1] = False  # an empty sequence
    old = rng.normal(-1.0, 0.3, (B, L)).astype(np.float32)
    return ids, mask, old


@pytest.mark.parametrize("ids_dtype", [torch.int64, torch.int32])
def test_pack_rows_matches_numpy(ids_dtype):
    ids, mask, old = _batch(0)
    B, L = ids.shape
    logits = torch.zeros((B, L, 1000), dtype=torch.bfloat16, device="cuda")
    pb = pack_token_batch(logits, torch.as_tensor(ids, device="cuda", dtype=ids_dtype),
                          torch.as_tensor(mask, device="cuda"), np.ones(B), [3, 3],
                          old_logprobs=torch.as_tensor(old, device="cuda"))
    want_idx, want_t, want_old, lens = [], [], [], []
    for b in range(B):
        n = 0
        for l in range(1, L):
            if mask[b, l]:
                want_idx.append(b * L + l - 1)
                want_t.append(ids[b, l])
                want_old.append(old[b, l])
                n += 1
        lens.append(n)
    assert pb.n_rows == len(want_idx)
    assert np.array_equal(pb.row_index.cpu().numpy(), want_idx)
    assert np.array_equal(pb.target.cpu().numpy(), want_t)
    assert np.array_equal(pb.old_lp.cpu().numpy(), np.array(want_old, np.float32))
    assert np.array_equal(np.diff(pb.seq_offsets.cpu().numpy()), lens)


def test_loss_through_device_packer():
    ids, mask, old = _batch(1, B=8, L=64, V=32000)
    B, L = ids.shape
    V = 32000
    logits = (torch.randn((B, L, V), device="cuda") * 2).to(torch.bfloat16)
    rewards = np.random.default_rng(2).integers(0, 2, B).astype(np.float32)
    cfg = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl",
                        kl_coef=0.01, loss_agg_mode="token-mean")
    pb = pack_token_batch(logits, torch.as_tensor(ids, device="cuda"),
                          torch.as_tensor(mask, device="cuda"), rewards, [4, 4],
                          old_logprobs=torch.as_tensor(old, device="cuda"),
                          ref_logprobs=torch.as_tensor(old, device="cuda"))
    a = RFTLoss(cfg)(pb)
    idx = pb.row_index
    compact = pack_arrays(logits.reshape(B * L, V)[idx].contiguous(), pb.target.cpu().numpy(),
                          np.diff(pb.seq_offsets.cpu().numpy()), [4, 4], rewards,
                          old_lp=pb.old_lp.cpu().numpy(), ref_lp=pb.ref_lp.cpu().numpy())
    b = RFTLoss(cfg)(compact)
    assert torch.equal(a.stats, b.stats)
    assert torch.equal(a.dlogits, b.dlogits)
