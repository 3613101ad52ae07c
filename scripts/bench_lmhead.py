"""Throughput of the fused LM-head logprob forward (tg_lmhead_logprob_fwd) at
Qwen2.5 shapes: TFLOP/s of the logits GEMM (2 T V d) against the measured bf16
peak, with cuBLAS (torch.matmul into materialised logits) timed beside it;
plus the training step from hidden states (loss + d hidden + d W), vocabulary
chunked through tg_lmhead_dlogits, against the unfused GEMM + loss + GEMMs.

    python scripts/bench_lmhead.py [--rows 16384] [--dim 1536] [--vocab 151936]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2505_17826_b200 import lmhead_logprob_fwd, logprob_fwd, pack_arrays  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=int, default=16384)
    p.add_argument("--dim", type=int, default=1536)
    p.add_argument("--vocab", type=int, default=151936)
    p.add_argument("--chunk", type=int, default=16384, help="vocabulary chunk of the backward")
    a = p.parse_args()
    T, d, V = a.rows, a.dim, a.vocab
    h = torch.randn(T, d, device="cuda").to(torch.bfloat16)
    w = (torch.randn(V, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
    y = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
    flops = 2.0 * T * V * d
    ms = timed(lambda: lmhead_logprob_fwd(h, w, y))
    ms_cublas = timed(lambda: torch.matmul(h, w.T))
    # unfused baseline: cuBLAS writes the bf16 logits, the streaming logprob kernel reads them
    logits = torch.matmul(h, w.T)
    import numpy as np
    batch = pack_arrays(logits, y.cpu().numpy(), [T], [1], np.zeros(1, np.float32))

    def unfused():
        torch.matmul(h, w.T, out=logits)
        logprob_fwd(batch)
    ms_unfused = timed(unfused)
    # the RFT loss forward from hidden states vs GEMM + the loss from logits
    from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, lmhead_loss_fwd
    rl = RFTLoss(RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl",
                               kl_coef=0.001, loss_agg_mode="token-mean"))
    n_seq = max(1, T // 2048)
    lens, groups = [T // n_seq] * n_seq, [n_seq]
    rew = np.random.default_rng(0).integers(0, 2, n_seq).astype(np.float32)
    tgt_h = y.cpu().numpy()
    ms_loss_fused = timed(lambda: lmhead_loss_fwd(h, w, rl, tgt_h, lens, groups, rew), reps=5)
    lbatch = pack_arrays(logits, tgt_h, lens, groups, rew)

    def loss_unfused():
        torch.matmul(h, w.T, out=logits)
        rl(lbatch, dlogits=None)
    ms_loss_unfused = timed(loss_unfused, reps=5)
    # training step from hidden states: loss + d hidden + d W.  Chunked
    # (tg_lmhead_dlogits recompute + two GEMMs per vocabulary chunk, no [T, V]
    # buffer) against the unfused step (GEMM -> logits, the fused loss kernel
    # in place, then the two gradient GEMMs over the full [T, V] dlogits).
    from paper_2505_17826_b200 import lmhead_dlogits, lmhead_loss_fwd_bwd
    ms_train_chunked = timed(lambda: lmhead_loss_fwd_bwd(h, w, rl, tgt_h, lens, groups, rew,
                                                         chunk_cols=a.chunk), reps=3)
    dh_u = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    dw_u = torch.empty(V, d, dtype=torch.bfloat16, device="cuda")

    def train_unfused():
        torch.matmul(h, w.T, out=logits)
        rl(lbatch, dlogits="inplace")
        torch.mm(logits, w, out=dh_u)
        torch.mm(logits.T, h, out=dw_u)
    ms_train_unfused = timed(train_unfused, reps=3)
    fo = lmhead_loss_fwd(h, w, rl, tgt_h, lens, groups, rew, row_coef=True)
    nc = min(a.chunk, V)
    dzb = torch.empty(T, nc, dtype=torch.bfloat16, device="cuda")
    ms_dz = timed(lambda: lmhead_dlogits(h, w, fo.target, fo.lse, fo.row_coef, 0, nc, out=dzb))
    # the two backward GEMMs of one chunk: tcgen05 (tg_lmhead_grad_*) vs cuBLAS
    from paper_2505_17826_b200 import lmhead_grad_hidden, lmhead_grad_weight
    dzc = (torch.randn(T, nc, device="cuda") * 1e-3).to(torch.bfloat16)
    dh_buf = torch.zeros(T, d, dtype=torch.float32, device="cuda")
    dw_buf = torch.empty(nc, d, dtype=torch.bfloat16, device="cuda")
    ms_gh = timed(lambda: lmhead_grad_hidden(dzc, w, 0, dh_buf, accumulate=True))
    ms_gw = timed(lambda: lmhead_grad_weight(dzc, h, dw_buf))
    from paper_2505_17826_b200 import lmhead_grad_chunk
    ms_gc = timed(lambda: lmhead_grad_chunk(dzc, h, w, 0, dh_buf, dw_buf, accumulate=True))
    ms_gh_cublas = timed(lambda: torch.addmm(dh_buf, dzc, w[:nc], out_dtype=torch.float32))
    ms_gw_cublas = timed(lambda: torch.mm(dzc.t(), h, out=dw_buf))
    gflop_c = 2.0 * T * nc * d / 1e9
    del dzb, dzc
    lp_f, _, lse_f = lmhead_logprob_fwd(h, w, y)
    # train_unfused left dlogits in the logits buffer: recompute the logits first
    torch.matmul(h, w.T, out=logits)
    lp_u, _, lse_u, _ = logprob_fwd(batch)
    dlse = float((lse_f - lse_u).abs().max())
    peak = peak_sus = None
    try:
        mp = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        peak, peak_sus = mp["bf16_tflops"], mp.get("bf16_tflops_sustained")
    except Exception:
        pass
    out = {"kernel": "k_lmhead_logprob", "rows": T, "dim": d, "vocab": V, "ms": ms,
           "tflops": flops / ms / 1e9, "peak_tflops": peak,
           "frac": (flops / ms / 1e9 / peak) if peak else None,  # vs the burst peak
           "peak_tflops_sustained": peak_sus,
           "frac_of_sustained": (flops / ms / 1e9 / peak_sus) if peak_sus else None,
           "cublas_gemm_only_ms": ms_cublas, "cublas_tflops": flops / ms_cublas / 1e9,
           "tokens_per_s": T / ms * 1e3, "unfused_cublas_plus_logprob_ms": ms_unfused,
           "speedup_vs_unfused": ms_unfused / ms,
           "max_abs_lse_diff_vs_unfused_bf16_logits": dlse,
           "loss_fwd_from_hidden_ms": ms_loss_fused,
           "loss_fwd_unfused_gemm_plus_loss_ms": ms_loss_unfused,
           "train_step_chunked_ms": ms_train_chunked, "train_chunk_cols": a.chunk,
           "train_step_unfused_ms": ms_train_unfused,
           "dlogits_kernel_ms_per_chunk": ms_dz,
           "dlogits_kernel_tflops": 2.0 * T * nc * d / ms_dz / 1e9,
           "grad_hidden_ms_per_chunk": ms_gh, "grad_hidden_tflops": gflop_c / ms_gh,
           "grad_hidden_cublas_tflops": gflop_c / ms_gh_cublas,
           "grad_weight_ms_per_chunk": ms_gw, "grad_weight_tflops": gflop_c / ms_gw,
           "grad_weight_cublas_tflops": gflop_c / ms_gw_cublas,
           "grad_chunk_one_launch_ms": ms_gc, "grad_chunk_tflops": 2 * gflop_c / ms_gc,
           "grad_pair_cublas_ms": ms_gh_cublas + ms_gw_cublas,
           "peak_note": "frac = vs the burst bf16 peak (an isolated kernel)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
