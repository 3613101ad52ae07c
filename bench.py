#!/usr/bin/env python
"""bench.py -- fused GRPO logprob + loss fwd/bwd throughput on B200.

Workload (BASELINE.json configs[1]): GRPO loss at Qwen2.5-1.5B shapes --
vocab 151,936, 64 prompts x 8 rollouts, 2,048-token responses = 1,048,576
trainable rows per GPU per step, bf16 logits, fp32 arithmetic.  Loss =
GRPO advantage (group mean / std) + PPO clip (0.2 / 0.28) + low_var_kl (k3,
0.001) + masked token-mean, gradient d loss / d logits written in bf16.

The step's logits are 318.6 GB, more than one B200 holds, so a step runs as 8
micro-batches of 8 groups (131,072 rows, 39.8 GB) each.  All micro-batches
read one resident synthetic logits buffer (N(0, 2^2) + a +13.5 bump at the
target, seeded) and write dlogits out of place to a second 39.8 GB buffer;
per-micro-batch targets are shared, rewards / old / ref logprobs differ.
Every micro-batch still streams its full 2V bytes per row in and 2V out:
the working set (80 GB) is ~600x the 126 MB L2, so no L2 flush is needed.

One process per GPU (torchrun for N > 1); each rank processes its own
1,048,576-row batch (weak scaling) and NCCL allreduces only the 32-double
statistics vector per step.  `value` = rows of all ranks / max-over-ranks
device time.  `e2e` = the same metric through the public API with pinned
HOST logits: H2D of the logits + metadata and D2H of dlogits + stats inside
the timed region, one e2e step = the same 1,048,576 rows (64 calls, 3-deep
copy / compute overlap).

`--variant c1|c3|c4|c5` runs the per-GPU workloads of BASELINE configs[0],
[2], [3], [4] (V = 32,000; PPO + k3 + entropy at 4,096 tokens; GRPO + SFT mix;
ragged long-CoT through row_index); `grpo_two_pass`, `opmd_kimi`,
`opmd_pairwise` measure the two-pass / sequence-coupled routes,
`opmd_kimi_unscaled` / `opmd_pairwise_unscaled` the single-pass coupled route
(unscaled gradient + per-row scales) and `anchor` the fused regularizer_g path
(6V bytes per row).  Kernel A/B: TG_LOSS_LIB selects a library build
(scripts/gpu_libab.sh).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--variant V]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tokens/sec of fused GRPO logprob+loss fwd/bwd at 1/2/4/8 B200; HBM GB/s vs peak"
UNIT = "tokens/s"
V = 151936
BUMP = 13.5
# behaviour-policy logprob = lp + N(0, sigma^2).  SURVEY.md 8(d) asks for a PPO
# clip fraction of about 5-20 % at eps = 0.2 / 0.28; its sigma = 0.05 gives
# ~0 % (ratios within exp(+-0.15)), sigma = 0.15 gives ~6 %.
OLD_LP_SIGMA = 0.15
ALGO_BYTES_PER_ROW = 4 * V + 24  # 2V read + 2V write + 24 B side data
WORKLOAD = "grpo_ppo_clip_k3_token_mean_qwen2.5_1.5b_shapes"
VARIANT_WORKLOAD = {
    "grpo": WORKLOAD,
    "c1": "configs[0]: GRPO loss, 8 prompts x 8 x 512 tokens, vocab 32,000 (the CPU "
          "reference's case) on 1 GPU",
    "c3": "configs[2] per-GPU shard: ppo_clip_k3_entropy, 16 prompts x 8 x 4096 tokens "
          "(128 x 8 over 8 GPUs)",
    "c4": "configs[3]: mixed GRPO + SFT NLL (50/50 sequences) at configs[1] shapes",
    "c5": "configs[4] per-GPU shard: long-CoT 32 groups x 16 ragged responses <= 8192, "
          "10 % interior mask-false spans, row_index gather (256 x 16 over 8 GPUs)",
}
_BASE_LOSS = "grpo adv + ppo_clip(0.2,0.28) + low_var_kl(0.001) + token-mean"
VARIANT_LOSS = {"grpo": _BASE_LOSS, "c1": _BASE_LOSS, "c3": _BASE_LOSS + " + entropy(0.001)",
                "c4": _BASE_LOSS + " on RL seqs + SFT NLL (weight 1) on expert seqs",
                "c5": _BASE_LOSS,
                "anchor": "opmd_simple(tau 1) + regularizer_g anchor KL (beta 0.1), fused (6V)"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--groups", type=int, default=64)
    p.add_argument("--group-size", type=int, default=8)
    p.add_argument("--resp-len", type=int, default=2048)
    p.add_argument("--mb-groups", type=int, default=8, help="groups per micro-batch")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--e2e-groups", type=int, default=0,
                   help="groups per e2e step (0 = the whole step's groups, as the device metric)")
    p.add_argument("--cpu-rows", type=int, default=256)
    p.add_argument("--quiet", action="store_true")
    p.add_argument("--variant", default="grpo",
                   choices=["grpo", "grpo_two_pass", "opmd_kimi", "opmd_pairwise", "sft",
                            "opmd_kimi_unscaled", "opmd_pairwise_unscaled", "anchor",
                            "c1", "c3", "c4", "c5"],
                   help="loss variant (the headline metric is 'grpo' = configs[1]; c3 / c4 / c5 "
                        "are the per-GPU shards of BASELINE configs[2..4]; the others measure "
                        "the two-pass / sequence-coupled routes)")
    a = p.parse_args()
    global V, BUMP, ALGO_BYTES_PER_ROW
    # per-GPU shards of the multi-GPU configs (weak scaling: fixed work per GPU)
    if a.variant == "c1":    # configs[0]: the CPU oracle's case, 8 x 8 x 512 at V = 32,000
        V, BUMP = 32000, 12.0
        ALGO_BYTES_PER_ROW = 4 * V + 24
        a.groups, a.group_size, a.resp_len, a.mb_groups = 8, 8, 512, 8
    elif a.variant == "c3":    # configs[2]: 128 x 8 rollouts x 4096 tokens over 8 GPUs
        a.groups, a.group_size, a.resp_len, a.mb_groups = 16, 8, 4096, 4
    elif a.variant == "c5":  # configs[4]: 256 x 16 rollouts, <= 8192 ragged tokens, 8 GPUs
        a.groups, a.group_size, a.resp_len, a.mb_groups = 32, 16, 8192, 2
    return a


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            d = json.loads(f.read_text())
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# clocks sampling during the timed region

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "power.draw,clocks.mem")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, power, mem, reasons = [], [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
            if len(parts) >= 9:
                try:
                    power.append(float(parts[7]))
                    mem.append(float(parts[8]))
                except ValueError:
                    pass
        out = {"sm_mhz": statistics.median(sm) if sm else None,
               "sm_max_mhz": max(smax) if smax else None,
               "reasons": sorted(reasons), "samples": len(sm)}
        if power:
            out["power_w"] = statistics.median(power)
            out["mem_mhz"] = statistics.median(mem)
        return out


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port (numpy float64), bounded sample

def cpu_sample(seed: int, rows: int, group_size: int):
    from oracle import rft_oracle as O
    rng = np.random.default_rng(seed)
    per = max(1, rows // group_size)
    T = per * group_size
    tgt = rng.integers(0, V, T)
    x = rng.normal(0, 2.0, (T, V))
    x[np.arange(T), tgt] += BUMP
    x = x.astype(np.float32).astype(np.float64)
    lp = O.row_forward(x, tgt)[1]
    b = O.Batch(logits=x, target=tgt, seq_offsets=np.arange(0, T + 1, per),
                group_offsets=np.array([0, group_size]),
                reward=rng.integers(0, 2, group_size).astype(np.float64),
                old_lp=lp + rng.normal(0, OLD_LP_SIGMA, T), ref_lp=lp + rng.normal(0, 0.1, T))
    return b


def oracle_cfg():
    from oracle import rft_oracle as O
    return O.Config(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="k3", kl_coef=0.001,
                    loss_agg_mode="token-mean", clip_lo=0.2, clip_hi=0.28)


def cpu_run(args_tuple):
    seed, rows, gsize = args_tuple
    from oracle import rft_oracle as O
    b = cpu_sample(seed, rows, gsize)
    dz = np.empty((b.n_rows, V), np.float32)
    t0 = time.perf_counter()
    O.single_pass_blocked(b, oracle_cfg(), dz_out=dz, block=32)
    return b.n_rows, time.perf_counter() - t0


def cpu_baseline(rows: int, gsize: int):
    n, dt = cpu_run((1234, rows, gsize))
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle/rft_oracle.single_pass_blocked (numpy f64, 1 thread) on {n} rows "
                      f"x V={V} (1 group x {gsize} seqs), same loss config; {dt:.2f} s"}


def run_reference(args):
    """--impl reference: the oracle port on all host cores (the reference is
    pure Python and cannot run on the GPU box)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    try:
        avail = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except Exception:
        avail = 64 << 30
    per_worker = args.cpu_rows * V * 4 * 8  # rough peak bytes of one worker
    workers = max(1, min(cores, int(0.5 * avail // per_worker), 64))
    ctx = mp.get_context("fork")
    rates = []
    with ctx.Pool(workers) as pool:
        for step in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = pool.map(cpu_run, [(1000 + step * workers + i, args.cpu_rows, args.group_size)
                                     for i in range(workers)])
            dt = time.perf_counter() - t0
            if step >= args.warmup:
                rates.append(sum(r[0] for r in res) / dt)
    value = statistics.median(rates)
    rows = workers * (args.cpu_rows // args.group_size) * args.group_size
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * rows / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "vocab": V,
                                        "sample_rows_per_step": rows},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": f"{workers} processes x {args.cpu_rows} rows x V={V} of the "
                                   "oracle port (numpy f64) per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, logprob_fwd, pack_arrays
    from paper_2505_17826_b200 import _native as N
    from paper_2505_17826_b200.distributed import allreduce_stats

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; TG_BENCH_BACKEND=gloo lets a multi-rank smoke run share
    # a single GPU (NCCL refuses two ranks on one device) -- plumbing only
    backend = os.environ.get("TG_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    L = N.lib()

    G, K, Lr = args.groups, args.group_size, args.resp_len
    mbg = min(args.mb_groups, G)
    n_mb = G // mbg
    mb_rows = mbg * K * Lr  # logits buffer rows (c5: padded layout of the ragged batch)
    B = G * K
    cfg = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl",
                        kl_coef=0.001, loss_agg_mode="token-mean", clip_lo=0.2, clip_hi=0.28)
    if args.variant == "grpo_two_pass":
        cfg = cfg.with_(force_two_pass=True)
    elif args.variant in ("opmd_kimi", "opmd_pairwise", "opmd_kimi_unscaled",
                          "opmd_pairwise_unscaled"):
        cfg = RFTLossConfig(policy_loss_fn=args.variant.replace("_unscaled", ""), tau=1.0)
    elif args.variant == "sft":
        cfg = RFTLossConfig.from_variant("SFT")
    elif args.variant == "anchor":  # regularizer_g: OPMD_SIMPLE + beta * KL(p || anchor)
        cfg = RFTLossConfig.from_variant("OPMD_SIMPLE", tau=1.0, beta=0.1)
    elif args.variant == "c3":  # PPO clip + low_var_kl + entropy bonus
        cfg = cfg.with_(entropy_loss_fn="default", entropy_coef=0.001)
    elif args.variant == "c4":  # GRPO + SFT NLL on expert sequences in the same batch
        cfg = cfg.with_(sft_weight=1.0)
    loss = RFTLoss(cfg)
    two_pass = args.variant in ("grpo_two_pass", "opmd_kimi", "opmd_pairwise")
    # coupled loss in one pass (TG_FLAG_UNSCALED_GRAD, route 4): p - e_y rows + row scales
    unscaled = args.variant.endswith("_unscaled")
    algo_bytes_row = (6 * V + 24) if (two_pass or args.variant == "anchor") else ALGO_BYTES_PER_ROW

    # ---- resident synthetic inputs (outside timing) ----
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    logits = torch.empty((mb_rows, V), dtype=torch.bfloat16, device=dev)
    for r0 in range(0, mb_rows, 8192):
        logits[r0:r0 + 8192].normal_(0.0, 2.0, generator=gen)
    rng = np.random.default_rng(1234 + rank)
    tgt = rng.integers(0, V, mb_rows)
    tgt_d = torch.as_tensor(tgt, device=dev)
    logits[torch.arange(mb_rows, device=dev), tgt_d] += BUMP
    dz = torch.empty_like(logits)
    anchor = None
    if args.variant == "anchor":  # the anchor policy's logits: the same rows + N(0, 0.3^2)
        anchor = torch.empty_like(logits)
        for r0 in range(0, mb_rows, 8192):
            anchor[r0:r0 + 8192].normal_(0.0, 0.3, generator=gen)
            anchor[r0:r0 + 8192] += logits[r0:r0 + 8192]
    lens = [Lr] * (mbg * K)
    gsz = [K] * mbg
    probe = pack_arrays(logits, tgt, lens, gsz, np.zeros(mbg * K, np.float32))
    lp_true = logprob_fwd(probe)[0].cpu().numpy().astype(np.float64)

    def mb_layout(m):
        """(lens, row_index, seq_kind) of micro-batch m.  c5: ragged long-CoT
        responses (lognormal lengths, 64..8192) with ~10 % of rows in interior
        mask-false spans of 8..64 rows, read in place from the padded buffer
        through row_index; c4: the second half of the groups are SFT sequences."""
        if args.variant == "c5":
            lrng = np.random.default_rng(1236 + 1000 * rank + m)
            L = np.clip(np.exp(lrng.normal(np.log(3000.0), 0.8, mbg * K)), 64, Lr).astype(int)
            keep = []
            off = 0
            for n in L:
                mask = np.ones(n, bool)
                masked = 0
                while masked < 0.1 * n:
                    run = int(lrng.integers(8, 65))
                    start = int(lrng.integers(0, max(1, n - run)))
                    masked += int(mask[start:start + run].sum())
                    mask[start:start + run] = False
                keep.append(np.nonzero(mask)[0] + off)
                off += n
            return [len(k) for k in keep], np.concatenate(keep), None
        kind = None
        if args.variant == "c4":
            kind = np.repeat((np.arange(mbg) >= mbg // 2).astype(np.uint8), K)
        return lens, None, kind

    batches, outs = [], []
    T = n_sft = 0
    for m in range(n_mb):
        rew = rng.integers(0, 2, mbg * K).astype(np.float32)
        if m == 0:
            rew[:K] = 1.0  # an all-equal group (A = 0, std = 0)
        lens_m, ridx, kind = mb_layout(m)
        rows = np.arange(mb_rows) if ridx is None else ridx
        old = (lp_true[rows] + rng.normal(0, OLD_LP_SIGMA, rows.size)).astype(np.float32)
        ref = (lp_true[rows] + rng.normal(0, 0.1, rows.size)).astype(np.float32)
        b = pack_arrays(logits, tgt[rows], lens_m, gsz, rew, old_lp=old, ref_lp=ref,
                        seq_kind=kind, row_index=ridx, anchor_logits=anchor)
        batches.append(b)
        outs.append(None)
        T += int(rows.size)
        n_sft += 0 if kind is None else int(kind.sum())
    route = loss.route(batches[0], unscaled=unscaled)
    assert route == (4 if unscaled else
                     1 if not two_pass else (2 if args.variant == "grpo_two_pass" else 3)), route
    # (anchor: route 1 = the fused anchor path, 6V bytes per row)
    n_tok_g, n_seq_g, n_sft_g = world * T, world * B, world * n_sft
    stats_all = torch.zeros((n_mb, N.NSTAT), dtype=torch.float64, device=dev)

    def step():
        for m in range(n_mb):
            outs[m] = loss(batches[m], dlogits=dz, n_tok_global=n_tok_g, n_seq_global=n_seq_g,
                           n_sft_seq_global=n_sft_g, out=outs[m], unscaled=unscaled)
        st = torch.stack([o.stats for o in outs]).sum(0)
        return allreduce_stats(st)

    for _ in range(args.warmup):
        st = step()
    torch.cuda.synchronize()
    s0 = step().cpu().numpy()
    torch.cuda.synchronize()

    # ---- timed region ----
    n_ev = args.steps * n_mb
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n_ev)]
    for a, b_ in evs:  # materialise the event handles
        a.record()
        b_.record()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    launches0 = L.tg_launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record()
    k = 0
    for _ in range(args.steps):
        for m in range(n_mb):
            L.tg_set_timing_events(evs[k][0].cuda_event, evs[k][1].cuda_event)
            k += 1
            outs[m] = loss(batches[m], dlogits=dz, n_tok_global=n_tok_g, n_seq_global=n_seq_g,
                           n_sft_seq_global=n_sft_g, out=outs[m], unscaled=unscaled)
        st = allreduce_stats(torch.stack([o.stats for o in outs]).sum(0))
    t_end.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = L.tg_launch_count() - launches0
    clk = clocks.stop()
    prof_out = os.environ.get("TG_FUSED_PROF_OUT")
    if prof_out and hasattr(L, "tg_debug_fused_prof"):  # instrumented library only
        import ctypes
        buf = (ctypes.c_ulonglong * (1024 * 16))()
        L.tg_debug_fused_prof(buf, 1024)
        arr = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16)
        np.save(prof_out, arr[:int((arr[:, 6] > 0).sum()) or 1024])
    ms = t_start.elapsed_time(t_end)
    fused_ms = [a.elapsed_time(b_) for a, b_ in evs]
    tmax = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms = float(tmax.item())
    stats = st.cpu().numpy()
    value = world * T * args.steps / (ms / 1000.0)

    # ---- roofline of the dominant kernel (k_fused_tma) ----
    peak, peak_src = peaks()
    f_ms = statistics.mean(fused_ms)
    rows_per_launch = T / n_mb
    achieved = rows_per_launch * algo_bytes_row / (f_ms / 1000.0) / 1e9
    # DRAM bytes per launch from the committed `ncu --set full` capture of the
    # same kernel at this vocabulary, scaled from its row count to this launch's
    # (the kernel streams rows independently, so bytes / row is size-invariant)
    traffic = None
    tf = ROOT / "profiles" / "fused_traffic.json"
    if tf.exists():
        try:
            d = json.loads(tf.read_text())
            if int(d.get("vocab", 0)) == V:
                traffic = float(d["dram_bytes_per_row"]) * rows_per_launch
        except Exception:
            traffic = None

    # ---- e2e: public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, loss, dev, world, rank, n_tok_g, n_seq_g)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline(args.cpu_rows, K)
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "port", "sample": repr(ex)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": VARIANT_WORKLOAD.get(args.variant,
                                                        f"{args.variant}_qwen2.5_1.5b_shapes"),
                       "vocab": V, "prompts": G, "repeats": K,
                       "response_len": Lr if args.variant != "c5" else f"ragged <= {Lr}",
                       "rows_per_gpu_per_step": T,
                       "micro_batches": n_mb, "rows_per_micro_batch": T // n_mb,
                       "loss": VARIANT_LOSS.get(args.variant, args.variant),
                       "l2": f"inputs larger than L2 ({2 * mb_rows * V * 2 / 1e9:.1f} GB "
                             "working set)",
                       "parallelism": f"dp{world} (groups sharded by rank; stats allreduce)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("k_fused_tma<anchor>" if args.variant == "anchor" else
                                    "k_fused_tma" if not two_pass else "k_fwd..k_bwd (two-pass)"),
                         "kernel_ms": f_ms,
                         "algorithmic_bytes_per_launch": rows_per_launch * algo_bytes_row,
                         "peak_source": peak_src,
                         "frac_of_8tbs_nominal": achieved / 8000.0},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "check": {"loss": float(stats[0]), "n_tok": float(stats[N.STAT["n_tok"]]),
                      "nonfinite": float(stats[N.STAT["nonfinite"]]),
                      "clipfrac": float(stats[N.STAT["clip_count"]] /
                                        max(stats[N.STAT["n_tok_rl"]], 1)),
                      "mean_lp": float(stats[N.STAT["sum_lp"]] / max(stats[N.STAT["n_tok"]], 1)),
                      "stats_match_warm": bool(np.allclose(s0, stats))},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(args, loss, dev, world, rank, n_tok_g, n_seq_g):
    """Public API with HOST buffers.  A step is `e2e_groups` (default: all of the
    step's groups, i.e. the same 1,048,576 rows as the device metric) RFTLoss calls, one
    GRPO group (8 x 2048 rows, 5 GB of bf16 logits) each: the group's logits
    and metadata are copied H2D from pinned memory on a copy stream, the loss
    runs on the compute stream (dlogits in place), and dlogits + the stats
    vector are copied D2H on a second copy stream.  Three device slots and
    three pinned in/out buffers rotate, so the H2D of group i+1, the kernel of
    group i and the D2H of group i-1 overlap (PCIe is full duplex)."""
    import torch

    from paper_2505_17826_b200.packing import PackedBatch

    K, Lr = args.group_size, args.resp_len
    ng = args.e2e_groups if args.e2e_groups > 0 else args.groups
    nbuf = min(3, ng)
    # pinned host memory: 2 * nbuf * rows * V * 2 bytes per rank (30 GB at the
    # defaults).  With many ranks per box, shrink the rotation depth, then the
    # per-call response length (whole groups are kept), to stay within a share
    # of the host's free memory -- the metric is rows/s either way.
    try:
        import psutil
        budget = 0.4 * psutil.virtual_memory().available / max(world, 1)
    except Exception:  # pragma: no cover
        budget = float("inf")
    if 2 * nbuf * K * Lr * V * 2 > budget and nbuf > 2:
        nbuf = 2
    while 2 * nbuf * K * Lr * V * 2 > budget and Lr > 256:
        Lr //= 2
    rows = K * Lr
    rng = np.random.default_rng(99 + rank)
    host_in = torch.empty((nbuf, rows, V), dtype=torch.bfloat16, pin_memory=True)
    host_out = torch.empty((nbuf, rows, V), dtype=torch.bfloat16, pin_memory=True)
    dev_in = [torch.empty((rows, V), dtype=torch.bfloat16, device=dev) for _ in range(nbuf)]
    gen = torch.Generator(device=dev)
    gen.manual_seed(7 + rank)
    for i in range(nbuf):  # synthetic host logits, generated on device once (setup)
        dev_in[0].normal_(0.0, 2.0, generator=gen)
        host_in[i].copy_(dev_in[0])
    torch.cuda.synchronize(dev)
    tmeta = [torch.as_tensor(rng.integers(0, V, rows).astype(np.int32)).pin_memory()
             for _ in range(nbuf)]
    fmeta = [torch.as_tensor(np.stack([rng.normal(-1.0, 0.05, rows),
                                       rng.normal(-1.0, 0.1, rows)]).astype(np.float32)
                             ).pin_memory() for _ in range(nbuf)]
    dev_meta = [torch.empty((2, rows), dtype=torch.float32, device=dev) for _ in range(nbuf)]
    dev_tgt = [torch.empty(rows, dtype=torch.int32, device=dev) for _ in range(nbuf)]
    s_in, s_cmp, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    host_stats = torch.empty((ng, 32), dtype=torch.float64, pin_memory=True)
    so = torch.as_tensor(np.arange(0, rows + 1, Lr, dtype=np.int32), device=dev)
    go = torch.as_tensor(np.array([0, K], np.int32), device=dev)
    rw = torch.as_tensor(rng.integers(0, 2, K).astype(np.float32), device=dev)
    h2d_bytes = ng * (rows * V * 2 + 3 * rows * 4)  # logits + target + old_lp + ref_lp
    d2h_bytes = ng * (rows * V * 2 + 32 * 8)        # dlogits + stats

    def one_step():
        free = [None] * nbuf
        for i in range(ng):
            b = i % nbuf
            with torch.cuda.stream(s_in):
                if free[b] is not None:
                    s_in.wait_event(free[b])
                dev_in[b].copy_(host_in[b], non_blocking=True)
                dev_meta[b].copy_(fmeta[b], non_blocking=True)
                dev_tgt[b].copy_(tmeta[b], non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ready)
                pb = PackedBatch(logits=dev_in[b], target=dev_tgt[b], seq_offsets=so,
                                 group_offsets=go, reward=rw, old_lp=dev_meta[b][0],
                                 ref_lp=dev_meta[b][1], vocab=V, n_rows=rows, n_seqs=K,
                                 n_groups=1, n_rl_rows=rows, n_rl_seqs=K, max_rows_per_seq=Lr)
                out = loss(pb, dlogits="inplace", n_tok_global=n_tok_g, n_seq_global=n_seq_g,
                           stream=s_cmp)
                done = torch.cuda.Event()
                done.record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(done)
                host_out[b].copy_(dev_in[b], non_blocking=True)
                host_stats[i].copy_(out.stats, non_blocking=True)
                free[b] = torch.cuda.Event()
                free[b].record(s_out)
        torch.cuda.synchronize(dev)

    one_step()  # warm
    times = []
    for _ in range(2):
        t0 = time.perf_counter()
        one_step()
        times.append(time.perf_counter() - t0)
    dt = statistics.median(times)
    return {"value": ng * rows / dt, "unit": UNIT, "h2d_bytes_per_step": h2d_bytes,
            "d2h_bytes_per_step": d2h_bytes,
            "note": f"{ng} RFTLoss calls x {rows} rows per step, pinned host logits in and "
                    f"dlogits + stats out, {nbuf}-deep copy/compute overlap; PCIe-bound"}


if __name__ == "__main__":
    sys.exit(main())
