import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from _cases import make_case, oracle_cfg
from oracle import rft_oracle as O
from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, logprob_fwd
import test_gpu_tight_parity as T
for name in ["bf16_cl2_ppo_k3_entropy", "bf16_cl2_opmd_simple"]:
    V, dtype, cl, cfg = T.FD_CASES[name]
    batch, packed = make_case(sum(name.encode()) % 1000, V, [9, 7, 8, 6], [2, 2], dtype=dtype)
    lp, _, _, _ = logprob_fwd(packed)
    packed.old_lp = lp.clone()
    batch.old_lp = lp.double().cpu().numpy()
    loss = RFTLoss(cfg)
    out = loss(packed, dlogits="new")
    g = out.dlogits.double().cpu().numpy()
    ref = O.general_loss(batch, oracle_cfg(cfg))
    print(name, "loss kernel", out.stats_dict()["loss"], "oracle", O.stats_dict(ref["stats"])["loss"])
    fwd = loss(packed, dlogits=None).stats_dict()
    print("fwd-only loss", fwd["loss"], "ent_loss", fwd["entropy_loss"], out.stats_dict()["entropy_loss"])
    t = 13
    row = packed.logits[t].float().clone(); y = int(packed.target[t]); row[y] = -float("inf")
    for v in [y] + torch.topk(row, 3).indices.tolist():
        h = 0.125
        z0 = float(packed.logits[t, v])
        Ls = []
        for sgn in (1, -1):
            b2 = O.Batch(**{**batch.__dict__}); b2.logits = batch.logits.copy(); b2.logits[t, v] = z0 + sgn * h
            Ls.append(O.general_loss(b2, oracle_cfg(cfg), want_dz=False)["stats"][0])
            packed.logits[t, v] = z0 + sgn * h
            Ls.append(loss(packed, dlogits=None).stats_dict()["loss"])
            packed.logits[t, v] = z0
        print(v, "g_kernel", g[t, v], "g_oracle", ref["dz"][t, v], "fd_oracle", (Ls[0] - Ls[2]) / (2 * h), "fd_kernel", (Ls[1] - Ls[3]) / (2 * h))
