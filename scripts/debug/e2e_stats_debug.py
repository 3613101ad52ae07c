import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import bench as Bm
from paper_2505_17826_b200 import RFTLoss, RFTLossConfig
from paper_2505_17826_b200 import _native as N
sys.argv = ["bench.py", "--e2e-groups", "12"]
args = Bm.parse()
args.resp_len = int(sys.argv_len) if False else 2048
dev = torch.device("cuda", 0)
cfg = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl",
                    kl_coef=0.001, loss_agg_mode="token-mean", clip_lo=0.2, clip_hi=0.28)
loss = RFTLoss(cfg)
# monkeypatch the check to print differences
orig_equal = torch.equal
def eq(a, b):
    r = orig_equal(a, b)
    if not r and a.dim() == 1 and a.numel() == 32:
        d = (a.double() - b.double().cpu() if a.device.type == "cpu" else a.double() - b.double())
        for i in np.nonzero(d.cpu().numpy())[0]:
            print(N.STAT_NAMES[i], float(a[i]), float(b[i]))
    return r
torch.equal = eq
print(Bm.run_e2e(args, loss, dev, 1, 0, 1048576, 512, 12))
