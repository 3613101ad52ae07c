"""Throughput of the anchor-KL route (regularizer_g, algorithms.py:193-217:
OPMD_SIMPLE + beta * anchor KL, route 2 = forward + backward streaming over the
logits and the anchor logits, 10V bytes per row): 16,384 rows at V = 151,936.

    python scripts/bench_anchor.py [V] [rows] [bf16|fp32]
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, pack_arrays
V = int(sys.argv[1]) if len(sys.argv) > 1 else 151936
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
DT = torch.float32 if len(sys.argv) > 3 and sys.argv[3] == "fp32" else torch.bfloat16
K = 8
L = T // K
z=(torch.randn(T,V,device='cuda')*2).to(DT)
q=(z.float()+0.3*torch.randn(T,V,device='cuda')).to(DT)
y=np.random.default_rng(0).integers(0,V,T)
b=pack_arrays(z,y,[L]*K,[K],np.arange(K,dtype=np.float32)%2,anchor_logits=q)
loss=RFTLoss(RFTLossConfig.from_variant("OPMD_SIMPLE",tau=1.0,beta=0.1))
dz=torch.empty_like(z)
for _ in range(3): loss(b,dlogits=dz)
torch.cuda.synchronize()
a,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): loss(b,dlogits=dz)
e.record(); torch.cuda.synchronize()
ms=a.elapsed_time(e)/5
prof_out = __import__("os").environ.get("TG_FUSED_PROF_OUT")
if prof_out:  # instrumented library (--variant=prof): per-CTA cycle counters
    import ctypes
    from paper_2505_17826_b200 import _native as N
    L = N.lib()
    buf = (ctypes.c_ulonglong * (1024 * 16))()
    L.tg_debug_fused_prof(buf, 1024)
    arr = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16)
    np.save(prof_out, arr[:int((arr[:, 6] > 0).sum()) or 1024])
E = z.element_size()  # bytes per logit: 6V = 3 E V (z, za read; dz written)
print(json.dumps({"route":loss.route(b),"cl":loss.cluster_size(b),"rows":T,"ms":ms,"rows_per_s":T/ms*1e3,
                  "GBs_10V":T*5*E*V/ms/1e6,"GBs_6V":T*3*E*V/ms/1e6}))
