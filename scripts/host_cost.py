import time, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2505_17826_b200 import RFTLoss, RFTLossConfig, pack_arrays
cfg = RFTLossConfig(advantage_fn="grpo", policy_loss_fn="ppo_clip", kl_fn="low_var_kl", kl_coef=1e-3, loss_agg_mode="token-mean")
loss = RFTLoss(cfg)
V=32000; T=32768
z = torch.randn(T, V, device='cuda').to(torch.bfloat16)
rng = np.random.default_rng(0)
lens=[512]*64; b = pack_arrays(z, rng.integers(0,V,T), lens, [8]*8, rng.integers(0,2,64).astype(np.float32), old_lp=np.full(T,-5,np.float32), ref_lp=np.full(T,-5,np.float32))
dz = torch.empty_like(z)
out=None
for _ in range(5): out = loss(b, dlogits=dz, out=out)
torch.cuda.synchronize()
# host cost: tiny batch
zs = z[:64]
bs = pack_arrays(zs, rng.integers(0,V,64), [8]*8, [8], rng.integers(0,2,8).astype(np.float32), old_lp=np.full(64,-5,np.float32), ref_lp=np.full(64,-5,np.float32))
o2=None
for _ in range(20): o2 = loss(bs, dlogits=dz[:64], out=o2)
torch.cuda.synchronize()
t=time.perf_counter(); n=500
for _ in range(n): o2 = loss(bs, dlogits=dz[:64], out=o2)
t1=time.perf_counter(); torch.cuda.synchronize(); t2=time.perf_counter()
print(f"host per call {1e6*(t1-t)/n:.1f} us (sync tail {1e6*(t2-t1):.0f} us)")
# full c1 call: host vs device
a,e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); t=time.perf_counter()
for _ in range(50): out = loss(b, dlogits=dz, out=out)
t1=time.perf_counter(); e.record(); torch.cuda.synchronize()
print(f"c1 call: device {a.elapsed_time(e)/50*1e3:.1f} us per call, host {1e6*(t1-t)/50:.1f} us per call")
# graph replay of the c1 call
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(2): out = loss(b, dlogits=dz, out=out)
torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
with torch.cuda.graph(g):
    out = loss(b, dlogits=dz, out=out)
torch.cuda.synchronize()
for _ in range(3): g.replay()
torch.cuda.synchronize()
a.record()
for _ in range(50): g.replay()
e.record(); torch.cuda.synchronize()
print(f"c1 graph replay: {a.elapsed_time(e)/50*1e3:.1f} us per call")
