"""EA accumulate only (bkfac_ea_accumulate_batch) on cfg4's 32 factors: stage time, and a
target for ncu captures of the symmetric short-K GEMM."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2210_08494_b200 import binding
cfg = synth.cfg4_vgg_sharded()
fac = [(f.n, f.r, f.c, binding.BKFAC_FACTOR_DENSE_EA) for f in cfg.factors]
ctx = binding.Context(fac, [], device=0)
items = [dict(factor=g, K=torch.zeros((f.n, f.n), device="cuda"), M=torch.randn(f.c, f.n, device="cuda"), rho=0.95)
         for g, f in enumerate(cfg.factors)]
for _ in range(3):
    ctx.bkfac_ea_batch(items)
torch.cuda.synchronize()
if len(sys.argv) > 1 and sys.argv[1] == "time":
    ctx.bkfac_profile_enable(True)
    for _ in range(20):
        ctx.bkfac_ea_batch(items)
    torch.cuda.synchronize()
    for s in ctx.bkfac_profile_read():
        print(f"{s['name']:16s} {s['ms'] / 20:8.4f} ms/call  {s['flops'] / 20 / 1e9:8.2f} GFLOP  {s['bytes'] / 20 / 1e6:8.1f} MB")
print("ok")
