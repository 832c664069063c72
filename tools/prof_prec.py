"""Preconditioning only (bkfac_precondition) on cfg4's 16 layers with random rank-r
representations: per-stage event times, and a target for ncu captures of its GEMMs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2210_08494_b200 import binding
cfg = synth.cfg4_vgg_sharded()
fac = [(f.n, f.r, f.c, 0) for f in cfg.factors]
lay = [(L.d_G, L.d_A, cfg.factors[L.g_index].r, cfg.factors[L.a_index].r) for L in cfg.layers]
ctx = binding.Context(fac, lay, device=0)
dev = "cuda"
rep = []
for f in cfg.factors:
    U = torch.linalg.qr(torch.randn(f.n, f.r, device=dev))[0].t().contiguous()
    D = torch.sort(torch.rand(f.r, device=dev) * 5, descending=True)[0]
    rep.append((U, D))
items = []
for li, L in enumerate(cfg.layers):
    J = torch.randn(L.d_G, L.d_A, device=dev) * 0.1
    (UG, DG), (UA, DA) = rep[L.g_index], rep[L.a_index]
    items.append(dict(layer=li, U_G=UG, D_G=DG, lambda_G=0.1, U_A=UA, D_A=DA, lambda_A=0.1, J=J,
                      S=torch.empty_like(J)))
for _ in range(3):
    ctx.bkfac_precondition(items)
torch.cuda.synchronize()
if len(sys.argv) > 1 and sys.argv[1] == "time":
    ctx.bkfac_profile_enable(True)
    for _ in range(20):
        ctx.bkfac_precondition(items)
    torch.cuda.synchronize()
    tot = 0.0
    for s in ctx.bkfac_profile_read():
        print(f"{s['name']:16s} {s['ms'] / 20:8.4f} ms/step  launches {s['launches'] / 20:.0f}  "
              f"{s['flops'] / 20 / 1e9:8.2f} GFLOP  {s['bytes'] / 20 / 1e6:8.1f} MB")
        tot += s['ms'] / 20
    print(f"total {tot:.4f} ms")
print("ok")
