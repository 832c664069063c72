import sys, os
sys.path.insert(0, '/root/repo')
import torch
from paper_2210_08494_b200 import binding
n, c, r = 100, 8, 10
ctx = binding.Context([(n, r, c, 0)], [], device=0)
U = torch.zeros((r, n), device="cuda"); D = torch.zeros(r, device="cuda")
U[torch.arange(r), torch.arange(r)] = 1.0
Uo = torch.zeros_like(U); Do = torch.zeros_like(D)
Mn = torch.full((c, n), float("nan"), device="cuda")
ctx.bkfac_profile_enable(True)
ctx.bkfac_brand_update([dict(factor=0, U_in=U, D_in=D, M=Mn, U_out=Uo, D_out=Do, alpha=0.0, beta=1.0)])
print("check", ctx.bkfac_check())
print("Do", Do[:4].tolist(), "Uo nan", torch.isnan(Uo).any().item())
for s in ctx.bkfac_profile_read(): print(s['name'], s['launches'])
