"""One Brand update of a chosen shape (for ncu on the eigensolver kernels)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2210_08494_b200 import binding
n, c, r, count = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 256, 220, 1)))
ctx = binding.Context([(n, r, c, 0)] * count, [], device=0)
ups = []
for i in range(count):
    U = torch.linalg.qr(torch.randn(n, r, device="cuda"))[0].t().contiguous()
    D = torch.sort(torch.rand(r, device="cuda"), descending=True)[0]
    M = torch.randn(c, n, device="cuda") * 0.1
    ups.append(dict(factor=i, U_in=U, D_in=D, M=M, U_out=torch.empty_like(U), D_out=torch.empty_like(D), alpha=0.95, beta=0.05))
for _ in range(2):
    ctx.bkfac_brand_update(ups)
torch.cuda.synchronize()
print("ok")
