"""One Brand step on a cfg4-shaped factor batch (m = r + c = 476 cores), for ncu captures
of the tridiagonalisation (ncu -k regex:sytrd)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2210_08494_b200 import binding
n, c, r, nf = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (577, 256, 220, 8)))
ctx = binding.Context([(n, r, c, 0)] * nf, [], device=0)
ups = []
for f in range(nf):
    U = torch.linalg.qr(torch.randn(n, r, device="cuda"))[0].t().contiguous()
    D = torch.sort(torch.rand(r, device="cuda"), descending=True)[0]
    M = torch.randn(c, n, device="cuda") * 0.1
    ups.append(dict(factor=f, U_in=U, D_in=D, M=M, U_out=torch.empty_like(U), D_out=torch.empty_like(D),
                    alpha=0.95, beta=0.05))
for _ in range(3):
    ctx.bkfac_brand_update(ups)
torch.cuda.synchronize()
print("ok")
if len(sys.argv) > 5 and sys.argv[5] == "time":
    ctx.bkfac_profile_enable(True)
    for _ in range(20):
        ctx.bkfac_brand_update(ups)
    torch.cuda.synchronize()
    for s in ctx.bkfac_profile_read():
        if s["name"].startswith(("eig", "chol")):
            print(f"{s['name']:14s} {s['ms'] / max(s['calls'], 1):8.4f} ms/call")
