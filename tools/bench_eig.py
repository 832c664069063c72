"""Per-stage timing of the Brand update (eigensolver stages) on batches of factors."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2210_08494_b200 import binding

def run(name, n, c, r, count, reps=5):
    ctx = binding.Context([(n, r, c, 0)] * count, [], device=0)
    U = [torch.linalg.qr(torch.randn(n, r, device="cuda"))[0].t().contiguous() for _ in range(count)]
    D = [torch.sort(torch.rand(r, device="cuda"), descending=True)[0] for _ in range(count)]
    M = [torch.randn(c, n, device="cuda") * 0.1 for _ in range(count)]
    Uo = [torch.empty_like(u) for u in U]; Do = [torch.empty_like(d) for d in D]
    ups = [dict(factor=i, U_in=U[i], D_in=D[i], M=M[i], U_out=Uo[i], D_out=Do[i], alpha=0.95, beta=0.05)
           for i in range(count)]
    ctx.bkfac_brand_update(ups); torch.cuda.synchronize()
    ctx.bkfac_profile_enable(True)
    for _ in range(reps):
        ctx.bkfac_brand_update(ups)
    st = ctx.bkfac_profile_read()
    torch.cuda.synchronize()
    out = {s["name"]: round(s["ms"] / reps, 3) for s in st}
    print(json.dumps({"case": name, "n": n, "c": c, "r": r, "count": count, "ms": out}), flush=True)

run("brand m476 x1", 577, 256, 220, 1)
run("brand m476 x23", 577, 256, 220, 23)
run("dense n256 x1", 256, 256, 220, 1)
run("dense n256 x9", 256, 256, 220, 9)
run("brand m96 x1", 256, 32, 64, 1)
if "--big" in sys.argv:
    run("brand m1536 x1", 4097, 1024, 512, 1, reps=1)
