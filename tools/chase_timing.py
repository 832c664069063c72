"""Phase cycle sums of the bulge-chase kernel (BKFAC_CHASE_TIMING build, factor 0's CTA):
runs one cfg5-shaped factor's Brand step and prints cycles per task by phase."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2210_08494_b200 import binding
lib = binding.load()
n, c, r = 4097, 1024, 512
ctx = binding.Context([(n, r, c, 0)] * 4, [], device=0)
ctx.bkfac_set_option(binding.BKFAC_OPT_TWO_STAGE, 2)   # the chase runs on the two-stage path only
f = synth.random_case(n, c, r, seed=5, k=256, decay=0.98, sigma=0.02)
items = []
for i in range(4):
    U = torch.from_numpy(np.ascontiguousarray(synth.phantom_basis(n, r).T)).cuda()
    items.append(dict(factor=i, U_in=U, D_in=torch.zeros(r, device="cuda"),
                      M=torch.from_numpy(np.ascontiguousarray(f.batch(i).T)).cuda(),
                      U_out=torch.empty_like(U), D_out=torch.empty(r, device="cuda"), alpha=0.0, beta=1.0))
ctx.bkfac_brand_update(items); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
lib.bkfac_debug_chase(buf, 1)
ctx.bkfac_brand_update(items); torch.cuda.synchronize()
lib.bkfac_debug_chase(buf, 0)
v = list(buf); nt = max(v[5], 1)
names = ["wait", "loads", "E part", "D part", "publish"] if len(sys.argv) < 2 else ["wait+sync", "stage+nx issue", "compute", "store+shift"]
print("tasks", nt, "kernel cycles", v[6], "per task:", {nm: round(v[i] / nt) for i, nm in enumerate(names)})
