"""Phase cycle sums of the band reduction's panel kernel (BKFAC_PANEL_TIMING build, factor 0's
CTA, thread 0): runs configs[4]-shaped factors' Brand steps on the two-stage path and prints
cycles per column step by phase."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2210_08494_b200 import binding
lib = binding.load()
n, c, r = 4097, 1024, 512
nf = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ctx = binding.Context([(n, r, c, 0)] * nf, [], device=0)
ctx.bkfac_set_option(binding.BKFAC_OPT_TWO_STAGE, 2)
f = synth.random_case(n, c, r, seed=5, k=256, decay=0.98, sigma=0.02)
items = []
for i in range(nf):
    U = torch.from_numpy(np.ascontiguousarray(synth.phantom_basis(n, r).T)).cuda()
    items.append(dict(factor=i, U_in=U, D_in=torch.zeros(r, device="cuda"),
                      M=torch.from_numpy(np.ascontiguousarray(f.batch(i % 4).T)).cuda(),
                      U_out=torch.empty_like(U), D_out=torch.empty(r, device="cuda"), alpha=0.0, beta=1.0))
ctx.bkfac_brand_update(items); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
lib.bkfac_debug_chase(buf, 1)
ctx.bkfac_brand_update(items); torch.cuda.synchronize()
lib.bkfac_debug_chase(buf, 0)
v = list(buf); nt = max(v[5], 1)
names = ["partial sums + warp reduce", "barrier", "tau + T column (warp 0)", "apply + publish"]
print("column steps", nt, "thread 0, cycles per step:", {nm: round(v[i] / nt) for i, nm in enumerate(names)})
print("thread 256: partial sums", round(v[7] / nt), "barrier", round(v[6] / nt), "apply + publish", round(v[4] / nt))
