"""Per-phase cycle breakdown of the tiled tridiagonalisation (BKFAC_SYT_TIMING build)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_08494_b200 import binding
n, c, r = (int(x) for x in sys.argv[1:4])
ctx = binding.Context([(n, r, c, 0)], [], device=0)
U = torch.linalg.qr(torch.randn(n, r, device="cuda"))[0].t().contiguous()
D = torch.sort(torch.rand(r, device="cuda"), descending=True)[0]
M = torch.randn(c, n, device="cuda") * 0.1
ups = [dict(factor=0, U_in=U, D_in=D, M=M, U_out=torch.empty_like(U), D_out=torch.empty_like(D), alpha=0.95, beta=0.05)]
ctx.bkfac_brand_update(ups)
torch.cuda.synchronize()
lib = binding.load()
lib.bkfac_debug_eig_scratch.restype = ctypes.c_void_p
lib.bkfac_debug_eig_scratch.argtypes = [ctypes.c_void_p, ctypes.c_int]
ptr = lib.bkfac_debug_eig_scratch(ctx.h, 0)
# the timing sums were overwritten by invit (Y is its output); rerun only sytrd is not
# possible from here, so the timing build skips invit's writes to Y rows 0..63 -- instead
# we read them right after a run with BKFAC_SYT_TIMING where invit is disabled
buf = (ctypes.c_ulonglong * 128)()
lib.bkfac_debug_d2h.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
lib.bkfac_debug_d2h(ctypes.addressof(buf), ctypes.c_void_p(ptr), 128 * 8)
a = np.array(buf, dtype=np.int64).reshape(8, 16)
m = r + c
for q in range(8):
    if a[q, :9].sum() <= 0: continue
    tot = a[q, :9].sum()
    print(f"CTA {q}: per step cycles: (a)owner {a[q,0]/(m-2):.0f}  sync1 {a[q,1]/(m-2):.0f}  tiles {a[q,2]/(m-2):.0f}  sync2 {a[q,3]/(m-2):.0f}  merged: loads {a[q,5]/(m-2):.0f} sum1 {a[q,6]/(m-2):.0f} x+yzero {a[q,7]/(m-2):.0f} sum2 {a[q,8]/(m-2):.0f} finish {a[q,4]/(m-2):.0f}  total {tot/(m-2):.0f}")
