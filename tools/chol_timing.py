"""Per-phase cycle sums of the tiled Cholesky (BKFAC_CHOL_TIMING build), CTA 0 of each
launch of one Brand update (two CholeskyQR passes)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_08494_b200 import binding
n, c, r = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (577, 256, 220)
ctx = binding.Context([(n, r, c, 0)], [], device=0)
U = torch.linalg.qr(torch.randn(n, r, device="cuda"))[0].t().contiguous()
D = torch.sort(torch.rand(r, device="cuda"), descending=True)[0]
M = torch.randn(c, n, device="cuda") * 0.1
ups = [dict(factor=0, U_in=U, D_in=D, M=M, U_out=torch.empty_like(U), D_out=torch.empty_like(D), alpha=0.95, beta=0.05)]
ctx.bkfac_brand_update(ups); torch.cuda.synchronize()
lib = binding.load()
lib.bkfac_debug_chol.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.bkfac_debug_chol(None, 1); torch.cuda.synchronize()
ctx.bkfac_brand_update(ups); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
lib.bkfac_debug_chol(ctypes.addressof(buf), 0)
names = ["load", "diag", "trsm", "trail", "-", "inv1", "inv2", "out"]
a = np.array(buf, dtype=np.float64)
print("cycles (2 launches):", {k: int(v) for k, v in zip(names, a)}, "total", int(a.sum()))
