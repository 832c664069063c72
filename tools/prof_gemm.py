"""One tcgen05 GEMM launch of a chosen hot-path shape (for ncu --set full)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2210_08494_b200 import binding
shape = sys.argv[1] if len(sys.argv) > 1 else "prec_out"
S = {"prec_out": (False, True, 4097, 16384, 1024), "proj": (True, False, 512, 1024, 16385),
     "rotate": (False, False, 16385, 512, 1536), "ea": (False, True, 4609, 4609, 256)}
ta, tb, M, N, K = S[shape]
A = torch.randn((M, K) if ta else (K, M), device="cuda")
B = torch.randn((K, N) if tb else (N, K), device="cuda")
C = torch.zeros((N, M), device="cuda")
ws = torch.empty(16 * M * N, device="cuda")
for _ in range(3):
    binding.bkfac_gemm(ta, tb, 1.0, A, B, 0.0, C, ws=ws)
torch.cuda.synchronize()
print("ok", shape)
