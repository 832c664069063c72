"""Diagnostic: probe the tcgen05 GEMM's operand mappings with one-hot A and index-coded B."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_08494_b200 import binding

M = N = 128; K = 32
def colmaj_to_torch(X):  # X is math (rows x cols) -> torch (cols, rows)
    return torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
for ta in (False, True):
    for tb in (False, True):
        print(f"=== ta={ta} tb={tb}")
        # op(B)(k, j) = 1000 k + j + 1  (exact in 3xTF32)
        opB = (1000.0 * np.arange(K)[:, None] + np.arange(N)[None, :] + 1).astype(np.float32)
        Bm = opB.T if tb else opB            # stored matrix (math orientation)
        for (i, k) in [(0, 0), (1, 0), (0, 1), (5, 3), (40, 9), (100, 31), (33, 8)]:
            opA = np.zeros((M, K), np.float32); opA[i, k] = 1.0
            Am = opA.T if ta else opA
            A = colmaj_to_torch(Am); B = colmaj_to_torch(Bm)
            C = torch.zeros((N, M), device="cuda")
            binding.bkfac_gemm(ta, tb, 1.0, A, B, 0.0, C)
            torch.cuda.synchronize()
            Cm = C.cpu().numpy().T   # math M x N
            rows = np.nonzero(np.abs(Cm).sum(1))[0]
            desc = []
            for rr in rows[:3]:
                v = Cm[rr]
                nz = np.nonzero(v)[0]
                dec = [(int(round(v[j] - 1)) // 1000, int(round(v[j] - 1)) % 1000, j) for j in nz[:4]]
                desc.append(f"row {rr}: nnz {len(nz)} first (k,jval,jpos) {dec}")
            print(f" A({i},{k})=1 -> rows {list(rows[:6])} | " + " ; ".join(desc))
