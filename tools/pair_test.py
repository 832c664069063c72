import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2210_08494_b200 import binding
torch.manual_seed(0)
for (ta, tb, M, N, K) in [(False, False, 256, 128, 64), (False, False, 300, 200, 100), (True, False, 513, 260, 777),
                          (False, True, 1000, 333, 250), (True, True, 700, 129, 1025), (False, False, 4096, 4096, 4096)]:
    A = torch.randn((M, K) if ta else (K, M), device="cuda")
    B = torch.randn((K, N) if tb else (N, K), device="cuda")
    C = torch.zeros((N, M), device="cuda")
    binding.bkfac_gemm(ta, tb, 1.0, A, B, 0.0, C)
    torch.cuda.synchronize()
    Ad = A.double().t() if ta else A.double()
    # math: C(MxN) = op(A) op(B); our tensors are col-major transposes
    opA = (A.double() if ta else A.double().t())   # M x K
    opB = (B.double().t() if tb else B.double())    # hmm
    Am = A.double().cpu().numpy(); Bm = B.double().cpu().numpy()
    a = Am if ta else Am.T          # M x K  (A stored as (K,M) col-major MxK when not ta)
    bb = Bm.T if tb else Bm         # ... B stored (N,K) col-major KxN when not tb -> math B = Bm.T? 
    ref = None
    Cm = C.double().cpu().numpy().T   # M x N
    # try both orientations for B and A to be robust in this ad-hoc check
    best = 1e9
    for a_ in (Am, Am.T):
        for b_ in (Bm, Bm.T):
            if a_.shape[0] == M and b_.shape[1] == N and a_.shape[1] == b_.shape[0]:
                r = a_ @ b_
                best = min(best, np.abs(Cm - r).max() / max(np.abs(r).max(), 1e-30))
    print(ta, tb, M, N, K, "rel err", best, flush=True)
