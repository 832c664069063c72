"""MMA-warp cycle breakdown of the tcgen05 GEMM (BKFAC_TC_TIMING build)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2210_08494_b200 import binding
lib = binding.load()
lib.bkfac_debug_tc.argtypes = [ctypes.c_void_p, ctypes.c_int]
for (ta, tb, M, N, K, beta) in [(False, False, 8192, 8192, 8192, 0.0), (False, True, 4097, 16384, 1024, 0.0),
                                (False, True, 4609, 4609, 256, 0.0), (False, True, 4609, 4609, 256, 0.95),
                                (False, True, 4608, 4608, 256, 0.95),
                                (False, False, 4609, 220, 476, 0.0), (False, False, 4609, 256, 220, 0.0),
                                (True, False, 256, 256, 4609, 0.0), (False, False, 128, 128, 32, 0.0),
                                (False, False, 128, 128, 256, 0.0), (False, False, 4096, 128, 32, 0.0)]:
    A = torch.randn((M, K) if ta else (K, M), device="cuda")
    B = torch.randn((K, N) if tb else (N, K), device="cuda")
    C = torch.zeros((N, M), device="cuda")
    binding.bkfac_gemm(ta, tb, 1.0, A, B, beta, C); torch.cuda.synchronize()
    lib.bkfac_debug_tc(None, 1); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); binding.bkfac_gemm(ta, tb, 1.0, A, B, beta, C); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    buf = (ctypes.c_ulonglong * (148 * 8))()
    lib.bkfac_debug_tc(ctypes.addressof(buf), 0)
    a = np.array(buf, dtype=np.float64).reshape(148, 8)
    cyc = ms * 1e-3 * 1.9e9
    nch = a[:, 3].mean()
    print(f"{M}x{N}x{K} ta={ta} tb={tb} beta={beta}: {ms:.3f} ms ~{cyc:.0f} cyc; per CTA chunks {nch:.0f}; per chunk: "
          f"wait tempty {a[:,0].mean()/nch:.0f}  wait full {a[:,1].mean()/nch:.0f}  issue {a[:,2].mean()/nch:.0f}  "
          f"(total cyc/chunk {cyc/nch:.0f})")
