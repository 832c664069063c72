"""GEMM micro-benchmark: the tcgen05 3xTF32 kernel vs the SIMT baseline on the hot
path's shapes (CUDA events, warm-up, median of repeats)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2210_08494_b200 import binding

SHAPES = [  # name, ta, tb, M, N, K
    ("cfg5 proj UtM 16385", True, False, 512, 1024, 16385),
    ("cfg5 resid M-UP 16385", False, False, 16385, 1024, 512),
    ("cfg5 gram RtR 16385", True, False, 1024, 1024, 16385),
    ("cfg5 rotate [UQ]V 16385", False, False, 16385, 512, 1536),
    ("cfg5 prec proj J^T U_A", True, False, 16384, 512, 4097),
    ("cfg5 prec out", False, True, 4097, 16384, 1024),
    ("cfg4 EA MMt 4609", False, True, 4609, 4609, 256),
    ("square 8192", False, False, 8192, 8192, 8192),
]

def run(path, ta, tb, M, N, K, reps=10):
    A = torch.randn((M, K) if ta else (K, M), device="cuda")
    B = torch.randn((K, N) if tb else (N, K), device="cuda")
    C = torch.zeros((N, M), device="cuda")
    ws = torch.empty(16 * M * N, device="cuda")
    for _ in range(2):
        binding.bkfac_gemm(ta, tb, 1.0, A, B, 0.0, C, ws=ws, path=path)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); binding.bkfac_gemm(ta, tb, 1.0, A, B, 0.0, C, ws=ws, path=path); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    return ms, 2.0 * M * N * K / ms / 1e9

out = []
for name, ta, tb, M, N, K in SHAPES:
    row = {"shape": name, "M": M, "N": N, "K": K}
    for path, key in ((binding.BKFAC_GEMM_TCGEN05, "tc"), (binding.BKFAC_GEMM_SIMT, "simt")):
        if key == "simt" and (M * N * K > 3e11 or "--tc-only" in sys.argv):
            continue
        ms, tf = run(path, ta, tb, M, N, K)
        row[key + "_ms"] = round(ms, 4); row[key + "_tflops"] = round(tf, 2)
    print(json.dumps(row), flush=True)
