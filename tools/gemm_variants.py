"""Times the hot-path GEMM shapes of configs[4] on the library build named by BKFAC_LIB
(tuning variants, tools/build_variants.sh): CUDA events, median of repeats, batched like the
stage (nb problems per call through bkfac_gemm's single-problem entry is not batched, so each
shape runs once per call)."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2210_08494_b200 import binding

SHAPES = [  # name, ta, tb, M, N, K, beta
    ("prec_out 4097x16384 K1024", False, True, 4097, 16384, 1024, 1.0),
    ("prec_out 16385x4096 K1024", False, True, 16385, 4096, 1024, 1.0),
    ("prec_proj Y=J U_A", True, False, 16384, 512, 4097, 0.0),
    ("prec_proj Xt=J^T U_G", False, False, 4097, 512, 16384, 0.0),
    ("resid 16385x1024 K512", False, False, 16385, 1024, 512, 1.0),
    ("qmul 16385x1024 K1024", False, True, 16385, 1024, 1024, 0.0),
    ("gram 1024x1024 K16385", True, False, 1024, 1024, 16385, 0.0),
    ("square 8192", False, False, 8192, 8192, 8192, 0.0),
]


def run(ta, tb, M, N, K, beta, reps=7):
    A = torch.randn((M, K) if ta else (K, M), device="cuda")
    B = torch.randn((K, N) if tb else (N, K), device="cuda")
    C = torch.zeros((N, M), device="cuda")
    ws = torch.empty(16 * M * N, device="cuda") if M * N <= 2 ** 22 else None
    for _ in range(2):
        binding.bkfac_gemm(ta, tb, 1.0, A, B, beta, C, ws=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); binding.bkfac_gemm(ta, tb, 1.0, A, B, beta, C, ws=ws); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    return ms, 2.0 * M * N * K / ms / 1e9


lib = os.path.basename(os.environ.get("BKFAC_LIB", "libbkfac.so"))
for name, ta, tb, M, N, K, beta in SHAPES:
    ms, tf = run(ta, tb, M, N, K, beta)
    print(json.dumps({"lib": lib, "shape": name, "ms": round(ms, 4), "tflops": round(tf, 1)}), flush=True)
