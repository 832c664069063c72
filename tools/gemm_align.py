"""Times the preconditioning GEMM shapes of configs[4] with the caller's odd leading
dimensions (scalar loader path) and with the same matrices padded to a multiple of 32
(16-byte loader path): CUDA events, median of repeats."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2210_08494_b200 import binding

SHAPES = [  # name, ta, tb, M, N, K, beta
    ("prec_out 4097x16384 K1024", False, True, 4097, 16384, 1024, 1.0),
    ("prec_out 16385x4096 K1024", False, True, 16385, 4096, 1024, 1.0),
    ("prec_proj Y=J^T U_A 16384x512 K4097", True, False, 16384, 512, 4097, 0.0),
    ("prec_proj Xt=J U_G 4097x512 K16384", False, False, 4097, 512, 16384, 0.0),
    ("prec_proj Y=J^T U_A 4096x512 K16385", True, False, 4096, 512, 16385, 0.0),
    ("prec_proj Xt=J U_G 16385x512 K4096", False, False, 16385, 512, 4096, 0.0),
]


def pad(x):
    return (x + 31) // 32 * 32


def run(ta, tb, M, N, K, beta, aligned, reps=7):
    lib = binding.load()
    ra, ca = (M, K) if ta else (K, M)          # A tensor shape (rows, cols): ld = cols
    rb, cb = (K, N) if tb else (N, K)
    lda = pad(ca) if aligned else ca
    ldb = pad(cb) if aligned else cb
    A = torch.randn(ra * lda, device="cuda")
    B = torch.randn(rb * ldb, device="cuda")
    C = torch.zeros(N * M, device="cuda")
    ws = torch.empty(16 * M * N, device="cuda") if M * N <= 2 ** 22 else None
    wsb = 0 if ws is None else ws.numel() * 4

    def call():
        rc = lib.bkfac_gemm(int(ta), int(tb), M, N, K, 1.0, A.data_ptr(), lda, B.data_ptr(), ldb,
                            beta, C.data_ptr(), M, 0 if ws is None else ws.data_ptr(), wsb,
                            binding.BKFAC_GEMM_TCGEN05, 0)
        assert rc == 0, rc
    for _ in range(2):
        call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); call(); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    return ms, 2.0 * M * N * K / ms / 1e9


for name, ta, tb, M, N, K, beta in SHAPES:
    row = {"shape": name}
    for al in (False, True):
        ms, tf = run(ta, tb, M, N, K, beta, al)
        row["aligned" if al else "odd_ld"] = {"ms": round(ms, 4), "tflops": round(tf, 1)}
    print(json.dumps(row), flush=True)
