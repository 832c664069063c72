"""Diagnostic: orthonormality of U_out and GEMM accuracy, tcgen05 3xTF32 vs SIMT fp32."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, synth
from tests._util import lowrank_rel_err
from tests.gpu_helpers import gpu_brand
from paper_2210_08494_b200 import binding

for (n, c, r) in [(577, 256, 220), (2000, 250, 350), (2000, 300, 450)]:
    f = synth.random_case(n, c, r, seed=1000 + n + c + r, k=min(n, 2 * c), decay=0.9)
    M0, M1 = f.batch(0).astype(np.float64), f.batch(1).astype(np.float64)
    U0 = synth.phantom_basis(n, r)
    Uo, Do = O.brand_update(U0, np.zeros(r), M0, 0.0, 1.0, r)
    U32 = Uo.astype(np.float32).astype(np.float64); D32 = Do.astype(np.float32).astype(np.float64)
    for path in ("tc", "simt"):
        os.environ["BKFAC_GEMM"] = path
        ctx = binding.Context([(n, r, c, 0)], [], device=0)
        Ug, Dg = gpu_brand(ctx, 0, U32, D32, M1, 0.95, 0.05)
        Uo2, Do2 = O.brand_update(U32, D32, M1, 0.95, 0.05, r)
        orth = np.abs(Ug.T @ Ug - np.eye(r)).max()
        print(f"n={n} c={c} r={r} {path}: orth {orth:.2e} rec {lowrank_rel_err(Uo2, Do2, Ug, Dg):.2e}")
rng = np.random.default_rng(0)
for (M, N, K) in [(2000, 450, 750), (4609, 220, 476), (256, 256, 4609)]:
    A = torch.from_numpy(rng.standard_normal((K, M)).astype(np.float32)).cuda()
    B = torch.from_numpy(rng.standard_normal((N, K)).astype(np.float32)).cuda()
    ref = (A.double().cpu().numpy().T @ B.double().cpu().numpy().T)
    for path in (binding.BKFAC_GEMM_TCGEN05, binding.BKFAC_GEMM_SIMT):
        C = torch.zeros((N, M), device="cuda")
        binding.bkfac_gemm(False, False, 1.0, A, B, 0.0, C, path=path)
        torch.cuda.synchronize()
        d = C.double().cpu().numpy().T - ref
        print(f"gemm {M}x{N}x{K} path {path}: rel rms {np.sqrt((d**2).mean()/(ref**2).mean()):.2e} max {np.abs(d).max()/np.abs(ref).max():.2e}")
    # emulate 3xTF32 in numpy (rna hi, truncated lo read) for reference
