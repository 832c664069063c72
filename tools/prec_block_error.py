"""Error of bkfac_precondition against the fp64 oracle as a function of the output GEMM's TMEM
accumulation block length (BKFAC_OPT_PREC_BLOCK), on the shape of
tests/test_gpu_parity.py::test_precondition_output_block_length (or d_G d_A r_G r_A [blocks...]
from the command line): normwise on S and on the
components inside span(U_G) x span(U_A).  A measurement tool (it calls the oracle, like the
tests do); prints one JSON line."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import oracle as O
    import __graft_entry__ as g
    g.build()
    from paper_2210_08494_b200 import binding
    from tests.gpu_helpers import to_dev, to_dev_cols
    dG, dA, rG, rA = [int(a) for a in sys.argv[1:5]] if len(sys.argv) >= 5 else (700, 1300, 512, 512)
    blocks = [int(a) for a in sys.argv[5:]] or [1, 2, 4, 8, 16, 32]
    rng = np.random.default_rng(99)
    UG, _ = np.linalg.qr(rng.standard_normal((dG, rG)))
    UA, _ = np.linalg.qr(rng.standard_normal((dA, rA)))
    DG = np.sort(rng.random(rG) * 5)[::-1]
    DA = np.sort(rng.random(rA) * 5)[::-1]
    J = (0.1 * rng.standard_normal((dG, dA))).astype(np.float32)
    lam = 0.01
    f32 = lambda x: x.astype(np.float32).astype(np.float64)
    UGf, UAf = f32(UG), f32(UA)
    So = O.precondition(J.astype(np.float64), UGf, f32(DG), lam, UAf, f32(DA), lam,
                        continuation=False, lam_relative=False)
    Po = UGf.T @ So @ UAf
    out = {"shape": [dG, dA, rG, rA], "lambda": lam, "blocks": {}}
    for block in blocks:
        ctx = binding.Context([], [(dG, dA, rG, rA)], device=0)
        ctx.bkfac_set_option(binding.BKFAC_OPT_PREC_BLOCK, block)
        S = torch.empty((dG, dA), dtype=torch.float32, device="cuda")
        ctx.bkfac_precondition([dict(layer=0, U_G=to_dev_cols(UG), D_G=to_dev(DG), lambda_G=lam,
                                     U_A=to_dev_cols(UA), D_A=to_dev(DA), lambda_A=lam,
                                     J=to_dev(J), S=S, flags=0)])
        torch.cuda.synchronize()
        Sg = S.double().cpu().numpy()
        Pg = UGf.T @ Sg @ UAf
        out["blocks"][str(32 * block)] = {
            "rel_err_S": float(np.linalg.norm(Sg - So) / np.linalg.norm(So)),
            "rel_err_subspace": float(np.linalg.norm(Pg - Po) / np.linalg.norm(Po)),
            "mean_signed_err_subspace_over_rms": float(np.mean((Pg - Po) * np.sign(Po)) / np.sqrt(np.mean(Po ** 2)))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
