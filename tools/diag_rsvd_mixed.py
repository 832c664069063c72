"""Diagnostic: per-shape RSVD parity in batched vs single-factor calls."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, synth
from tests._util import lowrank_rel_err
from tests.gpu_helpers import from_dev_cols, to_dev_cols
from paper_2210_08494_b200 import binding

shapes = [(300, 40, 10), (64, 64, 0), (900, 100, 10), (64, 54, 10), (577, 220, 10)]
def run(batched):
    ctx = binding.Context([(n, r, 32, 1) for (n, r, _) in shapes], [], device=0)
    Ks, items, outs = [], [], []
    for i, (n, r, ro) in enumerate(shapes):
        f = synth.random_case(n, 32, r, seed=500 + i, k=min(n, 24), decay=0.9)
        K = torch.zeros((n, n), dtype=torch.float32, device="cuda")
        for k in range(6):
            ctx.bkfac_ea_batch([dict(factor=i, K=K, M=to_dev_cols(f.batch(k)), rho=0.9 if k else 0.0)])
        U = torch.empty((r, n), device="cuda"); D = torch.empty((r,), device="cuda")
        items.append(dict(factor=i, K=K, oversample=ro, power_iters=2, seed=7 + i, counter=1, U_out=U, D_out=D))
        Ks.append(K); outs.append((U, D))
    if batched:
        ctx.bkfac_rsvd_batch(items)
    else:
        for it in items:
            ctx.bkfac_rsvd_batch([it])
    torch.cuda.synchronize()
    print("check", ctx.bkfac_check())
    for (n, r, ro), K, (U, D), it in zip(shapes, Ks, outs, items):
        Kg = K.double().cpu().numpy()
        Uo, Do = O.rsvd_overwrite(Kg, r, ro, 2, it["seed"], 1)
        Ug = from_dev_cols(U)
        print(f"batched={batched} n={n} r={r} ro={ro} err={lowrank_rel_err(Uo, Do, Ug, D.double().cpu().numpy()):.3e} "
              f"orth={np.abs(Ug.T@Ug-np.eye(r)).max():.2e} D0={float(D[0]):.4e}/{Do[0]:.4e} Dr={float(D[-1]):.4e}/{Do[-1]:.4e}")
run(True); run(False)
