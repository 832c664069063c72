"""Diagnostic: run the cfg4 stack to the first RSVD step, then time each factor's RSVD
overwrite alone and report the eigenvalue spectrum/gaps it produced."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2210_08494_b200 import BKFACStack  # noqa: E402

cfg = synth.cfg4_vgg_sharded()
factors = [(f.n, f.r, f.c) for f in cfg.factors]
layers = [(l.d_G, l.d_A, l.g_index, l.a_index) for l in cfg.layers]
st = BKFACStack(factors, layers, cfg.rho, cfg.lam, rsvd_every=10**9, oversample=10, power_iters=2)
st.rsvd_every = 0
Mp, Jp = bench.device_inputs(cfg, st.my_factors, st.my_layers, 2, torch.device("cuda:0"))
# keep the dense factors accumulating (rsvd_every huge => K maintained)
st.rsvd_every = 10**9
for k in range(25):
    st.step(Mp[k % 2], Jp[k % 2])
torch.cuda.synchronize()
for i, g in enumerate(st.my_factors):
    n, r, _ = factors[g]
    ro = min(10, n - r)
    U = torch.empty((r, n), device="cuda")
    D = torch.empty((r,), device="cuda")
    st.ctx.bkfac_profile_enable(True)
    st.ctx.bkfac_rsvd_overwrite(i, st.K[i], ro, 2, 1234 + g, 0, U, D)
    prof = {s["name"]: s["ms"] for s in st.ctx.bkfac_profile_read()}
    st.ctx.bkfac_profile_enable(False)
    d = D.double().cpu().numpy()
    gaps = -np.diff(d)
    K = st.K[i].double()
    ev = torch.linalg.eigvalsh(K).cpu().numpy()[::-1][:r]
    print(f"factor {g:2d} n={n:5d} r={r:3d} l={r+ro:3d} cluster={prof.get('eig_cluster', 0):8.3f}ms "
          f"sytrd={prof.get('eig_sytrd', 0):7.3f} D0={d[0]:.4g} Dr={d[-1]:.4g} "
          f"min_gap/D0={gaps.min()/max(d[0],1e-30):.2e} maxrel_vs_eigh={np.max(np.abs(d-ev))/ev[0]:.2e}",
          flush=True)
