import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import bench
from paper_2210_08494_b200 import BKFACStack
cfg = bench.make_workload("cfg4")
factors = [(f.n, f.r, f.c) for f in cfg.factors]
layers = [(l.d_G, l.d_A, l.g_index, l.a_index) for l in cfg.layers]
st = BKFACStack(factors, layers, cfg.rho, cfg.lam, rsvd_every=cfg.rsvd_every, full_rank=True)
Mp, Jp = bench.device_inputs(cfg, st.my_factors, st.my_layers, 2, torch.device("cuda:0"))
for i in range(6):
    st.step(Mp[i % 2], Jp[i % 2])
torch.cuda.synchronize()
for g in st.my_factors:
    U, D = st.state(g)
    D = D.double().cpu().numpy()
    tol = 1e-7 * D[0]
    lens = []; cur = 1
    for gap in -np.diff(D):
        if gap <= tol: cur += 1
        else:
            if cur > 1: lens.append(cur)
            cur = 1
    if cur > 1: lens.append(cur)
    print(g, factors[g], len(D), "D0 %.3g Dmin %.3g" % (D[0], D[-1]), "zeros", int((D <= tol).sum()), "clusters", sorted(lens)[-4:])
