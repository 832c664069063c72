"""Small end-to-end driver for compute-sanitizer (memcheck / racecheck / synccheck): the
configs[0] toy stack for a few chained steps (Brand init + steps, preconditioning) and one
configs[1]-shaped Brand step with its dense EA accumulate and an RSVD overwrite, plus a
two-stage eigensolver factor (core m = 96) -- every kernel family of the library once."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2210_08494_b200 import BKFACStack, binding
from tests.gpu_helpers import to_dev, to_dev_cols

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = synth.cfg1_toy()
st = BKFACStack([(f.n, f.r, f.c) for f in cfg.factors],
                [(l.d_G, l.d_A, l.g_index, l.a_index) for l in cfg.layers], cfg.rho, cfg.lam)
for k in range(steps):
    st.step({i: to_dev_cols(f.batch(k)) for i, f in enumerate(cfg.factors)}, {0: to_dev(cfg.layers[0].grad(k))})
torch.cuda.synchronize()
assert st.check()[0] == 0
c2 = synth.cfg2_conv()
f = c2.factors[0]
st2 = BKFACStack([(f.n, f.r, f.c)], [], c2.rho, c2.lam, rsvd_every=2)
for k in range(3):   # init, Brand + EA, RSVD overwrite + Brand + EA
    st2.step({0: to_dev_cols(f.batch(k))})
torch.cuda.synchronize()
assert st2.check()[0] == 0
ctx = binding.Context([(300, 64, 32, 0)], [], device=0)
ctx.bkfac_set_option(binding.BKFAC_OPT_TWO_STAGE, 2)
g = synth.random_case(300, 32, 64, seed=3, k=40)
U = to_dev_cols(synth.phantom_basis(300, 64)); D = torch.zeros(64, device="cuda")
Uo, Do = torch.empty_like(U), torch.empty_like(D)
ctx.bkfac_brand_update([dict(factor=0, U_in=U, D_in=D, M=to_dev_cols(g.batch(0)), U_out=Uo, D_out=Do,
                             alpha=0.0, beta=1.0)])
torch.cuda.synchronize()
assert ctx.bkfac_check()[0] == 0
print("sanitize_run ok")
