"""Profiling driver for one configs[4] (cfg5) step's library calls, each inside an NVTX range
("brand", "prec") so that ncu can pick a stage's kernels:
  ncu --nvtx --nvtx-include "prec/" -k regex:gemm_tc -c 4 ... python tools/prof_cfg5.py
Warm-up steps run first (outside the ranges).  --blocks selects how many of the 24
transformer blocks are set up (default all)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=24)
    ap.add_argument("--warm", type=int, default=2)
    ap.add_argument("--stage-nvtx", action="store_true",
                    help="library NVTX ranges per stage (BKFAC_OPT_NVTX) instead of brand/prec")
    args = ap.parse_args()
    import torch
    import synth
    import bench
    from paper_2210_08494_b200 import BKFACStack
    cfg = synth.cfg5_transformer(blocks=args.blocks)
    factors = [(f.n, f.r, f.c) for f in cfg.factors]
    layers = [(l.d_G, l.d_A, l.g_index, l.a_index) for l in cfg.layers]
    st = BKFACStack(factors, layers, cfg.rho, cfg.lam)
    dev = torch.device("cuda:0")
    M_pool, J_pool = bench.device_inputs(cfg, st.my_factors, st.my_layers, 2, dev)
    for i in range(args.warm):
        st.step(M_pool[i % 2], J_pool[i % 2])
    torch.cuda.synchronize()
    from paper_2210_08494_b200 import binding
    if args.stage_nvtx:
        st.ctx.bkfac_set_option(binding.BKFAC_OPT_NVTX, 1)
    push = (lambda name: None) if args.stage_nvtx else torch.cuda.nvtx.range_push
    pop = (lambda: None) if args.stage_nvtx else torch.cuda.nvtx.range_pop
    # one more step, its two library calls in NVTX ranges (same order as BKFACStack._step)
    k = st.k
    ups = []
    for i, g in enumerate(st.my_factors):
        c, nx = st.cur[i], 1 - st.cur[i]
        ups.append(dict(factor=i, U_in=st.U[i][c], D_in=st.D[i][c], M=M_pool[k % 2][g],
                        U_out=st.U[i][nx], D_out=st.D[i][nx], alpha=st.rho, beta=1 - st.rho))
    push("brand")
    st.ctx.bkfac_brand_update(ups)
    torch.cuda.synchronize()
    pop()
    for i in range(len(st.my_factors)):
        st.cur[i] = 1 - st.cur[i]
    items = []
    for lj, li in enumerate(st.my_layers):
        dG, dA, g, a = st.layers[li]
        UG, DG = st.state(g)
        UA, DA = st.state(a)
        items.append(dict(layer=lj, U_G=UG, D_G=DG, lambda_G=st.lam, U_A=UA, D_A=DA, lambda_A=st.lam,
                          J=J_pool[k % 2][li], S=st.S2[0][li]))
    push("prec")
    st.ctx.bkfac_precondition(items)
    torch.cuda.synchronize()
    pop()
    assert st.check()[0] == 0
    print("prof_cfg5 ok")


if __name__ == "__main__":
    main()
