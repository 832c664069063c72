"""NEXT-f4 driver: the §4.2 error protocol on the GPU at the paper's
"FC layer 0" shape (VGG16_bn fc0: A 513, Gamma 512; n_BS = 256, r = 220, rho = 0.95,
lambda = 0.1; synth's cfg4 generator for that layer), averaged over --runs re-seeded
streams (the paper averages 5 runs, :794).  Writes the per-algorithm window averages of
metrics (1)-(4), the per-update curves and the wall time to a JSON file.

usage: python tools/f4_protocol.py [--runs 5] [--burn-in 60] [--window 30] [--out PATH]
"""
import argparse
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=5)
    ap.add_argument("--burn-in", type=int, default=60)
    ap.add_argument("--window", type=int, default=30)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_f4_error_protocol.json"))
    args = ap.parse_args()
    import torch
    import synth
    from paper_2210_08494_b200 import error_protocol as EP
    cfg = synth.cfg4_vgg_sharded()
    li = [l.name for l in cfg.layers].index("fc0")
    L = cfg.layers[li]
    fA0, fG0 = cfg.factors[L.a_index], cfg.factors[L.g_index]
    algos = EP.paper_algorithms()
    runs, t_all = [], time.time()
    for run in range(args.runs):
        fA = dataclasses.replace(fA0, seed=fA0.seed + 7777 * run)
        fG = dataclasses.replace(fG0, seed=fG0.seed + 7777 * run)
        lay = dataclasses.replace(L, seed=L.seed + 7777 * run)
        torch.cuda.synchronize()
        t0 = time.time()
        out = EP.run(fA, fG, lay, r=fA.r, rho=cfg.rho, lam=cfg.lam, burn_in=args.burn_in,
                     window=args.window, algos=algos, oversample=cfg.oversample,
                     power_iters=cfg.power_iters, seed=run)
        torch.cuda.synchronize()
        runs.append((out, time.time() - t0))
        print(f"run {run}: {time.time() - t0:.1f} s", flush=True)
    names = [a.name for a in algos]
    avg = {n: [sum(EP.summary(o)[n][m] for o, _ in runs) / len(runs) for m in range(4)] for n in names}
    curves = {n: [[sum(o[n][t][m] for o, _ in runs) / len(runs) for m in range(4)]
                  for t in range(args.window)] for n in names}
    res = {
        "protocol": "PAPER.md §4.2 (:774-784), synthetic stand-in for VGG16_bn FC layer 0 K-factors",
        "shape": {"d_A": fA0.n, "d_G": fG0.n, "n_BS": fA0.c, "r": fA0.r, "rho": cfg.rho,
                  "lambda": cfg.lam, "signal_rank": fA0.k, "decay": fA0.decay, "sigma": fA0.sigma},
        "time_unit": "one K-factor update (= T_updt = 10 optimizer steps); periods of :782 / 10",
        "burn_in_updates": args.burn_in, "window_updates": args.window, "runs": args.runs,
        "metrics": ["m1 ||A~^-1 - A_ref^-1||_F/||A_ref^-1||_F", "m2 same for Gamma",
                    "m3 ||s~ - s_ref||_F/||s_ref||_F", "m4 1 - cos(s~, s_ref)"],
        "window_average": avg,
        "per_update_mean_over_runs": curves,
        "wall_s_per_run": [round(t, 2) for _, t in runs],
        "device": torch.cuda.get_device_name(0),
    }
    json.dump(res, open(args.out, "w"), indent=1)
    print(f"{'algorithm':14s} {'m1':>10s} {'m2':>10s} {'m3':>10s} {'m4':>10s}")
    for n in names:
        print(f"{n:14s} " + " ".join(f"{v:10.3e}" for v in avg[n]))
    print(f"total {time.time() - t_all:.1f} s")


if __name__ == "__main__":
    main()
