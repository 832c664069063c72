"""Dense EA accumulate (a8) micro-benchmark: K <- rho K + (1-rho) M M^T over the cfg4
factor set and single large factors (CUDA events, median)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2210_08494_b200 import binding
import bench


def time_ea(shapes, rho, reps=10):
    ctx = binding.Context([(n, min(r, n), c, binding.BKFAC_FACTOR_DENSE_EA) for (n, r, c) in shapes], [])
    Ks = [torch.zeros((n, n), device="cuda") for (n, _, _) in shapes]
    Ms = [torch.randn((c, n), device="cuda") for (n, _, c) in shapes]
    items = [dict(factor=i, K=Ks[i], M=Ms[i], rho=rho) for i in range(len(shapes))]
    flush = torch.empty(128 * 1024 * 1024, device="cuda")
    for _ in range(3):
        ctx.bkfac_ea_batch(items)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ctx.bkfac_ea_batch(items); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    fl = sum(2.0 * n * n * c for (n, _, c) in shapes)
    by = sum(4.0 * (n * n * (2 if rho else 1) + n * c) for (n, _, c) in shapes)
    return dict(ms=round(ms, 4), tflops=round(fl / ms / 1e9, 1), gbs=round(by / ms / 1e6, 1))


cfg = bench.make_workload("cfg4")
ONCE = "--once" in sys.argv
fs = [(f[0], f[1], f[2]) for f in cfg.factors] if isinstance(cfg.factors[0], tuple) else \
     [(f.n, f.r, f.c) for f in cfg.factors]
if ONCE:   # profiling: 4 launches of the cfg4 EA batch
    fs0 = [(f[0], f[1], f[2]) for f in cfg.factors] if isinstance(cfg.factors[0], tuple) else \
          [(f.n, f.r, f.c) for f in cfg.factors]
    print(time_ea(fs0, 0.95, reps=1))
    sys.exit(0)
for name, shapes in (("cfg4 all 32", fs), ("one 4609", [(4609, 220, 256)]),
                     ("five 4609", [(4609, 220, 256)] * 5), ("one 4608", [(4608, 220, 256)])):
    for rho in (0.95, 0.0):
        print(json.dumps(dict(case=name, rho=rho, **time_ea(shapes, rho))), flush=True)
