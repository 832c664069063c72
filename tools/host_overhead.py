"""Host enqueue time of one stack step vs its device time (cfg4 by default): is the step
launch-bound?"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2210_08494_b200 import BKFACStack

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
cfg = bench.make_workload(cfgname)
factors = [(f.n, f.r, f.c) for f in cfg.factors]
layers = [(l.d_G, l.d_A, l.g_index, l.a_index) for l in cfg.layers]
stack = BKFACStack(factors, layers, cfg.rho, cfg.lam, rsvd_every=cfg.rsvd_every,
                   oversample=cfg.oversample, power_iters=cfg.power_iters)
M_pool, J_pool = bench.device_inputs(cfg, stack.my_factors, stack.my_layers, 2, torch.device("cuda:0"))
for i in range(4):
    stack.step(M_pool[i % 2], J_pool[i % 2])
torch.cuda.synchronize()
for prof in (False, True):
    stack.ctx.bkfac_profile_enable(prof)
    N = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # keep the GPU busy first so the host runs ahead: host time = pure enqueue cost
    big = torch.empty(1 << 28, device="cuda")
    for _ in range(40):
        big.mul_(1.0)
    e0.record()
    t0 = time.perf_counter()
    for i in range(N):
        stack.step(M_pool[i % 2], J_pool[i % 2])
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    # device time of the same steps without the busy prefix
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for i in range(N):
        stack.step(M_pool[i % 2], J_pool[i % 2])
    f1.record()
    torch.cuda.synchronize()
    if prof:
        stack.ctx.bkfac_profile_read()
    print(f"profiling={prof}: host enqueue {1e3 * (t1 - t0) / N:.3f} ms/step, "
          f"device (back-to-back) {f0.elapsed_time(f1) / N:.3f} ms/step, launches/step "
          f"{stack.launches() / max(1, stack.k):.1f}")

# ---- CUDA-graph replay of a (non-RSVD) step: two graphs (U ping-pong parity x input pool)
stack.ctx.bkfac_profile_enable(False)
while stack.rsvd_every and (stack.k % stack.rsvd_every in (0, 1, 2)):
    stack.step(M_pool[stack.k % 2], J_pool[stack.k % 2])
torch.cuda.synchronize()
graphs = []
s = torch.cuda.Stream()
for par in range(2):
    g = torch.cuda.CUDAGraph()
    i = stack.k
    with torch.cuda.graph(g, stream=s):
        stack.step(M_pool[i % 2], J_pool[i % 2], stream=torch.cuda.current_stream())
    graphs.append((g, i % 2))
torch.cuda.synchronize()
# the captures advanced the schedule by two steps without running them: replay both
for g, _ in graphs:
    g.replay()
torch.cuda.synchronize()
code = stack.check()[0]
N = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(N):
    graphs[i % 2][0].replay()
e1.record()
torch.cuda.synchronize()
print(f"graph replay: {e0.elapsed_time(e1) / N:.3f} ms/step (status {code}, {stack.check()[0]})")
