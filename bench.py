#!/usr/bin/env python
"""B-KFAC hot-path benchmark (driver contract).

A "step" is one pass of the whole hot path over one batch of synthetic input: the
Brand update of every K-factor the rank owns (SURVEY §8(a) a0-a6, a6'), the dense EA
accumulate and -- every T_RSVD steps -- the RSVD overwrite (a7, a8), the
preconditioning of every owned layer (a9), and for N > 1 the NCCL all-gather of the
preconditioned gradients (§8(e)).

Default workload: BASELINE.json configs[4], the transformer-MLP stack the metric's
1/2/4/8-GPU figures are quoted on (24 blocks x (4097->16384, 16385->4096): 96 K-factors,
48 layers, n_BS = 1024, r = 512, rho = 0.97, lambda = 0.01), the same workload at every
GPU count (strong scaling).  ``--config cfg1|cfg2|cfg3|cfg4|cfg5r8`` selects another
BASELINE config; with an RSVD schedule (cfg2, cfg4) the timed window starts on an
overwrite step, so it always holds ceil(steps / T_RSVD) overwrites.

value = Brand factor-updates/s over the whole job (all ranks); the line also carries
preconditioned layers/s.  ``--impl reference`` times the fp64 oracle (the reference arm
of this tier) on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "Brand factor-updates/s + preconditioned layers/s, % roofline, 1/2/4/8 B200"
UNIT = "factor-updates/s"
L2_FLUSH_BYTES = 512 << 20


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=25)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-sets", type=int, default=2,
                    help="device input sets of the e2e leg, used round robin (uploads run ahead)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ignore-status", action="store_true",
                    help="tuning runs of deliberately broken library variants: report stage times anyway")
    ap.add_argument("--cpu-budget-s", type=float, default=25.0)
    ap.add_argument("--pool", type=int, default=2, help="distinct input batches kept on device")
    ap.add_argument("--full-rank", action="store_true",
                    help="NEXT-f1: keep all r + c eigenpairs per step and precondition with them")
    ap.add_argument("--factored", action="store_true",
                    help="NEXT-f2: precondition from the factored gradient G A^T (Algorithm 8)")
    ap.add_argument("--correct-every", type=int, default=0,
                    help="NEXT-f3 (B-KFAC-C): light correction (Alg 6) every T steps")
    ap.add_argument("--phi-crc", type=float, default=0.5, help="n_crc / r of the light correction")
    ap.add_argument("--pipeline", type=int, default=-1,
                    help="> 0: pipelined steps (Brand(k) beside the preconditioning of step k-1, "
                         "the persistent GEMM grids split PIPELINE : 148 - PIPELINE SMs); 0 off; "
                         "-1 (default) auto: stack.pipeline_sms(factors on this rank)")
    ap.add_argument("--no-graphs", action="store_true",
                    help="launch every step eagerly instead of replaying CUDA graphs")
    ap.add_argument("--opt", action="append", default=[],
                    help="library option NAME=VALUE (bkfac_set_option, e.g. TWO_STAGE=2); tuning runs")
    return ap.parse_args()


# ------------------------------------------------------------------------------ helpers

def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0, "_source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def make_workload(name: str):
    import synth
    if name not in synth.CONFIGS:
        raise SystemExit(f"unknown config {name}")
    return synth.CONFIGS[name]()


def device_inputs(cfg, my_factors, my_layers, pool: int, device):
    """Per-step inputs generated ON DEVICE outside the timed region, same recipe as
    synth.FactorSpec.batch (L diag(s) W + sigma N) but drawn with torch's CUDA RNG.  M and J
    live in buffers whose leading dimension is padded to 32 floats (stack.padded)."""
    import torch
    from paper_2210_08494_b200.stack import padded
    M_pool = [dict() for _ in range(pool)]
    J_pool = [dict() for _ in range(pool)]
    for g in my_factors:
        f = cfg.factors[g]
        gen = torch.Generator(device=device)
        gen.manual_seed(f.seed)
        G = torch.randn((f.n, f.k), generator=gen, device=device, dtype=torch.float32)
        L, R = torch.linalg.qr(G)
        L = L * torch.sign(torch.diagonal(R))[None, :]
        s = f.decay ** torch.arange(f.k, device=device, dtype=torch.float32)
        for p in range(pool):
            W = torch.randn((f.k, f.c), generator=gen, device=device)
            N = torch.randn((f.n, f.c), generator=gen, device=device)
            M = (L * s[None, :]) @ W + f.sigma * N            # n x c
            M_pool[p][g] = padded(f.c, f.n, device, zero=False)   # (c, n) == col-major n x c
            M_pool[p][g].copy_(M.t())
        del G, L, R
    for li in my_layers:
        l = cfg.layers[li]
        gen = torch.Generator(device=device)
        gen.manual_seed(l.seed)
        for p in range(pool):
            J_pool[p][li] = padded(l.d_G, l.d_A, device, zero=False)
            J_pool[p][li].copy_(l.grad_std * torch.randn((l.d_G, l.d_A), generator=gen, device=device))
    torch.cuda.synchronize()
    return M_pool, J_pool


def roofline_from_stages(stages, peaks, clocks):
    """Dominant stage (largest event-timed share of the step) against its bound."""
    if not stages:
        return None, []
    # the EA accumulate runs on a side stream beside the tridiagonalisation (library default,
    # option BKFAC_OPT_EA_MODE != 1): off the critical path, so it is not the dominant stage
    side = {"gemm_ea"}
    total = sum(s["ms"] for s in stages if s["name"] not in side)
    stages = sorted(stages, key=lambda s: -s["ms"])
    top = [s for s in stages if s["name"] not in side][0]
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12          # TFLOP/s, FFMA on CUDA cores
    name = top["name"]
    sec = top["ms"] / 1e3
    if name.startswith("gemm_") and top.get("path") == "tc":
        tf32 = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))) * 0.5
        bound, peak, unit, achieved = "tensor", tf32 / 3.0, "TFLOP/s", top["flops"] / sec / 1e12
    elif name.startswith("gemm_") or name.startswith("eig_") or name.startswith("chol"):
        bound, peak, unit, achieved = "alu", fp32_peak, "TFLOP/s", top["flops"] / sec / 1e12
    else:
        bound, peak, unit, achieved = "hbm", float(peaks["hbm_gbs"]), "GB/s", top["bytes"] / sec / 1e9
    roof = {"bound": bound, "achieved": round(achieved, 4), "peak": round(peak, 3), "unit": unit,
            "frac": round(achieved / peak, 5) if peak else None, "traffic": None,
            "kernel": name, "share_of_step": round(top["ms"] / total, 4) if total else None,
            "launches_per_step": None,
            "side_stream_stages": sorted(side & {s["name"] for s in stages}),
            "peak_source": peaks["_source"] +
            ("; fp32 CUDA-core peak = 148 SM x 128 FMA x 2 x sm_max" if bound == "alu" else "")}
    table = [{"stage": s["name"], "ms": round(s["ms"], 4),
              "share": None if s["name"] in side else round(s["ms"] / total, 4),
              "gflop": round(s["flops"] / 1e9, 3), "gbytes": round(s["bytes"] / 1e9, 4),
              "launches": s["launches"]} for s in stages]
    return roof, table


def traffic_lookup(kernel_stage: str, workload: str):
    """DRAM bytes per launch of the stage's kernel from the committed ncu launch list, when
    that list was taken on this workload (else None)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(workload, {}).get(kernel_stage)
    except (OSError, ValueError, AttributeError):
        return None


# ------------------------------------------------------------------------------ CPU oracle

def oracle_sample(cfg, budget_s: float):
    """Time the fp64 oracle as it stands on a bounded sample of the workload: one layer per
    distinct layer shape (smallest first) -- its A and Gamma Brand updates and its
    preconditioning -- until the time budget is spent.  Input generation is not timed.
    Returns (factor_updates, layers, seconds, extrapolated full-step seconds, description)."""
    import numpy as np
    import oracle as O
    rng = np.random.default_rng(0)

    def inputs(f):
        U, _ = np.linalg.qr(rng.standard_normal((f.n, f.r)))
        return U, np.sort(rng.random(f.r))[::-1], f.batch(1).astype(np.float64)

    layers = list(cfg.layers)
    if not layers:   # factor-only workload (cfg2)
        f = cfg.factors[0]
        U, D, M = inputs(f)
        t0 = time.perf_counter()
        O.brand_update(U, D, M, cfg.rho, 1 - cfg.rho, f.r)
        dt = time.perf_counter() - t0
        return 1, 0, dt, dt * len(cfg.factors), f"1 Brand update of n={f.n}, fp64 numpy"
    shapes = {}
    for li, l in enumerate(layers):
        key = (cfg.factors[l.a_index].n, cfg.factors[l.g_index].n, l.d_G, l.d_A)
        shapes.setdefault(key, []).append(li)
    times, counts = {}, {}
    spent = 0.0
    passes = 0
    # passes over the distinct shapes (smallest first) until ~10 s of oracle work (at least
    # one full pass unless the budget runs out first); per-shape time = mean over passes
    while True:
        done_pass = True
        for key, lis in sorted(shapes.items(), key=lambda kv: kv[0][0] + kv[0][1]):
            if spent > budget_s and times:
                done_pass = False
                break
            l = layers[lis[0]]
            fa, fg = cfg.factors[l.a_index], cfg.factors[l.g_index]
            ia, ig = inputs(fa), inputs(fg)
            J = l.grad(1).astype(np.float64)
            t0 = time.perf_counter()
            UA, DA = O.brand_update(*ia, cfg.rho, 1 - cfg.rho, fa.r)
            UG, DG = O.brand_update(*ig, cfg.rho, 1 - cfg.rho, fg.r)
            O.precondition(J, UG, DG, cfg.lam, UA, DA, cfg.lam)
            dt = time.perf_counter() - t0
            times[key] = times.get(key, 0.0) + dt
            counts[key] = counts.get(key, 0) + 1
            spent += dt
        passes += done_pass
        if not done_pass or spent >= min(10.0, budget_s):
            break
    total = sum(times.values())
    nupd = 2 * sum(counts.values())
    times = {key: t / counts[key] for key, t in times.items()}
    step_s = 0.0
    kref, tref = max(times.items(), key=lambda kv: kv[1])
    for key, lis in shapes.items():
        if key in times:
            step_s += times[key] * len(lis)
        else:   # unsampled shapes: O(n^2 (r + c)) model relative to the slowest sample
            scale = (key[0] ** 2 + key[1] ** 2) / max(kref[0] ** 2 + kref[1] ** 2, 1)
            step_s += tref * scale * len(lis)
    lay = len(times)
    desc = (f"{lay} of {len(layers)} layers (one per distinct shape, smallest first), "
            f"{max(passes, 1)} pass(es) within ~10 s (budget {budget_s:.0f}s): 2 Brand updates + 1 "
            f"preconditioning each, fp64 numpy oracle; full-step time extrapolated by layer counts"
            + ("" if lay == len(shapes) else "; unsampled shapes scaled by n^2"))
    return nupd, sum(counts.values()), total, step_s, desc


def oracle_thread_ratio(cfg):
    """Wall time of one oracle Brand update of the workload's smallest Brand-path factor at 1
    BLAS thread over the same at all threads: scales the all-cores baseline to one core."""
    import numpy as np
    import oracle as O
    from threadpoolctl import threadpool_limits
    f = min(cfg.factors, key=lambda x: (x.r + x.c >= x.n, x.n))
    rng = np.random.default_rng(7)
    U, _ = np.linalg.qr(rng.standard_normal((f.n, f.r)))
    D = np.sort(rng.random(f.r))[::-1]
    M = f.batch(1).astype(np.float64)
    t = {}
    for nt in (None, 1):
        with threadpool_limits(limits=nt, user_api="blas"):
            t0 = time.perf_counter()
            O.brand_update(U, D, M, cfg.rho, 1 - cfg.rho, f.r)
            t[nt] = time.perf_counter() - t0
    return t[None] / t[1], f"one Brand update of n={f.n}: {t[None]:.2f} s at all threads, {t[1]:.2f} s at 1 thread"


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [d.get("num_threads", 1) for d in threadpool_info() if d.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return 1


# ------------------------------------------------------------------------------ arms

def run_reference(args, rank, world):
    """Reference arm of this tier: the fp64 oracle as it stands on the host cores."""
    if rank != 0:
        return
    cfg = make_workload(args.config)
    import numpy as np
    import oracle as O
    layers = list(cfg.layers)
    n_f = len(cfg.factors)
    n_l = len(layers)
    per_step = []
    upd_total = 0
    t_total = 0.0
    rng = np.random.default_rng(1)
    for step in range(args.warmup + args.steps):
        # one layer per step (cycling): its 2 Brand updates + its preconditioning
        if layers:
            l = layers[step % n_l]
            fis = (l.a_index, l.g_index)
        else:
            l = None
            fis = (step % n_f,)
        inputs = []
        for fi in fis:
            f = cfg.factors[fi]
            U, _ = np.linalg.qr(rng.standard_normal((f.n, f.r)))
            inputs.append((U, np.sort(rng.random(f.r))[::-1], f.batch(step).astype(np.float64), f.r))
        J = l.grad(step).astype(np.float64) if l is not None else None
        t0 = time.perf_counter()
        reps = [O.brand_update(U, D, M, cfg.rho, 1 - cfg.rho, r) for (U, D, M, r) in inputs]
        if l is not None:
            O.precondition(J, reps[1][0], reps[1][1], cfg.lam, reps[0][0], reps[0][1], cfg.lam)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            per_step.append(dt)
            upd_total += len(fis)
            t_total += dt
    value = upd_total / t_total
    cores = blas_threads()
    sample = (f"per step: one layer of the {cfg.name} stack (cycling) = {len(fis)} Brand "
              f"update(s) + {'1 preconditioning' if layers else 'no layer'}, fp64 numpy oracle")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * t_total / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name + ("+f1_full_rank" if args.full_rank else "")
                                   + ("+f2_factored" if args.factored else "")
                                   + (f"+f3_correct{args.correct_every}_phi{args.phi_crc:g}"
                                      if args.correct_every else ""),
                       "factors": n_f, "layers": n_l,
                       "sample": "one layer (2 factor updates + preconditioning) per step"},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2210_08494_b200 import BKFACStack, SlotGather

    device = torch.device(f"cuda:{local_rank}")
    torch.cuda.set_device(device)
    cfg = make_workload(args.config)
    factors = [(f.n, f.r, f.c) for f in cfg.factors]
    layers = [(l.d_G, l.d_A, l.g_index, l.a_index) for l in cfg.layers]
    stack = BKFACStack(factors, layers, cfg.rho, cfg.lam, rsvd_every=cfg.rsvd_every,
                       oversample=cfg.oversample, power_iters=cfg.power_iters,
                       device=local_rank, rank=rank, world=world, full_rank=args.full_rank,
                       correct_every=args.correct_every, phi_crc=args.phi_crc)
    from paper_2210_08494_b200 import binding as _bd
    for o in args.opt:
        name, val = o.split("=")
        stack.ctx.bkfac_set_option(getattr(_bd, "BKFAC_OPT_" + name.upper()), int(val))
    gather = SlotGather(layers, stack.owned_layers_all, rank, device) if world > 1 and layers else None
    if gather is not None:
        # precondition straight into the send slots; step k's all-gather (buffer set k & 1)
        # overlaps step k + 1's compute
        stack.bind_outputs([gather.send_views(0), gather.send_views(1)])
    M_pool, J_pool = device_inputs(cfg, stack.my_factors, stack.my_layers, args.pool, device)
    in_bytes = sum(4 * t.numel() for t in M_pool[0].values()) + sum(4 * t.numel() for t in J_pool[0].values())
    # inputs larger than L2 (configs[4]: 17 GB per step on one GPU, 2 GB per rank at 8): no
    # flush needed between steps; smaller workloads flush L2 (512 MiB write) between steps
    use_flush = in_bytes < 2 * (126 << 20)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=device) if use_flush else None
    stream = torch.cuda.current_stream()

    use_graphs = not args.no_graphs

    if args.pipeline < 0:
        from paper_2210_08494_b200 import pipeline_sms
        args.pipeline = 0 if (args.factored or args.correct_every) \
            else pipeline_sms(len(stack.my_factors))
    if args.pipeline:
        stack.set_pipeline(args.pipeline)

    def one_step(i, graph, profile=False):
        # pipelined: this call preconditions (and writes the S of) step k - 1
        ks = stack.k - 1 if args.pipeline else stack.k
        b = ks & 1
        if gather is not None and ks >= 0:
            gather.finish(b)          # step k - 2's gather on this buffer set has completed
        S = stack.step(M_pool[i % args.pool], None if args.factored else J_pool[i % args.pool],
                       graph=graph, factored=args.factored, profile=profile)
        if gather is not None and ks >= 0:
            gather.start(b)

    # warm-up (>= 3 steps also captures the two CUDA graphs of a non-RSVD step: the U/D
    # ping-pong parity and the input pool alternate together).  With an RSVD schedule the
    # warm-up is extended so that the timed window starts on an overwrite step: the window
    # then holds ceil(K / T_RSVD) overwrites (never none).
    warm = args.warmup
    T = cfg.rsvd_every
    if T and warm % T != 0:
        warm += T - warm % T
    for i in range(warm):
        one_step(i, use_graphs)
    torch.cuda.synchronize()
    code, bad, info = stack.check()
    if code != 0 and not args.ignore_status:
        raise SystemExit(f"device status error after warm-up (factor {bad})")

    def timed(first, nsteps, graph, profile=False):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(nsteps)]
        stage_acc = {}
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(nsteps):
            if use_flush:
                if gather is not None:          # no collective overlaps the (untimed) flush
                    gather.finish(0); gather.finish(1)
                flush.zero_()                   # L2 flush between timed steps (not timed)
            r0 = stack.ctx.bkfac_profile_count() if profile else 0
            stack.last_profile_range = None
            ev[i][0].record(stream)
            one_step(first + i, graph, profile)
            ev[i][1].record(stream)
            if profile:
                # the stage events of this step: a profiled graph's record range (re-recorded
                # by every replay), or the records an eager (RSVD) step appended
                rng = stack.last_profile_range or (r0, stack.ctx.bkfac_profile_count())
                torch.cuda.synchronize()
                for st_ in stack.ctx.bkfac_profile_read(rng):
                    acc = stage_acc.setdefault(st_["name"], dict(st_, ms=0.0, flops=0.0, bytes=0.0,
                                                                 launches=0, calls=0))
                    for key_ in ("ms", "flops", "bytes", "launches", "calls"):
                        acc[key_] += st_[key_]
        # the last steps' all-gathers still in flight belong to the timed work
        tail = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        tail[0].record(stream)
        if gather is not None:
            gather.finish(0); gather.finish(1)
        tail[1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return (sum(a.elapsed_time(b) for a, b in ev) + tail[0].elapsed_time(tail[1]),
                list(stage_acc.values()))

    # headline: K steps (RSVD steps included at their schedule), profiling off
    sampler = ClockSampler(local_rank)
    sampler.start()
    ms, _ = timed(warm, args.steps, use_graphs)
    clocks = sampler.stop()
    n_rsvd = sum(1 for k in range(warm, warm + args.steps) if T and k % T == 0)
    # stage table + roofline: the next K steps again with the library's per-stage CUDA events
    # on the launching streams.  With graphs these events are nodes of separately captured
    # "profiled" graphs (the same kernels; the event nodes add little), so the stage times
    # are graph-replay times like the headline's; launch counts come from an eager step.
    stack.ctx.bkfac_profile_enable(True)
    first_prof = warm + args.steps
    if T:   # same RSVD phase as the headline window
        first_prof += (T - first_prof % T) % T
        for i in range(warm + args.steps, first_prof):
            one_step(i, use_graphs)
    ms_prof, stages = timed(first_prof, args.steps, use_graphs, profile=True)
    stack.ctx.bkfac_profile_enable(False)
    l0 = stack.launches()
    one_step(first_prof + args.steps, False)      # one eager step: launches per step
    torch.cuda.synchronize()
    launches = (stack.launches() - l0) * args.steps
    t = torch.tensor([ms, float(launches)], dtype=torch.float64, device=device)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms, launches = float(tmax[0]), int(tsum[1])
    code, bad, info = stack.check()
    if code != 0 and not args.ignore_status:
        raise SystemExit(f"device status error in the timed region (factor {bad})")

    n_f, n_l = len(cfg.factors), len(cfg.layers)
    sec = ms / 1e3
    value = n_f * args.steps / sec
    layers_per_s = n_l * args.steps / sec

    # ---- e2e through the public API with host buffers (pinned), copies timed
    e2e = None
    if args.pipeline:
        stack.flush()
        stack.set_pipeline(0)     # the e2e leg runs the unpipelined schedule
    if not args.no_e2e:
        e2e = run_e2e(args, stack, gather, cfg, device, stream, world, M_pool, J_pool)

    if rank != 0:
        return
    peaks = load_peaks()
    for s in stages:
        s["path"] = "tc" if stack_uses_tc(stack) else "simt"
    roof, table = roofline_from_stages(stages, peaks, clocks)
    if roof is not None:
        variant = ((args.full_rank or args.factored or args.correct_every) and "+variant") or ""
        roof["traffic"] = traffic_lookup(roof["kernel"], cfg.name + variant)
        roof["launches_per_step"] = round(next(s["launches"] for s in stages
                                               if s["name"] == roof["kernel"]) / args.steps, 2)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        upd, lay, ssec, step_s, desc = oracle_sample(cfg, args.cpu_budget_s)
        cpu = {"value": round(n_f / step_s, 4), "unit": UNIT, "cores": blas_threads(),
               "kind": "oracle", "sample": desc + f"; sample took {ssec:.1f}s",
               "measured_updates_per_s_on_sample": round(upd / ssec, 4),
               "host_cpu_count": os.cpu_count()}
        try:
            ratio, rdesc = oracle_thread_ratio(cfg)
            cpu["value_1_thread"] = round(n_f / step_s * ratio, 4)
            cpu["value_1_thread_how"] = "all-threads value x (t_all / t_1) measured on " + rdesc
        except Exception as exc:   # threadpoolctl missing: report the all-cores figure only
            cpu["value_1_thread"] = None
            cpu["value_1_thread_how"] = f"unavailable: {exc}"
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "weak" if not layers else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "layers_per_s": round(layers_per_s, 3),
            "config": {"workload": cfg.name + ("+f1_full_rank" if args.full_rank else "")
                                   + ("+f2_factored" if args.factored else "")
                                   + (f"+f3_correct{args.correct_every}_phi{args.phi_crc:g}"
                                      if args.correct_every else ""),
                       "factors": n_f, "layers": n_l,
                       "n_BS": cfg.factors[0].c, "rho": cfg.rho, "lambda": cfg.lam,
                       "rsvd_every": cfg.rsvd_every, "rsvd_steps_in_window": n_rsvd,
                       "parallelism": f"layer-shard x{world}",
                       "l2": ("flushed between timed steps (512 MiB write)" if use_flush else
                              f"inputs larger than L2 ({in_bytes / 2**30:.1f} GiB per step per rank), no flush"),
                       "allgather": ("per-slot NCCL all-gather of step k overlapped with step k+1 "
                                     "(preconditioned straight into the send slots)") if gather else None,
                       "inputs": "device-resident pool of %d synthetic batches" % args.pool},
            "roofline": roof, "stages": table, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks,
            "launch_mode": "cuda-graph replay (non-RSVD steps)" if use_graphs else "eager",
            "profiled_pass_ms_per_step": round(ms_prof / args.steps, 4),
            "profiled_pass": ("graph replays with the library's stage events as graph nodes"
                              if use_graphs else "eager launches with stage events")}
    if args.opt:
        line["library_options"] = args.opt
    if args.pipeline:
        line["pipeline"] = {"prec_sms": args.pipeline, "schedule": (
            "step k runs Brand(k) beside the preconditioning of step k-1 (second stream, "
            "persistent GEMM grids split %d : %d SMs); every timed step does one Brand update of "
            "every factor and one preconditioning of every layer" % (args.pipeline, 148 - args.pipeline))}
    print(json.dumps(line), flush=True)


def stack_uses_tc(stack) -> bool:
    try:
        return b"tcgen05" in stack.ctx.lib.bkfac_build_info()
    except Exception:
        return False


def run_e2e(args, stack, gather, cfg, device, stream, world, M_pool, J_pool):
    """Same metric through the public API with HOST inputs: per step, pinned host -> device
    copies of the step's M and J, the step, and a device -> host read of S."""
    import torch
    import torch.distributed as dist
    from paper_2210_08494_b200.stack import padded, full_rows
    steps = max(1, min(args.e2e_steps, args.steps))
    # host inputs: the headline's own synthetic batches (synth recipe, device pool batch 0)
    # copied to pinned host memory -- every factor's M (so the eigensolver sees the same
    # spectra as the headline) and one gradient per layer shape (J ~ N(0, var) throughout)
    # host buffers have the device buffers' padded layout (leading dimension a multiple of
    # 32), so every copy is one contiguous DMA of the whole buffer
    host_M = {g: full_rows(M_pool[0][g]).cpu().pin_memory() for g in stack.my_factors}
    host_J, host_S = {}, {}
    for li in stack.my_layers:
        l = cfg.layers[li]
        key = (l.d_G, l.d_A)
        if key not in host_J:
            host_J[key] = full_rows(J_pool[0][li]).cpu().pin_memory()
            host_S[key] = torch.empty(tuple(host_J[key].shape), dtype=torch.float32).pin_memory()
    # NB device input sets, used round robin: the host->device copies of steps i+1 .. i+NB-1
    # run back to back on the copy stream while step i computes (with NB = 2 the next upload
    # could only start when the step two back had finished, which serialises copies and
    # compute once the copies are the longer of the two); step i's S is read back on a second
    # copy stream while step i+1 computes (the stack's two S sets, by step parity)
    NB = max(2, args.e2e_sets)
    dev_M = [{g: padded(cfg.factors[g].c, cfg.factors[g].n, device, zero=False)
              for g in stack.my_factors} for _ in range(NB)]
    dev_J = [{li: padded(cfg.layers[li].d_G, cfg.layers[li].d_A, device, zero=False)
              for li in stack.my_layers} for _ in range(NB)]
    h2d = sum(4 * full_rows(t).numel() for t in dev_M[0].values()) + \
        (0 if args.factored else sum(4 * full_rows(t).numel() for t in dev_J[0].values()))
    d2h = sum(4 * host_S[(cfg.layers[li].d_G, cfg.layers[li].d_A)].numel() for li in stack.my_layers)
    use_graphs = not args.no_graphs
    up, down = torch.cuda.Stream(device=device), torch.cuda.Stream(device=device)
    ev_up = [torch.cuda.Event() for _ in range(NB)]
    ev_done = [torch.cuda.Event() for _ in range(NB)]
    ev_down = [torch.cuda.Event() for _ in range(2)]

    def upload(j):
        b = j % NB
        with torch.cuda.stream(up):
            up.wait_event(ev_done[b])             # step j-NB (same buffers) has finished
            for g, t in dev_M[b].items():
                full_rows(t).copy_(host_M[g], non_blocking=True)
            if not args.factored:
                for li, t in dev_J[b].items():
                    l = cfg.layers[li]
                    full_rows(t).copy_(host_J[(l.d_G, l.d_A)], non_blocking=True)
            ev_up[b].record(up)

    def run(n):
        for j in range(min(NB - 1, n)):
            upload(j)
        for j in range(n):
            b = j % NB
            sb = stack.k & 1
            stream.wait_event(ev_up[b])
            stream.wait_event(ev_down[sb])        # S set sb was read back (step j-2)
            if gather is not None:
                gather.finish(sb)
            S = stack.step(dev_M[b], None if args.factored else dev_J[b], graph=use_graphs,
                           factored=args.factored)
            if gather is not None:
                gather.start(sb)
            ev_done[b].record(stream)
            if j + NB - 1 < n:
                upload(j + NB - 1)
            with torch.cuda.stream(down):
                down.wait_event(ev_done[b])
                for li, s_ in S.items():
                    l = cfg.layers[li]
                    hs = host_S[(l.d_G, l.d_A)]
                    if s_.stride(0) == hs.shape[1]:
                        hs.copy_(full_rows(s_), non_blocking=True)
                    else:   # S bound to packed send slots (N > 1)
                        hs[:, :l.d_A].copy_(s_, non_blocking=True)
                ev_down[sb].record(down)
        if gather is not None:
            gather.finish(0); gather.finish(1)
        torch.cuda.synchronize()

    run(2 * NB)             # untimed: captures the graphs of every (U parity, input set) pair
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(steps)
    sec = time.perf_counter() - t0

    # the link bound of this leg: the same copies (H2D of the inputs and D2H of S on their
    # two streams, concurrently) with no compute, wall clock per step
    def copies_only(n):
        for j in range(n):
            b = j & 1
            with torch.cuda.stream(up):
                for g, t in dev_M[b].items():
                    full_rows(t).copy_(host_M[g], non_blocking=True)
                if not args.factored:
                    for li, t in dev_J[b].items():
                        l = cfg.layers[li]
                        full_rows(t).copy_(host_J[(l.d_G, l.d_A)], non_blocking=True)
            with torch.cuda.stream(down):
                for li in stack.my_layers:
                    l = cfg.layers[li]
                    s_ = stack.S2[b][li]
                    hs = host_S[(l.d_G, l.d_A)]
                    if s_.stride(0) == hs.shape[1]:
                        hs.copy_(full_rows(s_), non_blocking=True)
                    else:
                        hs[:, :l.d_A].copy_(s_, non_blocking=True)
        torch.cuda.synchronize()
    copies_only(1)
    t1 = time.perf_counter()
    copies_only(steps)
    link_sec = time.perf_counter() - t1
    t = torch.tensor([sec, link_sec], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec, link_sec = float(t[0]), float(t[1])
        hd = torch.tensor([h2d, d2h], dtype=torch.float64, device=device)
        dist.all_reduce(hd, op=dist.ReduceOp.SUM)
        h2d, d2h = int(hd[0]), int(hd[1])
    return {"value": round(len(cfg.factors) * steps / sec, 3), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps,
            "ms_per_step": round(1e3 * sec / steps, 3),
            "copies_only_ms_per_step": round(1e3 * link_sec / steps, 3),
            "link_frac": round(link_sec / sec, 4),
            "input_sets": NB,
            "timing": "wall clock around every step's pinned-host H2D copies, the step and the D2H read of S "
                      "(uploads of the next input sets and the read-back of step i-1 overlapped with step i "
                      "on two copy streams), max over ranks; "
                      "copies_only_ms_per_step: the same H2D + D2H copies with no compute (the PCIe bound "
                      "of this leg), link_frac = copies-only time / e2e time"}


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world == 1 and args.gpus > 1:
        raise SystemExit("--gpus N > 1 must be launched with torch.distributed.run (one rank per GPU)")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
