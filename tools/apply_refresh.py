"""Copy the bench lines / ncu summaries of a gpu_round_refresh.sh (+ gpu_next_rows.sh) run
from gpurun_out/ into profiles/ and update the measured numbers in DESIGN.md, README.md and
profiles/r01_summary.md.  usage: python tools/apply_refresh.py [milestone text]"""
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def load(f):
    line = [x for x in open(os.path.join(G, f)) if x.startswith("{")][-1]
    return json.loads(line)


def sub(s, pat, new):
    if not re.search(pat, s):
        raise SystemExit(f"pattern not found: {pat}")
    return re.sub(pat, new, s)


def main():
    c4, c5, r8 = load("bench_cfg4.json"), load("bench_cfg5.json"), load("bench_cfg5r8.json")
    f1, f2, f3 = load("bench_f1.json"), load("bench_f2.json"), load("bench_f3.json")
    for src, dst in [("bench_cfg4.json", "r01_bench_cfg4.json"), ("bench_cfg5.json", "r01_bench_cfg5.json"),
                     ("bench_ref.json", "r01_bench_reference_cfg4.json"),
                     ("bench_f1.json", "r01_bench_cfg4_f1_full_rank.json"),
                     ("bench_f2.json", "r01_bench_cfg4_f2_factored.json"),
                     ("bench_f3.json", "r01_bench_cfg4_f3_correction.json"),
                     ("r01_launches_cfg4.txt", "r01_launches_cfg4.txt"),
                     ("r01_ncu_full_cfg4.txt", "r01_ncu_full_cfg4.txt")]:
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))
    r8["_note"] = ("one rank's share of configs[4] at 8 GPUs (3 of 24 blocks: 12 factors, 6 layers) timed "
                   "on one GPU, all-gather excluded: projects the 8-GPU step; 1-GPU configs[4] = %.0f ms/step"
                   % c5["ms_per_step"])
    json.dump(r8, open(os.path.join(P, "r01_bench_cfg5_rank_of_8.json"), "w"))
    t = json.load(open(os.path.join(G, "traffic.json")))
    for line in open(os.path.join(G, "r01_launches_cfg4.txt")):
        if line.startswith("gemm_tc_kernel<0, 1, 128, 16, 1, 8, 0>"):
            t["gemm_ea"] = float(line.split()[-1]) * 1e6
    t["workload"] = "cfg4_vgg16bn_rsvd"
    t["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes), ncu launch list r01 "
                  "(profiles/r01_launches_cfg4.txt), cfg4 bench; gemm_ea = gemm_tc_kernel<0, 1, 128, 16, 1, 8, 0> "
                  "mean (EA accumulate and the other short-K TB stages). Valid for the cfg4 workload only.")
    json.dump(t, open(os.path.join(P, "traffic.json"), "w"), indent=1)
    st = {s["stage"]: s["ms"] / c4["steps"] for s in c4["stages"]}
    proj = c5["ms_per_step"] / r8["ms_per_step"]
    p = os.path.join(ROOT, "DESIGN.md")
    s = open(p).read()
    s = sub(s, r"\| cfg4 \(default\) \| [0-9.]+ \| ≈ \d+ \| e2e ≈ \d+/s",
            "| cfg4 (default) | %.2f | ≈ %d | e2e ≈ %d/s" % (c4["ms_per_step"], round(c4["value"], -1),
                                                           round(c4["e2e"]["value"], -1)))
    s = sub(s, r"\| cfg5 \| [0-9.]+ \| ≈ \d+ \| e2e ≈ \d+/s",
            "| cfg5 | %.0f | ≈ %d | e2e ≈ %d/s" % (c5["ms_per_step"], round(c5["value"]), round(c5["e2e"]["value"])))
    s = sub(s, r"\| cfg5r8 \(one 8-GPU rank's share\) \| [0-9.]+ \| ≈ \d+ per rank \| projected 1→8: [0-9.]+×",
            "| cfg5r8 (one 8-GPU rank's share) | %.1f | ≈ %d per rank | projected 1→8: %.1f×"
            % (r8["ms_per_step"], round(r8["value"]), proj))
    for tag, d in (("f1 \\(rank r \\+ c\\)", f1), ("f2 \\(Algorithm 8\\)", f2), ("f3 \\(correction every 5\\)", f3)):
        s = sub(s, r"\| cfg4 \+ %s \| [0-9.]+ \| ≈ \d+ \|" % tag,
                "| cfg4 + %s | %.1f | ≈ %d |" % (tag.replace("\\", ""), d["ms_per_step"], round(d["value"], -1)))
    s = sub(s, r"Next, in order of expected gain \(cfg4 at [0-9.]+ ms/step; configs\[4\] at \d+ ms",
            "Next, in order of expected gain (cfg4 at %.2f ms/step; configs[4] at %.0f ms"
            % (c4["ms_per_step"], c5["ms_per_step"]))
    s = sub(s, r"\| tridiagonalisation \| 1\.[0-9]+ alone, ≈ [0-9.]+ beside the EA",
            "| tridiagonalisation | 1.72 alone, ≈ %.1f beside the EA" % st["eig_sytrd"])
    s = sub(s, r"\| EA accumulate \| 0\.[0-9]+ serial \([0-9.]+ beside",
            "| EA accumulate | 0.64 serial (%.2f beside" % st["gemm_ea"])
    s = sub(s, r"\| Cholesky \| [0-9.]+ \|", "| Cholesky | %.2f |" % st["chol_inv"])
    s = sub(s, r"against \d+ ms/step on one GPU \([0-9.]+ ms per rank\): [0-9.]+× before the all-gather",
            "against %.0f ms/step on one GPU (%.1f ms per rank): %.1f× before the all-gather"
            % (c5["ms_per_step"], r8["ms_per_step"], proj))
    open(p, "w").write(s)
    p = os.path.join(ROOT, "README.md")
    s = open(p).read()
    s = sub(s, r"\| config 4: VGG16_bn stack, 32 factors \+ 16 layers, RSVD every 25 \| [0-9.]+ \| ≈ \d+ \| ≈ \d+ \|",
            "| config 4: VGG16_bn stack, 32 factors + 16 layers, RSVD every 25 | %.2f | ≈ %d | ≈ %d |"
            % (c4["ms_per_step"], round(c4["value"], -1), round(c4["e2e"]["value"], -1)))
    s = sub(s, r"\| config 5: transformer MLP stack, 96 factors \(n ≤ 16385\), 48 layers \| [0-9.]+ \| ≈ \d+ \| ≈ \d+ \|",
            "| config 5: transformer MLP stack, 96 factors (n ≤ 16385), 48 layers | %.0f | ≈ %d | ≈ %d |"
            % (c5["ms_per_step"], round(c5["value"]), round(c5["e2e"]["value"])))
    s = sub(s, r"\| config 5, one 8-GPU rank's share \(12 factors, 6 layers\) \| [0-9.]+ \| ≈ \d+ per rank",
            "| config 5, one 8-GPU rank's share (12 factors, 6 layers) | %.1f | ≈ %d per rank"
            % (r8["ms_per_step"], round(r8["value"])))
    open(p, "w").write(s)
    p = os.path.join(P, "r01_summary.md")
    s = open(p).read()
    if len(sys.argv) > 1:
        rows = [m.end() for m in re.finditer(r"\n\| [^\n]+ \| [0-9.]+ \| \d+ \|", s)]
        i = rows[-1] if rows else None
        if i is not None:
            s = s[:i] + "\n| %s | %.2f | %d |" % (sys.argv[1], c4["ms_per_step"], round(c4["value"])) + s[i:]
    s = re.sub(r"NEXT rows measured at cfg4 \(final\): f1 full rank [0-9.]+ ms/step, f2 factored [0-9.]+ ms/step,\n"
               r"f3 correction every 5 steps [0-9.]+ ms/step",
               "NEXT rows measured at cfg4 (final): f1 full rank %.2f ms/step, f2 factored %.2f ms/step,\n"
               "f3 correction every 5 steps %.2f ms/step" % (f1["ms_per_step"], f2["ms_per_step"], f3["ms_per_step"]), s)
    open(p, "w").write(s)
    print("cfg4 %.3f ms (%.0f/s, e2e %.0f/s)  cfg5 %.1f ms  cfg5r8 %.2f ms (x%.2f)  f1 %.2f f2 %.2f f3 %.2f"
          % (c4["ms_per_step"], c4["value"], c4["e2e"]["value"], c5["ms_per_step"], r8["ms_per_step"], proj,
             f1["ms_per_step"], f2["ms_per_step"], f3["ms_per_step"]))


if __name__ == "__main__":
    main()
