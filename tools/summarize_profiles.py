"""Summaries of an ncu launch list (gpu__time_duration + dram bytes per launch) and of an
ncu --set full report, written under profiles/ for the round.

usage: python tools/summarize_profiles.py LAUNCHES.csv FULL.ncu-rep ROUND_TAG
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# kernel-name prefix -> bench stage tag whose roofline line the traffic belongs to
STAGE_OF = {
    "sytrd_tiled_kernel": "eig_sytrd",
    "chol_smem_kernel": "chol_inv",
    "chol_tiled_kernel": "chol_inv",
    "invit_kernel": "eig_invit",
    "bisect_kernel": "eig_bisect",
    "cluster_kernel": "eig_cluster",
}


def short(name: str) -> str:
    n = name.replace("void ", "").replace("bkfac::", "")
    return n.split("(")[0]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = short(r[ki])
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0) / 1e3        # ns -> us
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    return agg


def main():
    csv_path, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    allk = launches(csv_path)
    # the library's kernels only: torch (input generation, the L2 flush) and cuSOLVER (the
    # bench's input bases) kernels run outside the timed region
    ours = ("sytrd", "gemm_", "chol_", "bisect", "invit", "cluster", "backtr", "ew_", "prec_",
            "nonfinite", "philox", "colidx")
    agg = {k: v for k, v in allk.items() if k.startswith(ours)}
    other = {k: v for k, v in allk.items() if k not in agg}
    tot = sum(v[1] for v in agg.values())
    out = [f"# {tag} launch list (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
           "dram__bytes_write.sum --clock-control none)",
           "# command: python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e   (cfg4, 1 GPU)",
           "# whole process (init, warm-up incl. graph captures, 3 graph-replayed + 3 profiled steps);",
           "# cold-cache serialised launches: compare SHARES, not absolute times",
           f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'share':>6s} {'dram_MB/launch':>14s}"]
    traffic = {}
    for k, (n, us, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k[:60]:60s} {n:8d} {us:10.1f} {100 * us / tot:5.1f}% {by / max(n, 1) / 1e6:14.2f}")
        for pre, stage in STAGE_OF.items():
            if k.startswith(pre):
                t = traffic.setdefault(stage, [0, 0.0])
                t[0] += n
                t[1] += by
    # the EA accumulate: the symmetric gemm_tc variant with 8 epilogue warps
    # template args <TA, TB, BN, NLW, DEPTH, EPI, PAIR>: TB = 1 with EPI = 8
    ea = [v for k, v in agg.items() if k.startswith("gemm_tc_kernel<0, 1,")
          and k.split("<")[1].rstrip(">").split(",")[5].strip() == "8"]
    if ea:
        traffic["gemm_ea"] = [sum(v[0] for v in ea), sum(v[2] for v in ea)]
    out.append("# not the library's (outside the timed region): " + ", ".join(
        f"{k[:40]} x{v[0]}" for k, v in sorted(other.items(), key=lambda kv: -kv[1][1])))
    tj = {k: v[1] / max(v[0], 1) for k, v in traffic.items()}
    tj["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes), ncu launch list "
                   f"{tag}, cfg4 bench; gemm_ea = mean over the 8-epilogue-warp <0,1> launches "
                   "(EA accumulate and the other short-K TB stages)")
    open(os.path.join(ROOT, "profiles", f"{tag}_launches_cfg4.txt"), "w").write("\n".join(out) + "\n")
    json.dump(tj, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    # --set full summary
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) > 2:
        h = rows[0]
        want = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                "sm__warps_active.avg.per_cycle_active", "launch__grid_size", "launch__block_size",
                "launch__cluster_dim_x", "launch__registers_per_thread",
                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
        stalls = [n for n in h if "average_warps_issue_stalled" in n and n.endswith("per_issue_active.ratio")]
        lines = [f"# {tag} ncu --set full summary (bench.py cfg4, launches 60-69 of the matched kernels)"]
        for r in rows[2:]:
            lines.append(f"## {r[h.index('Kernel Name')][:90]}")
            for w in want:
                if w in h:
                    lines.append(f"  {w:80s} {r[h.index(w)]}")
            top = sorted(((float(r[h.index(n)] or 0), n) for n in stalls), reverse=True)[:4]
            lines.append("  top stalls (per issue): " + ", ".join(
                f"{n.split('stalled_')[1].split('_per')[0]} {v:.2f}" for v, n in top))
        open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_cfg4.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(out[:22]))


if __name__ == "__main__":
    main()
