"""Text summary of one or more ncu --set full reports (run where ncu is): key metrics and
top stall reasons per captured launch.  usage: ncu_full_summary.py OUT.txt TITLE REP..."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.per_cycle_active", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "launch__registers_per_thread",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "lts__t_bytes.sum.per_second", "dram__bytes.sum.per_second",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]

out, title, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
lines = [f"# {title}"]
for rep in reps:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    h = rows[0]
    stalls = [n for n in h if "average_warps_issue_stalled" in n and n.endswith("per_issue_active.ratio")]
    for r in rows[2:]:
        lines.append(f"## {r[h.index('Kernel Name')][:100]}   [{rep.split('/')[-1]}]")
        for w in WANT:
            if w in h:
                lines.append(f"  {w:80s} {r[h.index(w)]}")
        top = sorted(((float(r[h.index(n)] or 0), n) for n in stalls), reverse=True)[:4]
        lines.append("  top stalls (per issue): " + ", ".join(
            f"{n.split('stalled_')[1].split('_per')[0]} {v:.2f}" for v, n in top))
open(out, "w").write("\n".join(lines) + "\n")
print(f"{len(lines)} lines -> {out}")
