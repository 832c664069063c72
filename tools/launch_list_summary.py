"""ncu launch-list CSV (gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum per
launch) -> the text list kept under profiles/ plus per-kernel totals and shares.
usage: python tools/launch_list_summary.py LAUNCHES.csv OUT.txt "header line" """
import csv
import re
import sys
from collections import defaultdict

src, out, header = sys.argv[1], sys.argv[2], sys.argv[3]
rows = []
with open(src, newline="") as f:
    lines = [l for l in f if not l.startswith("==")]
rd = csv.reader(lines)
head = next(rd)
ix = {n: i for i, n in enumerate(head)}
per = {}
for r in rd:
    if len(r) != len(head):
        continue
    key = int(r[ix["ID"]])
    d = per.setdefault(key, {"kernel": r[ix["Kernel Name"]]})
    val = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    name = r[ix["Metric Name"]]
    if name.startswith("gpu__time"):
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(unit, 1e-3)
        d["us"] = val * scale
    else:
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1e-6)
        d["rd" if "read" in name else "wr"] = val * scale
ids = sorted(per)
tot = sum(per[i].get("us", 0.0) for i in ids)
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
text = [f"# {header}", "# columns: id, kernel, duration_us, dram_read_MB, dram_write_MB"]
for i in ids:
    d = per[i]
    k = re.sub(r"^void |bkfac::|\(.*$", "", d["kernel"])
    text.append(f"{i}, {k}, {d.get('us', 0):.1f}, {d.get('rd', 0):.1f}, {d.get('wr', 0):.1f}")
    a = agg[k]
    a[0] += 1; a[1] += d.get("us", 0); a[2] += d.get("rd", 0); a[3] += d.get("wr", 0)
text.append("")
text.append(f"# per kernel: launches, total_ms, share of the listed kernel time ({tot / 1e3:.1f} ms), dram_read_GB, dram_write_GB")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    text.append(f"# {k}: {a[0]}, {a[1] / 1e3:.2f}, {a[1] / tot:.3f}, {a[2] / 1e3:.2f}, {a[3] / 1e3:.2f}")
open(out, "w").write("\n".join(text) + "\n")
print(f"{len(ids)} launches, {tot / 1e3:.1f} ms")
