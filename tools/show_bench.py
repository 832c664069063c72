"""Prints a bench.py JSON line's headline and per-stage table (ms per step)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["ms_per_step"], d["value"], d.get("roofline"))
K = d["steps"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for s in d.get("stages", [])[:n]:
    tf = s["gflop"] / s["ms"] if s["ms"] else 0
    print(f"{s['stage']:24s} {s['ms'] / K:8.2f} ms  {s['gflop'] / K:9.1f} GF  {tf:7.1f} TF/s")
