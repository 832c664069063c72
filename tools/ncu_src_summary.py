"""Summarise an ncu --page source --csv dump: stall reasons and hottest SASS lines."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address']
for n, start in enumerate(hi):
    end = hi[n + 1] - 1 if n + 1 < len(hi) else len(rows)
    h = rows[start]
    data = [r for r in rows[start + 1:end] if len(r) == len(h)]
    iS = h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[iS] or 0) for r in data)
    cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
    agg = {c: sum(int(r[h.index(c)] or 0) for r in data if r[h.index(c)].isdigit()) for c in cols}
    print(f"kernel #{n}: samples {tot}")
    print("  stalls:", sorted(agg.items(), key=lambda kv: -kv[1])[:8])
    for r in sorted(data, key=lambda r: -int(r[iS] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
        print("  ", r[0][-5:], r[iS], r[1][:100])
