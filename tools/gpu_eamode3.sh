#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for m in ${MODES:-0 3}; do
  BKFAC_EA_MODE=$m timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_m$m.log 2>&1
  python - <<PY
import json
l=[x for x in open("gpurun_out/bench_m$m.log") if x.startswith("{")][-1]
d=json.loads(l); print("mode $m", d["ms_per_step"], [(s["stage"], round(s["ms"]/d["steps"],3)) for s in d["stages"]][:4])
PY
done
